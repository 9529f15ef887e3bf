#!/usr/bin/env bash
set -x
O=gpurun_out/r2e
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "dropout or mask or autograd or contract" 2>&1 | tail -15 > $O/pytest_sel.log
tail -15 $O/pytest_sel.log
timeout 600 python bench.py --steps 10 --warmup 3 --dropout 0.1 --no-cpu-baseline > $O/bench_c3_drop.json 2> $O/bench_c3_drop.err; cat $O/bench_c3_drop.json; tail -3 $O/bench_c3_drop.err
timeout 900 ncu --set full --clock-control none -k regex:"dropmask|dkdv" -s 2 -c 2 -o $O/ncu_drop python bench.py --steps 1 --warmup 3 --dropout 0.1 --no-cpu-baseline --e2e-steps 0 > $O/ncu_drop.log 2>&1; tail -3 $O/ncu_drop.log
