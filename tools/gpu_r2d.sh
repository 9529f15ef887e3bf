#!/usr/bin/env bash
set -x
O=gpurun_out/r2d
mkdir -p $O
timeout 600 python -m pytest tests/test_mha_gpu.py -q -x -k "autograd or dropout" 2>&1 | tail -30 > $O/pytest_sel.log
tail -30 $O/pytest_sel.log
timeout 600 python -m pytest tests -m gpu -q -k "dropout or mask" 2>&1 | tail -15 > $O/pytest_drop.log
tail -15 $O/pytest_drop.log
timeout 600 python bench.py --steps 10 --warmup 3 --dropout 0.1 --no-cpu-baseline > $O/bench_c3_drop.json 2> $O/bench_c3_drop.err; cat $O/bench_c3_drop.json; tail -3 $O/bench_c3_drop.err
