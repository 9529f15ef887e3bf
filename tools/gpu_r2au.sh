#!/usr/bin/env bash
# dK/dV dropout PRMT lane masks, final form: full GPU suite, dropout and C3 bench lines
O=gpurun_out/r2au
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do
  timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/d$rep.json 2>/dev/null; python tools/bench_summary.py $O/d$rep.json "drop"
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/c3.json 2>/dev/null; python tools/bench_summary.py $O/c3.json "c3"
