#!/usr/bin/env bash
# run-time dispatch knobs at C3: forward L2 group budget, dK/dV tail waves
O=gpurun_out/r2bb
mkdir -p $O
run() { env "$@" timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "$*"; }
for rep in 1 2; do
  run X=default
  run VATTN_L2_GROUP_MB_FWD=32
  run VATTN_L2_GROUP_MB_FWD=128
  run VATTN_L2_GROUP_MB_FWD=0
  run VATTN_DKDV_TAIL_WAVES=2.5
  run VATTN_DKDV_TAIL_WAVES=5
  run VATTN_L2_GROUP_MB_BWD=64
done
