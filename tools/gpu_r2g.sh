#!/usr/bin/env bash
O=gpurun_out/r2g
mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:dropmask -s 1 -c 1 -o $O/ncu_mask python bench.py --steps 1 --warmup 1 --dropout 0.1 --no-cpu-baseline --e2e-steps 0 > $O/ncu_mask.log 2>&1; tail -2 $O/ncu_mask.log
