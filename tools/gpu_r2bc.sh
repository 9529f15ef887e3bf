#!/usr/bin/env bash
# source-level stall profile (SASS + CUDA lines) of the C3 forward and dK/dV kernels
O=gpurun_out/r2bc
mkdir -p $O
for k in mha_fwd_sm100_kernel mha_bwd_dkdv_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $O/$k \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/$k.log 2>&1
  ncu -i $O/$k.ncu-rep --page source --csv --print-source sass > $O/${k}_sass.csv 2>/dev/null
  ncu -i $O/$k.ncu-rep --page source --csv --print-source cuda > $O/${k}_cuda.csv 2>/dev/null
  rm -f $O/$k.ncu-rep
done
ls -la $O
