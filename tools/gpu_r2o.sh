#!/usr/bin/env bash
O=gpurun_out/r2o
mkdir -p $O
for pr in 0 1; do
  VATTN_DKDV_PAIR=$pr timeout 600 python tools/time_variants.py --configs c3,c3_nc,c5 --steps 20 2>&1 | sed "s/^/pair=$pr /" | tee -a $O/variants.txt
done
timeout 300 python -m pytest tests/test_mha_gpu.py -q -x 2>&1 | tail -2
