#!/usr/bin/env bash
O=gpurun_out/r2ae
mkdir -p $O
VATTN_DQ_PERSIST=1 timeout 600 python -m pytest tests/test_mha_gpu.py -q -x -k "dq_modes or workers or golden" 2>&1 | tail -1
for rep in 1 2; do for pe in 0 1; do VATTN_DQ_PERSIST=$pe timeout 600 python tools/time_variants.py --configs c4,c2_512,c2_1k,c3 --steps 20 2>&1 | sed "s/^/persist=$pe /" | tee -a $O/variants.txt; done; done
