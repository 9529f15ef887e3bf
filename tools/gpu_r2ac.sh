#!/usr/bin/env bash
O=gpurun_out/r2ac
mkdir -p $O
timeout 600 python -m pytest tests/test_mha_gpu.py -q -x 2>&1 | tail -2 | tee $O/pytest.log
for rep in 1 2; do timeout 900 python tools/time_variants.py --configs c3,c3_nc,c2_4k,c4 --steps 20 2>&1 | tee -a $O/variants.txt; done
