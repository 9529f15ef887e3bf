#!/usr/bin/env bash
O=gpurun_out/r2v
mkdir -p $O
VATTN_LIB=tools/variants/onepoly.so timeout 600 python -m pytest tests/test_mha_gpu.py tests/test_random_gpu.py -q -x 2>&1 | tail -3 | tee $O/pytest.log
for rep in 1 2; do timeout 600 python tools/time_variants.py --configs c3,c3_nc,c2_4k,c4,c5 --steps 20 onepoly 2>&1 | tee -a $O/variants.txt; done
