#!/usr/bin/env bash
O=gpurun_out/r2l
mkdir -p $O
timeout 900 python -m pytest tests/test_mha_gpu.py tests/test_contract_gpu.py -q -x 2>&1 | tail -2
VATTN_LIB=tools/variants/wg4d128.so timeout 900 python -m pytest tests/test_mha_gpu.py -q -x 2>&1 | tail -2
timeout 900 python tools/time_variants.py --configs c3,c3_nc,c2_4k,c4 --steps 20 wg4d128 2>&1 | tee $O/variants.txt
