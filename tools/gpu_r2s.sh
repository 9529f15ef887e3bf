#!/usr/bin/env bash
O=gpurun_out/r2s
mkdir -p $O
timeout 600 python -m pytest tests/test_mha_gpu.py tests/test_random_gpu.py tests/test_contract_gpu.py -q -x 2>&1 | tail -4 | tee $O/pytest.log
timeout 900 python tools/time_variants.py --configs c4,c2_1k,c2_4k,c2_16k,c3,c3_nc --steps 20 2>&1 | tee $O/variants.txt
