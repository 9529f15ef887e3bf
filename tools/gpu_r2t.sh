#!/usr/bin/env bash
O=gpurun_out/r2t
mkdir -p $O
VATTN_LIB=tools/variants/dbg.so timeout 300 python tools/debug_pair.py 1,2,384,128,1 2,2,1000,128,0 1,2,1024,64,1 4,16,2048,128,1 2>&1 | tee $O/debug.txt
rm -f tools/variants/dbg.so
timeout 900 python -m pytest tests/test_mha_gpu.py tests/test_random_gpu.py tests/test_contract_gpu.py tests/test_stress_gpu.py tests/test_full_size_gpu.py -q -x 2>&1 | tail -4 | tee $O/pytest.log
for w in 0 8 16 24; do VATTN_DQ_WORKERS=$w timeout 600 python tools/time_variants.py --configs c3,c3_nc,c4,c2_1k --steps 20 2>&1 | sed "s/^/W=$w /" | tee -a $O/variants.txt; done
