#!/usr/bin/env bash
O=gpurun_out/r2ah
mkdir -p $O
VATTN_DKDV_PERSIST=1 VATTN_LIB=tools/variants/dbg.so timeout 300 python tools/debug_pair.py 1,2,384,64,1 1,1,256,128,0 2,3,1000,128,1 4,8,512,64,0 2,16,1024,64,1,bf16 2>&1 | tee $O/debug.txt
rm -f tools/variants/dbg.so
VATTN_DKDV_PERSIST=1 timeout 1200 python -m pytest tests/test_mha_gpu.py tests/test_random_gpu.py tests/test_stress_gpu.py tests/test_full_size_gpu.py tests/test_contract_gpu.py -q -x 2>&1 | tail -2 | tee $O/pytest.log
for rep in 1 2; do for pe in 0 1; do VATTN_DKDV_PERSIST=$pe timeout 600 python tools/time_variants.py --configs c4,c2_512,c2_1k,c2_4k,c3 --steps 20 2>&1 | sed "s/^/persist=$pe /" | tee -a $O/variants.txt; done; done
for pe in 0 1; do VATTN_DKDV_PERSIST=$pe timeout 600 python bench.py --config c4x24 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "c4x24 persist=$pe"; done
