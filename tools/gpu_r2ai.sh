#!/usr/bin/env bash
O=gpurun_out/r2ai
mkdir -p $O
VATTN_FWD_PERSIST=1 VATTN_LIB=tools/variants/dbg.so timeout 300 python tools/debug_pair.py 1,2,384,64,1 1,1,256,128,0 2,3,1000,128,1 16,16,512,64,0 8,16,1024,64,1 2,16,1000,128,0,bf16 2>&1 | tee $O/debug.txt
rm -f tools/variants/dbg.so
VATTN_FWD_PERSIST=1 timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee $O/pytest.log
for rep in 1 2; do for pe in 0 1; do VATTN_FWD_PERSIST=$pe timeout 600 python tools/time_variants.py --configs c4,c2_512,c2_1k,c3 --steps 20 2>&1 | grep libvattn | sed "s/^/fpersist=$pe /" | tee -a $O/variants.txt; done; done
for pe in 0 1; do VATTN_FWD_PERSIST=$pe timeout 600 python bench.py --config c4x24 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "c4x24 fpersist=$pe"; done
