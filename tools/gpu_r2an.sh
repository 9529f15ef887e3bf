#!/usr/bin/env bash
# causal persistent kernels: zigzag longest-first vs static round robin over the dispatch order
O=gpurun_out/r2an
mkdir -p $O
timeout 900 python -m pytest tests/test_mha_gpu.py -q -x -k "persistent or workers or golden or random" 2>&1 | tail -1 | tee $O/pytest.log
VATTN_DKDV_PERSIST=1 VATTN_FWD_PERSIST=1 timeout 900 python -m pytest tests/test_random_gpu.py tests/test_full_size_gpu.py -q -x 2>&1 | tail -1 | tee -a $O/pytest.log
for rep in 1 2; do timeout 900 python tools/time_variants.py --configs c4,c2_1k,c3 --steps 20 rrstatic 2>&1 | tee -a $O/v.txt; done
for pe in 1; do VATTN_DKDV_PERSIST=$pe VATTN_FWD_PERSIST=$pe timeout 900 python tools/time_variants.py --configs c3,c5 --steps 10 rrstatic 2>&1 | sed "s/^/forced /" | tee -a $O/v.txt; done
for lib in paper_2502_12784_b200/libvattn_b200.so tools/variants/rrstatic.so; do VATTN_LIB=$lib timeout 600 python bench.py --config c4x24 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "c4x24 $lib"; done
