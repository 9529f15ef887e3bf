#!/usr/bin/env bash
set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python -m pytest tests/test_mha_gpu.py tests/test_contract_gpu.py -q -x 2>&1 | tail -5 > $O/pytest_sel.log
tail -5 $O/pytest_sel.log
timeout 900 python tools/time_variants.py --configs c3,c2_4k,c4 --steps 20 base 2>&1 | tee $O/variants.txt
timeout 600 python bench.py --steps 10 --warmup 3 --dropout 0.1 --no-cpu-baseline --e2e-steps 0 > $O/bench_c3_drop.json 2> $O/bench_c3_drop.err; cat $O/bench_c3_drop.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['kernels_ms'])"
