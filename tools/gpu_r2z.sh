#!/usr/bin/env bash
O=gpurun_out/r2z
mkdir -p $O
timeout 900 python -m pytest tests/test_mha_gpu.py tests/test_contract_gpu.py tests/test_random_gpu.py -q -x -k "dropout or drop or mask or digest" 2>&1 | tail -3 | tee $O/pytest.log
timeout 900 python -m pytest tests/test_full_size_gpu.py -q -x -k "dropout" 2>&1 | tail -2 | tee -a $O/pytest.log
timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_drop.json 2>/dev/null
python -c "import json;d=json.load(open('$O/bench_drop.json'));print(d['value'], d['ms_per_step'], d['kernels_ms'])"
timeout 600 ncu --set full --clock-control none -k "regex:mha_dropmask_kernel" -s 1 -c 1 -o $O/mask python bench.py --dropout 0.1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $O/ncu.log 2>&1
