#!/usr/bin/env bash
O=gpurun_out/r2aa
mkdir -p $O
timeout 900 python -m pytest tests/test_mha_gpu.py tests/test_contract_gpu.py tests/test_random_gpu.py tests/test_traditional_gpu.py -q -x -k "dropout or drop or mask or digest" 2>&1 | tail -2 | tee $O/pytest.log
timeout 900 python -m pytest tests/test_full_size_gpu.py -q -x -k "dropout" 2>&1 | tail -1 | tee -a $O/pytest.log
for lib in paper_2502_12784_b200/libvattn_b200.so tools/variants/maskalu.so paper_2502_12784_b200/libvattn_b200.so tools/variants/maskalu.so; do
VATTN_LIB=$lib timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_drop.json 2>/dev/null
python -c "import json;d=json.load(open('$O/bench_drop.json'));print('$lib', round(d['value'],1), round(d['ms_per_step'],3), 'mask', round(d['kernels_ms']['dropmask'],3))"
done
