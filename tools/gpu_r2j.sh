#!/usr/bin/env bash
O=gpurun_out/r2j
mkdir -p $O
timeout 900 python -m pytest tests/test_mha_gpu.py tests/test_contract_gpu.py tests/test_host_slabs_gpu.py -q -x 2>&1 | tail -5 > $O/pytest_sel.log
cat $O/pytest_sel.log
timeout 900 python tools/time_variants.py --configs c4,c2_1k,c2_4k,c2_16k,c3 --steps 20 wg2 base 2>&1 | tee $O/variants.txt
