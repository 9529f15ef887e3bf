#!/usr/bin/env bash
# CTA-pair dK/dV (cta_group::2) first run: parity, then timing pair vs single.
O=gpurun_out/r2n
mkdir -p $O
timeout 300 python -m pytest tests/test_mha_gpu.py -q -x 2>&1 | tail -15 | tee $O/pytest_pair.log
timeout 600 python -m pytest tests/test_mha_gpu.py tests/test_contract_gpu.py tests/test_random_gpu.py -q -x 2>&1 | tail -5 | tee $O/pytest_pair_all.log
for pr in 0 1; do
  VATTN_DKDV_PAIR=$pr timeout 600 python tools/time_variants.py --configs c3,c3_nc,c5 --steps 20 2>&1 | tail -3 | sed "s/^/pair=$pr /" | tee -a $O/variants.txt
done
