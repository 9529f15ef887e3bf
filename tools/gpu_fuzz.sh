#!/usr/bin/env bash
# One-off randomized soak of the final code paths against the binary64 oracle:
# default, CTA-pair dK/dV, overlapped dQ workers, per-tile dQ, recompute dQ.
O=gpurun_out/fuzz
mkdir -p $O
for cfg in "" "VATTN_DKDV_PAIR=1" "VATTN_DQ_WORKERS=12" "VATTN_DQ_PERSIST=0" "VATTN_DQ_MODE=0"; do
  env $cfg VATTN_FUZZ_SEEDS=1000:1150 timeout 1200 python -m pytest tests/test_random_gpu.py -q -k "vs_binary64" 2>&1 | tail -2 | sed "s/^/[$cfg] /" | tee -a $O/fuzz.txt
done
