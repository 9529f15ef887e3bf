#!/usr/bin/env bash
# Hang-fix evidence on the final code: schedule-fuzzer soak, legacy (round-1) barrier
# protocol vs the per-parity fix, 10 runs each; then the plain build for 200 fwd+bwd
# launches each at (4,32,4096,64) causal fp16 and C3, digests checked for stability.
O=gpurun_out/r2ax
mkdir -p $O
bash tools/stress_soak.sh 10 $O/soak > $O/soak_summary.txt 2>&1; grep -E "failed|MISSING" $O/soak_summary.txt
grep -h "watchdog" $O/soak/stress_legacy_*.log | head -3
timeout 900 python tests/stress_child.py '[[4,32,4096,64,1,"fp16",0.0]]' 200 > $O/plain_d64_200.log 2>&1; echo "d64 x200 rc=$?"; tail -1 $O/plain_d64_200.log | cut -c1-200
timeout 1200 python tests/stress_child.py '[[4,16,8192,128,1,"bf16",0.0]]' 200 > $O/plain_c3_200.log 2>&1; echo "C3 x200 rc=$?"; tail -1 $O/plain_c3_200.log | cut -c1-200
