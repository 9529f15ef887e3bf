#!/usr/bin/env bash
# d = 64, N > 1024: dQ by recompute (default) vs materialised dS^T + persistent dQ GEMM
O=gpurun_out/r2al
mkdir -p $O
for rep in 1 2; do for m in 0 1; do VATTN_DQ_MODE=$m timeout 900 python tools/time_variants.py --configs c2_2k,c2_4k,c2_8k,c2_16k --steps 10 2>&1 | grep libvattn | sed "s/^/mode=$m /" | tee -a $O/v.txt; done; done
