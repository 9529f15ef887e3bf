#!/usr/bin/env bash
O=gpurun_out/r2k
mkdir -p $O
VATTN_LIB=tools/variants/dsdirect.so timeout 600 python -m pytest tests/test_mha_gpu.py -q -x -k "golden or f64 or binary64" 2>&1 | tail -3
timeout 900 python tools/time_variants.py --configs c3,c4,c2_1k --steps 20 dsdirect 2>&1 | tee $O/variants.txt
