#!/usr/bin/env bash
O=gpurun_out/r2i
mkdir -p $O
timeout 300 python tools/cta_timeline.py 8 16 1024 64 1 2>&1 | tee $O/cta_c4.txt
timeout 300 python tools/cta_timeline.py 4 32 4096 64 0 2>&1 | tee $O/cta_c2_4k.txt
timeout 300 python tools/trace_bwd.py 8 16 1024 64 1 100 2>&1 | tee $O/trace_c4.txt
