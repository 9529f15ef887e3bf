#!/usr/bin/env bash
# knob sweep on the final code: K/V ring depth (d=128 fwd), dK/dV tail waves, fwd L2 group
O=gpurun_out/r2ag
mkdir -p $O
timeout 900 python tools/time_variants.py --configs c3,c3_nc,c5 --steps 20 st3 st5 2>&1 | tee $O/stages.txt
for tw in 0 2 3.5 5; do VATTN_DKDV_TAIL_WAVES=$tw timeout 600 python tools/time_variants.py --configs c3,c5 --steps 20 none 2>&1 | grep libvattn | sed "s/^/tail=$tw /" | tee -a $O/tail.txt; done
for g in 32 64 128; do VATTN_L2_GROUP_MB_FWD=$g timeout 600 python tools/time_variants.py --configs c3,c5,c2_4k --steps 20 none 2>&1 | grep libvattn | sed "s/^/l2=$g /" | tee -a $O/l2.txt; done
