#!/usr/bin/env bash
# C4 / C2 (d = 64) where-does-the-time-go: CTA timelines, dK/dV + fwd traces, ncu of the forward.
O=gpurun_out/r2q
mkdir -p $O
timeout 300 python tools/cta_timeline.py 8 16 1024 64 1 2>&1 | tail -30 | tee $O/cta_c4.txt
timeout 300 python tools/trace_bwd.py 8 16 1024 64 1 0 2>&1 | tail -40 | tee $O/trace_c4.txt
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:mha_fwd_sm100_kernel" -s 3 -c 1 -o $O/fwd_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_fwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:mha_bwd_dkdv_kernel" -s 3 -c 1 -o $O/dkdv_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_dkdv.log 2>&1
ls -la $O
