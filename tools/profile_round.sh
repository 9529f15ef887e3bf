#!/usr/bin/env bash
# Profile the hot path on one B200 (run under gpurun): launch list of the bench
# command and one `ncu --set full` capture per hot kernel.  Outputs go to
# gpurun_out/ (scratch); tools/ncu_summary.py turns them into profiles/*.md.
#   bash tools/profile_round.sh [config] [tag]
set -u
CFG=${1:-c3}
TAG=${2:-r1}
OUT=gpurun_out/prof_${TAG}_${CFG}
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > "$OUT/gpu.txt"
# launch list (cold-cache, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --config "$CFG" --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > "$OUT/launches_bench.log" 2>&1
# one full capture per hot kernel (skip the warm-up launches)
for k in ${KERNELS:-mha_fwd_sm100_kernel mha_bwd_dkdv_kernel mha_bwd_dq_tail_kernel mha_bwd_dq_kernel mha_bwd_preprocess_kernel}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 \
        -o "$OUT/$k" python bench.py --config "$CFG" --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
        > "$OUT/$k.log" 2>&1
done
ls -la "$OUT"
