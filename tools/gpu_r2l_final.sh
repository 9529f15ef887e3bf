#!/usr/bin/env bash
# Round-2 evidence on the final code: GPU tests, smoke, bench lines, sweep, soak, launch
# lists + ncu --set full summaries (reports summarised on the box and deleted: gpurun
# returns at most 64 MiB).  compute-sanitizer is closed on the GPU pool since r2i.
set -x
O=gpurun_out/r2l
mkdir -p $O/profiles
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv | tee $O/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee $O/smoke.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; cut -c1-300 $O/bench_c3.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --config c4x24 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4x24.json 2> $O/bench_c4x24.err
timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c3_dropout0.1.json 2> $O/bench_c3_drop.err
timeout 900 python bench.py --config c5 --split bh --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c5_bh.json 2> $O/bench_c5_bh.err
timeout 1500 python tools/sweep.py --steps 10 --tag r2l --out $O/profiles > $O/sweep.log 2>&1; tail -3 $O/sweep.log
bash tools/stress_soak.sh 6 $O/soak > $O/soak_summary.txt 2>&1; cat $O/soak_summary.txt
bash tools/profile_round.sh c3 r2l > $O/profile_round.log 2>&1
KERNELS="mha_bwd_dq_kernel mha_fwd_sm100_kernel mha_bwd_dkdv_kernel" bash tools/profile_round.sh c2_4k r2l > $O/profile_round_c2.log 2>&1
for d in gpurun_out/prof_r2l_c3 gpurun_out/prof_r2l_c2_4k; do
  cfg=${d##*prof_r2l_}
  VATTN_PROFILES_DIR=$O/profiles python tools/ncu_summary.py $d r2l $cfg > $O/ncu_summary_$cfg.log 2>&1
done
rm -rf gpurun_out/prof_r2l_*
du -sh gpurun_out
