#!/usr/bin/env bash
# Round-2 evidence run: soak (legacy vs fixed barrier protocol), sanitizers, GPU tests,
# smoke, bench lines (C3, C4x24, reference arm, split bh at 1 GPU), launch list.
set -x
O=gpurun_out/r2c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -40 > $O/pytest_gpu.log
tail -8 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err; cat $O/bench_c3.json; tail -3 $O/bench_c3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; cat $O/bench_ref.json
timeout 600 python bench.py --config c4x24 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c4x24.json 2> $O/bench_c4x24.err; cat $O/bench_c4x24.json; tail -3 $O/bench_c4x24.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_bench.log 2>&1; tail -2 $O/ncu_bench.log
bash tools/stress_soak.sh 6 $O/soak > $O/soak_summary.txt 2>&1
cat $O/soak_summary.txt
for tool in synccheck racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tests/stress_child.py '[[1,2,384,64,1,"fp16",0.0],[1,1,256,128,0,"bf16",0.0],[1,1,300,128,1,"bf16",0.2],[1,2,200,64,0,"fp16",0.1]]' 1 > $O/san_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RESULT" $O/san_$tool.txt | head -3
done
