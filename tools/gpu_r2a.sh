#!/usr/bin/env bash
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out/r2a
bash tools/stress_soak.sh 4 gpurun_out/r2a/soak > gpurun_out/r2a/soak_summary.txt 2>&1
cat gpurun_out/r2a/soak_summary.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/r2a/pytest_gpu.log
tail -15 gpurun_out/r2a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r2a/bench_c3.json 2> gpurun_out/r2a/bench_c3.err; cat gpurun_out/r2a/bench_c3.json; tail -3 gpurun_out/r2a/bench_c3.err
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tests/stress_child.py '[[1,2,384,64,1,"fp16",0.0],[1,1,256,128,0,"bf16",0.0]]' 1 > gpurun_out/r2a/san_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -5 gpurun_out/r2a/san_$tool.txt
done
