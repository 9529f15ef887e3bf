#!/usr/bin/env bash
set -x
mkdir -p gpurun_out/r2b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for tool in synccheck racecheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tests/stress_child.py '[[1,2,384,64,1,"fp16",0.0],[1,1,256,128,0,"bf16",0.0],[1,1,300,128,1,"bf16",0.2],[1,2,200,64,0,"fp16",0.1]]' 1 > gpurun_out/r2b/san_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "SUMMARY|RESULT" gpurun_out/r2b/san_$tool.txt | head -3
  VATTN_DQ_MODE=0 timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tests/stress_child.py '[[1,1,256,128,1,"bf16",0.0],[1,2,384,64,0,"fp16",0.0]]' 1 > gpurun_out/r2b/san_${tool}_dq0.txt 2>&1
  echo "$tool dq0 rc=$?"; grep -E "SUMMARY|RESULT" gpurun_out/r2b/san_${tool}_dq0.txt | head -3
done
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/r2b/pytest_gpu.log
tail -25 gpurun_out/r2b/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r2b/bench_c3.json 2> gpurun_out/r2b/bench_c3.err; cat gpurun_out/r2b/bench_c3.json; tail -3 gpurun_out/r2b/bench_c3.err
timeout 600 python bench.py --config c4x24 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2b/bench_c4x24.json 2> gpurun_out/r2b/bench_c4x24.err; cat gpurun_out/r2b/bench_c4x24.json; tail -3 gpurun_out/r2b/bench_c4x24.err
