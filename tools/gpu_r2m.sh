#!/usr/bin/env bash
# Re-entry check of HEAD: GPU suite, smoke, bench line.
O=gpurun_out/r2m
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv | tee $O/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 | tee $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee $O/smoke.log
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; cut -c1-400 $O/bench_c3.json
timeout 900 python tools/time_variants.py --configs c3,c3_nc,c2_4k,c4 --steps 20 2>&1 | tail -20 | tee $O/variants.txt
