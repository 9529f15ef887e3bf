#!/usr/bin/env bash
# dK/dV dropout: L2 prefetch of the key-major keep words 0 / 1 / 2 (default) / 4 steps ahead
O=gpurun_out/r2ay
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "drop or mask" 2>&1 | tail -2
for rep in 1 2; do
  for lib in tools/variants/pf0.so tools/variants/pf1.so paper_2502_12784_b200/libvattn_b200.so tools/variants/pf4.so; do
    VATTN_LIB=$lib timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "drop $lib"
  done
done
