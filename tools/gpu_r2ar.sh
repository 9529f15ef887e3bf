#!/usr/bin/env bash
# forward dropout: keep bits staged through shared memory (cp.async) + PRMT lane masks
# vs HEAD (register prefetch, spills); C3 with and without dropout
O=gpurun_out/r2ar
mkdir -p $O
for rep in 1 2; do
  for lib in tools/variants/head.so paper_2502_12784_b200/libvattn_b200.so; do
    VATTN_LIB=$lib timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "drop $lib"
    VATTN_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "c3   $lib"
  done
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
