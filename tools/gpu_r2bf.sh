#!/usr/bin/env bash
# persistent dQ GEMM: producer prefetches the next item's first tiles under the epilogue
O=gpurun_out/r2bf
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do
  for cfg in c2_512 c2_1k c4 c3; do
    for lib in tools/variants/dqbase.so paper_2502_12784_b200/libvattn_b200.so; do
      VATTN_LIB=$lib timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "$cfg $lib"
    done
  done
done
