#!/usr/bin/env bash
# mask kernel: unroll of the per-key loop (8 default) and occupancy
O=gpurun_out/r2av
mkdir -p $O
for rep in 1 2; do
  for lib in paper_2502_12784_b200/libvattn_b200.so tools/variants/unroll4.so tools/variants/unroll16.so tools/variants/u16b8.so tools/variants/unroll32.so; do
    VATTN_LIB=$lib timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "drop $lib"
  done
done
