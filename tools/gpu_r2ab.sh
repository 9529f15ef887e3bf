#!/usr/bin/env bash
O=gpurun_out/r2ab
mkdir -p $O
for lib in paper_2502_12784_b200/libvattn_b200.so tools/variants/noprefetch.so paper_2502_12784_b200/libvattn_b200.so tools/variants/noprefetch.so; do
VATTN_LIB=$lib timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_drop.json 2>/dev/null
python tools/bench_summary.py $O/bench_drop.json $lib
done
