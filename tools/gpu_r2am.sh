#!/usr/bin/env bash
# round-1 final kernels vs the current ones, same box, interleaved
O=gpurun_out/r2am
mkdir -p $O
timeout 900 python tools/time_variants.py --configs c3,c3_nc,c2_4k,c4 --steps 20 r1final 2>&1 | tee $O/v.txt
for rep in 1 2; do for lib in paper_2502_12784_b200/libvattn_b200.so tools/variants/r1final.so; do VATTN_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "$lib"; done; done
