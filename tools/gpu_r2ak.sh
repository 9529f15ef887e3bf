#!/usr/bin/env bash
O=gpurun_out/r2ak
mkdir -p $O
for rep in 1 2; do
  for lib in paper_2502_12784_b200/libvattn_b200.so tools/variants/prepersist.so; do
    VATTN_LIB=$lib timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "drop $lib"
  done
done
timeout 900 python tools/time_variants.py --configs c3,c3_nc,c2_512,c2_4k,c4 --steps 20 prepersist 2>&1 | tee $O/variants.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
