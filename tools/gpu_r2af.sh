#!/usr/bin/env bash
O=gpurun_out/r2af
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1 | tee $O/pytest.log
for rep in 1 2; do
  for lib in paper_2502_12784_b200/libvattn_b200.so tools/variants/pdllate.so; do
    VATTN_LIB=$lib timeout 600 python bench.py --config c4x24 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "c4x24 $lib"
  done
done
timeout 900 python tools/time_variants.py --configs c4,c2_512,c2_1k,c3 --steps 20 pdllate 2>&1 | tee $O/variants.txt
