#!/usr/bin/env bash
# mask-kernel issue-balance variants (VATTN_DROPKEEP 0 / 1 / 2 = default build)
O=gpurun_out/r2ao
mkdir -p $O
for rep in 1 2; do
  for lib in tools/variants/dropkeep0.so tools/variants/dropkeep1.so paper_2502_12784_b200/libvattn_b200.so; do
    VATTN_LIB=$lib timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "drop $lib"
  done
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
