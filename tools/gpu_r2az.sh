#!/usr/bin/env bash
# Persistent dK/dV (VATTN_DKDV_PERSIST=1) vs one CTA per item at long N: C3 non-causal
# (equal items, unit-grouped round robin) and causal (zigzag)
O=gpurun_out/r2az
mkdir -p $O
for rep in 1 2; do
  for cfg in c3_nc c3; do
    for pe in 0 1; do
      VATTN_DKDV_PERSIST=$pe timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "$cfg persist=$pe"
    done
  done
done
