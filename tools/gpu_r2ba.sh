#!/usr/bin/env bash
# Persistent dK/dV over host-built dispatch-like item lists (VATTN_DKDV_LISTS=1, long heads)
# vs one CTA per item (=0): GPU suite, then C3 / C3 non-causal / C5 / dropout A/B
O=gpurun_out/r2ba
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for rep in 1 2; do
  for cfg in c3 c3_nc; do
    for li in 0 1; do
      VATTN_DKDV_LISTS=$li timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "$cfg lists=$li"
    done
  done
done
for li in 0 1; do
  VATTN_DKDV_LISTS=$li timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "drop lists=$li"
  VATTN_DKDV_LISTS=$li timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "c5 lists=$li"
done
