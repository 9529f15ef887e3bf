#!/usr/bin/env bash
# pair vs single dK/dV under the bench's own (power-capped) conditions, interleaved
O=gpurun_out/r2p
mkdir -p $O
for rep in 1 2; do for pr in 0 1; do
  VATTN_DKDV_PAIR=$pr timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > $O/bench_pair${pr}_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('$O/bench_pair${pr}_$rep.json'));print('pair=$pr', round(d['value'],1), d['ms_per_step'], d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernels_ms'].items() if k!='note'})"
done; done
