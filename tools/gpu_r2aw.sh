#!/usr/bin/env bash
# host pipeline: step in two phases (O/lse D2H during the backward, dO H2D during the forward) vs one
O=gpurun_out/r2aw
mkdir -p $O
timeout 900 python -m pytest tests/test_host_slabs_gpu.py tests/test_contract_gpu.py -q -x 2>&1 | tail -3
for rep in 1 2; do
  for split in 0 1; do
    VATTN_HOST_SPLIT=$split timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/b.json 2>/dev/null
    python -c "import json; d=json.load(open('$O/b.json')); print('split=$split', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['e2e'].get('ms_per_step',0),3))"
  done
done
