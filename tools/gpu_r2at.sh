#!/usr/bin/env bash
# dK/dV dropout: PRMT lane masks for the dV operand (vs selects); mask kernel ncu --set full
O=gpurun_out/r2at
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "drop or mask" 2>&1 | tail -3
for rep in 1 2; do
  for lib in tools/variants/strip0.so paper_2502_12784_b200/libvattn_b200.so; do
    VATTN_LIB=$lib timeout 600 python bench.py --dropout 0.1 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/b.json 2>/dev/null; python tools/bench_summary.py $O/b.json "drop $lib"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dropmask -s 3 -c 1 -o $O/mask \
  python bench.py --dropout 0.1 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu.log 2>&1
ncu -i $O/mask.ncu-rep --page raw --csv > $O/mask_raw.csv 2>/dev/null
ncu -i $O/mask.ncu-rep --page source --csv --print-source sass > $O/mask_src.csv 2>/dev/null
ncu -i $O/mask.ncu-rep --page details > $O/mask_details.txt 2>/dev/null
rm -f $O/mask.ncu-rep
