#!/usr/bin/env bash
O=gpurun_out/r2ap
mkdir -p $O
for lib in tools/variants/dropkeep0.so paper_2502_12784_b200/libvattn_b200.so; do
  n=$(basename $lib .so)
  VATTN_LIB=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:mha_dropmask -s 3 -c 1 -o $O/mask_$n \
    python bench.py --dropout 0.1 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/mask_$n.log 2>&1
done
ls -la $O
