#!/usr/bin/env bash
# Build experimental variants of libvattn_b200.so (tuning only; never shipped).
#   bash tools/build_variants.sh name1 "-DFLAG=.." name2 "-DFLAG=.." ...
# -> tools/variants/<name>.so  (load with VATTN_LIB=tools/variants/<name>.so)
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/variants
SRC=paper_2502_12784_b200/csrc
pids=()
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -cudart static \
       --expt-relaxed-constexpr $flags -shared $SRC/capi.cu $SRC/capi_host.cu -o tools/variants/$name.so &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
ls -la tools/variants
