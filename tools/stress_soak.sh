#!/usr/bin/env bash
# Schedule-fuzzer soak (run under gpurun): the legacy (round-1) barrier protocol vs the
# fixed one, both built with -DVATTN_STRESS_NS (tools/build_stress_legacy.sh, Makefile
# target libvattn_b200_stress.so).  Each run is one child process of
# tests/stress_child.py; a watchdog trap shows as a non-zero exit.
#   bash tools/stress_soak.sh <runs> [out_dir]
RUNS=${1:-5}
OUT=${2:-gpurun_out/soak}
mkdir -p "$OUT"
CFG_D64='[[2,4,2048,64,1,"fp16",0.0],[4,8,1024,64,0,"bf16",0.0]]'
for lib in tools/variants/stress_legacy.so paper_2502_12784_b200/libvattn_b200_stress.so; do
  name=$(basename $lib .so)
  if [ ! -f "$lib" ]; then  # a missing build must not read as a trapped run
    echo "$name: MISSING ($lib) -- build it first (tools/build_stress_legacy.sh / make)"
    continue
  fi
  fails=0
  for i in $(seq 1 $RUNS); do
    VATTN_LIB=$lib timeout 300 python tests/stress_child.py "$CFG_D64" 8 > "$OUT/${name}_$i.log" 2>&1
    rc=$?
    [ $rc -ne 0 ] && fails=$((fails+1))
    echo "$name run $i rc=$rc $(grep -c 'watchdog' $OUT/${name}_$i.log) watchdog-lines $(grep RESULT $OUT/${name}_$i.log | head -c 300)"
  done
  echo "$name: $fails / $RUNS runs failed"
done
