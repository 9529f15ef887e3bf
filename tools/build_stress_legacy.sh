#!/usr/bin/env bash
# Rebuild the round-1 barrier protocol under the schedule fuzzer, for the hang
# root-cause record: a copy of csrc/ with the two per-step-parity
# barrier pairs folded back into one barrier each --
#   dK/dV  p_full[s & 1][h][half] -> p_full[h][half]   (parity s & 1)
#   dQ     ds_full[j & 1]   -> ds_full          (parity j & 1)
# -> tools/variants/stress_legacy.so (load with VATTN_LIB=...).  Never shipped.
set -e
cd "$(dirname "$0")/.."
T=$(mktemp -d)
mkdir -p "$T/paper_2502_12784_b200" tools/variants
cp -r paper_2502_12784_b200/csrc "$T/paper_2502_12784_b200/"
cp -r include "$T/"
python - "$T/paper_2502_12784_b200/csrc/mha_bwd_sm100.cuh" <<'EOF'
import sys
p = sys.argv[1]
s = open(p).read()
subs = [
    ("p_full + kWG * kHv * (s & 1), (s >> 1) & 1,", "p_full, s & 1,", 2),
    ("mbar_arrive(p_full + kWG * kHv * (s & 1) + kHv * h + half)", "mbar_arrive(p_full + kHv * h + half)", 1),
    ("mbar_wait_mma(ds_full + (j & 1), (j >> 1) & 1)", "mbar_wait_mma(ds_full, j & 1)", 1),
    ("mbar_arrive(ds_full + (j & 1))", "mbar_arrive(ds_full)", 1),
]
for a, b, n in subs:
    assert s.count(a) == n, (a, s.count(a))
    s = s.replace(a, b)
open(p, "w").write(s)
EOF
SRC=$T/paper_2502_12784_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -cudart static \
     --expt-relaxed-constexpr -DVATTN_STRESS_NS=20000 -DVATTN_WATCHDOG_NS=4000000000ull -DVATTN_WATCHDOG_PRINT \
     -shared $SRC/capi.cu $SRC/capi_host.cu -o tools/variants/stress_legacy.so
rm -rf "$T"
ls -la tools/variants/stress_legacy.so
