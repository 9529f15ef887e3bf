#!/usr/bin/env bash
# Rebuild the round-1 barrier protocol under the schedule fuzzer, for the hang
# root-cause record: a copy of csrc/ with the two per-step-parity
# barrier pairs folded back into one barrier each --
#   dK/dV  p_full[g & 1][h][half] -> p_full[h][half]   (parity g & 1; g = the CTA's
#          step counter across its items)
#   dQ     ds_full[j & 1]   -> ds_full          (parity j & 1)
# -> tools/variants/stress_legacy.so (load with VATTN_LIB=...).  Never shipped.
# The patterns follow the current source; the build fails loudly if one stops matching.
set -e
cd "$(dirname "$0")/.."
T=$(mktemp -d)
mkdir -p "$T/paper_2502_12784_b200" tools/variants
cp -r paper_2502_12784_b200/csrc "$T/paper_2502_12784_b200/"
cp -r include "$T/"
python - "$T/paper_2502_12784_b200/csrc/mha_bwd_sm100.cuh" <<'PYEOF'
import re
import sys
p = sys.argv[1]
s = open(p).read()
subs = [  # (regex, replacement, expected count)
    (r"p_full \+ kWG \* kHv \* \(g & 1u\),\s*\(g >> 1\) & 1,", "p_full, g & 1,", 2),
    (r"arrive_mma\(p_full \+ kWG \* kHv \* \(g & 1u\) \+ kHv \* h \+ half\)", "arrive_mma(p_full + kHv * h + half)", 1),
    (r"mbar_wait_mma\(ds_full \+ \(j & 1\), \(j >> 1\) & 1\)", "mbar_wait_mma(ds_full, j & 1)", 1),
    (r"mbar_arrive\(ds_full \+ \(j & 1\)\)", "mbar_arrive(ds_full)", 1),
]
for a, b, n in subs:
    s, k = re.subn(a, b, s)
    assert k == n, (a, k)
open(p, "w").write(s)
PYEOF
SRC=$T/paper_2502_12784_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -cudart static \
     --expt-relaxed-constexpr -DVATTN_STRESS_NS=20000 -DVATTN_WATCHDOG_NS=4000000000ull -DVATTN_WATCHDOG_PRINT \
     -shared $SRC/capi.cu $SRC/capi_host.cu -o tools/variants/stress_legacy.so
rm -rf "$T"
ls -la tools/variants/stress_legacy.so
