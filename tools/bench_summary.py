"""Print one bench.py JSON line compactly: python tools/bench_summary.py <file> [label]"""
import json
import sys

d = json.load(open(sys.argv[1]))
label = sys.argv[2] if len(sys.argv) > 2 else ""
k = {a: round(b, 3) for a, b in d.get("kernels_ms", {}).items() if a != "note"}
print(label, round(d["value"], 1), round(d["ms_per_step"], 3), d.get("clocks", {}).get("sm_mhz"), k)
