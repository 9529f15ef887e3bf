"""Summarise a tools/profile_round.sh output directory into profiles/*.md.

    python tools/ncu_summary.py gpurun_out/prof_<tag>_<cfg> <tag> <cfg>

Writes profiles/<tag>_launches_<cfg>.md (+ the raw csv) and
profiles/<tag>_ncu_full_<cfg>.md, and records each kernel's per-launch DRAM
bytes in profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]

SHORT = {
    "mha_fwd_sm100_kernel": "fwd",
    "mha_bwd_dkdv_kernel": "bwd_dkdv",
    "mha_bwd_dq_kernel": "bwd_dq",
    "mha_bwd_dq_gemm_kernel": "bwd_dq_gemm",
    "mha_bwd_dq_tail_kernel": "bwd_dq_gemm",  # the persistent dQ GEMM (same role)
    "mha_bwd_preprocess_kernel": "bwd_preprocess",
}


def raw(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    return {n: (u, v) for n, u, v in zip(rows[0], rows[1], rows[2])}


def to_bytes(unit: str, v: str) -> float:
    x = float(v)
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def stalls(rep: str, top: int = 6) -> list:
    """Top warp-stall reasons over the whole kernel (source page, summed)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next((i for i, r in enumerate(rows) if "Address" in r or "Source" in r), None)
    if hdr_i is None:
        return []
    hdr = rows[hdr_i]
    cols = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
    tot = {}
    for r in rows[hdr_i + 1:]:
        for i in cols:
            try:
                tot[hdr[i]] = tot.get(hdr[i], 0) + int(r[i] or 0)
            except (ValueError, IndexError):
                pass
    s = sum(tot.values()) or 1
    return [(k[6:], v / s) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]]


def launches(path: str) -> list:
    text = open(path).read()
    lines = text[text.index('"ID"'):] if '"ID"' in text else text
    rows = list(csv.DictReader(io.StringIO(lines)))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        t = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        t_ms = t * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "nsecond": 1e-6}.get(unit, 1e-6)
        a = agg.setdefault(r["Kernel Name"].split("(")[0].strip(), [0, 0.0])
        a[0] += 1
        a[1] += t_ms
    return [(k, n, t) for k, (n, t) in agg.items()]


def main():
    d, tag, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
    prof = os.environ.get("VATTN_PROFILES_DIR", os.path.join(ROOT, "profiles"))  # (gpurun: a dir under gpurun_out)
    os.makedirs(prof, exist_ok=True)
    gpu = open(os.path.join(d, "gpu.txt")).read().strip().splitlines()[-1] if os.path.exists(os.path.join(d, "gpu.txt")) else ""
    # ---- launch list
    lp = os.path.join(d, "launches.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(prof, f"{tag}_launches_{cfg}.csv"))
        ls = launches(lp)
        tot = sum(t for _, _, t in ls) or 1
        with open(os.path.join(prof, f"{tag}_launches_{cfg}.md"), "w") as f:
            f.write(f"# {tag} launch list (ncu --metrics gpu__time_duration.sum --clock-control none), config {cfg}\n\n")
            f.write("Command: `python bench.py --config %s --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0`.\n" % cfg)
            f.write("Cold-cache, serialised launches -- compare SHARES, not absolutes.  GPU: %s\n\n" % gpu)
            f.write("| kernel | launches | mean ms | share |\n|---|---|---|---|\n")
            for k, n, t in ls:
                f.write(f"| `{k}` | {n} | {t / n:.3f} | {100 * t / tot:.1f}% |\n")
    # ---- full captures
    traffic_path = os.path.join(prof, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    tcfg = traffic.setdefault(cfg, {})
    with open(os.path.join(prof, f"{tag}_ncu_full_{cfg}.md"), "w") as f:
        f.write(f"# {tag} ncu --set full summaries (one launch each after 3 warm-up steps), config {cfg}\n\n")
        f.write("`ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 3 -c 1` "
                "(tools/profile_round.sh).  GPU: %s\n" % gpu)
        for k, short in SHORT.items():
            rep = os.path.join(d, f"{k}.ncu-rep")
            if not os.path.exists(rep):
                continue
            m = raw(rep)
            f.write(f"\n## {k}\n\n")
            for name in METRICS:
                if name in m:
                    u, v = m[name]
                    f.write(f"- `{name}` = {v} {u}\n")
            try:
                rb = to_bytes(*m["dram__bytes_read.sum"])
                wb = to_bytes(*m["dram__bytes_write.sum"])
                tcfg[f"{short}_dram_bytes"] = rb + wb
                f.write(f"- DRAM read+write per launch = {(rb + wb) / 1e6:.1f} MB\n")
            except (KeyError, ValueError):
                pass
            st = stalls(rep)
            if st:
                f.write("- top warp-stall reasons (share of samples): " +
                        ", ".join(f"{n} {100 * s:.1f}%" for n, s in st) + "\n")
    tcfg["source"] = f"profiles/{tag}_ncu_full_{cfg}.md (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch)"
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
