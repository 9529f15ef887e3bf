"""the reference's closed-form HBM traffic against ncu DRAM bytes.

    python tools/traffic_crosscheck.py [profiles/ncu_traffic.json] > profiles/<tag>_traffic_crosscheck.md

For each B200 kernel of C3 (BASELINE configs[2]) it prints the measured
`dram__bytes_read.sum + dram__bytes_write.sum` (one ncu --set full launch) beside the
two caching extremes of paper_2502_12784_b200.traffic.b200_hbm_model: every tensor
once (L2 absorbs all re-reads; the algorithmic bytes) and the reference's cache-less
closed form (attention.hpp:40-58, every visited tile pair re-reads its tiles).  It
also restates the reference's own element counts for the whole pass
(forward_fused_traffic / backward_fused_traffic, tile 128 x 128) in bytes.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_12784_b200 import traffic as tr  # noqa: E402


class Cfg:
    batch, heads, seq_len, head_dim, tile_rows, tile_cols, causal, acc_mode = 4, 16, 8192, 128, 128, 128, True, "fp32"


KEYS = {"fwd": "fwd_dram_bytes", "bwd_preprocess": "bwd_preprocess_dram_bytes", "bwd_dkdv": "bwd_dkdv_dram_bytes",
        "bwd_dq_gemm": "bwd_dq_gemm_dram_bytes"}


def rows(measured: dict):
    model = tr.b200_hbm_model(Cfg)
    out = []
    for k, m in model.items():
        got = measured.get(KEYS[k])
        out.append((k, m["l2_reuse"], m["cache_less"], got))
    return out


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "ncu_traffic.json")
    meas = json.load(open(path))["c3"]
    print("# SURVEY 8(f4): closed-form HBM traffic vs ncu DRAM bytes, C3 (4,16,8192,128) causal bf16\n")
    print(f"Measured: `{path}` ({meas.get('source', '')}).  Model: `traffic.b200_hbm_model` "
          "(bytes; 16-bit tensors 2 B, lse / D 4 B).\n")
    print("| kernel | every tensor once (L2 reuse) | reference closed form (cache-less) | ncu measured | measured / once | measured / cache-less |")
    print("|---|---|---|---|---|---|")
    tot = [0, 0, 0]
    for k, lo, hi, got in rows(meas):
        tot[0] += lo
        tot[1] += hi
        tot[2] += got or 0
        g = f"{got / 1e9:.3f} GB" if got else "n/a"
        print(f"| `{k}` | {lo / 1e9:.3f} GB | {hi / 1e9:.3f} GB | {g} | "
              f"{(got / lo if got else float('nan')):.3f} | {(got / hi if got else float('nan')):.3f} |")
    print(f"| **step** | {tot[0] / 1e9:.3f} GB | {tot[1] / 1e9:.3f} GB | {tot[2] / 1e9:.3f} GB | {tot[2] / tot[0]:.3f} | {tot[2] / tot[1]:.3f} |")
    ff, fb = tr.forward_fused_traffic(Cfg), tr.backward_fused_traffic(Cfg)
    print("\nThe reference's own TrafficCounter for the same config (element counts x 2 B; its backward "
          "re-runs the forward and reduce-adds fp32 dQ partials per tile pair):\n")
    print(f"- forward_fused: {ff.element_reads} element reads + {ff.element_writes} writes = "
          f"{2 * (ff.element_reads + ff.element_writes) / 1e9:.2f} GB")
    print(f"- backward_fused: {fb.element_reads} element reads + {fb.element_writes} writes = "
          f"{2 * (fb.element_reads + fb.element_writes) / 1e9:.2f} GB")
    print("\nReading: each kernel's measured bytes are at least its 'every tensor once' figure "
          "(the preprocess has nothing to re-read, so its two extremes coincide; the +1 % is ncu's "
          "sector granularity) and far below the reference's cache-less closed form.  The dK/dV "
          "kernel and the dQ GEMM are within 1 % of 'once': the 126 MB L2 absorbs every K/V and "
          "Q/dO re-read the reference's model charges to HBM, and their bytes are the dS^T round "
          "trip (the design's price for atomic-free deterministic dQ, DESIGN 2.2).  The forward is "
          "1.3x 'once': under longest-first grouping some K/V tiles are evicted before the last "
          "query block of a unit reads them (DESIGN 5, dispatch order).")

if __name__ == "__main__":
    main()
