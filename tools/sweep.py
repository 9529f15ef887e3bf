"""Throughput over every BASELINE.json config on one B200 (bench.py's C3 line is the
number of record; this is the supporting table).

    python tools/sweep.py [--steps 10] [--tag r1] [--out profiles]

configs[0] C1 (1,2,128,64) fp16 non-causal       -- launch-bound, parity shape
configs[1] C2 16k tokens, H=32, d=64, N=512..16k  -- non-causal fp16
configs[2] C3 (4,16,8192,128) causal bf16         -- north_star target (+ fp16, non-causal)
configs[3] C4 GPT-2-medium attention: (8,16,1024,64) x 24 layers, causal fp16: one step =
           24 forward then 24 backward (reverse order) on per-layer tensors, captured
           once as a CUDA graph and replayed (plus the eager time for comparison)
configs[4] C5 (1,64,32768,128) causal bf16 on one GPU (8 GPUs shard (b,h): 8 heads each)

Timing: CUDA events on the launching stream after 3 warm-up steps; inputs are
> L2 except C1/C4 per layer (C4's 24 layers together are ~1.5 GB).  TFLOPS use the
algorithmic count 14 B H N^2 d c (c = 1/2 causal).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2502_12784_b200 as vb  # noqa: E402
from bench import flops, measured_peaks  # noqa: E402

CONFIGS = [
    ("C1", 1, 2, 128, 64, False, torch.float16),
    ("C2 N=512", 32, 32, 512, 64, False, torch.float16),
    ("C2 N=1k", 16, 32, 1024, 64, False, torch.float16),
    ("C2 N=2k", 8, 32, 2048, 64, False, torch.float16),
    ("C2 N=4k", 4, 32, 4096, 64, False, torch.float16),
    ("C2 N=8k", 2, 32, 8192, 64, False, torch.float16),
    ("C2 N=16k", 1, 32, 16384, 64, False, torch.float16),
    ("C3", 4, 16, 8192, 128, True, torch.bfloat16),
    ("C3 fp16", 4, 16, 8192, 128, True, torch.float16),
    ("C3 non-causal", 4, 16, 8192, 128, False, torch.bfloat16),
    ("C5 (1 GPU)", 1, 64, 32768, 128, True, torch.bfloat16),
]


def kernel_ms():
    out = []
    for kind in (0, 1, 2):
        t, n = C.c_double(), C.c_int()
        vb.lib.vattn_profile_read(kind, C.byref(t), C.byref(n))
        out.append(t.value / max(n.value, 1))
    return out


def run_one(name, B, H, N, d, causal, dtype, steps):
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    q, k, v, do = (torch.randn((B, H, N, d), generator=g, device="cuda").to(dtype) for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty((B, H, N), device="cuda")
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    ws = torch.empty(vb.workspace_bytes(B, H, N, d, causal, dtype), dtype=torch.uint8, device="cuda")

    def step():
        vb.mha_forward(q, k, v, causal, out=o, lse=lse)
        vb.mha_backward(q, k, v, o, do, lse, causal, dq=dq, dk=dk, dv=dv, workspace=ws)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    vb.lib.vattn_profile_enable(1)  # per-kernel times from a separate profiled pass
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    fwd, dkdv, dqk = kernel_ms()
    vb.lib.vattn_profile_enable(0)
    ff, fb = flops(B, H, N, d, causal)
    return dict(config=name, shape=[B, H, N, d], causal=causal, dtype=str(dtype).split(".")[-1], ms=ms,
                tflops=(ff + fb) / ms / 1e9, fwd_ms=fwd, fwd_tflops=ff / fwd / 1e9, bwd_ms=ms - fwd,
                bwd_tflops=fb / (ms - fwd) / 1e9, dkdv_ms=dkdv, dq_ms=dqk)


def run_traditional(name, B, H, N, d, causal, dtype, steps):
    """The unfused three-pass forward (comparator) vs the fused forward."""
    from paper_2502_12784_b200 import traditional as tr
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    q, k, v = (torch.randn((B, H, N, d), generator=g, device="cuda").to(dtype) for _ in range(3))
    ws = torch.empty(tr.workspace_bytes(q, causal), dtype=torch.uint8, device="cuda")
    o = torch.empty_like(q)
    lse = torch.empty((B, H, N), device="cuda")

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    t_trad = timeit(lambda: tr.forward_traditional(q, k, v, causal, workspace=ws))
    t_fused = timeit(lambda: vb.mha_forward(q, k, v, causal, out=o, lse=lse))
    ff, _ = flops(B, H, N, d, causal)
    return dict(config=f"{name} forward: traditional vs fused", shape=[B, H, N, d], causal=causal,
                dtype=str(dtype).split(".")[-1], traditional_ms=t_trad, fused_ms=t_fused,
                speedup=t_trad / t_fused, traditional_tflops=ff / t_trad / 1e9, fused_tflops=ff / t_fused / 1e9,
                traditional_workspace_gb=ws.numel() / 1e9)


def run_c4(steps, layers=24):
    B, H, N, d, causal, dtype = 8, 16, 1024, 64, True, torch.float16
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    L = []
    for _ in range(layers):
        q, k, v, do = (torch.randn((B, H, N, d), generator=g, device="cuda").to(dtype) for _ in range(4))
        L.append(dict(q=q, k=k, v=v, do=do, o=torch.empty_like(q), lse=torch.empty((B, H, N), device="cuda"),
                      dq=torch.empty_like(q), dk=torch.empty_like(q), dv=torch.empty_like(q)))
    ws = torch.empty(vb.workspace_bytes(B, H, N, d, causal, dtype), dtype=torch.uint8, device="cuda")

    def step():
        for x in L:  # forward through the 24 layers
            vb.mha_forward(x["q"], x["k"], x["v"], causal, out=x["o"], lse=x["lse"])
        for x in reversed(L):  # backward in reverse layer order
            vb.mha_backward(x["q"], x["k"], x["v"], x["o"], x["do"], x["lse"], causal,
                            dq=x["dq"], dk=x["dk"], dv=x["dv"], workspace=ws)

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    eager = timeit(step)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        step()  # warm (attributes, descriptors) outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            step()
    torch.cuda.current_stream().wait_stream(s)
    graphed = timeit(graph.replay)
    ff, fb = flops(B, H, N, d, causal)
    tot = layers * (ff + fb)
    return dict(config=f"C4 GPT-2-medium x{layers} layers (CUDA graph)", shape=[B, H, N, d], causal=causal,
                dtype="float16", ms=graphed, tflops=tot / graphed / 1e9, eager_ms=eager,
                eager_tflops=tot / eager / 1e9, launches_per_step=layers * 4)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    args = ap.parse_args()
    burst, sust, src = measured_peaks()
    rows = []
    for cfg in CONFIGS:
        time.sleep(2)  # let clocks / power recover so the row does not inherit the previous row's state
        r = run_one(*cfg, steps=args.steps if cfg[0] != "C5 (1 GPU)" else max(2, args.steps // 4))
        rows.append(r)
        print(json.dumps(r), flush=True)
    r = run_c4(args.steps)
    rows.append(r)
    print(json.dumps(r), flush=True)
    trad = []
    for cfg in [c for c in CONFIGS if c[0] in ("C2 N=1k", "C2 N=4k", "C3", "C3 non-causal")]:
        t = run_traditional(*cfg, steps=max(2, args.steps // 2))
        trad.append(t)
        print(json.dumps(t), flush=True)
    name = torch.cuda.get_device_name()
    os.makedirs(args.out, exist_ok=True)
    with open(os.path.join(args.out, f"{args.tag}_sweep.json"), "w") as f:
        json.dump({"gpu": name, "peak_bf16_tflops": {"burst": burst, "sustained": sust, "source": src},
                   "rows": rows, "traditional_vs_fused": trad}, f, indent=1)
    with open(os.path.join(args.out, f"{args.tag}_sweep.md"), "w") as f:
        f.write(f"# {args.tag} throughput sweep over BASELINE.json configs ({name}, 1 GPU)\n\n")
        f.write("`python tools/sweep.py` -- CUDA events, 3 warm-up steps, 2 s idle before each config; TFLOPS = algorithmic "
                "14 B H N^2 d c / step time; % of the measured sustained bf16 peak "
                f"({sust} TF/s, MEASURED_PEAKS.json).\n\n")
        f.write("| config | shape (B,H,N,d) | causal | dtype | step ms | TFLOPS | % peak | fwd TFLOPS | bwd TFLOPS |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['config']} | {tuple(r['shape'])} | {r['causal']} | {r['dtype']} | {r['ms']:.3f} | "
                    f"{r['tflops']:.0f} | {100 * r['tflops'] / sust:.0f}% | "
                    f"{r.get('fwd_tflops', float('nan')):.0f} | {r.get('bwd_tflops', float('nan')):.0f} |\n")
        c4 = rows[-1]
        f.write(f"\nC4 eager (no graph): {c4['eager_ms']:.3f} ms per 24-layer step = {c4['eager_tflops']:.0f} TFLOPS; "
                f"graph replay {c4['ms']:.3f} ms = {c4['tflops']:.0f} TFLOPS ({c4['launches_per_step']} kernels).\n")
        f.write("\n## Fused vs traditional forward (the paper's comparison, SURVEY 8f-3)\n\n"
                "Traditional = `mha_forward_traditional` (S = QK^T in binary32 via cuBLAS, full-row softmax "
                "kernel, O = PV via cuBLAS; every key tile computed and masked, as the reference's "
                "`forward_traditional`).  TFLOPS use the same algorithmic count for both.\n\n"
                "| config | traditional ms | fused ms | speedup | traditional TFLOPS | fused TFLOPS | S+P workspace GB |\n"
                "|---|---|---|---|---|---|---|\n")
        for t in trad:
            f.write(f"| {t['config']} | {t['traditional_ms']:.3f} | {t['fused_ms']:.3f} | {t['speedup']:.1f}x | "
                    f"{t['traditional_tflops']:.0f} | {t['fused_tflops']:.0f} | {t['traditional_workspace_gb']:.1f} |\n")


if __name__ == "__main__":
    main()
