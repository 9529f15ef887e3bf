"""Forward-only TFLOPS over shapes (diagnostic): python tools/fwd_scan.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_12784_b200 as vb

SHAPES = [(4, 16, 8192, 128, True), (4, 16, 8192, 128, False), (4, 16, 4096, 128, False),
          (8, 16, 4096, 128, False), (4, 16, 2048, 128, False), (16, 16, 2048, 128, False),
          (4, 16, 16384, 128, True), (8, 16, 8192, 128, True), (2, 16, 8192, 128, True),
          (4, 16, 8192, 64, True), (4, 16, 8192, 64, False)]
if len(sys.argv) > 1:
    SHAPES = [tuple(json.loads(s)) for s in sys.argv[1:]]
for B, H, N, d, causal in SHAPES:
    DT = torch.float16 if os.environ.get("DT") == "fp16" else torch.bfloat16
    q, k, v = (torch.randn((B, H, N, d), device="cuda").to(DT) for _ in range(3))
    o = torch.empty_like(q); lse = torch.empty((B, H, N), device="cuda")
    f = lambda: vb.mha_forward(q, k, v, causal, out=o, lse=lse)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    fl = 4 * B * H * N * N * d * (0.5 if causal else 1.0)
    ctas = B * H * ((N + 255) // 256)
    print(f"B{B} H{H} N{N} d{d} causal={int(causal)} ctas={ctas} ctas/SM={ctas/148:.1f} fwd {ms:.3f} ms {fl/ms/1e9:.0f} TF", flush=True)
