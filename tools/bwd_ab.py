"""Backward-only timing (diagnostic A/B of library variants via VATTN_LIB):
python tools/bwd_ab.py [B H N d causal] -> ms per mha_backward (CUDA events, 40 launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_12784_b200 as vb
from bench import flops
B, H, N, d, causal = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (4, 16, 8192, 128, 1)
P = float(os.environ.get("DROP", "0"))
DT = torch.float16 if os.environ.get("DT") == "fp16" else torch.bfloat16
q, k, v, do = (torch.randn((B, H, N, d), device="cuda").to(DT) for _ in range(4))
o, lse = vb.mha_forward(q, k, v, bool(causal), dropout_p=P, seed=5)
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
ws = torch.empty(vb.workspace_bytes(B, H, N, d, bool(causal), DT), dtype=torch.uint8, device="cuda")
f = lambda: vb.mha_backward(q, k, v, o, do, lse, bool(causal), dq=dq, dk=dk, dv=dv, workspace=ws, dropout_p=P, seed=5)
for _ in range(3): f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(40): f()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 40
print(f"{os.path.basename(os.environ.get('VATTN_LIB', 'default'))}: bwd {ms:.3f} ms {flops(B, H, N, d, bool(causal))[1] / ms / 1e9:.0f} TF", flush=True)
