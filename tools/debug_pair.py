"""Debug aid: one fwd+bwd per shape in its own process, dQ/dK/dV vs a torch fp32 reference.
    python tools/debug_pair.py  B,H,N,d,causal[,bf16] ...
"""
import os
import subprocess
import sys

CHILD = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch
import paper_2502_12784_b200 as vb
B, H, N, d, causal = (int(x) for x in sys.argv[1].split(",")[:5])
dt = torch.bfloat16 if sys.argv[1].endswith("bf16") else torch.float16
g = torch.Generator(device="cuda"); g.manual_seed(0)
q, k, v, do = (torch.randn(B, H, N, d, generator=g, device="cuda").to(dt) for _ in range(4))
o, lse = vb.mha_forward(q, k, v, bool(causal))
dq, dk, dv = vb.mha_backward(q, k, v, o, do, lse, bool(causal))
torch.cuda.synchronize()
qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
s = qf @ kf.transpose(-1, -2) / d ** 0.5
if causal:
    s = s.masked_fill(torch.ones(N, N, device="cuda", dtype=torch.bool).triu(1), float("-inf"))
of = torch.softmax(s, -1) @ vf
of.backward(do.float())
def rel(a, b):
    return ((a.float() - b).norm() / b.norm()).item()
print(f"{sys.argv[1]}: o {rel(o, of.detach()):.2e} dq {rel(dq, qf.grad):.2e} dk {rel(dk, kf.grad):.2e} dv {rel(dv, vf.grad):.2e}", flush=True)
'''

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for case in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", CHILD, case], env=dict(os.environ, ROOT=root), capture_output=True, text=True,
                       timeout=120)
    out = (r.stdout + r.stderr).strip().splitlines()
    keep = [l for l in out if "watchdog" in l or ": o " in l or "Error" in l]
    print(f"[{case}] rc={r.returncode}", *keep[:12], sep="\n  ", flush=True)
