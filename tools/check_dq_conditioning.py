"""Why tiny-N dQ misses the binary64 bound (tools/gpu_fuzz.sh seeds 1026/1056/1078/1139):
compare the GPU dQ with (a) exact binary64 math and (b) the same math with D formed from
the 16-bit O, as the reference's compute_dpsum (attention_backward.cpp:44-57) does."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_12784_b200 as vb  # noqa: E402
from tests.gpu_util import workload  # noqa: E402
from tests.test_random_gpu import _case  # noqa: E402


def grads(q, k, v, do, causal, scale, o16=None):
    q, k, v, do = (x.double() for x in (q, k, v, do))
    N = q.shape[2]
    s = q @ k.transpose(-1, -2) * scale
    if causal:
        s = s.masked_fill(torch.ones(N, N, dtype=torch.bool).triu(1), float("-inf"))
    p = torch.softmax(s, -1)
    o = p @ v
    dp = do @ v.transpose(-1, -2)
    D = (do * (o if o16 is None else o16.double())).sum(-1, keepdim=True)
    ds = p * (dp - D) * scale
    return ds @ k


for seed in (1026, 1056, 1078, 1139):
    c = _case(seed)
    if c["p"] > 0:
        continue  # dropout cases: same mechanism, the keep bits only change P
    B, H, N, d = c["B"], c["H"], c["N"], c["d"]
    q, k, v, do = workload(seed, (B, H, N, d), c["dtype"])
    scale = c["scale"] if c["scale"] > 0 else d ** -0.5
    cfg = vb.AttnConfig(batch=B, heads=H, seq_len=N, head_dim=d, causal=c["causal"], softmax_scale=c["scale"])
    o, lse = vb.forward_fused(q, k, v, cfg)
    dq, _, _ = vb.backward_fused(q, k, v, do, lse, cfg, out=o)
    qc, kc, vc, doc = (x.cpu() for x in (q, k, v, do))
    exact = grads(qc, kc, vc, doc, c["causal"], scale)
    algo = grads(qc, kc, vc, doc, c["causal"], scale, o16=o.cpu())
    rel = lambda a, b: float((a.double() - b).norm() / b.norm())  # noqa: E731
    print(f"seed {seed} {c}: dQ fro_rel vs exact {rel(dq.cpu(), exact):.2e}, vs D-from-16-bit-O {rel(dq.cpu(), algo):.2e},"
          f" exact vs D-from-16-bit-O {rel(algo, exact):.2e}")
