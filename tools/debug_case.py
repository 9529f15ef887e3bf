import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_12784_b200 as vb
B, H, N, d, causal = (int(x) for x in sys.argv[1:6])
dt = torch.bfloat16 if len(sys.argv) > 6 and sys.argv[6] == "bf16" else torch.float16
q, k, v, do = (torch.randn(B, H, N, d, device="cuda").to(dt) for _ in range(4))
o, lse = vb.mha_forward(q, k, v, bool(causal))
torch.cuda.synchronize()
print("fwd ok", flush=True)
dq, dk, dv = vb.mha_backward(q, k, v, o, do, lse, bool(causal))
torch.cuda.synchronize()
print("bwd ok", flush=True)
