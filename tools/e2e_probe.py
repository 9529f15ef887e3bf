"""e2e (host-buffer mha_step_host) timing only (diagnostic): python tools/e2e_probe.py [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_12784_b200 as vb
from bench import flops
B, H, N, d, causal = 4, 16, 8192, 128, True
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
shape = (B, H, N, d)
hq, hk, hv, hdo = (torch.randn(shape).to(torch.bfloat16).pin_memory() for _ in range(4))
ho, hdq, hdk, hdv = (torch.empty(shape, dtype=torch.bfloat16).pin_memory() for _ in range(4))
hlse = torch.empty((B, H, N), dtype=torch.float32).pin_memory()
step = lambda: vb.mha_step_host(hq, hk, hv, hdo, causal, out=(ho, hlse, hdq, hdk, hdv))
step(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps): step()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
ff, fb = flops(B, H, N, d, causal)
print(f"e2e RAMP={os.environ.get('VATTN_HOST_RAMP','1')} SLABS={os.environ.get('VATTN_HOST_SLABS','auto')}: {ms:.2f} ms/step {(ff+fb)/ms/1e9:.0f} TF", flush=True)
