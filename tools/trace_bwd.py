"""Timeline of one backward CTA (debug build tools/libvattn_b200_trace.so).

usage: python tools/trace_bwd.py B H N d causal item
Prints, per query-tile step, the clock64 deltas between pipeline events.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_12784_b200 as vb  # noqa: E402  (for the config struct)

lib = C.CDLL(os.path.join(ROOT, "tools", "libvattn_b200_trace.so"))
B, H, N, d, causal, item = (int(x) for x in sys.argv[1:7])
dt = torch.bfloat16
q, k, v, do = (torch.randn(B, H, N, d, device="cuda").to(dt) for _ in range(4))
o = torch.empty_like(q)
lse = torch.empty(B, H, N, device="cuda")
cfg = vb._Cfg(B, H, N, d, causal, 0.0, 1)
vp = C.c_void_p
lib.mha_forward.argtypes = [C.POINTER(vb._Cfg)] + [vp] * 6
lib.mha_backward.argtypes = [C.POINTER(vb._Cfg)] + [vp] * 10 + [C.c_size_t, vp]
lib.mha_backward_workspace_bytes.argtypes = [C.POINTER(vb._Cfg)]
lib.mha_backward_workspace_bytes.restype = C.c_size_t
ws = torch.empty(lib.mha_backward_workspace_bytes(C.byref(cfg)), dtype=torch.uint8, device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
s = torch.cuda.current_stream().cuda_stream
assert lib.mha_forward(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), s) == 0


def bwd():
    assert lib.mha_backward(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
                            lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws.numel(), s) == 0


for _ in range(3):
    bwd()
torch.cuda.synchronize()
lib.vattn_trace_select(item)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
bwd()
e1.record()
torch.cuda.synchronize()
print(f"bwd total {e0.elapsed_time(e1):.3f} ms")
buf = (C.c_longlong * 4096)()
lib.vattn_trace_read(buf, 4096)
t = np.array(buf[:], dtype=np.int64)
t0 = t[3072]
n_q = (N + 127) // 128
kb = item % n_q
steps = (n_q - kb) if causal else n_q
print(f"item {item} kb {kb} steps {steps}; cycles relative to CTA start")
names_m = ["p_full", "dq_empty", "q_next", "ds_full", "dQ_iss"]
names_s = ["s_full", "P_done", "dp_full", "ds_free", "dS_done"]
names_q = ["sem_ok", "dq_full", "written", "released"]
print("step | MMA: " + " ".join(f"{x:>8}" for x in names_m) + " | dS: " + " ".join(f"{x:>8}" for x in names_s) +
      " | dQ: " + " ".join(f"{x:>8}" for x in names_q))
prev = None
for st in range(steps):
    m = [t[8 * st + j] - t0 if t[8 * st + j] else -1 for j in range(5)]
    sx = [t[1024 + 8 * st + j] - t0 if t[1024 + 8 * st + j] else -1 for j in range(5)]
    qx = [t[2048 + 8 * st + j] - t0 if t[2048 + 8 * st + j] else -1 for j in range(4)]
    print(f"{st:4d} | " + " ".join(f"{x:8d}" for x in m) + " | " + " ".join(f"{x:8d}" for x in sx) + " | " +
          " ".join(f"{x:8d}" for x in qx))
