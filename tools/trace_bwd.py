"""Timelines of one CTA of each kernel (debug build tools/libvattn_b200_trace.so).

usage: python tools/trace_bwd.py B H N d causal [block]
Prints per-iteration clock64 stamps (relative to the MMA loop start) for the
forward, dK/dV and dQ kernels of the same problem.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_12784_b200 as vb  # noqa: E402  (config struct only)

lib = C.CDLL(os.environ.get("VATTN_TRACE_LIB") or os.path.join(ROOT, "tools", "libvattn_b200_trace.so"))
B, H, N, d, causal = (int(x) for x in sys.argv[1:6])
block = int(sys.argv[6]) if len(sys.argv) > 6 else 0
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


def fwd():
    assert lib.mha_forward(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), s) == 0


def bwd():
    assert lib.mha_backward(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
                            lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws.numel(), s) == 0


for _ in range(3):
    fwd()
    bwd()
torch.cuda.synchronize()


def trace(kid, fn):
    lib.vattn_trace_select(kid, block)
    fn()
    torch.cuda.synchronize()
    buf = (C.c_longlong * 4096)()
    lib.vattn_trace_read(buf, 4096)
    return np.array(buf[:], dtype=np.int64)


def show(t, names_m, names_w, n_iter, width):
    t0 = t[3072]
    print("iter | MMA: " + " ".join(f"{x:>9}" for x in names_m) + " | WG: " + " ".join(f"{x:>9}" for x in names_w) + " | dt")
    prev = None
    for it in range(n_iter):
        m = [t[width * it + j] - t0 if t[width * it + j] else -1 for j in range(len(names_m))]
        w = [t[1024 + width * it + j] - t0 if t[1024 + width * it + j] else -1 for j in range(len(names_w))]
        dtv = (m[0] - prev) if prev is not None and m[0] >= 0 else 0
        prev = m[0] if m[0] >= 0 else prev
        print(f"{it:4d} | " + " ".join(f"{x:9d}" for x in m) + " | " + " ".join(f"{x:9d}" for x in w) + f" | {dtv}")


n_q = (N + 127) // 128
if "dq" not in sys.argv:
    print(f"== forward, block {block}")
    t = trace(0, fwd)
    t0 = t[3072]
    print("iter | MMA pv0_issued s0_issued pv1_issued s1_issued | tile0: s0 +ld +max +resc +q0 +q1 +q2 +q3 | tile1: s1 ... | dt")
    prev = None
    for it in range(min(n_q, 24)):
        m = [t[8 * it + k] - t0 for k in (0, 1, 4, 5)]
        rows = []
        for tt in range(2):
            s0 = t[1024 + 8 * it + 4 * tt]
            rel = [t[2048 + 8 * it + 4 * tt + k] - s0 for k in range(3)] + \
                  [t[1024 + 8 * it + 4 * tt + k] - s0 for k in (1, 2, 3)] + [t[2048 + 8 * it + 4 * tt + 3] - s0]
            rows.append(f"{s0 - t0:7d} " + " ".join(f"{x:5d}" for x in rel))
        dtv = m[0] - prev if prev is not None else 0
        prev = m[0]
        print(f"{it:3d} | " + " ".join(f"{x:7d}" for x in m) + " | " + " | ".join(rows) + f" | {dtv}")
    print(f"== dK/dV, block {block}")
    t = trace(1, bwd)
    show(t, ["p_full", "S_next", "ds_full"], ["s_full", "P_done", "dp_full", "dS_done", "s_full1", "P_done1", "dp_full1", "dS_done1"], min(n_q, 24), 8)
print(f"== dQ, block {block}")
t = trace(2, bwd)
show(t, ["ds_full", "v_next", "k_next2", "dQ_iss", "commit", "dP_iss", "S_iss"], ["s_full", "P_done", "dp_full", "dS_done"], min(n_q, 24), 8)
