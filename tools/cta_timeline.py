"""Per-CTA timelines of the hot kernels (debug build tools/libvattn_b200_trace.so):
SM-busy fraction, gaps between consecutive CTAs on one SM, head and tail idle.

usage: python tools/cta_timeline.py [B H N d causal]   (default C3)
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_12784_b200 as vb  # noqa: E402

lib = C.CDLL(os.path.join(ROOT, "tools", "libvattn_b200_trace.so"))
B, H, N, d, causal = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (4, 16, 8192, 128, 1)
q, k, v, do = (torch.randn(B, H, N, d, device="cuda").to(torch.bfloat16) for _ in range(4))
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


def step():
    assert lib.mha_forward(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(), s) == 0
    assert lib.mha_backward(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
                            lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ws.data_ptr(), ws.numel(), s) == 0


for _ in range(3):
    step()
torch.cuda.synchronize()
nq = (N + 127) // 128
grids = {0: ("fwd", B * H * ((N + 255) // 256)), 1: ("dK/dV", B * H * nq), 3: ("dQ GEMM", B * H * nq)}
buf = (C.c_ulonglong * (3 * 16384))()
for kid, (name, nb) in grids.items():
    lib.vattn_trace_select(kid, -1)
    lib.vattn_cta_read(buf, 16384)  # clear
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    lib.vattn_cta_read(buf, 16384)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(16384, 3)[:nb].astype(np.int64)
    st, en, sm = a[:, 0], a[:, 1], a[:, 2]
    ok = (st > 0) & (en > st)
    st, en, sm = st[ok], en[ok], sm[ok]
    t0, t1 = st.min(), en.max()
    span = t1 - t0
    gaps, heads, tails, busy = [], [], [], 0
    for m in np.unique(sm):
        sel = sm == m
        o_ = np.argsort(st[sel])
        s_, e_ = st[sel][o_], en[sel][o_]
        busy += (e_ - s_).sum()
        gaps += list(s_[1:] - e_[:-1])
        heads.append(s_[0] - t0)
        tails.append(t1 - e_[-1])
    nsm = len(np.unique(sm))
    g = np.array(gaps)
    print(f"{name:8s}: {ok.sum()} CTAs on {nsm} SMs, span {span / 1e3:.1f} us, SM busy {100 * busy / (nsm * span):.1f} %, "
          f"CTA {np.mean(en - st) / 1e3:.1f} us mean ({np.min(en - st) / 1e3:.1f}..{np.max(en - st) / 1e3:.1f}), "
          f"gap between CTAs mean {g.mean() / 1e3:.2f} us (p90 {np.percentile(g, 90) / 1e3:.2f}), "
          f"head mean {np.mean(heads) / 1e3:.1f} us, tail mean {np.mean(tails) / 1e3:.1f} us max {np.max(tails) / 1e3:.1f}",
          flush=True)
