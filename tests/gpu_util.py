"""Shared helpers for the GPU parity tests (tests only)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import pyoracle as po

# SURVEY 8(c) stated bounds (R = max(1, max|ref|)):
#   vs binary64 oracle, fp16 inputs: fro_rel <= 1e-3, max_abs <= 2e-3 R;  lse max_rel <= 1e-5
#   vs binary64 oracle, bf16 inputs: fro_rel <= 8e-3, max_abs <= 1.6e-2 R
#   vs reference backward_fused (FP16-ACC): fro_rel <= 3e-3, max_abs <= 1e-2 R
TOL = {
    torch.float16: dict(fro=1e-3, abs=2e-3),
    torch.bfloat16: dict(fro=8e-3, abs=1.6e-2),
}
LSE_MAX_REL = 1e-5


def bits_to_torch(bits: np.ndarray, dtype=torch.float16, device="cuda") -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(bits, np.uint16).view(np.int16)).view(dtype)
    return t.to(device)


def torch_to_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().cpu().view(torch.int16).numpy().view(np.uint16)


def widen(t: torch.Tensor) -> np.ndarray:
    return t.detach().double().cpu().numpy()


def workload(seed, shape, dtype=torch.float16, with_dout=True):
    """Reference workload (workload.hpp:10-17): streams 1/2/3/4 = Q/K/V/dO."""
    bf = dtype == torch.bfloat16
    ts = [bits_to_torch(po.normal16(seed, s, shape, bf16=bf), dtype) for s in (1, 2, 3, 4 if with_dout else 3)]
    return ts if with_dout else ts[:3]


def check_close(test: np.ndarray, ref: np.ndarray, dtype, what: str, fro=None, abs_=None):
    tol = TOL[dtype]
    fro = tol["fro"] if fro is None else fro
    abs_ = tol["abs"] if abs_ is None else abs_
    R = max(1.0, float(np.max(np.abs(ref))))
    fr = po.frobenius_rel(test, ref)
    ma = float(np.max(np.abs(test - ref)))
    assert np.all(np.isfinite(test)), f"{what}: non-finite values"
    assert fr <= fro, f"{what}: fro_rel {fr:.3e} > {fro:.1e}"
    assert ma <= abs_ * R, f"{what}: max_abs {ma:.3e} > {abs_:.1e} * {R:.2f}"
    return fr, ma


def check_lse(test: np.ndarray, ref: np.ndarray, what="lse", max_rel=LSE_MAX_REL):
    rel = np.abs(test - ref) / np.maximum(np.abs(ref), 1e-6)
    # near-zero lse values (early causal rows) are judged absolutely (test_forward.cpp:200-214)
    absd = np.abs(test - ref)
    bad = (rel > max_rel) & (absd > max_rel)
    assert not np.any(bad), f"{what}: max_rel {rel.max():.3e} (max_abs {absd.max():.3e})"


def torch_ref_grads(q, k, v, do, causal, scale=None):
    """fp32 torch reference (GPU) for sizes where the binary64 oracle is too slow."""
    qf, kf, vf, dof = (x.float().requires_grad_(True) for x in (q, k, v, do))
    scale = scale if scale else 1.0 / np.sqrt(q.shape[-1])
    s = torch.matmul(qf, kf.transpose(-1, -2)) * scale
    if causal:
        n = q.shape[2]
        mask = torch.ones(n, n, dtype=torch.bool, device=q.device).triu(1)
        s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    p = torch.softmax(s, dim=-1)
    o = torch.matmul(p, vf)
    o.backward(dof.detach())
    return o.detach(), lse.detach(), qf.grad, kf.grad, vf.grad


def softmax_scale32(d: int) -> float:
    """AttnConfig::scale() in binary32 (attention_forward.cpp:42-45), as the kernels use it."""
    return float(torch.tensor(1.0, dtype=torch.float32) / torch.sqrt(torch.tensor(float(d), dtype=torch.float32)))


def f64_ref(q, k, v, do, causal, scale=None, block=4096):
    """binary64 restatement of the oracle's attention_ref / attention_grad_ref
    (reference.cpp:26-167) for ONE (b, h) slice [N, d], run on the GPU in float64 and
    chunked over query blocks so that N = 32k fits (one 4096 x N block of S at a time).
    Inputs are the kernels' 16-bit tensors widened exactly.  Returns float64
    (O, lse, dQ, dK, dV); D = rowsum(dO o O) uses the binary64 O, as the oracle does."""
    q, k, v, do = (x.double() for x in (q, k, v, do))
    N, d = q.shape
    scale = softmax_scale32(d) if scale is None else scale
    o = torch.empty_like(q)
    lse = torch.empty(N, dtype=torch.float64, device=q.device)
    cols = torch.arange(N, device=q.device)

    def scores(r0, r1):
        s = (q[r0:r1] @ k.T) * scale
        if causal:
            rows = torch.arange(r0, r1, device=q.device)[:, None]
            s = s.masked_fill(cols[None, :] > rows, float("-inf"))
        return s

    for r0 in range(0, N, block):
        r1 = min(N, r0 + block)
        s = scores(r0, r1)
        m = s.max(dim=1, keepdim=True).values
        p = torch.exp(s - m)
        l_ = p.sum(dim=1, keepdim=True)
        o[r0:r1] = (p @ v) / l_
        lse[r0:r1] = (m + torch.log(l_)).squeeze(1)
        del s, p
    D = (do * o).sum(dim=1)
    dq = torch.empty_like(q)
    dk = torch.zeros_like(k)
    dv = torch.zeros_like(v)
    for r0 in range(0, N, block):
        r1 = min(N, r0 + block)
        p = torch.exp(scores(r0, r1) - lse[r0:r1, None])
        dv += p.T @ do[r0:r1]
        ds = p * (do[r0:r1] @ v.T - D[r0:r1, None])
        del p
        dq[r0:r1] = (ds @ k) * scale
        dk += (ds.T @ q[r0:r1]) * scale
        del ds
    return o, lse, dq, dk, dv
