"""The unfused three-pass forward on B200 -- the comparator of the paper's
"fused vs traditional" metric, mirroring vattn::forward_traditional
(reference proj/src/attention_forward.cpp:229-310).  Separate library
(libvattn_b200_traditional.so, cuBLAS GEMMs + a softmax kernel) so the fused path
never depends on cuBLAS.  Comparator only: not on the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import _Cfg, _cfg, _check, _raise, _stream, VATTN_EINVAL

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libvattn_b200_traditional.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build()")
        _lib = C.CDLL(LIB_PATH)
        _lib.mha_forward_traditional_workspace_bytes.argtypes = [C.POINTER(_Cfg)]
        _lib.mha_forward_traditional_workspace_bytes.restype = C.c_size_t
        _lib.mha_forward_traditional.argtypes = [C.POINTER(_Cfg)] + [C.c_void_p] * 6 + [C.c_size_t, C.c_void_p]
        _lib.mha_forward_traditional.restype = C.c_int
        _lib.vattn_traditional_last_error.restype = C.c_char_p
    return _lib


def workspace_bytes(q: torch.Tensor, causal: bool = False) -> int:
    return int(lib().mha_forward_traditional_workspace_bytes(C.byref(_cfg(q, causal, 0.0))))


def forward_traditional(q, k, v, causal: bool = False, softmax_scale: float = 0.0, dropout_p: float = 0.0,
                        seed: int = 0, workspace=None):
    """Three-pass forward on CUDA tensors [B, H, N, d] (d % 4 == 0): returns (out, lse)."""
    _check((q, k, v), q.shape, q.dtype, ("q", "k", "v"))
    B, H, N, d = q.shape
    cfg = _cfg(q, causal, softmax_scale, dropout_p, seed)
    need = int(lib().mha_forward_traditional_workspace_bytes(C.byref(cfg)))
    if need == 0:
        raise ValueError(f"forward_traditional: {lib().vattn_traditional_last_error().decode()}")
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=q.device)
    out = torch.empty_like(q)
    lse = torch.empty((B, H, N), dtype=torch.float32, device=q.device)
    rc = lib().mha_forward_traditional(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                       lse.data_ptr(), workspace.data_ptr(), workspace.numel(), _stream())
    if rc:
        raise (ValueError if rc == VATTN_EINVAL else RuntimeError)(
            f"forward_traditional: {lib().vattn_traditional_last_error().decode()}")
    return out, lse
