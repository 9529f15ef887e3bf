"""paper_2502_12784_b200 -- B200 (sm_100a) fused multi-head-attention training path.

Python mirror of the reference's operator API (arxiv 2502.12784, reference tree
/root/reference/proj) over the C ABI in ``include/vattn_b200.h``:

=====================  ==============================================================
this module            reference
=====================  ==============================================================
``AttnConfig``         ``vattn::AttnConfig`` (include/vattn/attention.hpp:11-26)
``forward_fused``      ``vattn::forward_fused`` (attention.hpp:51-52) -> (out, lse)
``backward_fused``     ``vattn::backward_fused`` (backward.hpp:56-59) -> (dq, dk, dv)
``mha_forward``        C ABI ``mha_forward`` on device tensors
``mha_backward``       C ABI ``mha_backward`` on device tensors (takes O)
``compute_dpsum``      ``vattn::compute_dpsum`` (backward.hpp:43), via the backward
``MHAFunction``        torch.autograd binding (the paper's PyTorch layer)
=====================  ==============================================================

Errors mirror the reference: ``ValueError`` where it throws std::invalid_argument,
``ArithmeticError`` for std::domain_error, ``NotImplementedError`` for
unsupported-here, ``RuntimeError`` for CUDA failures.  There is no CPU fallback:
the shared library is required, and importing this module fails loudly without it.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import torch

__all__ = [
    "AttnConfig", "forward_fused", "backward_fused", "mha_forward", "mha_backward",
    "workspace_bytes", "MHAFunction", "attention", "LIB_PATH", "lib",
    "mha_forward_host", "mha_backward_host", "mha_step_host", "compute_dpsum", "dropout_digest",
]

LIB_PATH = os.environ.get("VATTN_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libvattn_b200.so")

VATTN_OK, VATTN_EINVAL, VATTN_EDOMAIN, VATTN_EUNSUPPORTED, VATTN_ECUDA = range(5)
VATTN_F16, VATTN_BF16 = 0, 1


class _Cfg(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("heads", C.c_int32), ("seq_len", C.c_int32), ("head_dim", C.c_int32),
        ("causal", C.c_int32), ("softmax_scale", C.c_float), ("dtype", C.c_int32),
        ("dropout_p", C.c_float), ("seed", C.c_uint64), ("bh_offset", C.c_int32), ("bh_count", C.c_int32),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for this path)")
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    lib.mha_forward.argtypes = [C.POINTER(_Cfg), vp, vp, vp, vp, vp, vp]
    lib.mha_forward.restype = C.c_int
    lib.mha_backward_workspace_bytes.argtypes = [C.POINTER(_Cfg)]
    lib.mha_backward_workspace_bytes.restype = C.c_size_t
    lib.mha_backward.argtypes = [C.POINTER(_Cfg)] + [vp] * 10 + [C.c_size_t, vp]
    lib.mha_backward.restype = C.c_int
    lib.mha_forward_host.argtypes = [C.POINTER(_Cfg)] + [vp] * 6
    lib.mha_forward_host.restype = C.c_int
    lib.mha_backward_host.argtypes = [C.POINTER(_Cfg)] + [vp] * 10
    lib.mha_backward_host.restype = C.c_int
    lib.mha_step_host.argtypes = [C.POINTER(_Cfg)] + [vp] * 10
    lib.mha_step_host.restype = C.c_int
    lib.vattn_dropout_digest.argtypes = [C.POINTER(_Cfg), C.c_int, C.c_int, vp, vp]
    lib.vattn_dropout_digest.restype = C.c_int
    if hasattr(lib, "mha_dropout_mask_bytes"):  # (VATTN_LIB may point at an older build)
        lib.mha_dropout_mask_bytes.argtypes = [C.POINTER(_Cfg)]
        lib.mha_dropout_mask_bytes.restype = C.c_size_t
        lib.mha_forward_dropout_mask.argtypes = [C.POINTER(_Cfg)] + [vp] * 7
        lib.mha_forward_dropout_mask.restype = C.c_int
        lib.mha_backward_dropout_mask.argtypes = [C.POINTER(_Cfg)] + [vp] * 11 + [C.c_size_t, vp]
        lib.mha_backward_dropout_mask.restype = C.c_int
    lib.mha_dpsum.argtypes = [C.POINTER(_Cfg)] + [vp] * 4
    lib.mha_dpsum.restype = C.c_int
    if hasattr(lib, "mha_forward_ex"):  # ABI >= 4
        lib.mha_forward_ex.argtypes = [C.POINTER(_Cfg)] + [vp] * 8
        lib.mha_forward_ex.restype = C.c_int
        lib.mha_backward_workspace_bytes_mask.argtypes = [C.POINTER(_Cfg)]
        lib.mha_backward_workspace_bytes_mask.restype = C.c_size_t
        lib.vattn_map_cache_stats.argtypes = [C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
        lib.vattn_map_cache_stats.restype = None
    lib.vattn_last_error.restype = C.c_char_p
    lib.vattn_abi_version.restype = C.c_int
    lib.vattn_last_launch_count.restype = C.c_int
    return lib


lib = _load()


def _raise(rc: int, where: str):
    msg = f"{where}: {lib.vattn_last_error().decode()}"
    if rc == VATTN_EINVAL:
        raise ValueError(msg)
    if rc == VATTN_EDOMAIN:
        raise ArithmeticError(msg)
    if rc == VATTN_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


@dataclass
class AttnConfig:
    """vattn::AttnConfig (attention.hpp:11-26).  Tile sizes are validated for
    compatibility with the reference but the GPU tiles are fixed at 128."""
    batch: int = 1
    heads: int = 1
    seq_len: int = 0
    head_dim: int = 0
    tile_rows: int = 64
    tile_cols: int = 64
    causal: bool = False
    dropout_p: float = 0.0
    seed: int = 0
    softmax_scale: float = 0.0
    acc_mode: str = "fp32"  # AccMode (attention.hpp:9): reported in traffic/report only; the GPU accumulates in fp32

    def validate(self, strict_tiles: bool = True) -> None:
        """AttnConfig::validate (attention_forward.cpp:31-40).  ``strict_tiles=False``
        drops the reference's N % tile requirement, which the GPU path does not need."""
        def req(ok, msg):
            if not ok:
                raise ValueError(msg)
        req(self.batch >= 1 and self.heads >= 1, "AttnConfig: batch and heads must be positive")
        req(self.seq_len > 0 and self.head_dim > 0, "AttnConfig: seq_len and head_dim must be positive")
        req(self.tile_rows > 0 and self.tile_rows % 8 == 0, "AttnConfig: tile_rows must be a positive multiple of 8")
        req(self.tile_cols > 0 and self.tile_cols % 8 == 0, "AttnConfig: tile_cols must be a positive multiple of 8")
        req(self.head_dim % 4 == 0, "AttnConfig: head_dim must be a multiple of 4")
        if strict_tiles:
            req(self.seq_len % self.tile_rows == 0, "AttnConfig: seq_len must be a multiple of tile_rows")
            req(self.seq_len % self.tile_cols == 0, "AttnConfig: seq_len must be a multiple of tile_cols")
        req(0.0 <= self.dropout_p < 1.0, "AttnConfig: dropout_p must be in [0, 1)")
        req(str(self.acc_mode).lower() in ("fp16", "fp32"), "AttnConfig: acc_mode must be fp16 or fp32")

    def scale(self) -> float:
        """AttnConfig::scale (attention_forward.cpp:42-45), binary32."""
        if self.softmax_scale > 0.0:
            return float(self.softmax_scale)
        return float(torch.tensor(1.0, dtype=torch.float32) / torch.sqrt(torch.tensor(float(self.head_dim))))


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float16:
        return VATTN_F16
    if t.dtype == torch.bfloat16:
        return VATTN_BF16
    raise ValueError(f"tensors must be float16 or bfloat16, got {t.dtype}")


def _cfg(q: torch.Tensor, causal: bool, softmax_scale: float, dropout_p: float = 0.0, seed: int = 0,
         bh_slab: tuple[int, int, int, int] | None = None) -> _Cfg:
    """bh_slab = (B, H, bh_offset, bh_count): q is the [bh_count, 1, N, d] slab of a
    global (B, H) problem (dropout masks then use the global (b, h))."""
    if bh_slab is None:
        B, H, N, d = q.shape
        off = cnt = 0
    else:
        B, H, off, cnt = bh_slab
        N, d = q.shape[-2:]
    return _Cfg(B, H, N, d, 1 if causal else 0, float(softmax_scale), _dtype_code(q), float(dropout_p), int(seed),
                int(off), int(cnt))


def _check(ts, shape, dtype, names):
    for t, n in zip(ts, names):
        if t.shape != shape:
            raise ValueError(f"{n} shape {tuple(t.shape)} != {tuple(shape)}")
        if t.dtype != dtype:
            raise ValueError(f"{n} dtype {t.dtype} != {dtype}")
        if not t.is_cuda:
            raise ValueError(f"{n} must be a CUDA tensor (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError(f"{n} must be contiguous [B, H, N, d]")


def _stream(dev=None) -> int:
    """The current stream of `dev` (the tensors' device), not of the current device."""
    return torch.cuda.current_stream(dev).cuda_stream


def _check_out(t, shape, dtype, name, dev):
    """Caller-supplied output buffer: the kernels write every element of `shape`."""
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype:
        raise ValueError(f"{name}: expected {dtype} {tuple(shape)}, got {t.dtype} {tuple(t.shape)}")
    if not t.is_cuda or t.device != dev:
        raise ValueError(f"{name} must be a CUDA tensor on {dev}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _domain_check(status: torch.Tensor, where: str):
    """Synchronises on the status word; the reference throws std::domain_error here."""
    if int(status.item()) & 1:
        raise ArithmeticError(f"{where}: softmax: NaN score or fully masked row (l == 0) in a query row "
                              "(reference: std::domain_error, online_softmax.cpp:33-34 / 81-82)")


def _native_dim(d: int) -> int:
    if d <= 64:
        return 64
    if d <= 128:
        return 128
    raise NotImplementedError(f"head_dim {d} > 128 is not supported")


def _pad(t: torch.Tensor, dn: int) -> torch.Tensor:
    return t if t.shape[-1] == dn else torch.nn.functional.pad(t, (0, dn - t.shape[-1])).contiguous()


def mha_forward(q, k, v, causal: bool = False, softmax_scale: float = 0.0, out=None, lse=None,
                dropout_p: float = 0.0, seed: int = 0, bh_slab=None, drop_mask=None, check_domain: bool = False):
    """C ABI ``mha_forward`` on CUDA tensors [B, H, N, d] (d in {64, 128}).
    Returns (out, lse) with lse [B, H, N] fp32 natural-log.  ``dropout_p > 0``
    applies the reference's dropout (keep bits = vattn::dropout_keep(seed, b, h, row, col, p)).
    ``check_domain``: synchronise and raise ArithmeticError where the reference throws
    std::domain_error (a NaN / +inf score or an empty softmax row; C ABI mha_forward_ex)."""
    _check((q, k, v), q.shape, q.dtype, ("q", "k", "v"))
    B, H, N, d = q.shape
    dev = q.device
    if out is None:
        out = torch.empty_like(q)
    else:
        _check_out(out, q.shape, q.dtype, "out", dev)
    if lse is None:
        lse = torch.empty((B, H, N), dtype=torch.float32, device=dev)
    else:
        _check_out(lse, (B, H, N), torch.float32, "lse", dev)
    cfg = _cfg(q, causal, softmax_scale, dropout_p, seed, bh_slab)
    status = None
    with torch.cuda.device(dev):
        if drop_mask is not None:  # also keep the dropout keep bits for mha_backward(drop_mask=...)
            _check_mask(drop_mask, cfg)
        if check_domain:
            status = torch.zeros(1, dtype=torch.int32, device=dev)
        if drop_mask is not None or check_domain:
            rc = lib.mha_forward_ex(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                    lse.data_ptr(), None if drop_mask is None else drop_mask.data_ptr(),
                                    None if status is None else status.data_ptr(), _stream(dev))
        else:
            rc = lib.mha_forward(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                 lse.data_ptr(), _stream(dev))
    if rc:
        _raise(rc, "mha_forward")
    if status is not None:
        _domain_check(status, "mha_forward")
    return out, lse


def dropout_mask_bytes(q, causal: bool = False, dropout_p: float = 0.0, bh_slab=None) -> int:
    """Bytes of the keep-bit mask mha_forward(drop_mask=...) fills (0 without dropout)."""
    return int(lib.mha_dropout_mask_bytes(C.byref(_cfg(q, causal, 0.0, dropout_p, 0, bh_slab))))


def _check_mask(m, cfg):
    need = int(lib.mha_dropout_mask_bytes(C.byref(cfg)))
    if need == 0:
        raise ValueError("drop_mask given but keep-bit masks are off (dropout_p == 0 or VATTN_DROP_MASK=0)")
    if not m.is_cuda or m.numel() * m.element_size() < need or m.data_ptr() % 256:
        raise ValueError(f"drop_mask must be a 256-byte aligned CUDA buffer of >= {need} bytes")


def workspace_bytes(B, H, N, d, causal=False, dtype=torch.float16, dropout_p: float = 0.0,
                    external_mask: bool = False) -> int:
    """mha_backward workspace.  With dropout it includes a keep-bit mask region unless
    ``external_mask`` (the caller passes the forward's mask: mha_backward(drop_mask=...))."""
    cfg = _Cfg(B, H, N, d, 1 if causal else 0, 0.0, VATTN_BF16 if dtype == torch.bfloat16 else VATTN_F16,
               float(dropout_p), 0, 0, 0)
    if external_mask:
        return int(lib.mha_backward_workspace_bytes_mask(C.byref(cfg)))
    return int(lib.mha_backward_workspace_bytes(C.byref(cfg)))


def keep_mask_cap_bytes() -> int:
    """Largest keep-bit mask the autograd binding / backward_fused keep from forward to
    backward (VATTN_KEEP_MASK_MB, default 2048 MiB).  Larger masks are not kept: the
    backward then hashes the bits itself into its (transient) workspace."""
    return int(float(os.environ.get("VATTN_KEEP_MASK_MB", "2048")) * (1 << 20))


def mha_backward(q, k, v, o, dout, lse, causal: bool = False, softmax_scale: float = 0.0,
                 dq=None, dk=None, dv=None, workspace=None, dropout_p: float = 0.0, seed: int = 0, bh_slab=None,
                 drop_mask=None):
    """C ABI ``mha_backward`` on CUDA tensors.  Returns (dq, dk, dv).
    ``bh_slab=(B, H, offset, count)``: the tensors are units [offset, offset+count)
    of a global (B, H) problem (used by (b, h) sharding)."""
    _check((q, k, v, o, dout), q.shape, q.dtype, ("q", "k", "v", "o", "dout"))
    B, H, N, d = q.shape
    if lse.shape != (B, H, N) or lse.dtype != torch.float32 or not lse.is_contiguous():
        raise ValueError("lse must be a contiguous float32 [B, H, N] tensor")
    dev = q.device
    if lse.device != dev:
        raise ValueError(f"lse must be on {dev}")
    cfg = _cfg(q, causal, softmax_scale, dropout_p, seed, bh_slab)
    need = int(lib.mha_backward_workspace_bytes(C.byref(cfg)) if drop_mask is None
               else lib.mha_backward_workspace_bytes_mask(C.byref(cfg)))
    if need == 0:
        rc = lib.mha_backward(C.byref(cfg), *([None] * 10), 0, None)
        _raise(rc if rc else VATTN_EINVAL, "mha_backward")
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    elif not workspace.is_cuda or workspace.device != dev or not workspace.is_contiguous():
        raise ValueError(f"workspace must be a contiguous CUDA buffer on {dev}")
    grads = []
    for t, n in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        if t is None:
            t = torch.empty_like(q)
        else:
            _check_out(t, q.shape, q.dtype, n, dev)
        grads.append(t)
    dq, dk, dv = grads
    with torch.cuda.device(dev):
        if drop_mask is not None:  # the forward's keep bits (mha_forward(drop_mask=...))
            _check_mask(drop_mask, cfg)
            rc = lib.mha_backward_dropout_mask(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                               dout.data_ptr(), lse.data_ptr(), drop_mask.data_ptr(), dq.data_ptr(),
                                               dk.data_ptr(), dv.data_ptr(), workspace.data_ptr(),
                                               workspace.numel() * workspace.element_size(), _stream(dev))
        else:
            rc = lib.mha_backward(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                  dout.data_ptr(), lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                  workspace.data_ptr(), workspace.numel() * workspace.element_size(), _stream(dev))
    if rc:
        _raise(rc, "mha_backward")
    return dq, dk, dv


# -------------------------------------------------- host-buffer entry points --

def _check_host(ts, shape, dtype, names):
    for t, n in zip(ts, names):
        if tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            raise ValueError(f"{n}: expected {dtype} {tuple(shape)}, got {t.dtype} {tuple(t.shape)}")
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{n} must be a contiguous host (CPU) tensor")


def _host_empty(shape, dtype, like):
    t = torch.empty(shape, dtype=dtype)
    return t.pin_memory() if like.is_pinned() else t


def mha_forward_host(q, k, v, causal: bool = False, softmax_scale: float = 0.0, dropout_p: float = 0.0,
                     seed: int = 0, out=None, lse=None, bh_slab=None):
    """C ABI ``mha_forward_host``: host tensors in and out, PCIe copies pipelined
    against the kernels slab by slab.  Pinned inputs give full overlap."""
    _check_host((q, k, v), q.shape, q.dtype, ("q", "k", "v"))
    B, H, N, d = q.shape
    out = _host_empty(q.shape, q.dtype, q) if out is None else out
    lse = _host_empty((B, H, N), torch.float32, q) if lse is None else lse
    _check_host((out,), q.shape, q.dtype, ("out",))
    _check_host((lse,), (B, H, N), torch.float32, ("lse",))
    cfg = _cfg(q, causal, softmax_scale, dropout_p, seed, bh_slab)
    rc = lib.mha_forward_host(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                              lse.data_ptr(), _stream())
    if rc:
        _raise(rc, "mha_forward_host")
    return out, lse


def mha_backward_host(q, k, v, o, dout, lse, causal: bool = False, softmax_scale: float = 0.0,
                      dropout_p: float = 0.0, seed: int = 0, dq=None, dk=None, dv=None, bh_slab=None):
    """C ABI ``mha_backward_host`` on host tensors.  Returns (dq, dk, dv)."""
    _check_host((q, k, v, o, dout), q.shape, q.dtype, ("q", "k", "v", "o", "dout"))
    B, H, N, d = q.shape
    _check_host((lse,), (B, H, N), torch.float32, ("lse",))
    dq, dk, dv = (_host_empty(q.shape, q.dtype, q) if t is None else t for t in (dq, dk, dv))
    _check_host((dq, dk, dv), q.shape, q.dtype, ("dq", "dk", "dv"))
    cfg = _cfg(q, causal, softmax_scale, dropout_p, seed, bh_slab)
    rc = lib.mha_backward_host(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                               dout.data_ptr(), lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                               _stream())
    if rc:
        _raise(rc, "mha_backward_host")
    return dq, dk, dv


def mha_step_host(q, k, v, dout, causal: bool = False, softmax_scale: float = 0.0, dropout_p: float = 0.0,
                  seed: int = 0, out=None, bh_slab=None):
    """C ABI ``mha_step_host``: forward + backward on host tensors with Q, K, V, dO
    crossing PCIe once.  ``out`` = optional preallocated (o, lse, dq, dk, dv).
    Returns (o, lse, dq, dk, dv)."""
    _check_host((q, k, v, dout), q.shape, q.dtype, ("q", "k", "v", "dout"))
    B, H, N, d = q.shape
    if out is None:
        out = (_host_empty(q.shape, q.dtype, q), _host_empty((B, H, N), torch.float32, q),
               *(_host_empty(q.shape, q.dtype, q) for _ in range(3)))
    o, lse, dq, dk, dv = out
    _check_host((o, dq, dk, dv), q.shape, q.dtype, ("o", "dq", "dk", "dv"))
    _check_host((lse,), (B, H, N), torch.float32, ("lse",))
    cfg = _cfg(q, causal, softmax_scale, dropout_p, seed, bh_slab)
    rc = lib.mha_step_host(C.byref(cfg), q.data_ptr(), k.data_ptr(), v.data_ptr(), dout.data_ptr(), o.data_ptr(),
                           lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), _stream())
    if rc:
        _raise(rc, "mha_step_host")
    return o, lse, dq, dk, dv


def compute_dpsum(d_out, out):
    """vattn::compute_dpsum (backward.hpp:43): D = rowsum(dO o O) as [B, H, N] fp32
    (C ABI ``mha_dpsum``; head_dim 64 or 128)."""
    _check((d_out, out), out.shape, out.dtype, ("d_out", "out"))
    B, H, N, d = out.shape
    D = torch.empty((B, H, N), dtype=torch.float32, device=out.device)
    cfg = _cfg(out, False, 0.0)
    with torch.cuda.device(out.device):
        rc = lib.mha_dpsum(C.byref(cfg), out.data_ptr(), d_out.data_ptr(), D.data_ptr(), _stream(out.device))
    if rc:
        _raise(rc, "mha_dpsum")
    return D


def dropout_digest(cfg: "AttnConfig", traditional: bool = False) -> int:
    """The reference's ``mask_digest`` for ``cfg`` (its tile sizes decide the visited
    positions; ``traditional`` = every N x N position), bit-identical to the
    reference (C ABI ``vattn_dropout_digest``)."""
    c = _Cfg(cfg.batch, cfg.heads, cfg.seq_len, _native_dim(cfg.head_dim), 0 if traditional else int(cfg.causal),
             float(cfg.softmax_scale), VATTN_F16, float(cfg.dropout_p), int(cfg.seed), 0, 0)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    br, bc = (cfg.seq_len, cfg.seq_len) if traditional else (cfg.tile_rows, cfg.tile_cols)
    rc = lib.vattn_dropout_digest(C.byref(c), br, bc, out.data_ptr(), _stream())
    if rc:
        _raise(rc, "vattn_dropout_digest")
    return int(out.item()) & ((1 << 64) - 1)


# ----------------------------------------- reference-shaped operator API --

def _prep(cfg: AttnConfig, *ts):
    cfg.validate(strict_tiles=False)
    shape = (cfg.batch, cfg.heads, cfg.seq_len, cfg.head_dim)
    for t in ts:
        if tuple(t.shape) != shape:
            raise ValueError(f"tensor shape {tuple(t.shape)} does not match config {shape}")
    dn = _native_dim(cfg.head_dim)
    return [_pad(t.contiguous(), dn) for t in ts], dn


def forward_fused(q, k, v, cfg: AttnConfig):
    """vattn::forward_fused on CUDA tensors: returns (out, lse).  head_dim other
    than 64/128 is zero-padded (exact: padded columns add 0 to every dot product)."""
    (qp, kp, vp), dn = _prep(cfg, q, k, v)
    out, lse = mha_forward(qp, kp, vp, cfg.causal, cfg.scale(), dropout_p=cfg.dropout_p, seed=cfg.seed,
                           check_domain=True)
    return out[..., : cfg.head_dim].contiguous(), lse


def backward_fused(q, k, v, d_out, lse, cfg: AttnConfig, out=None):
    """vattn::backward_fused on CUDA tensors: returns (dq, dk, dv).  Like the
    reference (attention_backward.cpp:91-104) it recomputes O with the forward
    when ``out`` is not given."""
    (qp, kp, vp, dop), dn = _prep(cfg, q, k, v, d_out)
    mask = None
    if out is None:
        mb = dropout_mask_bytes(qp, cfg.causal, cfg.dropout_p)
        if 0 < mb <= keep_mask_cap_bytes():  # the recomputed forward keeps its keep bits for the backward
            mask = torch.empty(mb, dtype=torch.uint8, device=qp.device)
        op, _ = mha_forward(qp, kp, vp, cfg.causal, cfg.scale(), dropout_p=cfg.dropout_p, seed=cfg.seed,
                            drop_mask=mask, check_domain=True)
    else:
        op = _pad(out.contiguous(), dn)
    dq, dk, dv = mha_backward(qp, kp, vp, op, dop, lse.contiguous(), cfg.causal, cfg.scale(),
                              dropout_p=cfg.dropout_p, seed=cfg.seed, drop_mask=mask)
    d = cfg.head_dim
    return dq[..., :d].contiguous(), dk[..., :d].contiguous(), dv[..., :d].contiguous()


class MHAFunction(torch.autograd.Function):
    """torch.autograd binding: forward = mha_forward, backward = mha_backward."""

    @staticmethod
    def forward(ctx, q, k, v, causal=False, softmax_scale=0.0, dropout_p=0.0, seed=0):
        d = q.shape[-1]
        dn = _native_dim(d)
        qp, kp, vp = (_pad(x.contiguous(), dn) for x in (q, k, v))
        scale = softmax_scale if softmax_scale > 0 else 1.0 / math.sqrt(d)
        mask = None
        mb = dropout_mask_bytes(qp, causal, dropout_p)
        if 0 < mb <= keep_mask_cap_bytes():
            # keep the forward's keep bits: the backward skips re-hashing them (a bigger
            # mask is not kept -- the backward hashes the bits into its own workspace)
            mask = torch.empty(mb, dtype=torch.uint8, device=qp.device)
        o, lse = mha_forward(qp, kp, vp, causal, scale, dropout_p=dropout_p, seed=seed, drop_mask=mask)
        if mask is not None:
            ctx.save_for_backward(qp, kp, vp, o, lse, mask)
        else:
            ctx.save_for_backward(qp, kp, vp, o, lse)
        ctx.causal, ctx.scale, ctx.d, ctx.dropout_p, ctx.seed = causal, scale, d, dropout_p, seed
        return o[..., :d] if dn != d else o

    @staticmethod
    def backward(ctx, do):
        saved = ctx.saved_tensors
        qp, kp, vp, o, lse = saved[:5]
        mask = saved[5] if len(saved) > 5 else None
        dop = _pad(do.contiguous(), qp.shape[-1])
        dq, dk, dv = mha_backward(qp, kp, vp, o, dop, lse, ctx.causal, ctx.scale,
                                  dropout_p=ctx.dropout_p, seed=ctx.seed, drop_mask=mask)
        d = ctx.d
        return dq[..., :d], dk[..., :d], dv[..., :d], None, None, None, None


def attention(q, k, v, causal: bool = False, softmax_scale: float = 0.0, dropout_p: float = 0.0, seed: int = 0):
    """Differentiable fused attention on [B, H, N, d] fp16/bf16 CUDA tensors."""
    return MHAFunction.apply(q, k, v, causal, softmax_scale, dropout_p, seed)
