"""ctypes bindings for the parity checker (TEST INFRASTRUCTURE ONLY).

Two libraries, both built by ``oracle/Makefile``:

* ``oracle/_build/liboracle.so`` -- the C restatement (``vattn_oracle.c``) of the
  reference's path; always available.
* ``oracle/_ref/libvattn_ref.so`` -- the unmodified reference sources
  (``/root/reference/proj/src``) + ``ref_shim.cpp``; available where it was built
  (it travels to the GPU box inside the gpurun snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs import
this module.  The product path (``paper_2502_12784_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvattn_ref.so")

_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32, _u64, _f32 = C.c_int, C.c_uint64, C.c_float

_oracle = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        lib.vo_normal_tensor16.argtypes = [_u64, _u64, _u64, _i32, _u16p]
        lib.vo_normal_at.argtypes = [_u64, _u64]
        lib.vo_normal_at.restype = C.c_float
        lib.vo_f32_to_f16.argtypes = [C.c_float]
        lib.vo_f32_to_f16.restype = C.c_uint16
        lib.vo_f16_to_f32.argtypes = [C.c_uint16]
        lib.vo_f16_to_f32.restype = C.c_float
        lib.vo_f32_to_bf16.argtypes = [C.c_float]
        lib.vo_f32_to_bf16.restype = C.c_uint16
        lib.vo_widen16.argtypes = [_u16p, _u64, _i32, _f64p]
        lib.vo_attention_ref.argtypes = [_i32] * 5 + [_f32, _f64p, _f64p, _f64p, _f64p, _f64p]
        lib.vo_attention_grad_ref.argtypes = [_i32] * 5 + [_f32] + [_f64p] * 7
        lib.vo_forward_fused_fp32acc.argtypes = [_i32] * 7 + [_f32, _u16p, _u16p, _u16p, _u16p, _f32p]
        lib.vo_forward_fused_fp32acc.restype = C.c_int
        lib.vo_compute_dpsum.argtypes = [_i32] * 5 + [_u16p, _u16p, _f32p]
        lib.vo_dropout_keep.argtypes = [_u64] * 5 + [_f32]
        lib.vo_dropout_keep.restype = C.c_int
        lib.vo_position_hash.argtypes = [_u64] * 5
        lib.vo_position_hash.restype = C.c_uint64
        lib.vo_attention_ref_dropout.argtypes = [_i32] * 5 + [_f32, _f32, _u64] + [_f64p] * 5
        lib.vo_attention_grad_ref_dropout.argtypes = [_i32] * 5 + [_f32, _f32, _u64] + [_f64p] * 7
        lib.vo_forward_fused_fp32acc_dropout.argtypes = [_i32] * 7 + [_f32, _f32, _u64, _u16p, _u16p, _u16p, _u16p, _f32p]
        lib.vo_forward_fused_fp32acc_dropout.restype = C.c_int
        lib.vo_error_metrics.argtypes = [_f64p, _f64p, _u64, _f64p]
        lib.vo_frobenius_rel.argtypes = [_f64p, _f64p, _u64]
        lib.vo_frobenius_rel.restype = C.c_double
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.vr_last_error.restype = C.c_char_p
        lib.vr_normal_tensor_f16.argtypes = [_u64, _u64, _u64, _u16p]
        lib.vr_forward_fused.argtypes = [_i32] * 8 + [_f32, _u16p, _u16p, _u16p, _u16p, _f32p]
        lib.vr_backward_fused.argtypes = [_i32] * 7 + [_f32] + [_u16p] * 4 + [_f32p] + [_u16p] * 3
        lib.vr_compute_dpsum.argtypes = [_i32] * 4 + [_u16p, _u16p, _f32p]
        lib.vr_attention_ref.argtypes = [_i32] * 5 + [_f32] + [_f64p] * 5
        lib.vr_attention_grad_ref.argtypes = [_i32] * 5 + [_f32] + [_f64p] * 7
        lib.vr_dropout_keep.argtypes = [_u64] * 5 + [_f32]
        lib.vr_dropout_keep.restype = C.c_int
        _u64p = C.POINTER(C.c_uint64)
        lib.vr_forward_fused_dropout.argtypes = [_i32] * 8 + [_f32, _f32, _u64, _u16p, _u16p, _u16p, _u16p, _f32p, _u64p]
        lib.vr_backward_fused_dropout.argtypes = [_i32] * 7 + [_f32, _f32, _u64] + [_u16p] * 4 + [_f32p] + [_u16p] * 3 + [_u64p]
        lib.vr_attention_ref_dropout.argtypes = [_i32] * 5 + [_f32, _f32, _u64] + [_f64p] * 5
        lib.vr_attention_grad_ref_dropout.argtypes = [_i32] * 5 + [_f32, _f32, _u64] + [_f64p] * 7
        lib.vr_bench_units.argtypes = [_i32] * 5
        lib.vr_bench_units.restype = C.c_double
        lib.vr_traffic.argtypes = [_i32] * 8 + [_u64p]
        lib.vr_write_spat_f16.argtypes = [C.c_char_p, _i32, _u64p, _u16p]
        lib.vr_write_spat_f32.argtypes = [C.c_char_p, _i32, _u64p, _f32p]
        lib.vr_read_spat_check.argtypes = [C.c_char_p]
        _ref = lib
    return _ref


# ----------------------------------------------------------------- helpers --

def normal16(seed: int, stream: int, shape, bf16: bool = False) -> np.ndarray:
    """workload.hpp:10-17 normal_tensor_f16 (bf16=True: same normals, RNE to bf16)."""
    n = int(np.prod(shape))
    out = np.empty(n, np.uint16)
    oracle_lib().vo_normal_tensor16(seed, stream, n, 1 if bf16 else 0, out)
    return out.reshape(shape)


def widen(bits: np.ndarray, bf16: bool = False) -> np.ndarray:
    bits = np.ascontiguousarray(bits, np.uint16)
    out = np.empty(bits.size, np.float64)
    oracle_lib().vo_widen16(bits.reshape(-1), bits.size, 1 if bf16 else 0, out)
    return out.reshape(bits.shape)


def attention_ref(q, k, v, causal: bool, scale: float = 0.0, dropout_p: float = 0.0, seed: int = 0):
    """binary64 oracle forward (reference.cpp:26-80) on widened float64 inputs [B,H,N,d]."""
    B, H, N, d = q.shape
    out = np.empty((B, H, N, d), np.float64)
    lse = np.empty((B, H, N), np.float64)
    oracle_lib().vo_attention_ref_dropout(B, H, N, d, int(causal), scale, dropout_p, seed,
                                          np.ascontiguousarray(q, np.float64), np.ascontiguousarray(k, np.float64),
                                          np.ascontiguousarray(v, np.float64), out, lse)
    return out, lse


def attention_grad_ref(q, k, v, dout, causal: bool, scale: float = 0.0, dropout_p: float = 0.0, seed: int = 0):
    """binary64 analytic gradients (reference.cpp:82-167)."""
    B, H, N, d = q.shape
    dq = np.empty((B, H, N, d), np.float64)
    dk = np.empty_like(dq)
    dv = np.empty_like(dq)
    c = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
    oracle_lib().vo_attention_grad_ref_dropout(B, H, N, d, int(causal), scale, dropout_p, seed,
                                               c(q), c(k), c(v), c(dout), dq, dk, dv)
    return dq, dk, dv


def dropout_keep(seed, b, h, row, col, p) -> bool:
    """rng.cpp:46-49."""
    return bool(oracle_lib().vo_dropout_keep(seed, b, h, row, col, p))


def forward_fused_fp32acc(q16, k16, v16, causal: bool, br: int = 64, bc: int = 64, scale: float = 0.0,
                          dropout_p: float = 0.0, seed: int = 0):
    """Bit-exact restatement of forward_fused at FP32-ACC (attention_forward.cpp:110-227)."""
    B, H, N, d = q16.shape
    out = np.empty((B, H, N, d), np.uint16)
    lse = np.empty((B, H, N), np.float32)
    c = lambda a: np.ascontiguousarray(a, np.uint16)  # noqa: E731
    rc = oracle_lib().vo_forward_fused_fp32acc_dropout(B, H, N, d, br, bc, int(causal), scale, dropout_p, seed,
                                                       c(q16), c(k16), c(v16), out, lse)
    if rc == -1:
        raise ValueError("forward_fused: invalid config")
    if rc == -2:
        raise ArithmeticError("forward_fused: NaN score or fully masked row")
    return out, lse


def compute_dpsum(dout16, o16, bf16: bool = False):
    """attention_backward.cpp:44-57."""
    B, H, N, d = dout16.shape
    out = np.empty((B, H, N), np.float32)
    c = lambda a: np.ascontiguousarray(a, np.uint16)  # noqa: E731
    oracle_lib().vo_compute_dpsum(B, H, N, d, 1 if bf16 else 0, c(dout16), c(o16), out)
    return out


def error_metrics(test, ref):
    """reference.cpp:186-210 -> dict(mean_rel, max_rel, mean_abs, max_abs)."""
    t = np.ascontiguousarray(test, np.float64).reshape(-1)
    r = np.ascontiguousarray(ref, np.float64).reshape(-1)
    out = np.empty(4, np.float64)
    oracle_lib().vo_error_metrics(t, r, t.size, out)
    return dict(mean_rel=out[0], max_rel=out[1], mean_abs=out[2], max_abs=out[3])


def frobenius_rel(test, ref) -> float:
    t = np.ascontiguousarray(test, np.float64).reshape(-1)
    r = np.ascontiguousarray(ref, np.float64).reshape(-1)
    return float(oracle_lib().vo_frobenius_rel(t, r, t.size))


# -------------------------------------------------- reference (oracle/_ref) --

def ref_forward_fused(q16, k16, v16, causal, br=64, bc=64, acc_fp16=False, scale=0.0):
    B, H, N, d = q16.shape
    out = np.empty((B, H, N, d), np.uint16)
    lse = np.empty((B, H, N), np.float32)
    c = lambda a: np.ascontiguousarray(a, np.uint16)  # noqa: E731
    lib = ref_lib()
    rc = lib.vr_forward_fused(B, H, N, d, br, bc, int(causal), int(acc_fp16), scale, c(q16), c(k16), c(v16), out, lse)
    if rc:
        raise RuntimeError(lib.vr_last_error().decode())
    return out, lse


def ref_backward_fused(q16, k16, v16, dout16, lse, causal, br=64, bc=64, scale=0.0):
    B, H, N, d = q16.shape
    dq = np.empty((B, H, N, d), np.uint16)
    dk = np.empty_like(dq)
    dv = np.empty_like(dq)
    c = lambda a: np.ascontiguousarray(a, np.uint16)  # noqa: E731
    lib = ref_lib()
    rc = lib.vr_backward_fused(B, H, N, d, br, bc, int(causal), scale, c(q16), c(k16), c(v16), c(dout16),
                               np.ascontiguousarray(lse, np.float32), dq, dk, dv)
    if rc:
        raise RuntimeError(lib.vr_last_error().decode())
    return dq, dk, dv


def ref_attention_ref(q, k, v, causal, scale=0.0):
    B, H, N, d = q.shape
    out = np.empty((B, H, N, d), np.float64)
    lse = np.empty((B, H, N), np.float64)
    c = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
    rc = ref_lib().vr_attention_ref(B, H, N, d, int(causal), scale, c(q), c(k), c(v), out, lse)
    assert rc == 0
    return out, lse


def ref_attention_grad_ref(q, k, v, dout, causal, scale=0.0):
    B, H, N, d = q.shape
    dq = np.empty((B, H, N, d), np.float64)
    dk = np.empty_like(dq)
    dv = np.empty_like(dq)
    c = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
    rc = ref_lib().vr_attention_grad_ref(B, H, N, d, int(causal), scale, c(q), c(k), c(v), c(dout), dq, dk, dv)
    assert rc == 0
    return dq, dk, dv


def ref_normal_f16(seed, stream, count):
    out = np.empty(count, np.uint16)
    ref_lib().vr_normal_tensor_f16(seed, stream, count, out)
    return out


def ref_compute_dpsum(dout16, o16):
    B, H, N, d = dout16.shape
    out = np.empty((B, H, N), np.float32)
    c = lambda a: np.ascontiguousarray(a, np.uint16)  # noqa: E731
    rc = ref_lib().vr_compute_dpsum(B, H, N, d, c(dout16), c(o16), out)
    assert rc == 0
    return out


def ref_bench_units(N: int, d: int, causal: bool, units: int, threads: int) -> float:
    """Seconds for `units` x (forward_fused FP32-ACC + backward_fused) on `threads` host threads."""
    return float(ref_lib().vr_bench_units(N, d, int(causal), units, threads))


def ref_dropout_keep(seed, b, h, row, col, p) -> bool:
    return bool(ref_lib().vr_dropout_keep(seed, b, h, row, col, p))


def ref_forward_fused_dropout(q16, k16, v16, causal, dropout_p, seed, br=64, bc=64, acc_fp16=False, scale=0.0):
    B, H, N, d = q16.shape
    out = np.empty((B, H, N, d), np.uint16)
    lse = np.empty((B, H, N), np.float32)
    dig = C.c_uint64(0)
    c = lambda a: np.ascontiguousarray(a, np.uint16)  # noqa: E731
    lib = ref_lib()
    rc = lib.vr_forward_fused_dropout(B, H, N, d, br, bc, int(causal), int(acc_fp16), scale, dropout_p, seed,
                                      c(q16), c(k16), c(v16), out, lse, C.byref(dig))
    if rc:
        raise RuntimeError(lib.vr_last_error().decode())
    return out, lse, dig.value


def ref_backward_fused_dropout(q16, k16, v16, dout16, lse, causal, dropout_p, seed, br=64, bc=64, scale=0.0):
    B, H, N, d = q16.shape
    dq = np.empty((B, H, N, d), np.uint16)
    dk = np.empty_like(dq)
    dv = np.empty_like(dq)
    dig = C.c_uint64(0)
    c = lambda a: np.ascontiguousarray(a, np.uint16)  # noqa: E731
    lib = ref_lib()
    rc = lib.vr_backward_fused_dropout(B, H, N, d, br, bc, int(causal), scale, dropout_p, seed, c(q16), c(k16),
                                       c(v16), c(dout16), np.ascontiguousarray(lse, np.float32), dq, dk, dv,
                                       C.byref(dig))
    if rc:
        raise RuntimeError(lib.vr_last_error().decode())
    return dq, dk, dv, dig.value


def ref_attention_ref_dropout(q, k, v, causal, dropout_p, seed, scale=0.0):
    B, H, N, d = q.shape
    out = np.empty((B, H, N, d), np.float64)
    lse = np.empty((B, H, N), np.float64)
    c = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
    assert ref_lib().vr_attention_ref_dropout(B, H, N, d, int(causal), scale, dropout_p, seed, c(q), c(k), c(v),
                                              out, lse) == 0
    return out, lse


def ref_attention_grad_ref_dropout(q, k, v, dout, causal, dropout_p, seed, scale=0.0):
    B, H, N, d = q.shape
    dq = np.empty((B, H, N, d), np.float64)
    dk = np.empty_like(dq)
    dv = np.empty_like(dq)
    c = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
    assert ref_lib().vr_attention_grad_ref_dropout(B, H, N, d, int(causal), scale, dropout_p, seed, c(q), c(k),
                                                   c(v), c(dout), dq, dk, dv) == 0
    return dq, dk, dv


def ref_traffic_counts(which, B, H, N, d, br, bc, causal):
    """The reference library's TrafficCounter (7 fields) for a generated workload
    (ref_shim.cpp vr_traffic: 0/3 forward_fused FP32/FP16-ACC, 1/4 forward_traditional
    FP32/FP16-ACC, 2 backward_fused)."""
    out = (C.c_uint64 * 7)()
    rc = ref_lib().vr_traffic(which, B, H, N, d, br, bc, int(causal), out)
    if rc:
        raise RuntimeError(ref_lib().vr_last_error().decode())
    return tuple(out)
