"""SPAT tensor container: the reference's file format for moving
golden tensors between hosts (proj/include/vattn/tensor_io.hpp:9-29,
proj/src/tensor_io.cpp).  Layout: magic "SPAT", u8 version (1), u8 dtype code
(0 binary16, 1 binary32, 2 binary64), u8 rank (1..8), little-endian u64 dims, then
the little-endian payload.  Errors follow the reader's std::runtime_error cases
(bad magic / version / dtype / rank, zero or overflowing dims, truncated or trailing
bytes) as RuntimeError.  bf16 has no SPAT code (the reference is binary16-only):
bf16 tensors are refused rather than silently reinterpreted.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"SPAT"
VERSION = 1
_CODES = {np.dtype(np.float16): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}
_DTYPES = {0: np.dtype("<f2"), 1: np.dtype("<f4"), 2: np.dtype("<f8")}


def _to_numpy(t):
    try:
        import torch
        if isinstance(t, torch.Tensor):
            if t.dtype == torch.bfloat16:
                raise ValueError("write_spat: bf16 has no SPAT dtype code (binary16/32/64 only)")
            t = t.detach().cpu().numpy()
    except ImportError:
        pass
    return np.ascontiguousarray(t)


def write_spat(path: str, t) -> None:
    a = _to_numpy(t)
    if a.dtype not in _CODES:
        raise ValueError(f"write_spat: unsupported dtype {a.dtype}")
    if not 1 <= a.ndim <= 8:
        raise ValueError("write_spat: rank must be 1..8")
    with open(path, "wb") as f:
        f.write(MAGIC + bytes([VERSION, _CODES[a.dtype], a.ndim]))
        f.write(b"".join(struct.pack("<Q", int(s)) for s in a.shape))
        f.write(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes())


def read_spat(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 4 or data[:4] != MAGIC:
        raise RuntimeError(f"read_spat: bad magic in {path}")
    if len(data) < 7 or data[4] != VERSION:
        raise RuntimeError("read_spat: unsupported version")
    code, rank = data[5], data[6]
    if code > 2:
        raise RuntimeError("read_spat: unknown dtype code")
    if not 1 <= rank <= 8:
        raise RuntimeError("read_spat: unsupported rank")
    if len(data) < 7 + 8 * rank:
        raise RuntimeError("read_spat: truncated header")
    dims = struct.unpack_from(f"<{rank}Q", data, 7)
    count = 1
    for d in dims:
        if d == 0:
            raise RuntimeError("read_spat: zero dimension")
        count *= d
        if count > (1 << 40):
            raise RuntimeError("read_spat: dimension overflow")
    dt = _DTYPES[code]
    off = 7 + 8 * rank
    need = count * dt.itemsize
    if len(data) - off < need:
        raise RuntimeError("read_spat: truncated payload")
    if len(data) - off > need:
        raise RuntimeError("read_spat: trailing bytes after payload")
    return np.frombuffer(data, dtype=dt, count=count, offset=off).reshape(dims).astype(dt.newbyteorder("="))
