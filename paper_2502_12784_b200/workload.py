"""The reference's synthetic workload generator (SURVEY 8d "Synthetic inputs").

``normal_tensor_f16(seed, stream, dims)`` restates ``vattn::normal_tensor_f16``
(proj/include/vattn/workload.hpp:10-17) over ``vattn::normal_at``
(proj/src/rng.cpp:23-31): element i is a Box-Muller draw over two SplitMix64
counter hashes of ``hash_combine(seed, stream)``, narrowed to binary32 and then
RNE to binary16.  Streams 1/2/3/4 are Q/K/V/dO.  ``bf16=True`` rounds the same
binary32 normals to bfloat16 (RNE), the convention SURVEY 8d fixes for bf16
configs, which have no reference counterpart.

Vectorised numpy on the host: it produces test/report inputs, it is not on the
timed path (bench.py generates throughput inputs on the device).  Pinned
bit-for-bit to the reference library by tests/test_reports.py.
"""
from __future__ import annotations

import numpy as np
import torch

_M = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def mix64(x):
    """SplitMix64 finaliser (rng.cpp:8-13); uint64 arrays wrap modulo 2^64."""
    x = x + _GOLDEN
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def hash_combine(state, v):
    """rng.cpp:15-17."""
    state = np.uint64(state) if np.isscalar(state) else state
    return mix64(state ^ (v + _GOLDEN + (state << np.uint64(6)) + (state >> np.uint64(2))))


def _unit(bits):
    """bits_to_unit (rng.cpp:19-21): upper 53 bits to [0, 1)."""
    return (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def normal_f32(seed: int, stream: int, count: int, chunk: int = 1 << 22) -> np.ndarray:
    """normal_at(hash_combine(seed, stream), i) for i < count, as binary32."""
    with np.errstate(over="ignore"):
        base = hash_combine(np.uint64(seed), np.uint64(stream))
        out = np.empty(count, dtype=np.float32)
        for s in range(0, count, chunk):
            i = np.arange(s, min(count, s + chunk), dtype=np.uint64)
            a = mix64(hash_combine(base, np.uint64(2) * i))
            b = mix64(hash_combine(base, np.uint64(2) * i + np.uint64(1)))
            u1 = 1.0 - _unit(a)
            u2 = _unit(b)
            out[s:s + len(i)] = (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).astype(np.float32)
    return out


def normal_tensor_f16(seed: int, stream: int, dims, bf16: bool = False, device=None) -> torch.Tensor:
    """vattn::normal_tensor_f16 as a torch tensor (fp16, or bf16 with ``bf16=True``)."""
    dims = tuple(int(x) for x in dims)
    x = torch.from_numpy(normal_f32(seed, stream, int(np.prod(dims)))).reshape(dims)
    x = x.to(torch.bfloat16 if bf16 else torch.float16)
    return x.to(device) if device is not None else x
