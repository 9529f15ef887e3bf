"""Closed-form modeled-HBM traffic of the reference's passes.

The reference fills ``ForwardOutput.traffic`` / ``GradOutputs.traffic`` (a
``vattn::TrafficCounter``, proj/include/vattn/traffic.hpp:12-31) while it
emulates the tiles.  The GPU path does not emulate anything, so the counters are
restated here in closed form from the reference's own bookkeeping and reported by
the operator API; tests pin them to the reference library's counters.

* ``forward_fused`` (attention.hpp:40-50, attention_forward.cpp:110-227): 3 pass
  reads / 1 write; per (b, h): reads = N d + 2 Bc d T, writes = N d + N, with T the
  visited (query-tile, key-tile) pairs (causal: key tile kt is visited by query tile
  qt iff kt Bc <= qt Br + Br - 1, attention_forward.cpp:128).
* ``forward_traditional`` (attention.hpp:54-58): 5 / 3 passes; per (b, h):
  reads = 2 N d + N^2 + N^2 + N d, writes = N^2 + N^2 + N d + N.
* ``backward_fused`` (attention_backward.cpp:59-219): 10 / 5 passes; the forward
  recompute pre-pass (reads N d + 2 Bc d T), D written (N), then per key tile K, V
  (2 Bc d), per visited (kt, qt) Q, dO (2 Br d) + lse, D (2 Br) read and a dQ
  atomic add (Br d) written, dK, dV stored (2 Bc d), and the dQ finalisation
  (N d read + N d written).

``mma_invocations``, ``shuffle_events`` and ``convert_events`` count Volta
m8n8k4 / warp-shuffle / fp16<->fp32 conversion events of the emulated datapath,
which has no counterpart on Blackwell (out of scope); they are 0 here.
Measured DRAM bytes of the B200 kernels are in profiles/*_ncu_full_*.md.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass

FIELDS = ("matrix_pass_reads", "matrix_pass_writes", "element_reads", "element_writes",
          "mma_invocations", "shuffle_events", "convert_events")


@dataclass
class TrafficCounter:
    matrix_pass_reads: int = 0
    matrix_pass_writes: int = 0
    element_reads: int = 0
    element_writes: int = 0
    mma_invocations: int = 0
    shuffle_events: int = 0
    convert_events: int = 0

    def as_tuple(self):
        return tuple(getattr(self, f) for f in FIELDS)

    def as_dict(self):
        return asdict(self)


def visited_pairs(N: int, br: int, bc: int, causal: bool) -> int:
    """(query-tile, key-tile) pairs a fused pass visits for one (b, h)."""
    nq, nk = N // br, N // bc
    if not causal:
        return nq * nk
    return sum(min(nk, (qt * br + br - 1) // bc + 1) for qt in range(nq))


def _dims(cfg):
    return cfg.batch * cfg.heads, cfg.seq_len, cfg.head_dim, cfg.tile_rows, cfg.tile_cols, bool(cfg.causal)


def forward_fused_traffic(cfg) -> TrafficCounter:
    BH, N, d, br, bc, causal = _dims(cfg)
    T = visited_pairs(N, br, bc, causal)
    return TrafficCounter(3, 1, BH * (N * d + 2 * bc * d * T), BH * (N * d + N))


def forward_traditional_traffic(cfg) -> TrafficCounter:
    BH, N, d, _, _, _ = _dims(cfg)
    return TrafficCounter(5, 3, BH * (3 * N * d + 2 * N * N), BH * (2 * N * N + N * d + N))


def backward_fused_traffic(cfg) -> TrafficCounter:
    BH, N, d, br, bc, causal = _dims(cfg)
    T = visited_pairs(N, br, bc, causal)
    nk = N // bc
    reads = (N * d + 2 * bc * d * T) + 2 * bc * d * nk + T * (2 * br * d + 2 * br) + N * d
    writes = N + T * br * d + 2 * bc * d * nk + N * d
    return TrafficCounter(10, 5, BH * reads, BH * writes)
