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

``mma_invocations``, ``shuffle_events`` and ``convert_events`` count the events
of the reference's emulated Volta datapath.  The B200 kernels do not execute that
datapath, but the counts are pure functions of the config, so they are restated
too (the reports of ``reports.py`` then equal the reference's field for field):

* one m8n8k4 invocation per (k-step of 4, 8-row band, chunk of four 8-column
  sub-tiles) of a tile GEMM C[rows x cols] += A[rows x k] B[k x cols]
  (tile_pipeline.cpp:36-49, tile_pipeline.hpp:24-33): (k/4)(rows/8)ceil(cols/32);
  P.V and dS.K run on the head dim padded to 8 (``pad8``);
* forward, per visited pair: S = Q K^T and O += P V; FP32-ACC adds 2 Br/8 xor
  shuffle rounds (attention_forward.cpp:147-148), FP16-ACC converts S, O (twice)
  and P (:136-137, :151-152, :164-165);
* backward (FP16-ACC only), per visited pair: S, dV, dP, dQ, dK GEMMs and four
  Br Bc conversions (attention_backward.cpp:132-199), on top of the FP16-ACC
  forward pre-pass (:93-103);
* traditional: S = Q K^T and O = P V on the whole N x N tile, no events
  (attention_forward.cpp:253-300).
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


def _fp16_acc(cfg) -> bool:
    return str(getattr(cfg, "acc_mode", "fp32")).lower() in ("fp16", "fp16_acc")


def pad8(d: int) -> int:
    """detail::pad8: head dim rounded up to a multiple of 8."""
    return (d + 7) // 8 * 8


def mma_count(rows: int, cols: int, k: int) -> int:
    """m8n8k4 invocations of one tile GEMM (tile_pipeline.cpp:36-49)."""
    return (k // 4) * (rows // 8) * ((cols // 8 + 3) // 4)


def _forward_events(br, bc, d, T, fp16_acc):
    """(mma, shuffles, converts) of T visited forward pairs (attention_forward.cpp:126-173)."""
    mma = T * (mma_count(br, bc, d) + mma_count(br, pad8(d), bc))
    if fp16_acc:
        return mma, 0, T * (2 * br * bc + 2 * br * d)
    return mma, T * 2 * (br // 8), 0


def forward_fused_traffic(cfg) -> TrafficCounter:
    BH, N, d, br, bc, causal = _dims(cfg)
    T = visited_pairs(N, br, bc, causal)
    mma, shf, cvt = _forward_events(br, bc, d, T, _fp16_acc(cfg))
    return TrafficCounter(3, 1, BH * (N * d + 2 * bc * d * T), BH * (N * d + N), BH * mma, BH * shf, BH * cvt)


def forward_traditional_traffic(cfg) -> TrafficCounter:
    BH, N, d, _, _, _ = _dims(cfg)
    mma = mma_count(N, N, d) + mma_count(N, pad8(d), N)
    return TrafficCounter(5, 3, BH * (3 * N * d + 2 * N * N), BH * (2 * N * N + N * d + N), BH * mma)


def backward_fused_traffic(cfg) -> TrafficCounter:
    BH, N, d, br, bc, causal = _dims(cfg)
    T = visited_pairs(N, br, bc, causal)
    nk = N // bc
    reads = (N * d + 2 * bc * d * T) + 2 * bc * d * nk + T * (2 * br * d + 2 * br) + N * d
    writes = N + T * br * d + 2 * bc * d * nk + N * d
    pre_mma, _, pre_cvt = _forward_events(br, bc, d, T, True)  # the FP16-ACC recompute pre-pass
    dp = pad8(d)
    mma = pre_mma + T * (2 * mma_count(br, bc, d) + 2 * mma_count(bc, dp, br) + mma_count(br, dp, bc))
    cvt = pre_cvt + T * 4 * br * bc
    return TrafficCounter(10, 5, BH * reads, BH * writes, BH * mma, 0, BH * cvt)


# ------------------------------------------- closed forms vs measured DRAM bytes --
# the reference's element-traffic closed forms (attention.hpp:40-58,
# attention_backward.cpp:59-219) turned into BYTES (16-bit tensors 2 B, lse / D and the
# fp32 dQ partials 4 B) so they can be set beside the DRAM bytes ncu measures for the
# B200 kernels (profiles/ncu_traffic.json).  The closed forms model a cache-less HBM:
# every K / V (or Q / dO) tile is re-read for every visited tile pair, so they are the
# upper bound a kernel reaches only when no tile survives in L2; the algorithmic minimum
# reads and writes every tensor exactly once.

def fused_forward_hbm_bytes(cfg) -> dict:
    """Closed-form (cache-less) and minimum HBM bytes of the fused forward."""
    BH, N, d, br, bc, causal = _dims(cfg)
    T = visited_pairs(N, br, bc, causal)
    closed = BH * (2 * (N * d + 2 * bc * d * T) + 2 * N * d + 4 * N)
    minimum = BH * (2 * 4 * N * d + 4 * N)  # Q, K, V read, O written (16-bit) + lse (f32)
    return {"closed_form": closed, "minimum": minimum, "visited_pairs_per_bh": T}


def fused_backward_hbm_bytes(cfg) -> dict:
    """Closed-form bytes of the reference's backward without its forward pre-pass (the
    B200 backward takes O; its D kernel reads O and dO instead): D (N f32) written; per
    key tile K, V read and dK, dV written; per visited pair Q, dO (16-bit) and lse, D (f32)
    read and a Br x d fp32 dQ partial reduce-added; dQ finalised (read f32, write 16-bit).
    Minimum: Q, K, V, O, dO read, dQ, dK, dV written once, lse read, D round trip."""
    BH, N, d, br, bc, causal = _dims(cfg)
    T = visited_pairs(N, br, bc, causal)
    nk = N // bc
    reads = 2 * (2 * N * d) + 2 * (2 * bc * d * nk) + T * (2 * 2 * br * d + 4 * 2 * br) + 4 * N * d
    writes = 4 * N + 2 * (2 * bc * d * nk) + T * 4 * br * d + 2 * N * d
    closed = BH * (reads + writes)
    minimum = BH * (2 * 5 * N * d + 2 * 3 * N * d + 4 * N + 4 * N * 2)
    return {"closed_form": closed, "minimum": minimum, "visited_pairs_per_bh": T}


def b200_hbm_model(cfg) -> dict:
    """Per-kernel DRAM bytes of the B200 path (d = 128 dS-materialised backward) under two
    caching extremes, for the cross-check against ncu (tools/traffic_crosscheck.py):

    * ``l2_reuse``: every tensor crosses HBM exactly once per kernel (K / V / Q / dO
      re-reads across CTAs all hit the 126 MB L2) -- the kernel's algorithmic bytes,
      plus the dS^T tiles the dK/dV kernel writes and the dQ GEMM reads back (16-bit,
      128 x 128 per visited (query tile, key tile) pair);
    * ``cache_less``: the reference's closed-form accounting (attention.hpp:40-58):
      every visited tile pair re-reads its streamed operand tiles from HBM.

    Tile sizes are the B200 kernels' own: the forward CTA covers 256 query rows against
    128-key tiles, the backward 128 x 128."""
    BH, N, d = cfg.batch * cfg.heads, cfg.seq_len, cfg.head_dim
    causal = bool(cfg.causal)
    T = visited_pairs(N, 128, 128, causal)           # backward tile pairs per (b, h)
    Tf = visited_pairs(N, 256, 128, causal)          # forward (256-row CTA) pairs per (b, h)
    nd2 = 2 * N * d                                  # one 16-bit [N, d] tensor
    ds = T * 128 * 128 * 2
    out = {
        "fwd": {"l2_reuse": BH * (4 * nd2 + 4 * N),                       # Q, K, V in, O out, lse
                "cache_less": BH * (nd2 + Tf * 2 * 128 * d * 2 + nd2 + 4 * N)},
        "bwd_preprocess": {"l2_reuse": BH * (2 * nd2 + 4 * N + 8 * N),    # O, dO, lse in; D, lse2 out
                           "cache_less": BH * (2 * nd2 + 4 * N + 8 * N)},
        "bwd_dkdv": {"l2_reuse": BH * (4 * nd2 + 8 * N + 2 * nd2 + ds),   # K V Q dO, lse2 D, dK dV, dS^T
                     "cache_less": BH * (2 * nd2 + T * (2 * 128 * d * 2 + 8 * 128) + 2 * nd2 + ds)},
        "bwd_dq_gemm": {"l2_reuse": BH * (ds + nd2 + nd2),                # dS^T, K in; dQ out
                        "cache_less": BH * (ds + T * 128 * d * 2 + nd2)},
    }
    return out
