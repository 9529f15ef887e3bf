"""JSON / CSV run reports in the reference's schema.

The reference's tool emits one JSON report per forward / backward run and a CSV
table per sweep (proj/tools/vattn_main.cpp:94-139 builders, :163-304 commands).
This module produces the same documents from the B200 path so a pipeline that
consumes them keeps working; the command-line front end itself is out of scope.

* ``forward_report`` -- vattn_main.cpp:163-201: ``command``, ``config``,
  ``paths.fused.{traffic, mask_digest}``, optionally ``paths.traditional`` and, when a
  checker is given, ``errors_vs_oracle`` per path and ``verify``.
* ``backward_report`` -- :203-249: ``forward`` / ``backward`` sections and
  ``mask_digest_match``; FP32-ACC is rejected exactly as the reference's tool does
  (the tool, not the library, owns that rule).
* ``sweep_csv`` -- :251-303: header + one CRLF-terminated row per (n, d, acc, causal).

Everything except the ``errors_vs_oracle`` numbers is a function of the config
(closed-form counters from ``traffic.py``; the dropout digest from the kernel-side
``vattn_dropout_digest``), so those parts are byte-identical to the reference's
reports.  Verification needs a binary64 checker; this package ships none (the
oracle is test infrastructure), so callers pass one in: ``reference(q, k, v, cfg)
-> out`` for forward, ``reference_grad(q, k, v, d_out, cfg) -> (dq, dk, dv)`` for
backward (numpy float64 arrays).  Tolerances are the tool's own
(vattn_main.cpp:31-33).
"""
from __future__ import annotations

import json
import math
from collections import OrderedDict
from dataclasses import replace

import numpy as np
import torch

from . import AttnConfig, backward_fused, dropout_digest, forward_fused
from . import traffic as tf
from . import traditional as tr
from .workload import normal_tensor_f16

FORWARD_TOL_FP32 = 5e-3  # kForwardTolFp32 (vattn_main.cpp:31)
FORWARD_TOL_FP16 = 2e-2  # kForwardTolFp16 (:32)
BACKWARD_TOL = 2e-2      # kBackwardTol, per gradient tensor (:33)

CSV_HEADER = ("n,d,acc,causal,seed,mean_rel,max_rel,mean_abs,max_abs,matrix_pass_reads,matrix_pass_writes,"
              "element_reads,element_writes,mma_invocations,shuffle_events,convert_events")


def _f32(x: float) -> float:
    """A binary32 config field as the reference's report prints it (widened to double)."""
    return float(np.float32(x))


def _acc(cfg: AttnConfig) -> str:
    return "fp16" if str(cfg.acc_mode).lower() in ("fp16", "fp16_acc") else "fp32"


def config_json(cfg: AttnConfig) -> OrderedDict:
    """config_json (vattn_main.cpp:94-106)."""
    return OrderedDict([("batch", cfg.batch), ("heads", cfg.heads), ("n", cfg.seq_len), ("d", cfg.head_dim),
                        ("br", cfg.tile_rows), ("bc", cfg.tile_cols), ("causal", bool(cfg.causal)),
                        ("dropout", _f32(cfg.dropout_p)), ("seed", int(cfg.seed)), ("acc", _acc(cfg)),
                        ("softmax_scale", _f32(cfg.scale()))])


def traffic_json(t: tf.TrafficCounter) -> OrderedDict:
    """traffic_json (vattn_main.cpp:108-116)."""
    return OrderedDict((f, int(getattr(t, f))) for f in tf.FIELDS)


def error_metrics(test, ref) -> OrderedDict:
    """vattn::error_metrics (proj/src/reference.cpp:186-202): relative error with the
    denominator floored at 1e-6, over every element, in binary64."""
    t = np.asarray(test, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    if t.shape != r.shape:
        raise ValueError("error_metrics: shape mismatch")
    a = np.abs(t - r)
    rel = a / np.maximum(np.abs(r), 1e-6)
    return OrderedDict([("mean_rel", float(rel.mean())), ("max_rel", float(rel.max())),
                        ("mean_abs", float(a.mean())), ("max_abs", float(a.max()))])


def hex64(v: int) -> str:
    """hex64 (vattn_main.cpp:125-129)."""
    return "0x%x" % (int(v) & ((1 << 64) - 1))


def dumps(report) -> str:
    """emit (vattn_main.cpp:131-139): two-space indented JSON plus a newline."""
    return json.dumps(report, indent=2) + "\n"


def _digest(cfg: AttnConfig, traditional: bool = False) -> int:
    return dropout_digest(cfg, traditional) if cfg.dropout_p > 0.0 else 0


def _inputs(cfg: AttnConfig, device: str = "cuda"):
    """load_or_generate (vattn_main.cpp:145-157): streams 1/2/3 of ``cfg.seed``."""
    dims = (cfg.batch, cfg.heads, cfg.seq_len, cfg.head_dim)
    return [normal_tensor_f16(cfg.seed, s, dims, device=device) for s in (1, 2, 3)]


def _np(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def forward_report(cfg: AttnConfig, q=None, k=None, v=None, with_traditional: bool = False, reference=None):
    """run_forward (vattn_main.cpp:163-201) -> (report, ok, out).

    ``q, k, v`` default to the generated workload; ``reference`` (optional binary64
    checker) turns on verification, which -- as in the reference -- also runs the
    traditional path."""
    cfg.validate()
    if q is None:
        q, k, v = _inputs(cfg)
    out, _ = forward_fused(q, k, v, cfg)
    report = OrderedDict([("command", "forward"), ("config", config_json(cfg))])
    paths = report["paths"] = OrderedDict()
    paths["fused"] = OrderedDict([("traffic", traffic_json(tf.forward_fused_traffic(cfg))),
                                  ("mask_digest", hex64(_digest(cfg)))])
    ok = True
    if with_traditional or reference is not None:
        out_t, _ = tr.forward_traditional(q, k, v, cfg.causal, cfg.scale(), cfg.dropout_p, cfg.seed)
        paths["traditional"] = OrderedDict([("traffic", traffic_json(tf.forward_traditional_traffic(cfg))),
                                            ("mask_digest", hex64(_digest(cfg, traditional=True)))])
        if reference is not None:
            ref = np.asarray(reference(q, k, v, cfg), dtype=np.float64)
            mf, mt = error_metrics(_np(out), ref), error_metrics(_np(out_t), ref)
            paths["fused"]["errors_vs_oracle"] = mf
            paths["traditional"]["errors_vs_oracle"] = mt
            tol = FORWARD_TOL_FP16 if _acc(cfg) == "fp16" else FORWARD_TOL_FP32
            report["verify"] = OrderedDict([("tolerance_mean_rel", tol), ("fused_pass", mf["mean_rel"] <= tol),
                                            ("traditional_pass", mt["mean_rel"] <= 2.0 * tol)])
            ok = mf["mean_rel"] <= tol and mt["mean_rel"] <= 2.0 * tol
    return report, ok, out


def backward_report(cfg: AttnConfig, acc_explicit: bool = False, reference_grad=None):
    """run_backward (vattn_main.cpp:203-249) -> (report, ok, (dq, dk, dv)).

    The tool forces FP16-ACC (the reference backward's only mode) and rejects an
    explicit FP32-ACC request with ``ValueError`` (its exit code 2)."""
    if acc_explicit and _acc(cfg) == "fp32":
        raise ValueError("backward: only FP16-ACC is supported")
    cfg = replace(cfg, acc_mode="fp16")
    cfg.validate()
    q, k, v = _inputs(cfg)
    dout = normal_tensor_f16(cfg.seed, 4, q.shape, device=q.device)
    out, lse = forward_fused(q, k, v, cfg)
    dq, dk, dv = backward_fused(q, k, v, dout, lse, cfg, out=out)
    fwd_digest, bwd_digest = _digest(cfg), _digest(cfg)  # same visited positions, same hash
    report = OrderedDict([("command", "backward"), ("config", config_json(cfg))])
    report["forward"] = OrderedDict([("traffic", traffic_json(tf.forward_fused_traffic(cfg))),
                                     ("mask_digest", hex64(fwd_digest))])
    report["backward"] = OrderedDict([("traffic", traffic_json(tf.backward_fused_traffic(cfg))),
                                      ("mask_digest", hex64(bwd_digest))])
    report["mask_digest_match"] = fwd_digest == bwd_digest
    ok = True
    if reference_grad is not None:
        rq, rk, rv = (np.asarray(x, dtype=np.float64) for x in reference_grad(q, k, v, dout, cfg))
        m = OrderedDict([("dq", error_metrics(_np(dq), rq)), ("dk", error_metrics(_np(dk), rk)),
                         ("dv", error_metrics(_np(dv), rv))])
        report["backward"]["errors_vs_oracle"] = m
        ok = all(x["mean_rel"] <= BACKWARD_TOL for x in m.values()) and fwd_digest == bwd_digest
        report["verify"] = OrderedDict([("tolerance_mean_rel", BACKWARD_TOL), ("pass", ok)])
    return report, ok, (dq, dk, dv)


def _fmt(x) -> str:
    """A CSV cell as std::ostream prints it (default floatfield, precision 6)."""
    if isinstance(x, bool):
        return str(int(x))
    if isinstance(x, float):
        if x == 0.0:
            return "0"
        if math.isinf(x) or math.isnan(x):
            return ("-" if x < 0 else "") + ("inf" if math.isinf(x) else "nan")
        return "%g" % x
    return str(x)


def sweep_csv(n_list, d_list, acc_list=("fp32",), causal_list=(0,), seed: int = 1, reference=None):
    """run_sweep (vattn_main.cpp:251-303) -> (csv_text, ok): one forward per grid point
    at batch = heads = 1, tiles min(64, n); error columns are 0 without a checker."""
    if not n_list or not d_list or not acc_list or not causal_list:
        raise ValueError("sweep: empty parameter list")
    rows = [CSV_HEADER]
    ok = True
    for n in n_list:
        for d in d_list:
            for acc in acc_list:
                for causal in causal_list:
                    cfg = AttnConfig(batch=1, heads=1, seq_len=int(n), head_dim=int(d), tile_rows=min(64, int(n)),
                                     tile_cols=min(64, int(n)), causal=bool(causal), seed=seed, acc_mode=acc)
                    cfg.validate()
                    m = OrderedDict([("mean_rel", 0.0), ("max_rel", 0.0), ("mean_abs", 0.0), ("max_abs", 0.0)])
                    if reference is not None:
                        q, k, v = _inputs(cfg)
                        out, _ = forward_fused(q, k, v, cfg)
                        m = error_metrics(_np(out), reference(q, k, v, cfg))
                        tol = FORWARD_TOL_FP16 if _acc(cfg) == "fp16" else FORWARD_TOL_FP32
                        ok = ok and m["mean_rel"] <= tol
                    t = tf.forward_fused_traffic(cfg)
                    cells = [n, d, _acc(cfg), int(causal), seed, *m.values(), *t.as_tuple()]
                    rows.append(",".join(_fmt(c) for c in cells))
    return "".join(r + "\r\n" for r in rows), ok
