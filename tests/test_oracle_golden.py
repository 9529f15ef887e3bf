"""CPU: pin the C restatement (oracle/vattn_oracle.c) to the reference's own outputs.

The fixtures in tests/golden/ were produced by the unmodified reference
(oracle/gen_golden.py -> oracle/_ref).  Every comparison here is bit-exact.
"""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as po

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MANIFEST = json.load(open(os.path.join(GOLDEN, "manifest.json")))["cases"]
IDS = [c["name"] for c in MANIFEST]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def test_normal_generator_matches_reference():
    g = load("normals_seed1")
    for s in (1, 2, 3, 4):
        ours = po.normal16(1, s, (256,))
        assert np.array_equal(ours, g[f"stream{s}"]), s


@pytest.mark.parametrize("case", MANIFEST, ids=IDS)
def test_inputs_regenerate_bitwise(case):
    g = load(case["name"])
    shape = tuple(case["shape"])
    for stream, key in enumerate(("q", "k", "v", "dout"), start=1):
        assert np.array_equal(po.normal16(case["seed"], stream, shape), g[key]), key


@pytest.mark.parametrize("case", MANIFEST, ids=IDS)
def test_forward_fused_fp32acc_restatement_bitexact(case):
    g = load(case["name"])
    br, bc = case["tiles"]
    out, lse = po.forward_fused_fp32acc(g["q"], g["k"], g["v"], case["causal"], br, bc)
    assert np.array_equal(out, g["fwd32_out"])
    assert np.array_equal(lse.view(np.uint32), g["fwd32_lse"].view(np.uint32))


@pytest.mark.parametrize("case", MANIFEST, ids=IDS)
def test_binary64_oracle_restatement_bitexact(case):
    g = load(case["name"])
    q, k, v, do = (po.widen(g[x]) for x in ("q", "k", "v", "dout"))
    out, lse = po.attention_ref(q, k, v, case["causal"])
    assert np.array_equal(out, g["ref_out"])
    assert np.array_equal(lse, g["ref_lse"])
    dq, dk, dv = po.attention_grad_ref(q, k, v, do, case["causal"])
    assert np.array_equal(dq, g["ref_dq"])
    assert np.array_equal(dk, g["ref_dk"])
    assert np.array_equal(dv, g["ref_dv"])


@pytest.mark.parametrize("case", MANIFEST, ids=IDS)
def test_compute_dpsum_restatement_bitexact(case):
    g = load(case["name"])
    d = po.compute_dpsum(g["dout"], g["fwd32_out"])
    assert np.array_equal(d.view(np.uint32), g["dpsum_fwd32"].view(np.uint32))


def test_dpsum_examples():
    """test_backward.cpp:172-199: 30.0 exact and orthogonal rows 0 exact."""
    a = np.zeros((1, 1, 2, 4), np.uint16)
    b = np.zeros((1, 1, 2, 4), np.uint16)
    for j in range(4):
        a[0, 0, 0, j] = po.oracle_lib().vo_f32_to_f16(float(j + 1))
        b[0, 0, 0, j] = po.oracle_lib().vo_f32_to_f16(float(j + 1))
    a[0, 0, 1, 0] = po.oracle_lib().vo_f32_to_f16(1.0)
    b[0, 0, 1, 1] = po.oracle_lib().vo_f32_to_f16(1.0)
    d = po.compute_dpsum(a, b)
    assert d[0, 0, 0] == 30.0 and d[0, 0, 1] == 0.0


def test_half_rounding_edge_cases():
    """half.cpp:5-44 RNE contract: ties to even, overflow to inf, subnormals kept."""
    f = po.oracle_lib().vo_f32_to_f16
    assert f(1.0) == 0x3C00
    assert f(65504.0) == 0x7BFF
    assert f(65520.0) == 0x7C00  # rounds up to inf
    assert f(2.0 ** -24) == 0x0001  # smallest subnormal
    assert f(2.0 ** -25) == 0x0000  # tie to even -> 0
    assert f(1.0 + 2.0 ** -11) == 0x3C00  # tie to even
    assert f(1.0 + 3 * 2.0 ** -11) == 0x3C02
    assert po.oracle_lib().vo_f32_to_bf16(1.0 + 2.0 ** -8) == 0x3F80  # bf16 tie to even


def test_oracle_self_validation_finite_differences():
    """reference.cpp:169-184 / acceptance criterion 4: analytic grads vs central differences."""
    rng = np.random.default_rng(0)
    B, H, N, d = 1, 1, 8, 4
    q, k, v, do = (rng.standard_normal((B, H, N, d)) for _ in range(4))
    for causal in (False, True):
        dq, dk, dv = po.attention_grad_ref(q, k, v, do, causal)
        f = lambda qq, kk, vv: float((po.attention_ref(qq, kk, vv, causal)[0] * do).sum())  # noqa: E731
        eps = 1e-6
        for which, grad in ((0, dq), (1, dk), (2, dv)):
            base = [q, k, v]
            num = np.zeros_like(grad)
            for idx in np.ndindex(grad.shape):
                plus = [x.copy() for x in base]
                minus = [x.copy() for x in base]
                plus[which][idx] += eps
                minus[which][idx] -= eps
                num[idx] = (f(*plus) - f(*minus)) / (2 * eps)
            assert np.max(np.abs(num - grad)) <= 1e-6 * max(1.0, np.max(np.abs(grad))) * 10


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")
def test_restatement_matches_live_reference_random_config():
    """Cross-check against the live reference on a config not in the fixtures."""
    shape = (1, 3, 96, 24)
    q, k, v = (po.normal16(42, s, shape) for s in (1, 2, 3))
    for causal in (False, True):
        a = po.forward_fused_fp32acc(q, k, v, causal, 32, 48)
        b = po.ref_forward_fused(q, k, v, causal, 32, 48)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


# ---------------------------------------------------------------- dropout --
DROP = json.load(open(os.path.join(GOLDEN, "manifest.json")))["dropout_cases"]


def test_dropout_keep_matches_reference_grid():
    """rng.cpp:46-49 restated bit-exactly (seed 42, p 0.5, b 0, h 1)."""
    g = load("dropout_keep_seed42")["keep"]
    ours = np.array([[po.dropout_keep(42, 0, 1, i, j, 0.5) for j in range(64)] for i in range(64)], np.uint8)
    assert np.array_equal(ours, g)
    assert po.dropout_keep(42, 0, 1, 2, 3, 0.0)  # p = 0 short-circuit (test_forward.cpp:227)


def test_dropout_keep_rate():
    """acceptance criterion 9: keep rate 0.9 +/- 0.002 at p = 0.1 (sampled)."""
    kept = sum(po.dropout_keep(42, 0, 0, i // 300, i % 300, 0.1) for i in range(90000))
    assert abs(kept / 90000 - 0.9) <= 0.004


@pytest.mark.parametrize("case", DROP, ids=[c["name"] for c in DROP])
def test_dropout_restatements_bitexact(case):
    g = load(case["name"])
    p, ds = case["dropout_p"], case["dropout_seed"]
    br, bc = case["tiles"]
    N = case["shape"][2]
    mask = np.array([[po.dropout_keep(ds, 0, 0, i, j, p) for j in range(N)] for i in range(N)], np.uint8)
    assert np.array_equal(mask, g["mask_b0h0"])
    out, lse = po.forward_fused_fp32acc(g["q"], g["k"], g["v"], case["causal"], br, bc, dropout_p=p, seed=ds)
    assert np.array_equal(out, g["fwd32_out"])
    assert np.array_equal(lse.view(np.uint32), g["fwd32_lse"].view(np.uint32))
    q, k, v, do = (po.widen(g[x]) for x in ("q", "k", "v", "dout"))
    o, l = po.attention_ref(q, k, v, case["causal"], dropout_p=p, seed=ds)
    assert np.array_equal(o, g["ref_out"]) and np.array_equal(l, g["ref_lse"])
    dq, dk, dv = po.attention_grad_ref(q, k, v, do, case["causal"], dropout_p=p, seed=ds)
    assert np.array_equal(dq, g["ref_dq"]) and np.array_equal(dk, g["ref_dk"]) and np.array_equal(dv, g["ref_dv"])
