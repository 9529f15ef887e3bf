"""CPU: SURVEY 8f-4 -- the TrafficCounter closed forms and the SPAT container,
pinned to the unmodified reference library (oracle/_ref, test infrastructure)."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_2502_12784_b200 import AttnConfig, spat
from paper_2502_12784_b200 import traffic as tf

need_ref = pytest.mark.skipif(not po.ref_available(), reason="reference library not built here")


def ref_traffic(which, B, H, N, d, br, bc, causal):
    out = (C.c_uint64 * 7)()
    rc = po.ref_lib().vr_traffic(which, B, H, N, d, br, bc, int(causal), out)
    assert rc == 0, po.ref_lib().vr_last_error()
    return tuple(out)


CASES = [(1, 1, 64, 32, 16, 16, False), (1, 1, 64, 32, 16, 16, True), (2, 3, 128, 64, 64, 32, True),
         (1, 2, 96, 16, 32, 16, True), (1, 2, 96, 16, 16, 32, False), (2, 1, 64, 8, 64, 64, True),
         (1, 1, 80, 12, 16, 40, True), (1, 2, 120, 20, 40, 24, False)]  # d not a multiple of 8, odd chunks


@need_ref
@pytest.mark.parametrize("B,H,N,d,br,bc,causal", CASES)
def test_traffic_closed_forms_match_reference(B, H, N, d, br, bc, causal):
    """All seven counters, both accumulation modes, equal the reference library's."""
    for acc, cases in (("fp32", ((0, tf.forward_fused_traffic), (1, tf.forward_traditional_traffic))),
                       ("fp16", ((3, tf.forward_fused_traffic), (4, tf.forward_traditional_traffic),
                                 (2, tf.backward_fused_traffic)))):
        cfg = AttnConfig(batch=B, heads=H, seq_len=N, head_dim=d, tile_rows=br, tile_cols=bc, causal=causal,
                         acc_mode=acc)
        for which, fn in cases:
            ref = ref_traffic(which, B, H, N, d, br, bc, causal)
            assert fn(cfg).as_tuple() == ref, (which, acc, fn(cfg).as_tuple(), ref)


def test_traffic_causal_halves_visits():
    assert tf.visited_pairs(1024, 64, 64, False) == 256
    assert tf.visited_pairs(1024, 64, 64, True) == 16 * 17 // 2


@pytest.mark.parametrize("arr", [
    np.arange(24, dtype=np.float16).reshape(2, 3, 4) / 7,
    np.linspace(-3, 3, 30, dtype=np.float32).reshape(5, 6),
    np.array([1e-310, -0.0, np.inf], dtype=np.float64),
])
def test_spat_round_trip(tmp_path, arr):
    p = str(tmp_path / "t.spat")
    spat.write_spat(p, arr)
    back = spat.read_spat(p)
    assert back.dtype == arr.dtype and back.shape == arr.shape
    assert np.array_equal(back.view(np.uint8), np.ascontiguousarray(arr).view(np.uint8))


@need_ref
def test_spat_bytes_identical_to_reference(tmp_path):
    bits = po.normal16(1, 1, (1, 2, 8, 4))
    dims = (C.c_uint64 * 4)(1, 2, 8, 4)
    ref_p, our_p = str(tmp_path / "ref.spat"), str(tmp_path / "our.spat")
    assert po.ref_lib().vr_write_spat_f16(ref_p.encode(), 4, dims, np.ascontiguousarray(bits, np.uint16)) == 0
    spat.write_spat(our_p, bits.view(np.float16))
    assert open(ref_p, "rb").read() == open(our_p, "rb").read()
    f32 = np.random.default_rng(0).standard_normal((3, 5)).astype(np.float32)
    d2 = (C.c_uint64 * 2)(3, 5)
    assert po.ref_lib().vr_write_spat_f32(ref_p.encode(), 2, d2, f32) == 0
    spat.write_spat(our_p, torch.from_numpy(f32))
    assert open(ref_p, "rb").read() == open(our_p, "rb").read()
    assert po.ref_lib().vr_read_spat_check(our_p.encode()) == 0


@need_ref
def test_spat_errors_match_reference(tmp_path):
    good = str(tmp_path / "g.spat")
    spat.write_spat(good, np.ones((2, 2), np.float32))
    raw = open(good, "rb").read()
    bad = {
        "magic": b"SPAX" + raw[4:],
        "version": raw[:4] + b"\x02" + raw[5:],
        "dtype": raw[:5] + b"\x07" + raw[6:],
        "rank": raw[:6] + b"\x00" + raw[7:],
        "zero_dim": raw[:7] + (0).to_bytes(8, "little") + raw[15:],
        "truncated": raw[:-1],
        "trailing": raw + b"\x00",
    }
    for name, blob in bad.items():
        p = str(tmp_path / f"{name}.spat")
        open(p, "wb").write(blob)
        assert po.ref_lib().vr_read_spat_check(p.encode()) == 9, name  # std::runtime_error
        with pytest.raises(RuntimeError):
            spat.read_spat(p)
    with pytest.raises(ValueError):
        spat.write_spat(str(tmp_path / "bf.spat"), torch.zeros(2, dtype=torch.bfloat16))


def test_f4_closed_forms_bracket_ncu_dram_bytes():
    """the measured DRAM bytes of every B200 kernel (profiles/ncu_traffic.json,
    one ncu --set full launch each) lie between 'every tensor once' (minus 2 % for ncu's
    sector granularity) and the reference's cache-less closed form (attention.hpp:40-58)."""
    import json
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tools"))
    import traffic_crosscheck as tc
    meas = json.load(open(os.path.join(root, "profiles", "ncu_traffic.json")))["c3"]
    for name, once, cache_less, got in tc.rows(meas):
        assert got is not None, name
        assert 0.98 * once <= got <= max(cache_less, once) * 1.02, (name, once, cache_less, got)
    # the dS^T round trip: the dK/dV kernel and the dQ GEMM move what the model says
    r = {n: (o, g) for n, o, _, g in tc.rows(meas)}
    for k in ("bwd_dkdv", "bwd_dq_gemm"):
        o, g = r[k]
        assert abs(g / o - 1) < 0.03, (k, g / o)
