"""the run reports (paper_2502_12784_b200/reports.py) in the schema of the
reference's tool (proj/tools/vattn_main.cpp), the workload generator they use, and the
assertions of the reference's own report tests (proj/tests/cli_tests.cpp:51-191) on the
B200 path.  CPU tests pin the generator and the config-only parts (counters, CSV
shape) to the reference library; GPU tests run the fused kernels."""
import json

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_2502_12784_b200 import AttnConfig, spat
from paper_2502_12784_b200 import reports as rp
from paper_2502_12784_b200 import traffic as tf
from paper_2502_12784_b200.workload import normal_f32, normal_tensor_f16

need_ref = pytest.mark.skipif(not po.ref_available(), reason="reference library not built here")
gpu = pytest.mark.gpu


# ------------------------------------------------------------------- CPU --

@need_ref
@pytest.mark.parametrize("seed,stream,count", [(1, 1, 4096), (7, 4, 100003), (2**63 + 5, 3, 777)])
def test_workload_generator_bitwise_vs_reference(seed, stream, count):
    ours = normal_tensor_f16(seed, stream, (count,)).numpy().view(np.uint16)
    assert np.array_equal(ours, po.ref_normal_f16(seed, stream, count))


def test_workload_bf16_is_rne_of_the_same_normals():
    x = normal_f32(3, 2, 5000)
    b = normal_tensor_f16(3, 2, (5000,), bf16=True)
    assert torch.equal(b, torch.from_numpy(x).to(torch.bfloat16))
    assert np.array_equal(normal_tensor_f16(3, 2, (5000,)).numpy(), x.astype(np.float16))


def test_config_json_schema_and_order():
    cfg = AttnConfig(batch=2, heads=3, seq_len=128, head_dim=64, causal=True, dropout_p=0.1, seed=9)
    j = rp.config_json(cfg)
    assert list(j) == ["batch", "heads", "n", "d", "br", "bc", "causal", "dropout", "seed", "acc", "softmax_scale"]
    assert j["dropout"] == float(np.float32(0.1)) and j["softmax_scale"] == float(np.float32(0.125))
    assert j["acc"] == "fp32"
    assert rp.dumps({"a": 1}) == '{\n  "a": 1\n}\n'
    assert rp.hex64(0) == "0x0" and rp.hex64(-1) == "0xffffffffffffffff"


def test_error_metrics_matches_reference_definition():
    t = np.array([1.0, 0.0, -2.0, 1e-9])
    r = np.array([1.5, 0.0, -2.0, 0.0])
    m = rp.error_metrics(t, r)
    rel = np.array([0.5 / 1.5, 0.0, 0.0, 1e-9 / 1e-6])
    assert m["mean_rel"] == pytest.approx(rel.mean()) and m["max_rel"] == pytest.approx(rel.max())
    assert m["max_abs"] == 0.5 and m["mean_abs"] == pytest.approx((0.5 + 1e-9) / 4)


@need_ref
def test_sweep_csv_shape_and_counters():
    """cli_tests.cpp:120-171: header + one CRLF row per grid point, 16 columns, the
    FP16/FP32 convert/shuffle trade-off, counters equal to the reference library's."""
    text, ok = rp.sweep_csv([64, 128], [32, 64], ["fp16", "fp32"], [0, 1], seed=2)
    assert ok
    lines = text.split("\r\n")
    assert lines[-1] == "" and lines[0] == rp.CSV_HEADER
    rows = [ln.split(",") for ln in lines[1:-1]]
    assert len(rows) == 2 * 2 * 2 * 2 and all(len(r) == 16 for r in rows)
    for r in rows:
        n, d, acc, causal = int(r[0]), int(r[1]), r[2], int(r[3])
        ref = po.ref_traffic_counts(3 if acc == "fp16" else 0, 1, 1, n, d, min(64, n), min(64, n), causal)
        assert tuple(int(x) for x in r[9:]) == ref
        shuffles, converts = int(r[14]), int(r[15])
        assert (converts > 0 and shuffles == 0) if acc == "fp16" else (shuffles > 0 and converts == 0)
    with pytest.raises(ValueError):
        rp.sweep_csv([64], [], ["fp32"], [0])


def test_reports_reject_what_the_tool_rejects():
    with pytest.raises(ValueError):  # n = 100 is not a multiple of the 64 tile (cli_tests.cpp:77-80)
        rp.forward_report(AttnConfig(seq_len=100, head_dim=64))
    with pytest.raises(ValueError):  # backward --acc fp32 (cli_tests.cpp:82-85)
        rp.backward_report(AttnConfig(seq_len=64, head_dim=64, acc_mode="fp32"), acc_explicit=True)


# ------------------------------------------------------------------- GPU --

def _oracle_fwd(q, k, v, cfg):
    w = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
    return po.attention_ref(w(q), w(k), w(v), cfg.causal, cfg.scale(), cfg.dropout_p, cfg.seed)[0]


def _oracle_grad(q, k, v, do, cfg):
    w = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
    return po.attention_grad_ref(w(q), w(k), w(v), w(do), cfg.causal, cfg.scale(), cfg.dropout_p, cfg.seed)


@gpu
def test_forward_report_verify_and_pass_counts():
    cfg = AttnConfig(seq_len=64, head_dim=64, tile_rows=64, tile_cols=64, seed=7)
    rep, ok, _ = rp.forward_report(cfg, reference=_oracle_fwd)
    assert ok and rep["verify"]["fused_pass"] and rep["verify"]["traditional_pass"]
    j = json.loads(rp.dumps(rep))
    assert list(j) == ["command", "config", "paths", "verify"]
    assert j["paths"]["fused"]["traffic"]["matrix_pass_reads"] == 3
    assert j["paths"]["fused"]["traffic"]["matrix_pass_writes"] == 1
    assert j["paths"]["traditional"]["traffic"]["matrix_pass_reads"] == 5
    assert j["paths"]["traditional"]["traffic"]["matrix_pass_writes"] == 3
    assert "errors_vs_oracle" in j["paths"]["fused"]


@gpu
def test_forward_reports_byte_identical_across_runs():
    cfg = AttnConfig(seq_len=64, head_dim=32, tile_rows=64, tile_cols=64, seed=5, dropout_p=0.2)
    a, _, oa = rp.forward_report(cfg)
    b, _, ob = rp.forward_report(cfg)
    assert rp.dumps(a) == rp.dumps(b) and torch.equal(oa, ob)


@gpu
@need_ref
def test_forward_report_digest_and_counters_equal_reference():
    cfg = AttnConfig(batch=1, heads=2, seq_len=128, head_dim=64, causal=True, dropout_p=0.1, seed=3)
    rep, _, _ = rp.forward_report(cfg)
    dims = (1, 2, 128, 64)
    q, k, v = (po.normal16(3, s, dims) for s in (1, 2, 3))
    _, _, dig = po.ref_forward_fused_dropout(q, k, v, True, 0.1, 3)
    assert rep["paths"]["fused"]["mask_digest"] == rp.hex64(dig)
    assert tuple(rep["paths"]["fused"]["traffic"].values()) == po.ref_traffic_counts(0, 1, 2, 128, 64, 64, 64, 1)


@gpu
def test_backward_report_verify_and_digest_match():
    cfg = AttnConfig(seq_len=64, head_dim=64, tile_rows=64, tile_cols=64, seed=1)
    rep, ok, _ = rp.backward_report(cfg, reference_grad=_oracle_grad)
    assert ok and rep["mask_digest_match"] is True
    assert rep["backward"]["errors_vs_oracle"]["dq"]["mean_rel"] <= 0.01
    assert rep["config"]["acc"] == "fp16"
    rep, _, _ = rp.backward_report(AttnConfig(seq_len=64, head_dim=64, seed=3, dropout_p=0.1))
    assert rep["mask_digest_match"] is True and rep["forward"]["mask_digest"] != "0x0"


@gpu
def test_causal_report_halves_mma_count():
    dense, _, _ = rp.forward_report(AttnConfig(seq_len=128, head_dim=64))
    causal, _, _ = rp.forward_report(AttnConfig(seq_len=128, head_dim=64, causal=True), reference=_oracle_fwd)
    r = causal["paths"]["fused"]["traffic"]["mma_invocations"] / dense["paths"]["fused"]["traffic"]["mma_invocations"]
    assert 0.5 <= r <= 1.0


@gpu
def test_spat_inputs_reproduce_generated_workload(tmp_path):
    """cli_tests.cpp:173-191: SPAT files of the generated workload give the same O."""
    cfg = AttnConfig(seq_len=64, head_dim=32, tile_rows=64, tile_cols=64, seed=9)
    dims = (1, 1, 64, 32)
    for s, name in ((1, "q"), (2, "k"), (3, "v")):
        spat.write_spat(str(tmp_path / f"{name}.spat"), normal_tensor_f16(9, s, dims))
    q, k, v = (torch.from_numpy(spat.read_spat(str(tmp_path / f"{n}.spat"))).cuda() for n in "qkv")
    _, _, o1 = rp.forward_report(cfg, q, k, v)
    _, _, o2 = rp.forward_report(cfg)
    spat.write_spat(str(tmp_path / "o1.spat"), o1)
    spat.write_spat(str(tmp_path / "o2.spat"), o2)
    assert (tmp_path / "o1.spat").read_bytes() == (tmp_path / "o2.spat").read_bytes()
