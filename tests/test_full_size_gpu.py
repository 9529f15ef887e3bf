"""GPU: BASELINE.json's full-size configs (SURVEY 8c "large configs").  The C oracle
would take hours at these sizes, so each config is checked by properties that hold at
any size -- bitwise run-to-run determinism of O, lse, dQ, dK, dV -- and by sampled
(b, h) slices against the same binary64 math run in float64 on the GPU
(tests/gpu_util.f64_ref, the oracle's attention_ref / attention_grad_ref restated),
at the SURVEY 8(c) bounds unchanged (gpu_util.TOL, lse max_rel 1e-5)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12784_b200 as vb
    from tests.gpu_util import check_close, check_lse, f64_ref, widen


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


FULL = [
    # name, shape, causal, dtype, sampled (b, h) slices
    ("C3", (4, 16, 8192, 128), True, torch.bfloat16, [(0, 0), (3, 15)]),
    ("C2 N=16k", (1, 32, 16384, 64), False, torch.float16, [(0, 7)]),
    ("C5 one GPU", (1, 64, 32768, 128), True, torch.bfloat16, [(0, 63)]),
]


@pytest.mark.parametrize("name,shape,causal,dtype,samples", FULL, ids=[f[0] for f in FULL])
def test_full_size_determinism_and_sampled_parity(name, shape, causal, dtype, samples):
    g = torch.Generator(device="cuda")
    g.manual_seed(2026)
    q, k, v, do = (torch.randn(shape, generator=g, device="cuda").to(dtype) for _ in range(4))
    o, lse = vb.mha_forward(q, k, v, causal)
    dq, dk, dv = vb.mha_backward(q, k, v, o, do, lse, causal)
    o2, lse2 = vb.mha_forward(q, k, v, causal)
    g2 = vb.mha_backward(q, k, v, o2, do, lse2, causal)
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(lse, lse2)
    for a, b in zip((dq, dk, dv), g2):
        assert torch.equal(a, b)
    for b_, h_ in samples:
        ro, rlse, rdq, rdk, rdv = f64_ref(q[b_, h_], k[b_, h_], v[b_, h_], do[b_, h_], causal)
        for nm, t, r in (("O", o, ro), ("dQ", dq, rdq), ("dK", dk, rdk), ("dV", dv, rdv)):
            check_close(widen(t[b_, h_]), r.cpu().numpy(), dtype, f"{name} {nm} (b={b_},h={h_})")
        check_lse(lse[b_, h_].cpu().double().numpy(), rlse.cpu().numpy())
        del ro, rlse, rdq, rdk, rdv
        torch.cuda.empty_cache()


@pytest.mark.parametrize("shape,causal", [((4, 16, 8192, 128), True), ((2, 15, 8192, 128), True),
                                          ((1, 37, 4096, 128), True), ((2, 8, 4096, 64), False)],
                         ids=["C3", "BH30-G15", "BH37-prime", "d64-noncausal"])
def test_every_unit_equals_its_one_unit_slab(shape, causal):
    """Dispatch order (grouped longest-first forward, longest-first tail of the dK/dV and
    dQ grids) must not change which (b, h) unit a CTA computes: every unit of the full
    problem is bitwise equal to the same unit computed alone as a one-unit slab, where
    the mapping is trivial."""
    B, H, N, d = shape
    dtype = torch.bfloat16
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    q, k, v, do = (torch.randn(shape, generator=g, device="cuda").to(dtype) for _ in range(4))
    o, lse = vb.mha_forward(q, k, v, causal)
    dq, dk, dv = vb.mha_backward(q, k, v, o, do, lse, causal)
    flat = [t.reshape(B * H, 1, N, -1) for t in (q, k, v, do, o, dq, dk, dv)]
    lse_f = lse.reshape(B * H, 1, N)
    for u in range(B * H):
        qs, ks, vs, dos = (x[u:u + 1].contiguous() for x in flat[:4])
        sl = (B, H, u, 1)
        o1, l1 = vb.mha_forward(qs, ks, vs, causal, bh_slab=sl)
        g1 = vb.mha_backward(qs, ks, vs, o1, dos, l1, causal, bh_slab=sl)
        assert torch.equal(o1, flat[4][u:u + 1]) and torch.equal(l1, lse_f[u:u + 1]), u
        for name, a, r in zip(("dq", "dk", "dv"), g1, flat[5:]):
            assert torch.equal(a, r[u:u + 1]), (name, u)


def test_full_size_dropout_mask_paths_bitwise():
    """C3 with dropout p = 0.1 (the paper's benchmark setting): the forward-kept keep-bit
    mask and the backward's own mask kernel give bit-identical gradients, run to run."""
    B, H, N, d, causal, p, seed = 4, 16, 8192, 128, True, 0.1, 31337
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    q, k, v, do = (torch.randn((B, H, N, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    m = torch.empty(vb.dropout_mask_bytes(q, causal, p), dtype=torch.uint8, device="cuda")
    o1, l1 = vb.mha_forward(q, k, v, causal, dropout_p=p, seed=seed, drop_mask=m)
    g1 = vb.mha_backward(q, k, v, o1, do, l1, causal, dropout_p=p, seed=seed, drop_mask=m)
    o2, l2 = vb.mha_forward(q, k, v, causal, dropout_p=p, seed=seed)
    g2 = vb.mha_backward(q, k, v, o2, do, l2, causal, dropout_p=p, seed=seed)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for name, a, b in zip(("dq", "dk", "dv"), g1, g2):
        assert torch.equal(a, b), name
        assert torch.isfinite(a.float()).all(), name


def test_c4_24_layer_cuda_graph_bitwise_equals_eager():
    """BASELINE configs[3] (GPT-2-medium attention, (8, 16, 1024, 64) causal fp16, 24
    layers): the training step captured as ONE CUDA graph (24 forwards, then 24
    backwards in reverse, one shared workspace -- bench.py --config c4x24) replays to
    exactly the bytes of the eager step, twice in a row."""
    B, H, N, d, causal, dtype, layers = 8, 16, 1024, 64, True, torch.float16, 24
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    L = []
    for _ in range(layers):
        q, k, v, do = (torch.randn((B, H, N, d), generator=g, device="cuda").to(dtype) for _ in range(4))
        L.append(dict(q=q, k=k, v=v, do=do, o=torch.empty_like(q), lse=torch.empty((B, H, N), device="cuda"),
                      dq=torch.empty_like(q), dk=torch.empty_like(q), dv=torch.empty_like(q)))
    ws = torch.empty(vb.workspace_bytes(B, H, N, d, causal, dtype), dtype=torch.uint8, device="cuda")

    def step():
        for x in L:
            vb.mha_forward(x["q"], x["k"], x["v"], causal, out=x["o"], lse=x["lse"])
        for x in reversed(L):
            vb.mha_backward(x["q"], x["k"], x["v"], x["o"], x["do"], x["lse"], causal,
                            dq=x["dq"], dk=x["dk"], dv=x["dv"], workspace=ws)

    names = ("o", "lse", "dq", "dk", "dv")
    step()
    torch.cuda.synchronize()
    eager = [[x[n].clone() for n in names] for x in L]
    for x in L:  # poison the outputs: the replay must rewrite every byte
        for n in names:
            x[n].fill_(float("nan"))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            step()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        for x in L:
            for n in names:
                x[n].fill_(float("nan"))
        graph.replay()
        torch.cuda.synchronize()
        for li, x in enumerate(L):
            for n, ref in zip(names, eager[li]):
                assert torch.equal(x[n], ref), (li, n)
