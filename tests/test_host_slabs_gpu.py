"""GPU: the host-buffer entry points (mha_*_host) and (b, h) slab calls.

Both only re-partition independent (b, h) units, and every kernel is
deterministic, so the contract is BITWISE equality with one whole-problem call
on device tensors -- including dropout, whose keep masks must follow the
global (b, h) of each unit (reference rng.cpp:46-49 hashes b and h).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12784_b200 as vb
    from tests.gpu_util import workload


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


CASES = [
    (2, 3, 200, 64, True, torch.float16, 0.0),
    (3, 4, 1024, 128, True, torch.bfloat16, 0.0),   # several slabs, three device slots rotate
    (1, 40, 512, 64, False, torch.float16, 0.1),    # dropout: global (b, h) per slab
    (4, 16, 640, 128, False, torch.bfloat16, 0.0),
    (1, 1, 77, 128, False, torch.float16, 0.0),     # a single unit
]


def _device_ref(q, k, v, do, causal, p, seed=77):
    o, lse = vb.mha_forward(q, k, v, causal, dropout_p=p, seed=seed)
    dq, dk, dv = vb.mha_backward(q, k, v, o, do, lse, causal, dropout_p=p, seed=seed)
    return o, lse, dq, dk, dv


@pytest.mark.parametrize("B,H,N,d,causal,dtype,p", CASES)
@pytest.mark.parametrize("pinned", [True, False])
def test_host_entry_points_bitwise(B, H, N, d, causal, dtype, p, pinned):
    q, k, v, do = workload(41 + N, (B, H, N, d), dtype)
    ref = [t.cpu() for t in _device_ref(q, k, v, do, causal, p)]
    hq, hk, hv, hdo = (t.cpu() for t in (q, k, v, do))
    if pinned:
        hq, hk, hv, hdo = (t.pin_memory() for t in (hq, hk, hv, hdo))
    got = vb.mha_step_host(hq, hk, hv, hdo, causal, dropout_p=p, seed=77)
    for name, a, b in zip(("o", "lse", "dq", "dk", "dv"), got, ref):
        assert not a.is_cuda
        assert torch.equal(a, b), name
    o, lse = vb.mha_forward_host(hq, hk, hv, causal, dropout_p=p, seed=77)
    assert torch.equal(o, ref[0]) and torch.equal(lse, ref[1])
    g = vb.mha_backward_host(hq, hk, hv, o, hdo, lse, causal, dropout_p=p, seed=77)
    for name, a, b in zip(("dq", "dk", "dv"), g, ref[2:]):
        assert torch.equal(a, b), name


@pytest.mark.parametrize("dtype,p", [(torch.float16, 0.0), (torch.bfloat16, 0.2)])
def test_slab_calls_bitwise(dtype, p):
    B, H, N, d, causal = 2, 3, 384, 128, True
    q, k, v, do = workload(5, (B, H, N, d), dtype)
    ref = _device_ref(q, k, v, do, causal, p)
    flat = [t.reshape(B * H, 1, N, -1) if t.dim() == 4 else t.reshape(B * H, 1, N) for t in (q, k, v, do)]
    for lo, hi in ((0, 2), (2, 5), (5, 6)):
        sl = (B, H, lo, hi - lo)
        qs, ks, vs, dos = (x[lo:hi].contiguous() for x in flat)
        o, lse = vb.mha_forward(qs, ks, vs, causal, dropout_p=p, seed=77, bh_slab=sl)
        dq, dk, dv = vb.mha_backward(qs, ks, vs, o, dos, lse, causal, dropout_p=p, seed=77, bh_slab=sl)
        for name, a, r in zip(("o", "lse", "dq", "dk", "dv"), (o, lse, dq, dk, dv), ref):
            rf = r.reshape(B * H, *r.shape[2:])[lo:hi]
            assert torch.equal(a.reshape(rf.shape), rf), (name, lo, hi)


def test_host_errors():
    q = torch.zeros(1, 1, 64, 64, dtype=torch.float16)
    with pytest.raises(ValueError):
        vb.mha_step_host(q.cuda(), q, q, q)  # device tensor at the host boundary
    with pytest.raises(ValueError):
        vb.mha_forward_host(q, q, q[:, :, :32].contiguous())
    with pytest.raises(NotImplementedError):
        big = torch.zeros(1, 1, 64, 96, dtype=torch.float16)
        vb.mha_forward_host(big, big, big)


def test_host_slab_calls_bitwise_with_dropout():
    """Host-buffer entry points on a (b, h) slab (what a rank of a sharded run passes):
    dropout masks follow the global (b, h), so each slab equals its rows of the
    whole-problem device result."""
    B, H, N, d, causal, dtype, p = 2, 3, 320, 128, True, torch.bfloat16, 0.15
    q, k, v, do = workload(9, (B, H, N, d), dtype)
    ref = _device_ref(q, k, v, do, causal, p)
    flat = [t.reshape(B * H, 1, N, -1).cpu() for t in (q, k, v, do)]
    for lo, hi in ((0, 4), (4, 6)):
        sl = (B, H, lo, hi - lo)
        hq, hk, hv, hdo = (x[lo:hi].contiguous().pin_memory() for x in flat)
        got = vb.mha_step_host(hq, hk, hv, hdo, causal, dropout_p=p, seed=77, bh_slab=sl)
        o, lse = vb.mha_forward_host(hq, hk, hv, causal, dropout_p=p, seed=77, bh_slab=sl)
        g = vb.mha_backward_host(hq, hk, hv, o, hdo, lse, causal, dropout_p=p, seed=77, bh_slab=sl)
        for name, a, r in zip(("o", "lse", "dq", "dk", "dv"), got, ref):
            rf = r.reshape(B * H, *r.shape[2:])[lo:hi].cpu()
            assert torch.equal(a.reshape(rf.shape), rf), (name, lo, hi)
        for name, a, b in zip(("o", "lse", "dq", "dk", "dv"), (o, lse, *g), got):
            assert torch.equal(a, b), ("separate calls", name, lo, hi)
