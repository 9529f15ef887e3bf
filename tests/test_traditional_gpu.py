"""GPU: the unfused three-pass comparator (libvattn_b200_traditional.so,
vattn::forward_traditional, reference attention_forward.cpp:229-310) against the
binary64 oracle, with the same SURVEY 8(c) tolerances as the fused path, and its
dropout keep bits against the reference hash."""
import numpy as np
import pytest
import torch

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2502_12784_b200 as vb
    from paper_2502_12784_b200 import traditional as tr
    from tests.gpu_util import check_close, check_lse, widen, workload


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("B,H,N,d,causal,dtype", [
    (1, 2, 128, 64, False, torch.float16),
    (2, 2, 256, 128, True, torch.bfloat16),
    (1, 3, 200, 64, True, torch.float16),   # ragged N
    (1, 1, 72, 32, False, torch.float16),   # head_dim the fused path pads
])
def test_traditional_vs_binary64(B, H, N, d, causal, dtype):
    q, k, v = workload(5 + N, (B, H, N, d), dtype, with_dout=False)
    o, lse = tr.forward_traditional(q, k, v, causal)
    torch.cuda.synchronize()
    ro, rlse = po.attention_ref(widen(q), widen(k), widen(v), causal)
    check_close(widen(o), ro, dtype, "traditional O")
    check_lse(lse.cpu().double().numpy(), rlse)


def test_traditional_matches_fused_within_tolerance():
    q, k, v = workload(9, (2, 4, 512, 128), torch.bfloat16, with_dout=False)
    o_t, lse_t = tr.forward_traditional(q, k, v, True)
    o_f, lse_f = vb.mha_forward(q, k, v, True)
    check_close(widen(o_t), widen(o_f), torch.bfloat16, "traditional vs fused O")
    check_lse(lse_t.cpu().double().numpy(), lse_f.cpu().double().numpy())


def test_traditional_dropout_mask_bitwise():
    B, H, N, d, p, seed = 1, 2, 64, 64, 0.3, 4242
    q = torch.zeros(B, H, N, d, dtype=torch.float16, device="cuda")
    v = torch.eye(N, d, dtype=torch.float16, device="cuda").expand(B, H, N, d).contiguous()
    o, _ = tr.forward_traditional(q, q, v, False, dropout_p=p, seed=seed)
    kept = (o != 0).cpu().numpy()
    for h in range(H):
        want = np.array([[po.dropout_keep(seed, 0, h, i, j, p) for j in range(N)] for i in range(N)])
        assert np.array_equal(kept[0, h], want), h
