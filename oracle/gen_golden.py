"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE.  Run here (where /root/reference exists):

    make -C oracle && python oracle/gen_golden.py

Every array in a fixture is produced by the reference library itself through
oracle/ref_shim.cpp: inputs by vattn::normal_tensor_f16 (workload.hpp:10-17),
outputs by forward_fused / backward_fused / compute_dpsum / attention_ref /
attention_grad_ref.  The shapes follow the reference's own tests
(test_forward.cpp, test_backward.cpp, acceptance.cpp) plus BASELINE config 1.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as po  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

# name, (B, H, N, d), causal, (br, bc), seed, source
CASES = [
    ("c1_noncausal_b1h2n128d64", (1, 2, 128, 64), False, (64, 64), 1, "BASELINE.json configs[0]"),
    ("causal_n64d32_t16x32", (1, 1, 64, 32), True, (16, 32), 27, "test_forward.cpp:200-214 / test_backward.cpp:75-90"),
    ("noncausal_n64d32_t32", (1, 1, 64, 32), False, (32, 32), 5, "test_backward.cpp:62-73"),
    ("causal_b2h1n128d128", (2, 1, 128, 128), True, (64, 64), 3, "acceptance.cpp grid (d=128) + causal"),
    ("noncausal_n256d64_h2", (1, 2, 256, 64), False, (64, 64), 7, "acceptance.cpp grid n=256"),
    ("odd_d20_b2h3n64", (2, 3, 64, 20), False, (32, 64), 7, "test_forward.cpp:54 (d=20, b2 h3)"),
    ("causal_d16_n64", (1, 1, 64, 16), True, (16, 16), 11, "test_backward.cpp:110-127"),
]


def make_case(name, shape, causal, tiles, seed, source):
    B, H, N, d = shape
    br, bc = tiles
    q = po.ref_normal_f16(seed, 1, B * H * N * d).reshape(shape)
    k = po.ref_normal_f16(seed, 2, B * H * N * d).reshape(shape)
    v = po.ref_normal_f16(seed, 3, B * H * N * d).reshape(shape)
    do = po.ref_normal_f16(seed, 4, B * H * N * d).reshape(shape)
    o32, lse32 = po.ref_forward_fused(q, k, v, causal, br, bc, acc_fp16=False)
    qd, kd, vd, dod = (po.widen(x) for x in (q, k, v, do))
    o64, lse64 = po.ref_attention_ref(qd, kd, vd, causal)
    dq64, dk64, dv64 = po.ref_attention_grad_ref(qd, kd, vd, dod, causal)
    # backward_fused consumes the lse of a forward at its own (FP16-ACC) mode, as
    # tools/vattn_main.cpp:207-219 and test_backward.cpp do.
    o16, lse16 = po.ref_forward_fused(q, k, v, causal, br, bc, acc_fp16=True)
    dq16, dk16, dv16 = po.ref_backward_fused(q, k, v, do, lse16, causal, br, bc)
    dpsum = po.ref_compute_dpsum(do, o32)
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"),
        q=q, k=k, v=v, dout=do,
        fwd32_out=o32, fwd32_lse=lse32,
        ref_out=o64, ref_lse=lse64,
        ref_dq=dq64, ref_dk=dk64, ref_dv=dv64,
        fwd16_lse=lse16, bwd16_dq=dq16, bwd16_dk=dk16, bwd16_dv=dv16,
        dpsum_fwd32=dpsum,
    )
    return dict(name=name, shape=list(shape), causal=causal, tiles=[br, bc], seed=seed, source=source)


# dropout cases: name, shape, causal, tiles, input seed, dropout_p, dropout seed, source
DROP_CASES = [
    ("drop_p10_n64d32", (1, 1, 64, 32), False, (32, 32), 23, 0.1, 33, "test_forward.cpp:238-253"),
    ("drop_p10_causal_n64d16", (1, 1, 64, 16), True, (32, 32), 13, 0.1, 77, "test_backward.cpp:129-146"),
    ("drop_p25_b2h2n128d64", (2, 2, 128, 64), False, (64, 64), 5, 0.25, 1234, "SURVEY 8f-1 (paper grid p)"),
]


def make_drop_case(name, shape, causal, tiles, seed, p, dseed, source):
    B, H, N, d = shape
    br, bc = tiles
    q, k, v, do = (po.ref_normal_f16(seed, s, B * H * N * d).reshape(shape) for s in (1, 2, 3, 4))
    o32, lse32, dig32 = po.ref_forward_fused_dropout(q, k, v, causal, p, dseed, br, bc, acc_fp16=False)
    qd, kd, vd, dod = (po.widen(x) for x in (q, k, v, do))
    o64, lse64 = po.ref_attention_ref_dropout(qd, kd, vd, causal, p, dseed)
    dq64, dk64, dv64 = po.ref_attention_grad_ref_dropout(qd, kd, vd, dod, causal, p, dseed)
    o16, lse16, dig16 = po.ref_forward_fused_dropout(q, k, v, causal, p, dseed, br, bc, acc_fp16=True)
    dq16, dk16, dv16, digb = po.ref_backward_fused_dropout(q, k, v, do, lse16, causal, p, dseed, br, bc)
    assert dig16 == digb and dig32 == dig16
    # the keep mask of every position of head (0, 0), as the reference decides it
    mask = np.array([[po.ref_dropout_keep(dseed, 0, 0, i, j, p) for j in range(N)] for i in range(N)], np.uint8)
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"), q=q, k=k, v=v, dout=do, mask_b0h0=mask,
        fwd32_out=o32, fwd32_lse=lse32, ref_out=o64, ref_lse=lse64, ref_dq=dq64, ref_dk=dk64, ref_dv=dv64,
        fwd16_lse=lse16, bwd16_dq=dq16, bwd16_dk=dk16, bwd16_dv=dv16, digest=np.uint64(dig32))
    return dict(name=name, shape=list(shape), causal=causal, tiles=[br, bc], seed=seed, dropout_p=p,
                dropout_seed=dseed, source=source)


def main():
    if not po.ref_available():
        raise SystemExit("oracle/_ref/libvattn_ref.so missing: run `make -C oracle` where /root/reference exists")
    os.makedirs(OUT, exist_ok=True)
    manifest = [make_case(*c) for c in CASES]
    drop_manifest = [make_drop_case(*c) for c in DROP_CASES]
    # dropout_keep grid (rng.cpp:46-49) for seed 42, p = 0.5, (b, h) = (0, 1)
    np.savez_compressed(os.path.join(OUT, "dropout_keep_seed42.npz"),
                        keep=np.array([[po.ref_dropout_keep(42, 0, 1, i, j, 0.5) for j in range(64)]
                                       for i in range(64)], np.uint8))
    # Generator pin: the first 256 binary16 normals of (seed 1, stream 1..4).
    np.savez_compressed(os.path.join(OUT, "normals_seed1.npz"),
                        **{f"stream{s}": po.ref_normal_f16(1, s, 256) for s in (1, 2, 3, 4)})
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(dict(generator="oracle/gen_golden.py", reference="/root/reference/proj (vattn, compiled by oracle/Makefile)",
                       cases=manifest, dropout_cases=drop_manifest), f, indent=1)
    print(f"wrote {len(manifest)} cases to {OUT}")


if __name__ == "__main__":
    main()
