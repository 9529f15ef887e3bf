"""Child process of the schedule-fuzzer soak (tests/test_stress_gpu.py, tools/stress_soak.py).

    VATTN_LIB=<lib.so> python tests/stress_child.py '<json list of configs>' <iterations>

Runs `iterations` forward + backward steps of every config on cuda:0 through the
library named by VATTN_LIB and prints one line ``RESULT {json}``: per config the
SHA-1 of (O, lse, dQ, dK, dV) bytes and whether every iteration gave the same
bytes.  The fuzzer only delays warps, so a correct barrier protocol returns the
bytes of the plain build; a race shows as a different or unstable digest, and a
hang as the watchdog's launch failure (non-zero exit).
Config = [B, H, N, d, causal, "bf16"|"fp16", dropout_p].
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2502_12784_b200 as vb  # noqa: E402


def digest(ts):
    h = hashlib.sha1()
    for t in ts:
        h.update(t.contiguous().view(torch.uint8).cpu().numpy().tobytes())
    return h.hexdigest()


def main():
    cfgs = json.loads(sys.argv[1])
    iters = int(sys.argv[2])
    out = {}
    for c in cfgs:
        B, H, N, d, causal, dt, p = c
        dtype = torch.bfloat16 if dt == "bf16" else torch.float16
        g = torch.Generator(device="cuda")
        g.manual_seed(1234)
        q, k, v, do = (torch.randn((B, H, N, d), generator=g, device="cuda").to(dtype) for _ in range(4))
        mask = None
        if p > 0:
            mask = torch.empty(vb.dropout_mask_bytes(q, bool(causal), p), dtype=torch.uint8, device="cuda")
        digs = set()
        for it in range(iters):
            o, lse = vb.mha_forward(q, k, v, bool(causal), dropout_p=p, seed=7, drop_mask=mask if it % 2 else None)
            dq, dk, dv = vb.mha_backward(q, k, v, o, do, lse, bool(causal), dropout_p=p, seed=7,
                                         drop_mask=mask if it % 2 else None)
            torch.cuda.synchronize()
            digs.add(digest((o, lse, dq, dk, dv)))
        out[json.dumps(c)] = {"digest": sorted(digs)[0], "stable": len(digs) == 1}
    print("RESULT " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
