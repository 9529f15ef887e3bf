"""Time libvattn_b200 variants (tools/variants/*.so) on the bench configs.

    python tools/time_variants.py [--configs c3,c2_4k] [--steps 20] [variant ...]

Each variant runs in its own subprocess (VATTN_LIB=<so>); prints per-kernel
milliseconds (CUDA events on the launching stream, vattn_profile hooks) and
fwd+bwd TFLOPS.  Tuning aid only -- bench.py is the number of record.
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch, ctypes as C
import paper_2502_12784_b200 as vb
from bench import CONFIGS, flops
out = {}
for name in os.environ["CFGS"].split(","):
    B, H, N, d, causal, dt, _ = CONFIGS[name]
    dtype = torch.bfloat16 if dt == "bf16" else torch.float16
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    q, k, v, do = (torch.randn((B, H, N, d), generator=g, device="cuda").to(dtype) for _ in range(4))
    o = torch.empty_like(q); lse = torch.empty((B, H, N), device="cuda")
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    ws = torch.empty(vb.workspace_bytes(B, H, N, d, causal, dtype), dtype=torch.uint8, device="cuda")
    def step():
        vb.mha_forward(q, k, v, causal, out=o, lse=lse)
        vb.mha_backward(q, k, v, o, do, lse, causal, dq=dq, dk=dk, dv=dv, workspace=ws)
    for _ in range(3): step()
    torch.cuda.synchronize()
    steps = int(os.environ["STEPS"])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps): step()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    vb.lib.vattn_profile_enable(1)
    for _ in range(5): step()
    torch.cuda.synchronize()
    ks = []
    for kind in (0, 1, 2):
        t, n = C.c_double(), C.c_int()
        vb.lib.vattn_profile_read(kind, C.byref(t), C.byref(n)); ks.append(t.value / max(n.value, 1))
    vb.lib.vattn_profile_enable(0)
    ff, fb = flops(B, H, N, d, causal)
    out[name] = dict(ms=ms, fwd=ks[0], dkdv=ks[1], dq=ks[2], tflops=(ff + fb) / ms / 1e9,
                     fwd_tf=ff / ks[0] / 1e9, ok=bool(torch.isfinite(dq).all()))
print("RESULT " + json.dumps(out))
'''


def main():
    args = sys.argv[1:]
    cfgs, steps = "c3", "20"
    names = []
    i = 0
    while i < len(args):
        if args[i] == "--configs":
            cfgs = args[i + 1]; i += 2
        elif args[i] == "--steps":
            steps = args[i + 1]; i += 2
        else:
            names.append(args[i]); i += 1
    libs = [os.path.join(ROOT, "paper_2502_12784_b200", "libvattn_b200.so")]
    libs += [os.path.join(ROOT, "tools", "variants", n + ".so") for n in names] if names else \
        sorted(glob.glob(os.path.join(ROOT, "tools", "variants", "*.so")))
    for rep in range(2):
        for lib in libs:
            env = dict(os.environ, VATTN_LIB=lib, ROOT=ROOT, CFGS=cfgs, STEPS=steps)
            r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
            line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
            name = os.path.basename(lib)[:-3]
            if not line:
                print(f"{name:28s} FAILED rc={r.returncode} {r.stderr[-400:]}")
                continue
            res = json.loads(line[0][7:])
            for c, v in res.items():
                print(f"{name:28s} {c:8s} step {v['ms']:.3f} ms  {v['tflops']:7.1f} TF | fwd {v['fwd']:.3f} "
                      f"({v['fwd_tf']:.0f} TF) dkdv {v['dkdv']:.3f} dq {v['dq']:.3f} ok={v['ok']}", flush=True)


if __name__ == "__main__":
    main()
