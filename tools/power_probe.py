"""Clock / power under sustained load (diagnostic): python tools/power_probe.py [seconds]
Runs fwd-only, then fwd+bwd steps, each for ~T s, sampling nvidia-smi every 100 ms."""
import os, sys, subprocess, threading, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_12784_b200 as vb
from bench import flops

T = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
B, H, N, d, causal = 4, 16, 8192, 128, True


def sampler(stop, out):
    q = "clocks.sm,power.draw,clocks_throttle_reasons.active,temperature.gpu"
    p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            out.append(line.strip())
    p.terminate()


q, k, v, do = (torch.randn((B, H, N, d), device="cuda").to(torch.bfloat16) for _ in range(4))
o = torch.empty_like(q); lse = torch.empty((B, H, N), device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
ws = torch.empty(vb.workspace_bytes(B, H, N, d, causal, torch.bfloat16), dtype=torch.uint8, device="cuda")
fwd = lambda: vb.mha_forward(q, k, v, causal, out=o, lse=lse)
bwd = lambda: vb.mha_backward(q, k, v, o, do, lse, causal, dq=dq, dk=dk, dv=dv, workspace=ws)
ff, fb = flops(B, H, N, d, causal)
for name, fn, fl in (("fwd", fwd, ff), ("bwd", bwd, fb), ("step", lambda: (fwd(), bwd()), ff + fb)):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()
    th = threading.Thread(target=sampler, args=(stop, samples)); th.start()
    time.sleep(0.3)
    t0 = time.time(); n = 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    while time.time() - t0 < T:
        for _ in range(10): fn()
        n += 10
        torch.cuda.synchronize()
    b.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = a.elapsed_time(b) / n
    rows = [s.split(", ") for s in samples if s.count(",") >= 3]
    clk = [float(r[0]) for r in rows]; pw = [float(r[1]) for r in rows]
    reasons = sorted(set(r[2] for r in rows))
    print(f"{name}: {ms:.3f} ms/iter {fl/ms/1e9:.0f} TF | sm MHz median {statistics.median(clk):.0f} min {min(clk):.0f} "
          f"| power median {statistics.median(pw):.0f} W max {max(pw):.0f} | reasons {reasons} | temp {rows[-1][3]}", flush=True)
