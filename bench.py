"""bench.py -- fused MHA fwd+bwd throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]

A *step* is one pass of the hot path over the workload: mha_forward (O, lse)
followed by mha_backward (dQ, dK, dV) through the C ABI of
paper_2502_12784_b200/libvattn_b200.so.  Default workload = BASELINE configs[2]
("C3"): causal, batch 4, heads 16, seq 8192, head_dim 128, bf16 -- the config
that carries north_star's target (1 GPU, seq >= 4k, d = 128).

Multi-GPU (torchrun, one process per GPU), partitioned by (batch, head) with no
collective on the data path:
  --split batch (default, "weak"): every rank owns its own (batch, head) slab of a
      global batch of N x the per-GPU config;
  --split bh ("strong"): the config IS the global problem (e.g. --config c5 =
      BASELINE configs[4], (1, 64, 32768, 128) over 8 GPUs) and rank r owns heads
      shard_range(B*H, N, r); after timing the slabs are gathered to rank 0 over
      NCCL and sampled heads are verified there (north_star: NCCL only to gather
      results for verification).
Timing: W warm-up steps, then K steps between barrier + synchronize, CUDA
events on the launching stream, max over ranks.  Inputs (>= 4 x 128 MiB for
C3) exceed the 126 MB L2, so no explicit flush.  The roofline denominator is the
measured BURST bf16 peak when the timed window is short (< 1 s) and the SM clock
stayed >= 0.95 x max, the SUSTAINED one otherwise; both fractions are printed.

Reported: value = aggregate algorithmic TFLOPS (14 B H N^2 d c over all ranks /
max-rank time; c = 1/2 causal), e2e = the same metric through the public API
with host (pinned) buffers and the H2D/D2H copies inside the timed region,
roofline = the fused backward main kernel (dominant) against the measured bf16
tensor peak, cpu_baseline = the reference's CPU path (oracle/_ref) on a
bounded sample.  `--impl reference` times the reference CPU path itself.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MHA fwd+bwd TFLOPS and % of B200 tensor peak at 1/2/4/8 GPUs vs CPU ref"

CONFIGS = {
    # name: (B, H, N, d, causal, dtype, description)
    "c3": (4, 16, 8192, 128, True, "bf16", "BASELINE configs[2]: causal MHA fwd+bwd, d=128, B=4, H=16, N=8192, bf16"),
    "c2_512": (32, 32, 512, 64, False, "fp16", "BASELINE configs[1] point: 16k tokens, hidden 2048, d=64, N=512"),
    "c2_1k": (16, 32, 1024, 64, False, "fp16", "BASELINE configs[1] point: 16k tokens, hidden 2048, d=64, N=1024"),
    "c2_2k": (8, 32, 2048, 64, False, "fp16", "BASELINE configs[1] point: 16k tokens, hidden 2048, d=64, N=2048"),
    "c2_4k": (4, 32, 4096, 64, False, "fp16", "BASELINE configs[1] point: 16k tokens, hidden 2048, d=64, N=4096"),
    "c2_8k": (2, 32, 8192, 64, False, "fp16", "BASELINE configs[1] point: 16k tokens, hidden 2048, d=64, N=8192"),
    "c2_16k": (1, 32, 16384, 64, False, "fp16", "BASELINE configs[1] point: 16k tokens, hidden 2048, d=64, N=16384"),
    "c3_fp16": (4, 16, 8192, 128, True, "fp16", "BASELINE configs[2] in fp16: causal MHA fwd+bwd, d=128, B=4, H=16, N=8192"),
    "c3_nc": (4, 16, 8192, 128, False, "bf16", "BASELINE configs[2] shape, non-causal: d=128, B=4, H=16, N=8192, bf16"),
    "c4": (8, 16, 1024, 64, True, "fp16", "BASELINE configs[3] per layer: GPT-2-medium attention, causal"),
    "c5": (1, 64, 32768, 128, True, "bf16", "BASELINE configs[4] on one GPU: causal seq 32k, d=128, H=64"),
    "c4x24": (8, 16, 1024, 64, True, "fp16", "BASELINE configs[3]: GPT-2-medium attention training step, "
              "24 layers (24 forwards, then 24 backwards in reverse) captured as one CUDA graph, causal"),
    "c1": (1, 2, 128, 64, False, "fp16", "BASELINE configs[0]: the CPU oracle shape (launch-bound)"),
}
# configs whose step runs several attention layers (distinct tensors per layer)
LAYERS = {"c4x24": 24}


def flops(B, H, N, d, causal):
    c = 0.5 if causal else 1.0
    return 4.0 * B * H * N * N * d * c, 10.0 * B * H * N * N * d * c


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("bf16_tflops"), j.get("bf16_tflops_sustained"), "measured"
    return 1590.0, 1400.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 2 ms) during the timed region.
    The main thread waits for the timed work with wait_event() (polls with the GIL
    released) so this thread keeps sampling; only samples taken between mark_start()
    and mark_stop() count."""

    REASONS = {  # nvmlClocksEventReason* bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
    }

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._ready = threading.Event()
        self._t = None
        self.t0 = self.t1 = None

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._ready.set()  # NVML is up: the timed region may start
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((time.perf_counter(), sm, smax, r))
                self._stop.wait(0.002)
        except Exception as e:  # sampling is evidence, never fatal
            self.error = str(e)
        finally:
            self._ready.set()

    def __enter__(self):
        # NVML import + init can take longer than a short timed region: start sampling
        # first, and only return (start the clock) once it runs
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=30)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_stop(self):
        self.t1 = time.perf_counter()

    def summary(self):
        t0 = self.t0 if self.t0 is not None else -math.inf
        t1 = self.t1 if self.t1 is not None else math.inf
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[1] for s in inside]
        reasons = sorted({name for s in inside for bit, name in self.REASONS.items() if s[3] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[2] for s in inside),
                "sm_min_mhz": min(sm), "reasons": reasons, "samples": len(inside)}


def wait_event(ev):
    """Block until CUDA event `ev` completed, polling with short sleeps (releases the GIL,
    so the clock sampler thread runs while the timed kernels execute)."""
    while not ev.query():
        time.sleep(0.0005)


def cpu_reference_sample(d, causal, threads, n_cpu=1024):
    """Reference CPU path (oracle/_ref: forward_fused FP32-ACC + backward_fused)
    on `threads` (b,h) units of [1,1,n_cpu,d].  Returns (TFLOPS, seconds, sample text, kind)."""
    from oracle import pyoracle as po
    units = threads
    f, b = flops(1, 1, n_cpu, d, causal)
    if po.ref_available():
        secs = po.ref_bench_units(n_cpu, d, causal, units, threads)
        kind = "reference"
    else:  # oracle port: restated FP32-ACC forward + binary64 gradients, single thread
        import numpy as np
        shape = (1, 1, n_cpu, d)
        q, k, v, do = (po.normal16(1, s, shape) for s in (1, 2, 3, 4))
        units, threads = 1, 1
        t0 = time.perf_counter()
        po.forward_fused_fp32acc(q, k, v, causal)
        po.attention_grad_ref(po.widen(q), po.widen(k), po.widen(v), po.widen(do), causal)
        secs = time.perf_counter() - t0
        kind = "port"
    if secs <= 0:
        raise RuntimeError("reference CPU run failed")
    tflops = units * (f + b) / secs / 1e12
    sample = (f"{units} (b,h) units of [1,1,{n_cpu},{d}] {'causal' if causal else 'non-causal'} fp16, "
              f"forward_fused FP32-ACC + backward_fused on {threads} host threads, {secs:.2f} s; "
              f"algorithmic GFLOP/s is N-independent for the emulated tile loops")
    return tflops, secs, sample, kind, threads


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    B, H, N, d, causal, dt, desc = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    vals = []
    # Each step is a bounded sample (~0.5 s on 16 cores) so --steps 50 ends in well under a minute.
    for _ in range(args.warmup):
        cpu_reference_sample(d, causal, threads, n_cpu=128)
    info = None
    for _ in range(args.steps):
        info = cpu_reference_sample(d, causal, threads, n_cpu=256)
        vals.append(info[0])
    val = statistics.median(vals)
    tfl, secs, sample, kind, cores = info
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16 storage, f32 math (reference software model)",
        "data": "synthetic (vattn::normal_tensor_f16 streams)",
        "config": {"workload": desc, "cpu_sample": sample},
        "cpu_baseline": {"value": val, "unit": "TFLOPS", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": val, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def pick_peak(window_s, clk, peak_burst, peak_sust):
    """Roofline denominator for the timed window: the burst bf16 peak applies to a
    short window (< 1 s) run at >= 0.95 x the max SM clock, the sustained
    (power-capped) one to anything longer or slower."""
    sm, smax = clk.get("sm_mhz"), clk.get("sm_max_mhz")
    at_max = sm is not None and smax and sm >= 0.95 * smax
    if window_s < 1.0 and at_max:
        return peak_burst, "bf16_tflops (burst): timed window < 1 s at >= 0.95 x max SM clock"
    return peak_sust, "bf16_tflops_sustained: timed window >= 1 s or SM clock < 0.95 x max"


def verify_gather(vb, torch, shard, world, rank, inputs, outs, slab_units, bh_total, causal, slab_of):
    """--split bh: gather every rank's O, lse, dQ, dK, dV to rank 0 over NCCL (the only
    collective; after the timed region) and check sampled heads there: each sampled
    head owned by another rank must equal, bit for bit, rank 0's own recomputation of
    that head as a one-unit slab (units are independent and slab results are
    bit-identical to whole-problem units, capi.cu vattn_config.bh_*)."""
    q, k, v, do = inputs
    gathered = [shard.gather_to_rank0(t.reshape(t.shape[0], *t.shape[2:]), bh_total) for t in outs]
    if rank != 0:
        return None
    B, H = slab_of
    picks = sorted({shard.shard_range(bh_total, world, r)[0] for r in range(world)} |
                   {shard.shard_range(bh_total, world, r)[1] - 1 for r in range(world)})
    bad = []
    for u in picks:
        qs, ks, vs, dos = (x.reshape(bh_total, 1, *x.shape[2:])[u:u + 1] for x in (q, k, v, do))
        o1, l1 = vb.mha_forward(qs, ks, vs, causal, bh_slab=(B, H, u, 1))
        g1 = vb.mha_backward(qs, ks, vs, o1, dos, l1, causal, bh_slab=(B, H, u, 1))
        for name, a, b in zip(("o", "lse", "dq", "dk", "dv"), (o1, l1) + tuple(g1), gathered):
            if not torch.equal(a.reshape(b[u].shape), b[u]):
                bad.append(f"{name}[unit {u}]")
    return {"gathered_bytes": int(sum(t.numel() * t.element_size() for t in gathered)),
            "units_checked": picks, "bitwise_equal": not bad, "mismatch": bad}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--split", default="batch", choices=["batch", "bh"],
                    help="multi-GPU partition: batch = weak (each rank its own copy of the config), "
                         "bh = strong (the config's (batch, head) units split over the ranks)")
    ap.add_argument("--no-verify", action="store_true", help="--split bh: skip the NCCL gather + check")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--dropout", type=float, default=0.0, help="fused dropout p (reference keep masks); 0 = north_star")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # test hook: VATTN_BENCH_SHARED_GPU=1 runs every rank on the visible GPU(s) with gloo
    # (exercises the N > 1 path on a 1-GPU box; never used for reported numbers)
    shared = os.environ.get("VATTN_BENCH_SHARED_GPU") == "1"
    if shared:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2502_12784_b200 as vb
    from paper_2502_12784_b200 import shard

    B, H, N, d, causal, dt, desc = CONFIGS[args.config]
    dtype = torch.bfloat16 if dt == "bf16" else torch.float16
    dev = torch.device("cuda", local)
    strong = args.split == "bh"
    if strong:
        # the config is the global problem: every rank draws the same global inputs
        # (same seed) and keeps its contiguous (b, h) slab, a view in [B, H, N, d]
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234)
        full = [torch.randn((B, H, N, d), generator=gen, device=dev, dtype=torch.float32).to(dtype) for _ in range(4)]
        lo, hi = shard.shard_range(B * H, world, rank)
        n_loc = hi - lo
        if n_loc < 1:
            raise SystemExit(f"--split bh: {B * H} (batch, head) units cannot feed {world} ranks")
        q, k, v, do = (shard.slab(x, lo, hi).unsqueeze(1) for x in full)
        slab = (B, H, lo, n_loc)
        shape = (n_loc, 1, N, d)
        units_total = B * H
    else:
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234 + rank)  # each rank: its own (batch, head) slab of the global batch
        shape = (B, H, N, d)
        q, k, v, do = (torch.randn(shape, generator=gen, device=dev, dtype=torch.float32).to(dtype) for _ in range(4))
        full = None
        # this rank's (b, h) slab of the global [B*world, H] problem (dropout masks use global (b, h))
        slab = (B * world, H, rank * B * H, B * H) if world > 1 else None
        units_total = B * H * world
    layers = LAYERS.get(args.config, 1)
    if layers > 1 and strong:
        raise SystemExit("--split bh is for single-layer configs")
    n_units_rank = shape[0] * shape[1]
    stream = torch.cuda.current_stream()

    def buffers(q, k, v, do):
        return dict(q=q, k=k, v=v, do=do, o=torch.empty(shape, device=dev, dtype=dtype),
                    lse=torch.empty(shape[:3], device=dev, dtype=torch.float32),
                    dq=torch.empty(shape, device=dev, dtype=dtype), dk=torch.empty(shape, device=dev, dtype=dtype),
                    dv=torch.empty(shape, device=dev, dtype=dtype),
                    # dropout: the forward keeps its keep bits for the backward (as the autograd binding does)
                    mask=(torch.empty(vb.dropout_mask_bytes(q, causal, args.dropout, slab), dtype=torch.uint8,
                                      device=dev) if args.dropout > 0 else None))

    Ls = [buffers(q, k, v, do)]
    for _ in range(layers - 1):  # further layers: their own inputs (same shapes)
        Ls.append(buffers(*(torch.randn(shape, generator=gen, device=dev, dtype=torch.float32).to(dtype)
                            for _ in range(4))))
    mask = Ls[0]["mask"]
    ws = torch.empty(vb.workspace_bytes(n_units_rank, 1, N, d, causal, dtype, args.dropout,
                                        external_mask=mask is not None), dtype=torch.uint8, device=dev)
    o, lse, dq, dk, dv = (Ls[0][x] for x in ("o", "lse", "dq", "dk", "dv"))

    def step_eager():
        for x in Ls:  # forwards through the layers
            vb.mha_forward(x["q"], x["k"], x["v"], causal, out=x["o"], lse=x["lse"], dropout_p=args.dropout,
                           seed=1234, bh_slab=slab, drop_mask=x["mask"])
        for x in reversed(Ls):  # backwards in reverse layer order
            vb.mha_backward(x["q"], x["k"], x["v"], x["o"], x["do"], x["lse"], causal, dq=x["dq"], dk=x["dk"],
                            dv=x["dv"], workspace=ws, dropout_p=args.dropout, seed=1234, bh_slab=slab,
                            drop_mask=x["mask"])

    step = step_eager
    if layers > 1:
        # one CUDA graph per training step (C4 "capture as a CUDA Graph")
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cap):
            step_eager()  # smem opt-ins and tensor maps outside the capture
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=cap):
                step_eager()
        stream.wait_stream(cap)
        step = graph.replay

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- timed
    # (no per-kernel events inside the timed region: an event between two kernels
    # would break their programmatic-dependent-launch overlap)
    launches_per_step = 4 * layers  # per layer: fwd + (preprocess, dK/dV kernel, dQ kernel or dQ GEMM)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        clocks.mark_start()
        start.record(stream)
        for _ in range(args.steps):
            step()
        stop.record(stream)
        wait_event(stop)
        clocks.mark_stop()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    # per-kernel durations (roofline): a separate profiled pass, CUDA events on the
    # launching stream around each hot kernel
    import ctypes as C
    vb.lib.vattn_profile_enable(1)
    for _ in range(max(3, min(args.steps, 10))):
        step_eager()  # (n_prof steps)
    torch.cuda.synchronize()
    kern_ms = []
    n_prof = max(3, min(args.steps, 10))
    for kind in (0, 1, 2, 3, 4):  # VATTN_KERNEL_FWD, _BWD_DKDV, _BWD_DQ, _BWD_PRE, _DROPMASK
        t_ms, n_l = C.c_double(), C.c_int()
        vb.lib.vattn_profile_read(kind, C.byref(t_ms), C.byref(n_l))
        # per launch, except the keep-bit mask: per step (0 without dropout)
        kern_ms.append(t_ms.value / (n_prof * layers if kind == 4 else max(n_l.value, 1)))
    vb.lib.vattn_profile_enable(0)
    t = torch.tensor([ms] + kern_ms, device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, fwd_ms, dkdv_ms, dq_ms, pre_ms, mask_ms = t.tolist()
    ms_step = ms_max / args.steps
    f_unit_fwd, f_unit_bwd = flops(1, 1, N, d, causal)
    f_fwd, f_bwd = n_units_rank * f_unit_fwd, n_units_rank * f_unit_bwd  # one layer of this rank's work
    value = layers * units_total * (f_unit_fwd + f_unit_bwd) / (ms_step * 1e-3) / 1e12

    # --------------------------------------------------- gather + verify (bh)
    verify = None
    if strong and world > 1 and not args.no_verify:
        verify = verify_gather(vb, torch, shard, world, rank, (full[0], full[1], full[2], full[3]),
                               (o, lse, dq, dk, dv), n_loc, B * H, causal, (B, H))
    del full

    # ------------------------------------------------------------------ e2e
    # Public API with host buffers: mha_step_host (C ABI) takes pinned host Q, K, V, dO
    # and returns O, lse, dQ, dK, dV in host memory; the H2D / D2H copies run inside
    # the call (pipelined against the kernels slab by slab).
    hq, hk, hv, hdo = (x.cpu().pin_memory() for x in (q, k, v, do))
    ho, hdq, hdk, hdv = (torch.empty(shape, dtype=dtype).pin_memory() for _ in range(4))
    hlse = torch.empty(shape[:3], dtype=torch.float32).pin_memory()
    h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv, hdo))
    d2h = sum(x.numel() * x.element_size() for x in (ho, hlse, hdq, hdk, hdv))

    def e2e_step():
        for _ in range(layers):  # (every layer's tensors have the same size; layer 0's buffers stand in)
            vb.mha_step_host(hq, hk, hv, hdo, causal, dropout_p=args.dropout, seed=1234,
                             out=(ho, hlse, hdq, hdk, hdv), bh_slab=slab)

    e2e_ms = e2e_val = None
    if args.e2e_steps > 0:
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = te.item() / args.e2e_steps
        e2e_val = layers * units_total * (f_unit_fwd + f_unit_bwd) / (e2e_ms * 1e-3) / 1e12

    rc = 0
    if rank == 0:
        peak_burst, peak_sust, peak_src = measured_peaks()
        clk = clocks.summary()
        peak, peak_why = pick_peak(ms_max * 1e-3, clk, peak_burst, peak_sust)
        # dominant kernel: the key-major dK/dV kernel (4 of the 5 algorithmic
        # backward GEMMs: S^T, dP^T, dV, dK = 8 B H N^2 d c flops per launch)
        f_dkdv = 0.8 * f_bwd
        # dQ path the library chose: the workspace holds materialised dS^T tiles
        # (d = 128 under the cap) beyond lse2 + D (8 B per padded row)
        n_q = (N + 127) // 128
        base_ws = 2 * ((n_units_rank * n_q * 128 * 4 + 255) // 256 * 256)
        tiles = n_units_rank * (n_q * (n_q + 1) // 2 if causal else n_q * n_q)
        ds_bytes = tiles * 32768
        # (with dropout the workspace may also hold a keep-bit mask of BH * Npad^2 / 8 bytes)
        dq_mode = "dS-GEMM" if ws.numel() >= base_ws + ds_bytes else "recompute"
        achieved = f_dkdv / (dkdv_ms * 1e-3) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(args.config, {}).get("bwd_dkdv_dram_bytes")
            except Exception:
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": dt,
            "data": "synthetic (torch.randn, " + ("one global seed, per-rank slabs" if strong else "per-rank seed") + ")",
            "config": {"workload": desc, "units_per_gpu": n_units_rank, "units_total": units_total,
                       "batch": B if strong else B * world, "heads": H, "seq_len": N, "head_dim": d,
                       "causal": causal, "global_batch": B if strong else B * world,
                       "parallelism": (f"(batch,head) units split over {world} GPU(s) (strong), no collective"
                                       if strong else f"(batch,head) shards x{world} (weak), no collective"),
                       "l2": "inputs (4 x %d MiB per GPU per layer) exceed the 126 MB L2; no flush"
                             % (q.numel() * 2 >> 20) if layers * q.numel() * 8 > (126 << 20)
                             else "inputs smaller than L2: L2-resident between steps",
                       "flop_model": "fwd 4BHN^2d*c + bwd 10BHN^2d*c, c=1/2 causal" +
                                     (f", x {layers} layers per step (one CUDA graph)" if layers > 1 else ""),
                       "layers": layers,
                       "dropout_p": args.dropout},
            "pct_of_peak": value / world / peak,
            "pct_of_peak_burst": value / world / peak_burst,
            "pct_of_peak_sustained": value / world / peak_sust,
            "peak_used": peak_why,
            "kernels_ms": {"fwd": fwd_ms, "bwd_preprocess": pre_ms, "bwd_dkdv": dkdv_ms, "bwd_dq": dq_ms,
                           "dropmask": mask_ms,
                           "note": "separate profiled pass after the timed region (CUDA events around each "
                                   "launch, which also break the PDL overlap); the sum can exceed ms_per_step"},
            "fwd_tflops": f_fwd / (fwd_ms * 1e-3) / 1e12,
            "bwd_tflops": f_bwd / ((pre_ms + dkdv_ms + dq_ms) * 1e-3) / 1e12,
            "bwd_dq_mode": dq_mode,
            "dq_kernel": ({"kernel": ("mha_bwd_dq_gemm_kernel" if os.environ.get("VATTN_DQ_PERSIST") == "0"
                                      else "mha_bwd_dq_tail_kernel (persistent dQ GEMM)"), "bound": "hbm",
                           "achieved_gbs": ds_bytes / (dq_ms * 1e-3) / 1e9,
                           "bytes_note": "dS^T tiles streamed once (16-bit, 32 KiB per tile pair)"}
                          if dq_mode == "dS-GEMM" else
                          {"kernel": "mha_bwd_dq_kernel", "bound": "tensor",
                           "tflops_executed": 0.6 * f_bwd / (dq_ms * 1e-3) / 1e12}),
            "roofline": {"kernel": "mha_bwd_dkdv_kernel", "bound": "tensor", "achieved": achieved,
                         "peak": peak, "peak_kind": f"{peak_why} ({peak_src})",
                         "unit": "TFLOP/s", "frac": achieved / peak, "frac_of_burst": achieved / peak_burst,
                         "frac_of_sustained": achieved / peak_sust, "traffic": traffic,
                         "algorithmic": "8 B H N^2 d c flops per launch (S^T, dP^T, dV, dK GEMMs)"},
            "e2e": {"value": e2e_val, "unit": "TFLOPS", "h2d_bytes_per_step": layers * h2d,
                    "d2h_bytes_per_step": layers * d2h,
                    "ms_per_step": e2e_ms},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
        }
        if verify is not None:
            line["verify_gather"] = verify
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only (a reported baseline)
            try:
                tfl, secs, sample, kind, cores = cpu_reference_sample(d, causal, os.cpu_count() or 1)
                line["cpu_baseline"] = {"value": tfl, "unit": "TFLOPS", "cores": cores, "kind": kind,
                                        "extrapolated": N != 1024,
                                        "sample": sample + (f"; EXTRAPOLATED to N = {N}: the reference's emulated "
                                                            "tile loops run at an N-independent GFLOP/s, so the "
                                                            "rate of the N = 1024 sample is reported as the "
                                                            "full-size rate" if N != 1024 else "")}
            except Exception as e:  # reported baseline only
                line["cpu_baseline"] = {"value": None, "unit": "TFLOPS", "cores": 0, "kind": "unavailable",
                                        "sample": f"failed: {e}"}
        print(json.dumps(line))
        if verify is not None and not verify["bitwise_equal"]:
            print(f"verify_gather FAILED: {verify['mismatch']}", file=sys.stderr)
            rc = 1
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
