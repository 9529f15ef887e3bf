"""Pinned-host PCIe bandwidth (diagnostic): H2D alone, D2H alone, both at once."""
import torch
n = 512 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda"); d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a.record(); fn(); 
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
    return best
def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
t1 = timed(h2d); t2 = timed(d2h); t3 = timed(lambda: (h2d(), d2h()))
print(f"H2D {n/t1/1e6:.1f} GB/s  D2H {n/t2/1e6:.1f} GB/s  duplex {n/t3/1e6:.1f}+{n/t3/1e6:.1f} GB/s ({t3:.2f} ms for {n>>20} MiB each way)")
