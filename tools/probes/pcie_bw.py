"""Pinned host <-> device copy bandwidth on this box: H2D, D2H, and both at once
(the ceiling of the e2e lines), 512 MiB each, CUDA events."""
import torch
n = 512 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda"); d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event(); ev.record(cur)
    s1.wait_event(ev); s2.wait_event(ev)
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for chunk in (32 << 20, 8 << 20):
    def h2d_chunks():
        for o in range(0, n, chunk): d_in[o:o + chunk].copy_(h_in[o:o + chunk], non_blocking=True)
    print(f"H2D chunks {chunk >> 20} MiB: {n / timed(h2d_chunks) / 1e6:.1f} GB/s")
t = timed(lambda: d_in.copy_(h_in, non_blocking=True)); print(f"H2D {n / t / 1e6:.1f} GB/s ({t:.2f} ms)")
t = timed(lambda: h_out.copy_(d_out, non_blocking=True)); print(f"D2H {n / t / 1e6:.1f} GB/s ({t:.2f} ms)")
t = timed(both); print(f"H2D+D2H concurrent: {2 * n / t / 1e6:.1f} GB/s total ({t:.2f} ms for 512 MiB each way)")
