"""Time sa_map_peaks on a C5-shaped complex64 map (4 maps cycled, > L2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
rows, cols, k = 4096, 2048, int(os.environ.get("K", "8"))
g = torch.Generator(device="cuda").manual_seed(1)
maps = [torch.randn(rows, cols, dtype=torch.complex64, device="cuda", generator=g) for _ in range(4)]
for i in range(3):
    sa.map_peaks(maps[i], k)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
n = int(os.environ.get("ITERS", "20"))
for i in range(n):
    sa.map_peaks(maps[i % 4], k)
e1.record(); torch.cuda.synchronize()
print(f"map_peaks (python API, incl. D2H of k peaks) {e0.elapsed_time(e1) / n:.4f} ms")
