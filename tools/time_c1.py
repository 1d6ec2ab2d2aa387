"""Time the C1 NDFT (N = 64, 4097 complex128 vectors, fast and exact modes) on
device-resident inputs, CUDA events, 200 launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
for n, b in ((64, 4097), (256, 4097), (1024, 1024), (64, 65536)):
    x = torch.randn(b, n, dtype=torch.complex128, device="cuda"); y = torch.empty_like(x)
    for mode in ("fast", "exact"):
        for _ in range(5): sa.ndft_batch(x, out=y, mode=mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200): sa.ndft_batch(x, out=y, mode=mode)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 200
        print(f"n={n} batch={b} {mode}: {ms * 1e3:.1f} us  {b * n * n / ms / 1e9:.3f} T⊙/s")
