"""Time the batched NDFT (C2 shape) on device-resident inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
for dt in (torch.complex64, torch.complex128):
    x = torch.randn(65536, 1024, dtype=dt, device="cuda"); y = torch.empty_like(x)
    for _ in range(3): sa.ndft_batch(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): sa.ndft_batch(x, out=y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{str(dt)[6:]} {ms:.3f} ms  {65536*1024*1024*16/ms/1e9:.1f} TFLOP/s")
