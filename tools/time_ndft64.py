"""Time the batched fp64 NDFT (C2 shape, complex128) on device-resident inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
x = torch.randn(65536, 1024, dtype=torch.complex128, device="cuda"); y = torch.empty_like(x)
for _ in range(2): sa.ndft_batch(x, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): sa.ndft_batch(x, out=y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"complex128 {ms:.3f} ms  {65536*1024*1024*16/ms/1e9:.1f} TFLOP/s")
