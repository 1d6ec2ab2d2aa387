"""Time the C2 NDFT (65536 x 1024): complex128 DFMA vs int8 tensor cores, and
complex64 bf16 tensor cores vs int8 tensor cores."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
for dt, modes in ((torch.complex128, ("tc", "fast", "tc")), (torch.complex64, ("tc", "tc8", "tc", "tc8"))):
    x = torch.randn(65536, 1024, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    for mode in modes:
        for _ in range(2): sa.ndft_batch(x, out=y, mode=mode)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): sa.ndft_batch(x, out=y, mode=mode)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"C2 {str(dt)[6:]} {mode}: {ms:.3f} ms  {65536*1024*1024/ms/1e9:.1f} G⊙/s")
