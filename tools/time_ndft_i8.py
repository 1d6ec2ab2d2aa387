"""Time the complex128 C2 NDFT: DFMA fast kernel vs the int8 tensor-core path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
x = torch.randn(65536, 1024, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
for mode in ("tc", "fast", "tc"):
    for _ in range(2): sa.ndft_batch(x, out=y, mode=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): sa.ndft_batch(x, out=y, mode=mode)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"C2 c128 {mode}: {ms:.3f} ms  {65536*1024*1024/ms/1e9:.1f} G⊙/s")
