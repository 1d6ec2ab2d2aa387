"""C2 timing of the tensor-core NDFT vs the FFMA2 fast kernel (CUDA events)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1402_0532_b200 as sa
from paper_1402_0532_b200.workloads import c2_ndft
x = torch.from_numpy(c2_ndft().astype('complex64')).cuda()
y = torch.empty_like(x)
for mode in ("tc", "fast", "tc"):
    for _ in range(3): sa.ndft_batch(x, mode=mode, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): sa.ndft_batch(x, mode=mode, out=y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{mode}: {ms:.3f} ms  {65536 * 1024**2 / ms / 1e9:.3e} ⊙/s  tc-GEMM {2 * 65536 * 2048 * 8192 / ms / 1e9:.0f} TFLOP/s")
