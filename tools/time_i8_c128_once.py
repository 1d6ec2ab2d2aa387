"""One C2 complex128 tc NDFT after warm-up (for per-kernel launch lists under ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
dt = torch.complex64 if os.environ.get("SA_DT") == "c64" else torch.complex128
mode = os.environ.get("SA_MODE", "tc")
x = torch.randn(65536, 1024, dtype=dt, device="cuda")
y = torch.empty_like(x)
for _ in range(3): sa.ndft_batch(x, out=y, mode=mode)
torch.cuda.synchronize()
