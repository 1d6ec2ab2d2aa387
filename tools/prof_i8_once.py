import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
x = torch.randn(65536, 1024, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
for _ in range(3): sa.ndft_batch(x, out=y, mode="tc")
torch.cuda.synchronize()
