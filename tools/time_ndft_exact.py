"""Time the exact (value-identical) NDFT mode on a C2-shaped batch (fewer rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
rows = int(os.environ.get("ROWS", "8192"))
for dt in (torch.complex64, torch.complex128):
    x = torch.randn(rows, 1024, dtype=dt, device="cuda"); y = torch.empty_like(x)
    sa.ndft_batch(x, out=y, mode="exact")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): sa.ndft_batch(x, out=y, mode="exact")
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{str(dt)[6:]} exact {rows} x 1024: {ms:.2f} ms -> C2 (65536 rows) {ms * 65536 / rows:.1f} ms  "
          f"{rows*1024*1024/ms/1e9:.1f} T⊙/s")
