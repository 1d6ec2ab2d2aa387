"""C2 end to end through ndft_batch with pinned host in/out (as bench.py's e2e)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
x = torch.randn(65536, 1024, dtype=torch.complex64)
hin = x.pin_memory(); hout = torch.empty_like(hin).pin_memory()
xd = hin.cuda(); yd = torch.empty_like(xd)
mode = os.environ.get("MODE", "tc")
for name, f in (("device", lambda: sa.ndft_batch(xd, out=yd, mode=mode)), ("e2e", lambda: sa.ndft_batch(hin, out=hout, mode=mode))):
    for _ in range(2): f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"mode={mode} mib={sa.transforms.PIPELINE_MIB} ramp={sa.transforms.PIPELINE_RAMP} {name} {best:.3f} ms")
