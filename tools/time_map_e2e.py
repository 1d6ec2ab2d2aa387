"""C4 / C5 map end to end through ambiguity_map with pinned host in/out (as bench.py's e2e)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
from paper_1402_0532_b200.workloads import c4_scene, c5_scene
for name, sc, L, M in (("C4", c4_scene(), 1024, 512), ("C5", c5_scene(), 4096, 2048)):
    hs = torch.from_numpy(sc.surv).to(torch.complex64).pin_memory()
    hr = torch.from_numpy(sc.ref).to(torch.complex64).pin_memory()
    hout = torch.empty((L, M), dtype=torch.complex64).pin_memory()
    f = lambda: sa.ambiguity_map(hs, hr, L, M, out=hout)
    for _ in range(2): f()
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name} map e2e {best:.3f} ms")
