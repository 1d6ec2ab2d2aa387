"""Run one hot-path workload a few times at full config size (for ncu captures)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1402_0532_b200 as sa

what = sys.argv[1]
dt = torch.complex64 if (len(sys.argv) < 3 or sys.argv[2] == "c64") else torch.complex128
reps = 3
if what in ("ndft", "ndft_tc", "ndft_tc8"):
    x = torch.randn(65536, 1024, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    for _ in range(reps):
        sa.ndft_batch(x, out=y, mode={"ndft": "fast", "ndft_tc": "tc", "ndft_tc8": "tc8"}[what])
elif what in ("nlfft", "nlfft_dif"):
    x = torch.randn(4096, 65536, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    for _ in range(reps):
        sa.nfft_batch(x, out=y, variant="dif" if what == "nlfft_dif" else "dit")
elif what == "map":
    from paper_1402_0532_b200.workloads import c4_scene
    sc = c4_scene()
    s = torch.from_numpy(sc.surv).to(dt).cuda()
    r = torch.from_numpy(sc.ref).to(dt).cuda()
    for _ in range(reps):
        sa.ambiguity_map(s, r, 1024, 512)
elif what == "map5":
    from paper_1402_0532_b200.workloads import c5_scene
    sc = c5_scene()
    s = torch.from_numpy(sc.surv).to(dt).cuda()
    r = torch.from_numpy(sc.ref).to(dt).cuda()
    for _ in range(reps):
        sa.ambiguity_map(s, r, 4096, 2048)
elif what == "detect":
    g = torch.Generator(device="cuda").manual_seed(1)
    m = torch.randn(4096, 2048, dtype=dt, device="cuda", generator=g)
    for _ in range(reps):
        sa.map_peaks(m, 8)
torch.cuda.synchronize()
print("ok", what)
