import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1402_0532_b200 as sa
from paper_1402_0532_b200.workloads import c4_scene
sc = c4_scene()
s = torch.from_numpy(sc.surv).to(torch.complex64).cuda(); r = torch.from_numpy(sc.ref).to(torch.complex64).cuda()
for lag, dop, mode in (("mf", "nfft", "fast"), ("mf", "nfft", "exact"), ("exact", "fft", "fast"), ("exact", "nfft", "fast")):
    f = lambda: sa.ambiguity_map(s, r, 1024, 512, lag=lag, doppler=dop, mode=mode)
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    print(lag, dop, mode, f"{e0.elapsed_time(e1)/5:.3f} ms")
