"""Time the C4 map (lag stage alone and full map) on device-resident inputs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
from paper_1402_0532_b200 import _native
from paper_1402_0532_b200.workloads import c4_scene, c5_scene
C5 = os.environ.get("C5") == "1"
sc = c5_scene() if C5 else c4_scene()
L, M = (4096, 2048) if C5 else (1024, 512)
for dt in ((torch.complex64,) if C5 else (torch.complex64, torch.complex128)):
    s = torch.from_numpy(sc.surv).to(dt).cuda(); r = torch.from_numpy(sc.ref).to(dt).cuda()
    out = torch.empty((L, M), dtype=dt, device="cuda")
    z = torch.empty_like(out)
    d = _native.SA_C64 if dt == torch.complex64 else _native.SA_C128
    def lag():
        _native.check(_native.lib().sa_ambiguity_integrate(d, _native.ptr(s), _native.ptr(r), s.numel(), r.numel(), 0, L, M, 1, 0, _native.ptr(z), _native.stream_ptr()))
    def full():
        sa.ambiguity_map(s, r, L, M, out=out)
    for name, fn in (("lag", lag), ("map", full)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{'C5' if C5 else 'C4'} {str(dt)[6:]} {name} {ms:.4f} ms  lag {16*L*s.numel()/ms/1e9:.1f} TFLOP/s (16 flop/⊙)")
