"""C4 / C5 map: eager calls against a CUDA-graph replay of the same call (is the map launch-bound?)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
from paper_1402_0532_b200.workloads import c4_scene, c5_scene
for C5 in (False, True):
    sc = c5_scene() if C5 else c4_scene()
    L, M = (4096, 2048) if C5 else (1024, 512)
    s = torch.from_numpy(sc.surv).to(torch.complex64).cuda(); r = torch.from_numpy(sc.ref).to(torch.complex64).cuda()
    out = torch.empty((L, M), dtype=torch.complex64, device="cuda")
    def full():
        sa.ambiguity_map(s, r, L, M, out=out)
    def timeit(fn, n=50):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    eager = timeit(full)
    ref = out.clone()
    try:
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for _ in range(3): full()
        torch.cuda.current_stream().wait_stream(st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            full()
        out.zero_()
        g.replay(); torch.cuda.synchronize()
        same = torch.equal(out.view(torch.uint8), ref.view(torch.uint8))
        gr = timeit(g.replay)
        print(f"{'C5' if C5 else 'C4'} eager {eager:.4f} ms  graph {gr:.4f} ms  identical {same}")
    except Exception as ex:
        print(f"{'C5' if C5 else 'C4'} eager {eager:.4f} ms  graph capture failed: {ex!r}"[:600])
