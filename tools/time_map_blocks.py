"""Per-rank compute of the multi-GPU C5 map on one GPU: the block-sharded lag
stage of one rank (M/G Doppler blocks x all 4096 delay rows, z rows to G owner
blocks -- here all local) and that rank's Doppler NL-FFT (L/G rows), for
G = 1, 2, 4, 8, next to the delay-row-sharded alternative (L/G rows, all blocks)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1402_0532_b200 as sa
from paper_1402_0532_b200 import _native
from paper_1402_0532_b200.sharded import shard_rows
from paper_1402_0532_b200.workloads import c5_scene
sc = c5_scene()
L, M = 4096, 2048
s = torch.from_numpy(sc.surv).to(torch.complex64).cuda(); r = torch.from_numpy(sc.ref).to(torch.complex64).cuda()
ns = s.numel()

def timeit(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

for G in (1, 2, 4, 8):
    zs = [torch.empty((shard_rows(L, G, o)[1], M), dtype=torch.complex64, device="cuda") for o in range(G)]
    table = torch.tensor([z.data_ptr() for z in zs], dtype=torch.int64, device="cuda")
    q0, qc = shard_rows(M, G, 0)
    def lag_blocks():
        _native.check(_native.lib().sa_ambiguity_integrate_blocks(
            _native.SA_C64, _native.ptr(s), _native.ptr(r), ns, ns, 0, L, M, q0, qc, 1, _native.ptr(table), G,
            _native.stream_ptr()))
    rows = shard_rows(L, G, 0)[1]
    out = torch.empty((rows, M), dtype=torch.complex64, device="cuda")
    from paper_1402_0532_b200.twiddle import device_twiddles
    import ctypes
    tw = device_twiddles(M, _native.SA_C64, 0)
    def nlfft():  # the owner's Doppler NL-FFT on its blocked z rows (sa_doppler_nlfft_blocked)
        _native.check(_native.lib().sa_doppler_nlfft_blocked(_native.SA_C64, _native.ptr(zs[0]), _native.ptr(out),
                                                              rows, M, ctypes.c_void_p(tw), 1.0, _native.stream_ptr()))
    zl = torch.empty((rows, M), dtype=torch.complex64, device="cuda")
    def lag_rows():
        _native.check(_native.lib().sa_ambiguity_integrate(
            _native.SA_C64, _native.ptr(s), _native.ptr(r), ns, ns, 0, rows, M, 1, _native.SA_NDFT_FAST,
            _native.ptr(zl), _native.stream_ptr()))
    a, b, c = timeit(lag_blocks), timeit(nlfft), timeit(lag_rows)
    print(f"G={G}: block-sharded lag {a:.4f} ms + NL-FFT {b:.4f} ms = {a + b:.4f} ms | delay-row lag {c:.4f} ms")
