"""Time the 2^16 NL-FFT implementations (device-resident, CUDA events)."""
import os, sys, subprocess
code = r'''
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1402_0532_b200 as sa
for dt in (torch.complex64, torch.complex128):
    for var in ("dit", "dif"):
        x = torch.randn(4096, 65536, dtype=dt, device="cuda"); y = torch.empty_like(x)
        for _ in range(3): sa.nfft_batch(x, out=y, variant=var)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): sa.nfft_batch(x, out=y, variant=var)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        gb = 2 * x.numel() * x.element_size() / 1e9
        print(f"{str(dt)[6:]} {var} {ms:.3f} ms  {gb/ms*1e3:.0f} GB/s")
        del x, y
'''
impls = [sys.argv[sys.argv.index("--impl") + 1]] if "--impl" in sys.argv else ["2p", "cluster"]
for impl in impls:
    env = dict(os.environ, SA_NLFFT_IMPL=impl)
    out = subprocess.run(["timeout", "300", sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("impl", impl, "rc", out.returncode); print(out.stdout.strip(), out.stderr.strip()[-300:])
