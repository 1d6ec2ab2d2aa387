"""One C3 NL-FFT launch (after warm-up) for ncu: python tools/prof_nlfft_once.py [dit|dif] [c64|c128]"""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1402_0532_b200 as sa
var = sys.argv[1] if len(sys.argv) > 1 else "dit"
dt = torch.complex128 if (len(sys.argv) > 2 and sys.argv[2] == "c128") else torch.complex64
x = torch.randn(4096, 65536, dtype=dt, device="cuda"); y = torch.empty_like(x)
for _ in range(3): sa.nfft_batch(x, out=y, variant=var)
torch.cuda.synchronize()
