import os, sys, subprocess, json
code = r'''
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1402_0532_b200 as sa
x = torch.randn(4096, 65536, dtype=torch.complex64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): sa.nfft_batch(x, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): sa.nfft_batch(x, out=y)
e1.record(); torch.cuda.synchronize()
print(e0.elapsed_time(e1) / 10)
'''
for p in [0, 1, 2, 3, 4, 7]:
    env = dict(os.environ, SA_NLFFT64K_PROBE=str(p))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("probe", p, out.stdout.strip(), out.stderr.strip()[-200:])
