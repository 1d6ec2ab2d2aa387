"""Per-CTA phase timestamps of the int8 lag kernel: run with a library built with
-DSA_LAG_TS (tools/build_variant.sh ts "-DSA_LAG_TS"; SA_LIB_PATH=tools/variants/ts.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1402_0532_b200 as sa
from paper_1402_0532_b200 import _native
from paper_1402_0532_b200.workloads import c4_scene, c5_scene
c5 = os.environ.get("C5") == "1"
sc = c5_scene() if c5 else c4_scene()
L, M = (4096, 2048) if c5 else (1024, 512)
s = torch.from_numpy(sc.surv).to(torch.complex64).cuda(); r = torch.from_numpy(sc.ref).to(torch.complex64).cuda()
for _ in range(3): sa.ambiguity_map(s, r, L, M)
torch.cuda.synchronize()
sa.ambiguity_map(s, r, L, M); torch.cuda.synchronize()
lib = _native.lib()
buf = (ctypes.c_ulonglong * (M * 8))()
lib.sa_lag_ts_read(buf, M * 8)
t = np.array(buf, dtype=np.float64).reshape(M, 8)
t0 = t[:, 0].min()
t = (t - t0) / 1000.0  # us
names = ["start", "prologue done", "A landed", "B0 ready", "MMAs issued", "MMAs done", "end"]
print("kernel span %.1f us" % (t[:, 6].max()))
for i in range(1, 7):
    d = t[:, i] - t[:, i - 1]
    print(f"{names[i-1]:>14s} -> {names[i]:<14s} mean {d.mean():6.2f} us  median {np.median(d):6.2f}  max {d.max():6.2f}")
life = t[:, 6] - t[:, 0]
print(f"CTA lifetime mean {life.mean():.2f} us, start times: first {t[:,0].min():.1f} last {t[:,0].max():.1f}")
