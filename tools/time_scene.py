"""Scene synthesis at C5 size (2^22 + 1024 samples, 8 echoes, AWGN): device
build_signals (host numpy draws included) vs the reference's numpy evaluation
(the oracle restatement, bit-identical to radar.py on this host); plus the
device-vs-host error on the golden scenes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import oracle
from paper_1402_0532_b200 import scene
from test_oracle_golden import SCENES, scene_params
from test_gpu_scene import spec

golden = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/golden.npz"))
for name in SCENES:
    p = scene_params(golden, name)
    r, s = scene.build_signals(spec(scene, p))
    er = np.max(np.abs(r.samples.cpu().numpy() - golden[f"scn_{name}_ref"])) / np.max(np.abs(golden[f"scn_{name}_ref"]))
    es = np.max(np.abs(s.samples.cpu().numpy() - golden[f"scn_{name}_surv"])) / np.max(np.abs(golden[f"scn_{name}_surv"]))
    print(f"{name}: ref rel err {er:.2e}, surv rel err {es:.2e}")

g = np.random.default_rng(1402)
d, n = (1 << 22) + 1024, 1 << 22
echoes = tuple(scene.Echo(int(g.integers(0, 1000)), complex(g.uniform(-1, 1), g.uniform(-1, 1)),
                          float(g.uniform(-400, 400)) if k % 3 else 0.0) for k in range(8))
sp = scene.SceneSpec(echoes=echoes, fm=scene.FmSpec(duration_samples=d, seed=77),
                     noise=scene.NoiseSpec("awgn", snr_db=-20.0, seed=78), n=n, surv_gain=64.0)
for _ in range(2):
    scene.build_signals(sp, dtype=torch.complex64)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    scene.build_signals(sp, dtype=torch.complex64)
torch.cuda.synchronize()
gpu_ms = (time.perf_counter() - t0) / 3 * 1e3
t0 = time.perf_counter()
ref_o = oracle.scene_stereo_fm(d, 200_000.0, 0.25, 19_000.0, 77)
oracle.scene_surveillance(ref_o, [e.delay for e in echoes], [e.amplitude for e in echoes],
                          [e.doppler_hz for e in echoes], 200_000.0, {"kind": "awgn", "snr_db": -20.0, "seed": 78}, 64.0)
cpu_ms = (time.perf_counter() - t0) * 1e3
print(f"C5-size scene ({d} samples, 8 echoes, AWGN): device build_signals {gpu_ms:.1f} ms wall "
      f"(host numpy draws included), numpy {cpu_ms:.0f} ms")
