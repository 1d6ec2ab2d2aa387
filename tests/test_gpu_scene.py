"""Scene synthesis on the device vs the reference's own
outputs (tests/golden: radar.build_signals of three scenes -- AWGN, eps-
contaminated and noiseless with complex amplitudes and negative Doppler) and
the pinned oracle.  The device sin/cos differ from the host libm by an ulp or
two, so the bar is a tolerance, stated per test; the random streams are the
reference's own."""

import numpy as np
import pytest

import oracle
from test_oracle_golden import SCENES, scene_params

pytestmark = pytest.mark.gpu

TOL = 1e-12  # max |device - reference| / max |reference|; measured ~1e-15


def T():
    import torch
    return torch


def spec(sc, p):
    return sc.SceneSpec(echoes=tuple(sc.Echo(d, complex(a), f) for d, a, f in zip(p["delays"], p["amps"], p["dopp"])),
                        fm=sc.FmSpec(f_s=p["f_s"], duration_samples=p["dur"], k_f=p["k_f"], f_p=p["f_p"],
                                     seed=p["seed"]),
                        noise=sc.NoiseSpec(**p["noise"]), n=p["n"], surv_gain=p["gain"])


def close(got, want, tol=TOL):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert err <= tol, f"relative max error {err:.3e} > {tol:g}"
    return err


@pytest.mark.parametrize("name", SCENES)
def test_stereo_fm_golden(sa, golden, name):
    from paper_1402_0532_b200 import scene
    p = scene_params(golden, name)
    s = scene.gen_stereo_fm(spec(scene, p).fm)
    assert s.samples.dtype == T().complex128 and s.f_s == p["f_s"]
    close(s.samples.cpu().numpy(), golden[f"scn_{name}_ref"])


@pytest.mark.parametrize("name", SCENES)
def test_synth_surveillance_golden(sa, golden, name):
    """Echo mixture + noise + gain from the reference's own illuminator."""
    from paper_1402_0532_b200 import scene
    p = scene_params(golden, name)
    ref = T().from_numpy(golden[f"scn_{name}_ref"]).cuda()
    s = scene.synth_surveillance(spec(scene, p), ref)
    close(s.samples.cpu().numpy(), golden[f"scn_{name}_surv"])


@pytest.mark.parametrize("name", SCENES)
def test_build_signals_golden(sa, golden, name):
    from paper_1402_0532_b200 import scene
    p = scene_params(golden, name)
    r, s = scene.build_signals(spec(scene, p))
    close(r.samples.cpu().numpy(), golden[f"scn_{name}_ref"])
    close(s.samples.cpu().numpy(), golden[f"scn_{name}_surv"])
    r32, s32 = scene.build_signals(spec(scene, p), dtype=T().complex64)
    assert r32.samples.dtype == T().complex64 and s32.samples.dtype == T().complex64
    close(s32.samples.cpu().numpy(), golden[f"scn_{name}_surv"], 1e-6)


def test_scene_cpi_scale_vs_oracle(sa):
    """2^20 samples, 8 echoes, AWGN: device vs the pinned oracle restatement."""
    from paper_1402_0532_b200 import scene
    g = np.random.default_rng(1402)
    d, n = (1 << 20) + 1024, 1 << 20
    echoes = tuple(scene.Echo(int(g.integers(0, 1000)), complex(g.uniform(-1, 1), g.uniform(-1, 1)),
                              float(g.uniform(-400, 400)) if k % 3 else 0.0) for k in range(8))
    sp = scene.SceneSpec(echoes=echoes, fm=scene.FmSpec(duration_samples=d, seed=77),
                         noise=scene.NoiseSpec("awgn", snr_db=-20.0, seed=78), n=n, surv_gain=64.0)
    r, s = scene.build_signals(sp)
    ref_o = oracle.scene_stereo_fm(d, 200_000.0, 0.25, 19_000.0, 77)
    close(r.samples.cpu().numpy(), ref_o)
    surv_o = oracle.scene_surveillance(ref_o, [e.delay for e in echoes], [e.amplitude for e in echoes],
                                       [e.doppler_hz for e in echoes], 200_000.0,
                                       {"kind": "awgn", "snr_db": -20.0, "seed": 78}, 64.0)
    close(s.samples.cpu().numpy(), surv_o)


def test_scene_feeds_the_map(sa, golden):
    """Device-built signals go straight into ambiguity_map: the target rows
    peak where the reference's surface does (argmax per true row)."""
    from paper_1402_0532_b200 import scene
    p = scene_params(golden, "none_custom")
    r, s = scene.build_signals(spec(scene, p))
    n = p["n"]
    m = sa.ambiguity_map(s.samples[:n].contiguous(), r.samples, 64, n, mode="exact").cpu().numpy()
    ref_map = oracle.ambiguity_map(golden["scn_none_custom_surv"][:n], golden["scn_none_custom_ref"], 0, 64, n,
                                   nthreads=8)
    for l in p["delays"]:
        assert np.argmax(np.abs(m[l])) == np.argmax(np.abs(ref_map[l]))


def test_scene_contracts(sa):
    from paper_1402_0532_b200 import scene
    from paper_1402_0532_b200.errors import ContractError
    fm = scene.FmSpec(duration_samples=600, seed=1)
    r = scene.gen_stereo_fm(fm)
    with pytest.raises(ContractError, match="below n \\+ max delay"):
        scene.synth_surveillance(scene.SceneSpec(echoes=(scene.Echo(200),), fm=fm, n=512), r)
    with pytest.raises(ContractError, match="at most 64"):
        scene.synth_surveillance(scene.SceneSpec(echoes=tuple(scene.Echo(1) for _ in range(65)), fm=fm, n=512), r)
    with pytest.raises(ContractError, match="zero-power"):
        scene.synth_surveillance(scene.SceneSpec(echoes=(scene.Echo(3, 0j),), fm=fm, n=512,
                                                 noise=scene.NoiseSpec("awgn", snr_db=0.0)), r)
    with pytest.raises(ContractError, match="complex128"):
        scene.synth_surveillance(scene.SceneSpec(echoes=(scene.Echo(3),), fm=fm, n=512),
                                 r.samples.to(T().complex64))
