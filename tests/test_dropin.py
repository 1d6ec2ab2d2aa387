"""Drop-in into the UNMODIFIED reference package (signadd 0.1.0).

The reference is imported from baseline/_ref (pip-installed there, git-ignored,
travels to the GPU box) or, in the build container, from /root/reference.  The
CPU tests check the name patching and exception mapping; the GPU tests drive the
reference's own public API, CLI and detection pipeline through the B200 path and
compare with the reference's CPU results on the same inputs.
"""

import importlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


@pytest.fixture(scope="module")
def ref():
    for c in CANDIDATES:
        if os.path.isdir(os.path.join(c, "signadd")):
            if c not in sys.path:
                sys.path.insert(0, c)
            return importlib.import_module("signadd")
    pytest.skip("reference package not available (baseline/_ref not installed)")


@pytest.fixture()
def installed(ref):
    from paper_1402_0532_b200 import dropin
    dropin.install(ref)
    yield ref
    dropin.uninstall(ref)


def test_install_patches_every_binding(installed):
    ref = installed
    import signadd.ambiguity as amod
    import signadd.cli as cmod
    import signadd.detection as dmod
    import signadd.transforms as tmod
    assert ref.ndft is tmod.ndft is cmod.ndft is cmod._TRANSFORMS["ndft"]
    assert ref.nfft is tmod.nfft is amod.nfft is cmod._TRANSFORMS["nfft"]
    assert ref.compute_ambiguity is amod.compute_ambiguity is dmod.compute_ambiguity
    assert ref.lag_product_mf is amod.lag_product_mf
    assert ref.ndft.__module__ == "paper_1402_0532_b200.dropin"


def test_errors_are_reference_classes(installed):
    ref = installed
    for n in (1, 3, 12):
        with pytest.raises(ref.ContractError):
            ref.nfft(np.ones(n, complex))
    with pytest.raises(ref.DomainError):
        ref.ndft([np.nan, 1.0])
    with pytest.raises(ref.ContractError):
        ref.lag_product_mf(np.ones(8, complex), np.ones(8, complex), 8)


def test_uninstall_restores(ref):
    from paper_1402_0532_b200 import dropin
    before = ref.ndft
    dropin.install(ref)
    assert ref.ndft is not before
    dropin.uninstall(ref)
    assert ref.ndft is before


# --- GPU: the reference's public API / CLI / pipeline through the B200 path ----

@pytest.mark.gpu
def test_reference_api_through_dropin(installed, golden, sa):
    ref = installed
    for n in (8, 64, 256):
        s = ref.ndft(golden[f"ndft_x_{n}"])
        assert isinstance(s, ref.Spectrum) and s.transform_kind is ref.TransformKind.NDFT
        assert np.array_equal(s.bins, golden[f"ndft_y_{n}"])
        assert s.op_counts.complex_mf_ops == n * n
    c = ref.OpCounter()
    s = ref.nfft(golden["nfft_x_4096"], counter=c)
    assert np.array_equal(s.bins, golden["nfft_y_4096"])
    assert c.report().complex_mf_ops == 4096 * 13
    fs = 200_000.0
    a = ref.compute_ambiguity("eq12a", ref.ComplexSignal(golden["lag_surv"], fs),
                              ref.ComplexSignal(golden["lag_ref"], fs), 8, 64, transform_input_gain=16.0)
    assert isinstance(a, ref.AmbiguitySurface) and a.variant is ref.AmbiguityVariant.EQ12A
    assert np.array_equal(a.values, golden["eq12a_g16"])
    assert a.lag_op_counts.complex_mf_ops == 8 * 64


@pytest.mark.gpu
def test_reference_cli_transform_through_dropin(installed, golden, sa, tmp_path):
    ref = installed
    import signadd.cli as cmod
    out = str(tmp_path / "t")
    assert cmod.main(["transform", "--kind", "ndft", "--tone", "7", "--n", "64", "--out", out]) == 0
    rows = np.loadtxt(out + ".spectrum.csv", delimiter=",", skiprows=2)  # "# manifest", header
    got = rows[:, 1] + 1j * rows[:, 2]
    assert np.array_equal(got, golden["ndft_tone7_64"])  # repr() floats round-trip exactly
    assert int(np.argmax(rows[:, 3])) == 7


@pytest.mark.gpu
def test_reference_pipeline_eq12a_matches_cpu(ref, sa):
    """Scene synthesis (reference, CPU) -> eq12a surface: drop-in vs reference CPU."""
    from paper_1402_0532_b200 import dropin
    import signadd.detection as dmod
    scn = ref.two_targets_one_clutter(seed=3)  # reference defaults: n=4096, 64 delay bins
    cpu = dmod.surface_for_scenario(scn, "eq12a")
    dropin.install(ref)
    try:
        gpu = dmod.surface_for_scenario(scn, "eq12a")
    finally:
        dropin.uninstall(ref)
    assert gpu.values.shape == cpu.values.shape
    assert np.array_equal(gpu.values, cpu.values)  # value-identical (fp64, T == 1)
    assert gpu.op_counts == cpu.op_counts


@pytest.mark.gpu
def test_reference_classify_through_dropin(ref, sa):
    """detection.classify (reference) with find_peaks / sidelobe_floor_db on the GPU."""
    from paper_1402_0532_b200 import dropin
    import signadd.detection as dmod
    scn = ref.two_targets_one_clutter(seed=5, n=512, l_bins=64)
    sf = dmod.surface_for_scenario(scn, "eq12a")
    cpu = dmod.classify(sf, scn)
    cpu_floor = dmod.sidelobe_floor_db(sf, scn, (3, 4))
    dropin.install(ref)
    try:
        assert dmod.find_peaks.__module__ == "paper_1402_0532_b200.dropin"
        gpu = dmod.classify(sf, scn)
        gpu_floor = dmod.sidelobe_floor_db(sf, scn, (3, 4))
    finally:
        dropin.uninstall(ref)
    assert gpu == cpu  # statuses, overall, floor, peaks (reference Peak objects)
    assert gpu_floor == cpu_floor


@pytest.mark.gpu
def test_reference_exact_variants_through_dropin(ref, sa, golden):
    """compute_ambiguity for eq11 / eq12b / eq12c (and fft_exact, the CLI's
    'fft' transform) through the drop-in equal the reference's own CPU results."""
    from paper_1402_0532_b200 import dropin
    import signadd.cli as cmod
    fs = 200_000.0
    S, R = ref.ComplexSignal(golden["vx_surv"], fs), ref.ComplexSignal(golden["vx_ref"], fs)
    cpu = {v: ref.compute_ambiguity(v, S, R, 5, 256, transform_input_gain=2.0) for v in ("eq11", "eq12b", "eq12c")}
    x = golden["fftx_x_512"]
    cpu_fft = ref.fft_exact(x)
    dropin.install(ref)
    try:
        assert cmod._TRANSFORMS["fft"].__module__ == "paper_1402_0532_b200.dropin"
        for v, c in cpu.items():
            g = ref.compute_ambiguity(v, S, R, 5, 256, transform_input_gain=2.0)
            assert isinstance(g, ref.AmbiguitySurface) and g.variant is c.variant
            assert np.array_equal(g.values, c.values)
            assert g.op_counts == c.op_counts
        f = ref.fft_exact(x)
        assert np.array_equal(f.bins, cpu_fft.bins) and f.op_counts == cpu_fft.op_counts
        assert f.transform_kind is ref.TransformKind.FFT_EXACT
    finally:
        dropin.uninstall(ref)
