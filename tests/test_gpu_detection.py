"""Detection on the device map vs the reference golden vectors
and the pinned oracle: detection.find_peaks (detection.py:85-108), classify's
guard-box decision (:115-134) and sidelobe_floor_db (:148-171)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

DET_CASES = ["rnd_7x9", "ties_16x24", "flat_5x5", "one_1x1", "row_1x17", "col_17x1", "big_40x70"]


def T():
    import torch
    return torch


def dev(a):
    return T().from_numpy(np.ascontiguousarray(a)).cuda()


def as_rows(peaks):
    return np.array([(p.l, p.p, p.magnitude) for p in peaks], dtype=float).reshape(-1, 3)


@pytest.mark.parametrize("name", DET_CASES)
@pytest.mark.parametrize("k", [1, 3, 1000])
def test_find_peaks_golden(sa, golden, name, k):
    """complex128 surfaces: bitwise equal to the reference (positions, order, magnitudes)."""
    got = as_rows(sa.find_peaks(golden[f"det_{name}"], k))
    assert np.array_equal(got, golden[f"det_{name}_k{k}"])


def test_find_peaks_complex64_vs_oracle(sa):
    g = np.random.default_rng(71)
    v = ((g.integers(0, 5, (300, 257)) * np.exp(2j * np.pi * g.random((300, 257))))).astype(np.complex64)
    v[100:103, 50:53] = 9  # plateau: no strict maximum
    v[7, 0] = 11           # on the edge
    for k in (1, 17, 1024):
        assert np.array_equal(as_rows(sa.map_peaks(dev(v), k)), oracle.find_peaks(v, k, "f32"))


@pytest.mark.parametrize("shape", [(1024, 512), (4096, 2048), (33, 2049)])
def test_map_peaks_large_vs_oracle(sa, shape):
    """Full-size maps (C4 / C5 shapes, ragged tiles) with quantised magnitudes, so
    equal-magnitude maxima must come out in row-major order."""
    g = np.random.default_rng(shape[0])
    v = (g.integers(0, 50, shape) + 1j * g.integers(0, 50, shape)).astype(np.complex128)
    for k in (8, 300):
        assert np.array_equal(as_rows(sa.map_peaks(dev(v), k)), oracle.find_peaks(v, k))


@pytest.mark.parametrize("shape", [(4096, 2048), (97, 130), (1, 1), (1, 61), (61, 1), (65, 31), (130, 59)])
def test_map_peaks_complex64_dense_vs_oracle(sa, shape):
    """complex64 maps (the integer-key path): quantised magnitudes (ties, plateaus),
    a checkerboard of strict maxima (64 per 4 x 64 warp strip, the compaction
    limit) and a continuous map; k up to the per-warp limit and past it."""
    g = np.random.default_rng(shape[1])
    q = (g.integers(0, 12, shape) + 1j * g.integers(0, 12, shape)).astype(np.complex64)
    cb = np.zeros(shape, np.complex64)
    cb[::2, ::2] = (1 + g.integers(0, 3, cb[::2, ::2].shape)).astype(np.complex64)  # a strict max every 2 x 2
    c = (g.standard_normal(shape) + 1j * g.standard_normal(shape)).astype(np.complex64)
    for v in (q, cb, c):
        for k in (1, 8, 32, 33):
            assert np.array_equal(as_rows(sa.map_peaks(dev(v), k)), oracle.find_peaks(v, k, "f32"))


def test_map_peaks_on_c4_map(sa):
    """The C4 map straight from ambiguity_map (device) -> peaks, vs the oracle on the same map."""
    from paper_1402_0532_b200.workloads import c4_scene
    sc = c4_scene()
    m = sa.ambiguity_map(dev(sc.surv.astype(np.complex64)), dev(sc.ref.astype(np.complex64)), 1024, 512)
    got = as_rows(sa.map_peaks(m, 10))
    assert np.array_equal(got, oracle.find_peaks(m.cpu().numpy(), 10, "f32"))
    assert as_rows(sa.ambiguity_peaks(dev(sc.surv.astype(np.complex64)), dev(sc.ref.astype(np.complex64)),
                                      1024, 512, 10)).tolist() == got.tolist()


def test_scenario_classify_and_floor_golden(sa, golden):
    v, tb = golden["det_scn_values"], [tuple(int(x) for x in b) for b in golden["det_scn_true_bins"]]
    assert np.array_equal(as_rows(sa.find_peaks(v, len(tb))), golden["det_scn_peaks"])
    statuses, overall, floor, peaks = sa.classify_bins(v, tb)
    assert [s == "detected" for s in statuses] == list(golden["det_scn_statuses"])
    for g0, g1 in ((1, 1), (2, 2), (3, 5)):
        assert sa.sidelobe_floor_db(v, tb, (g0, g1)) == float(golden[f"det_scn_floor_{g0}_{g1}"])


def test_floor_maxima_vs_oracle(sa):
    """Guard boxes hanging off the row edges and wrapping around Doppler bin 0."""
    from paper_1402_0532_b200.detection import floor_maxima
    g = np.random.default_rng(5)
    v = g.standard_normal((200, 300)) + 1j * g.standard_normal((200, 300))
    centers = [(0, 0), (199, 299), (100, 1), (50, 298), (250, 10)]
    for guard, dt in (((2, 2), np.complex128), ((1, 7), np.complex128), ((4, 3), np.complex64)):
        vv = v.astype(dt)
        got = floor_maxima(dev(vv), centers, guard)
        want = oracle.map_floor(vv, centers, guard, "f64" if dt == np.complex128 else "f32")
        assert got == want


def test_detection_errors(sa):
    from paper_1402_0532_b200.errors import ContractError
    v = np.ones((4, 4), complex)
    with pytest.raises(ContractError):
        sa.map_peaks(v, 0)
    with pytest.raises(ContractError):
        sa.map_peaks(v, 1025)
    with pytest.raises(ContractError):
        sa.sidelobe_floor_db(v, [(1, 1)], (5, 5))  # guard covers the whole surface
    with pytest.raises(ContractError):
        sa.classify_bins(v, [(1, 1)], (0, 1))
    assert sa.map_peaks(v, 5) == []  # flat: no strict maxima
