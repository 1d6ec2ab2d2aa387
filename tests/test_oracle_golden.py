"""Pin the CPU oracle against golden vectors from the unmodified reference.

The golden file is produced by ``tests/golden/make_golden.py`` (reference
imported read-only); this module needs neither the reference nor a GPU.
fp64 comparisons are value-exact (``==``; signed zeros may differ, see
DESIGN.md "value identity").
"""

import hashlib

import numpy as np
import pytest

import oracle


def _eq(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    bad = np.flatnonzero(~(a == b))
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: {a.ravel()[bad[:3]]} vs {b.ravel()[bad[:3]]}"


def test_twiddle_hash_pin(golden):
    # transforms.py:108-146 restated in oracle.twiddle_table; hash-pinned
    for n, h in zip(golden["tw_sizes"], golden["tw_sha"]):
        t = oracle.twiddle_table(int(n))
        assert hashlib.sha256(t.tobytes()).hexdigest() == str(h), n
    _eq(oracle.twiddle_table(64), golden["tw_64"])


def test_mf_complex_golden(golden):
    _eq(oracle.mf_complex(golden["mf_a"], golden["mf_b"]), golden["mf_out"])


def test_mf_complex_known_answers():
    # test_operator.py:38-41, :162-168
    out = oracle.mf_complex([1 + 2j, 5 - 4j, 1 + 0j], [3 - 1j, 0j, 1j])
    _eq(out, [7 + 3j, 0j, 2j])
    a, b, c = 1 + 0j, 1 + 1j, 1 - 1j
    lhs = oracle.mf_complex(oracle.mf_complex(a, b), c)
    rhs = oracle.mf_complex(a, oracle.mf_complex(b, c))
    assert lhs == 6 + 0j and rhs == 5 + 0j


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 16, 64, 128, 256])
def test_ndft_golden(golden, n):
    _eq(oracle.ndft(golden[f"ndft_x_{n}"]), golden[f"ndft_y_{n}"])


def test_ndft_tones_and_c1(golden):
    tones = np.stack([oracle.unit_tone(k, 64) for k in range(64)])
    _eq(oracle.ndft(tones), golden["ndft_tones_64"])
    _eq(oracle.ndft(oracle.unit_tone(7, 64)), golden["ndft_tone7_64"])
    assert int(np.argmax(np.abs(golden["ndft_tone7_64"]))) == 7
    _eq(oracle.ndft(golden["c1_x"], nthreads=4), golden["c1_y"])
    _eq(oracle.ndft([1 + 0j, 0j]), golden["ndft_two_point"])
    _eq(oracle.ndft(golden["x_1024"]), golden["ndft_y_1024"])
    _eq(oracle.ndft(golden["nfft_edge_x"][:64]), golden["ndft_edge_y"])


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256, 512, 2048, 4096])
def test_nfft_golden(golden, n):
    _eq(oracle.nfft(golden[f"nfft_x_{n}"]), golden[f"nfft_y_{n}"])


def test_nfft_tones_edges_large(golden):
    tones = np.stack([oracle.unit_tone(k, 64) for k in range(64)])
    _eq(oracle.nfft(tones), golden["nfft_tones_64"])
    tones = np.stack([oracle.unit_tone(k, 512) for k in range(0, 512, 37)])
    _eq(oracle.nfft(tones), golden["nfft_tones_512"])
    _eq(oracle.nfft(golden["nfft_edge_x"]), golden["nfft_edge_y"])
    _eq(oracle.nfft(golden["x_1024"]), golden["nfft_y_1024"])
    r = np.random.default_rng(14020534)
    x16 = r.standard_normal(65536) + 1j * r.standard_normal(65536)
    y16 = oracle.nfft(x16)
    _eq(y16[::257], golden["nfft_65536_sample"])
    assert hashlib.sha256(y16.tobytes()).hexdigest() == str(golden["nfft_65536_sha"])


def test_lag_products_golden(golden):
    surv, ref = golden["lag_surv"], golden["lag_ref"]
    for i, l in enumerate(golden["lag_lags"]):
        _eq(oracle.lag_product_mf(surv, ref, int(l), 64), golden["lag_conj"][i])
        _eq(oracle.lag_product_mf(surv, ref, int(l), 64, conj=False), golden["lag_noconj"][i])
    _eq(oracle.lag_product_mf(surv, ref, 5, 40), golden["lag_short_n"])


def test_eq12a_golden(golden):
    surv, ref = golden["lag_surv"], golden["lag_ref"]
    # T == 1 (m == ns): the block-integrated map IS ambiguity_eq12a
    _eq(oracle.ambiguity_map(surv, ref, 0, 8, 64, gain=16.0), golden["eq12a_g16"])
    _eq(oracle.ambiguity_map(surv, ref, 0, 8, 64), golden["eq12a_g1"])
    _eq(oracle.ambiguity_map(surv, ref, 0, 4, 64, conj=False), golden["eq12a_noconj"])
    _eq(oracle.ambiguity_map(golden["eq12a_512_surv"], golden["eq12a_512_ref"], 0, 16, 512, gain=4.0,
                             nthreads=4), golden["eq12a_512"])


def test_block_map_golden(golden):
    rr, s = golden["map_surv"], golden["map_ref"]
    _eq(oracle.ambiguity_map(rr, s, 0, 40, 64, nthreads=4), golden["map_ns4096_m64"])
    _eq(oracle.ambiguity_map(rr, s, 100, 8, 64, gain=0.5, doppler="ndft"),
        golden["map_ns4096_m64_ndft_l100_g05"])


# --- DIF convention (no reference: parity unpinned; properties only) ---------

def test_dif_properties():
    g = np.random.default_rng(7)
    for _ in range(20):
        x = g.standard_normal(2) + 1j * g.standard_normal(2)
        _eq(oracle.nfft(x, "dif"), oracle.ndft(x))  # N=2 equals NDFT
    assert np.all(oracle.nfft(np.zeros((3, 16), complex), "dif") == 0)
    viol = [k for k in range(64) if int(np.argmax(np.abs(oracle.nfft(oracle.unit_tone(k, 64), "dif")))) != k]
    assert viol == []


def test_fp32_restatement_close():
    g = np.random.default_rng(3)
    x = g.standard_normal((4, 512)) + 1j * g.standard_normal((4, 512))
    y64 = oracle.nfft(x)
    y32 = oracle.nfft(x.astype(np.complex64), dtype="f32")
    err = np.max(np.abs(y32 - y64), axis=1) / np.sum(np.abs(y64), axis=1)
    assert np.all(err < 1e-4)


# --- detection (detection.py:85-171) ----------------------------

def test_abs_matches_numpy_simd_formula(golden):
    """The magnitude restatement equals np.abs as the reference host computed it."""
    assert np.array_equal(oracle.abs_np(golden["abs_z"]), golden["abs_m"])
    assert np.array_equal(oracle.abs_np(golden["abs_z32"], "f32"), golden["abs_m32"])


DET_CASES = ["rnd_7x9", "ties_16x24", "flat_5x5", "one_1x1", "row_1x17", "col_17x1", "big_40x70"]


@pytest.mark.parametrize("name", DET_CASES)
@pytest.mark.parametrize("k", [1, 3, 1000])
def test_find_peaks_golden(golden, name, k):
    got = oracle.find_peaks(golden[f"det_{name}"], k)
    assert np.array_equal(got, golden[f"det_{name}_k{k}"])


def test_scenario_detection_golden(golden):
    """Scene -> eq12a surface -> find_peaks / classify / sidelobe_floor_db (reference)."""
    v, tb = golden["det_scn_values"], golden["det_scn_true_bins"]
    pk = oracle.find_peaks(v, len(tb))
    assert np.array_equal(pk, golden["det_scn_peaks"])
    hits = [any(abs(l - l0) <= 2 and min(abs(p - p0) % v.shape[1], v.shape[1] - abs(p - p0) % v.shape[1]) <= 2
                for l, p, _ in pk) for l0, p0 in tb]
    assert hits == list(golden["det_scn_statuses"])
    for g0, g1 in ((1, 1), (2, 2), (3, 5)):
        gmax, out, n_out = oracle.map_floor(v, tb, (g0, g1))
        assert n_out > 0
        db = max(20.0 * np.log10(out / gmax), -300.0)
        assert db == float(golden[f"det_scn_floor_{g0}_{g1}"])


# --- exact-multiply variants ------------------------------------

@pytest.mark.parametrize("n", [2, 4, 8, 64, 512, 4096])
def test_fft_exact_golden(golden, n):
    _eq(oracle.fft_exact(golden[f"fftx_x_{n}"]), golden[f"fftx_y_{n}"])


def test_fft_exact_zero_golden(golden):
    x = np.zeros(16, complex)
    x[3] = -0.0 - 0.0j
    assert oracle.fft_exact(x).tobytes() == golden["fftx_zero16"].tobytes()  # signed zeros too


def test_lag_product_exact_golden(golden):
    sv, rf = golden["vx_surv"], golden["vx_ref"]
    for l in (0, 1, 37, 255):
        assert oracle.lag_product_exact(sv, rf, l, 256).tobytes() == golden[f"lagx_{l}"].tobytes()
    assert oracle.lag_product_exact(sv, rf, 5, 256, conj=False).tobytes() == golden["lagx_noconj_5"].tobytes()


@pytest.mark.parametrize("var", ["eq11", "eq12b", "eq12c"])
def test_exact_variant_surfaces_golden(golden, var):
    """T = 1 maps with the variant's lag product and Doppler transform equal the
    reference surfaces (gain 4 reaches only eq12c, ambiguity.py:224-239)."""
    sv, rf = golden["vx_surv"], golden["vx_ref"]
    lag = "exact" if var in ("eq11", "eq12c") else "mf"
    dop = "nfft" if var == "eq12c" else "fft"
    got = oracle.ambiguity_map(sv, rf, 0, 12, 256, gain=4.0 if var == "eq12c" else 1.0, lag=lag, doppler=dop)
    _eq(got, golden[f"amb_{var}"])
    got = oracle.ambiguity_map(sv, rf, 0, 6, 256, conj=False, lag="exact", doppler="nfft") if var == "eq12c" else None
    if got is not None:
        _eq(got, golden["amb_eq12c_noconj_g1"])


# --- scene synthesis (radar.py:179-275) -------------------------

SCENES = ["awgn_2t1c", "eps_4t2c", "none_custom"]


def scene_params(golden, name):
    """The golden scene as plain numbers (what the GPU tests rebuild it from)."""
    f_s, dur, k_f, f_p, seed = golden[f"scn_{name}_fm"]
    kind, snr, eps, s1, s2, nseed = [str(v) for v in golden[f"scn_{name}_noise"]]
    noise = {"kind": kind, "snr_db": float(snr), "eps": float(eps), "sigma1": float(s1), "sigma2": float(s2),
             "seed": int(nseed)}
    n, gain = golden[f"scn_{name}_n_gain"]
    return dict(f_s=float(f_s), dur=int(dur), k_f=float(k_f), f_p=float(f_p), seed=int(seed), noise=noise,
                n=int(n), gain=float(gain), delays=[int(v) for v in golden[f"scn_{name}_delays"]],
                amps=list(golden[f"scn_{name}_amps"]), dopp=[float(v) for v in golden[f"scn_{name}_dopp"]])


@pytest.mark.parametrize("name", SCENES)
def test_scene_oracle_golden(golden, name):
    """The evaluation order the scene kernels follow reproduces the reference bit for bit on the host."""
    p = scene_params(golden, name)
    ref = oracle.scene_stereo_fm(p["dur"], p["f_s"], p["k_f"], p["f_p"], p["seed"])
    _eq(ref, golden[f"scn_{name}_ref"])
    surv = oracle.scene_surveillance(golden[f"scn_{name}_ref"], p["delays"], p["amps"], p["dopp"], p["f_s"],
                                     p["noise"], p["gain"])
    _eq(surv, golden[f"scn_{name}_surv"])


@pytest.mark.parametrize("name", SCENES)
def test_scene_delay_bins_golden(golden, name):
    """scene.bistatic_delay_bins (host) = the reference's geometry (radar.py:195-199)."""
    from types import SimpleNamespace
    from paper_1402_0532_b200 import scene
    tx, rx = golden[f"scn_{name}_txrx"]
    f_s = float(golden[f"scn_{name}_fm"][0])
    got = [scene.bistatic_delay_bins(tuple(tx), tuple(rx), SimpleNamespace(x_km=x, y_km=y), f_s)
           for x, y in golden[f"scn_{name}_geom"]]
    assert got == [int(v) for v in golden[f"scn_{name}_delays"]]
