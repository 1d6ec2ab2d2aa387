"""Generate golden vectors from the UNMODIFIED reference (signadd 0.1.0).

Run here (the survey container), never on the GPU box:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference read-only from /root/reference/pkg/src and writes
``tests/golden/golden.npz`` (committed).  The tests pin the CPU oracle
(``oracle/``) against these vectors, and the GPU kernels against the oracle.

Inputs are seeded (numpy PCG64), so they can be regenerated anywhere.  Large
outputs are stored as a sha256 of their bytes plus a strided sample.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import signadd as sa  # noqa: E402  (the reference)

    g: dict[str, np.ndarray] = {}

    # --- twiddle tables (transforms.py:108-146), pinned by hash ---------------
    tw_sizes = [1, 2, 3, 4, 8, 12, 64, 512, 1024, 2048, 4096, 65536]
    g["tw_sizes"] = np.array(tw_sizes)
    g["tw_sha"] = np.array([sha(sa.twiddle_table(n).entries) for n in tw_sizes])
    g["tw_64"] = sa.twiddle_table(64).entries.copy()

    # --- operator (operator.py:118-207) ------------------------------------------
    rng = np.random.default_rng(20240817)
    a = rng.uniform(-10, 10, 2000) + 1j * rng.uniform(-10, 10, 2000)
    b = rng.uniform(-10, 10, 2000) + 1j * rng.uniform(-10, 10, 2000)
    edge = np.array([0.0, -0.0, 5e-324, -5e-324, 1e-310, 1.0, -1.0, 1e308, -1e308,
                     2.0 ** -1074 * 3, 0.5, -0.25])
    ea, eb = np.meshgrid(edge, edge)
    ea = (ea + 1j * ea[::-1]).ravel()
    eb = (eb + 1j * eb.T).ravel()
    # keep the sums finite: |a|+|b| must not overflow
    keep = (np.abs(ea.real) + np.abs(eb.real) < 1.7e308) & (np.abs(ea.imag) + np.abs(eb.imag) < 1.7e308) \
        & (np.abs(ea.imag) + np.abs(eb.real) < 1.7e308) & (np.abs(ea.real) + np.abs(eb.imag) < 1.7e308)
    ea, eb = ea[keep], eb[keep]
    g["mf_a"] = np.concatenate([a, ea, [1 + 2j, 5 - 4j, 1 + 0j, 1 + 0j, 1 + 1j]])
    g["mf_b"] = np.concatenate([b, eb, [3 - 1j, 0 + 0j, 0 + 1j, 1 + 1j, 1 - 1j]])
    g["mf_out"] = sa.mf_complex(g["mf_a"], g["mf_b"])

    # --- NDFT (transforms.py:223-251) ------------------------------------------
    rng = np.random.default_rng(61)
    for n in (1, 2, 3, 5, 8, 16, 64, 128, 256):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        g[f"ndft_x_{n}"] = x
        g[f"ndft_y_{n}"] = sa.ndft(x).bins
    g["ndft_tone7_64"] = sa.ndft(sa.unit_tone(7, 64)).bins
    g["ndft_tones_64"] = np.stack([sa.ndft(sa.unit_tone(k, 64)).bins for k in range(64)])
    g["ndft_two_point"] = sa.ndft([1 + 0j, 0 + 0j]).bins
    # C1 sample: tone row + CN(0,1) rows (seed 14020532 + 0), N=64
    c1 = np.random.default_rng(14020532)
    xs = (c1.standard_normal((32, 64)) + 1j * c1.standard_normal((32, 64))) / np.sqrt(2.0)
    g["c1_x"] = xs
    g["c1_y"] = np.stack([sa.ndft(v).bins for v in xs])
    # the survey's N=1024 pin: CN(0,1)/sqrt2 from default_rng(14020532)
    r = np.random.default_rng(14020532)
    x1024 = (r.standard_normal(1024) + 1j * r.standard_normal(1024)) / np.sqrt(2.0)
    g["ndft_y_1024"] = sa.ndft(x1024).bins
    g["nfft_y_1024"] = sa.nfft(x1024).bins
    g["x_1024"] = x1024

    # --- NL-FFT (transforms.py:254-298) ------------------------------------------
    rng = np.random.default_rng(61)
    for n in (2, 4, 8, 16, 32, 64, 128, 256, 512, 2048, 4096):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        g[f"nfft_x_{n}"] = x
        g[f"nfft_y_{n}"] = sa.nfft(x).bins
    g["nfft_tones_64"] = np.stack([sa.nfft(sa.unit_tone(k, 64)).bins for k in range(64)])
    g["nfft_tones_512"] = np.stack([sa.nfft(sa.unit_tone(k, 512)).bins for k in range(0, 512, 37)])
    # exact zeros / subnormals / mixed scales inside the flow graph
    z = rng.standard_normal(256) + 1j * rng.standard_normal(256)
    z[::7] = 0.0
    z[3::11] = 5e-324 - 5e-324j
    z[5::13] = 1e200 + 1e-200j
    g["nfft_edge_x"] = z
    g["nfft_edge_y"] = sa.nfft(z).bins
    g["ndft_edge_y"] = sa.ndft(z[:64]).bins
    # large: 2^16 (hash + sample), input from default_rng(14020532 + 2)
    r = np.random.default_rng(14020534)
    x16 = r.standard_normal(65536) + 1j * r.standard_normal(65536)
    y16 = sa.nfft(x16).bins
    g["nfft_65536_sha"] = np.array(sha(y16))
    g["nfft_65536_sample"] = y16[::257].copy()

    # --- lag product / eq12a (ambiguity.py:116-202) --------------------------------
    rng = np.random.default_rng(988)
    surv = rng.standard_normal(64) + 1j * rng.standard_normal(64)
    ref = np.exp(2j * np.pi * rng.random(64))
    g["lag_surv"] = surv
    g["lag_ref"] = ref
    lags = [0, 1, 3, 7, 31, 63]
    g["lag_lags"] = np.array(lags)
    g["lag_conj"] = np.stack([sa.lag_product_mf(surv, ref, l, 64) for l in lags])
    g["lag_noconj"] = np.stack([sa.lag_product_mf(surv, ref, l, 64, conjugate_ref=False) for l in lags])
    g["lag_short_n"] = sa.lag_product_mf(surv, ref, 5, 40)
    fs = 200_000.0
    s_surv = sa.ComplexSignal(surv, fs)
    s_ref = sa.ComplexSignal(ref, fs)
    g["eq12a_g16"] = sa.ambiguity_eq12a(s_surv, s_ref, 8, 64, transform_input_gain=16.0).values
    g["eq12a_g1"] = sa.ambiguity_eq12a(s_surv, s_ref, 8, 64).values
    g["eq12a_noconj"] = sa.ambiguity_eq12a(s_surv, s_ref, 4, 64, conjugate_ref=False).values
    sv = rng.standard_normal(512) + 1j * rng.standard_normal(512)
    rf = np.exp(2j * np.pi * rng.random(512))
    g["eq12a_512_surv"] = sv
    g["eq12a_512_ref"] = rf
    g["eq12a_512"] = sa.compute_ambiguity("eq12a", sa.ComplexSignal(sv, fs), sa.ComplexSignal(rf, fs), 16, 512,
                                          transform_input_gain=4.0).values

    # --- block-integrated map, composed from reference primitives ----
    ns, m = 4096, 64
    t = ns // m
    r = np.random.default_rng(14020535)
    s = np.exp(1j * 2 * np.pi * 0.05 * np.cumsum(r.standard_normal(ns)))
    rr = s.copy()
    rr[37:] += 0.02 * s[:-37] * np.exp(2j * np.pi * 1e-3 * np.arange(ns - 37))
    rr += np.sqrt(0.05) * (r.standard_normal(ns) + 1j * r.standard_normal(ns))
    g["map_surv"] = rr
    g["map_ref"] = s
    rows = []
    for l in range(40):
        y = sa.lag_product_mf(rr, s, l, ns).reshape(m, t)
        zz = np.zeros(m, dtype=complex)
        for k in range(t):  # sequential block sum, from +0
            zz += y[:, k]
        rows.append(sa.nfft(zz).bins)
    g["map_ns4096_m64"] = np.stack(rows)
    rows = []
    for l in range(8):
        y = sa.lag_product_mf(rr, s, 100 + l, ns).reshape(m, t)
        zz = np.zeros(m, dtype=complex)
        for k in range(t):
            zz += y[:, k]
        rows.append(sa.ndft(0.5 * zz).bins)
    g["map_ns4096_m64_ndft_l100_g05"] = np.stack(rows)

    # --- exact-multiply variants: fft_exact, lag_product_exact,
    #     eq11 / eq12b / eq12c surfaces ----------------------------------------
    r = np.random.default_rng(14020537)
    for n in (2, 4, 8, 64, 512, 4096):
        x = r.standard_normal(n) + 1j * r.standard_normal(n)
        g[f"fftx_x_{n}"] = x
        g[f"fftx_y_{n}"] = sa.fft_exact(x).bins
    xz = np.zeros(16, complex)
    xz[3] = -0.0 - 0.0j
    g["fftx_zero16"] = sa.fft_exact(xz).bins
    sv = r.standard_normal(256) + 1j * r.standard_normal(256)
    rf = np.exp(2j * np.pi * r.random(256))
    g["vx_surv"], g["vx_ref"] = sv, rf
    for l in (0, 1, 37, 255):
        g[f"lagx_{l}"] = sa.lag_product_exact(sv, rf, l, 256)
    g["lagx_noconj_5"] = sa.lag_product_exact(sv, rf, 5, 256, conjugate_ref=False)
    S, R = sa.ComplexSignal(sv, fs), sa.ComplexSignal(rf, fs)
    for var in ("eq11", "eq12b", "eq12c"):
        sf = sa.compute_ambiguity(var, S, R, 12, 256, transform_input_gain=4.0)
        g[f"amb_{var}"] = sf.values
        g[f"amb_{var}_counts"] = np.array([
            sf.lag_op_counts.sign_ops, sf.lag_op_counts.abs_ops, sf.lag_op_counts.add_ops,
            sf.lag_op_counts.complex_mf_ops, sf.lag_op_counts.complex_mul_ops,
            sf.transform_op_counts.sign_ops, sf.transform_op_counts.abs_ops, sf.transform_op_counts.add_ops,
            sf.transform_op_counts.complex_mf_ops, sf.transform_op_counts.complex_mul_ops])
    g["amb_eq12c_noconj_g1"] = sa.compute_ambiguity("eq12c", S, R, 6, 256, conjugate_ref=False).values

    # --- detection: magnitudes, find_peaks, classify, floor -----
    import signadd.detection as det
    r = np.random.default_rng(14020536)
    z = r.standard_normal(4096) * 10.0 ** r.integers(-6, 7, 4096) + 1j * (
        r.standard_normal(4096) * 10.0 ** r.integers(-6, 7, 4096))
    z[:4] = [0, 3.0, -4j, 1e-300 + 1e-300j]
    g["abs_z"] = z
    g["abs_m"] = np.abs(z)
    g["abs_z32"] = z.astype(np.complex64)
    g["abs_m32"] = np.abs(z.astype(np.complex64))

    def surf(values):
        return sa.AmbiguitySurface(values=np.asarray(values, dtype=complex), range_bin_m=1.0,
                                   doppler_bin_hz=1.0, variant=sa.AmbiguityVariant.EQ12A,
                                   sample_rate_hz=1.0)

    def peaks(values, k):
        return np.array([(pk.l, pk.p, pk.magnitude) for pk in det.find_peaks(surf(values), k)],
                        dtype=float).reshape(-1, 3)

    ph = lambda shape: np.exp(2j * np.pi * r.random(shape))
    cases = {
        "rnd_7x9": r.standard_normal((7, 9)) + 1j * r.standard_normal((7, 9)),
        "ties_16x24": r.integers(0, 4, (16, 24)) * ph((16, 24)),
        "flat_5x5": np.full((5, 5), 2.0 + 1j),
        "one_1x1": np.array([[0.5 - 0.25j]]),
        "row_1x17": r.standard_normal((1, 17)) + 0j,
        "col_17x1": r.standard_normal((17, 1)) * 1j,
        "big_40x70": (r.standard_normal((40, 70)) + 1j * r.standard_normal((40, 70))) * 1e3,
    }
    cases["ties_16x24"][3, 5] = 7 * ph(())  # an isolated strict maximum among plateaus
    for name, v in cases.items():
        g[f"det_{name}"] = np.asarray(v, dtype=complex)
        for k in (1, 3, 1000):
            g[f"det_{name}_k{k}"] = peaks(v, k)
    scn = sa.two_targets_one_clutter(seed=3, n=512, l_bins=64)
    sf = det.surface_for_scenario(scn, "eq12a")
    g["det_scn_values"] = sf.values
    g["det_scn_true_bins"] = np.array(sa.true_bins(scn) if hasattr(sa, "true_bins")
                                      else __import__("signadd.radar").radar.true_bins(scn))
    g["det_scn_peaks"] = peaks(sf.values, len(scn.obstacles))
    rep = det.classify(sf, scn)
    g["det_scn_statuses"] = np.array([s_ == "detected" for s_ in rep.statuses])
    for gd in ((1, 1), (2, 2), (3, 5)):
        g[f"det_scn_floor_{gd[0]}_{gd[1]}"] = np.array(det.sidelobe_floor_db(sf, scn, gd))

    # --- scene synthesis (radar.py) -----------------------------
    from signadd import radar
    scenes = {
        "awgn_2t1c": radar.two_targets_one_clutter(
            noise=radar.NoiseModel(kind="awgn", snr_db=-12.0, seed=31), seed=5, n=1024, l_bins=64),
        "eps_4t2c": radar.four_targets_two_clutters(
            noise=radar.NoiseModel(kind="eps_contaminated", eps=0.8, sigma1=0.3, sigma2=4.0, seed=7),
            seed=9, n=2048, l_bins=64),
        "none_custom": radar.Scenario(
            tx_km=(0.0, 10.0), rx_km=(0.0, 0.0),
            obstacles=(radar.Obstacle(10.0, 0.0, doppler_hz=-333.25, amplitude=0.3 - 0.2j),
                       radar.Obstacle(3.0, 4.0, doppler_hz=12.5, amplitude=-1.5 + 0.75j),
                       radar.Obstacle(28.0, 33.0, doppler_hz=0.0, amplitude=0.5j)),
            fm=radar.StereoFmConfig(duration_samples=4096 + 100, seed=13, k_f=0.6),
            n=4096, l_bins=64, surv_gain=3.0),
    }
    for name, scn in scenes.items():
        s_ref, s_surv = radar.build_signals(scn)
        g[f"scn_{name}_ref"] = s_ref.samples
        g[f"scn_{name}_surv"] = s_surv.samples
        g[f"scn_{name}_delays"] = np.array(scn.delay_bins())
        g[f"scn_{name}_amps"] = np.array([complex(o.amplitude) for o in scn.obstacles])
        g[f"scn_{name}_dopp"] = np.array([o.doppler_hz for o in scn.obstacles])
        g[f"scn_{name}_geom"] = np.array([[o.x_km, o.y_km] for o in scn.obstacles])
        g[f"scn_{name}_txrx"] = np.array([scn.tx_km, scn.rx_km])
        nz = scn.noise
        g[f"scn_{name}_noise"] = np.array([str(nz.kind.value), repr(nz.snr_db), repr(nz.eps), repr(nz.sigma1),
                                           repr(nz.sigma2), str(nz.seed)])
        fm = scn.fm
        g[f"scn_{name}_fm"] = np.array([fm.f_s, fm.duration_samples, fm.k_f, fm.f_p, fm.seed], dtype=float)
        g[f"scn_{name}_n_gain"] = np.array([scn.n, scn.surv_gain], dtype=float)

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
