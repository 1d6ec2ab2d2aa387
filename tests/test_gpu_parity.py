"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference golden vectors.  Mirrors the reference's hot-path tests
(test_operator.py, test_transforms.py, test_ambiguity.py) plus the batched
configs of BASELINE.json at oracle-sized subsets and full-size properties.
"""

import hashlib

import numpy as np
import pytest

import oracle
from parity import TOL_F32, TOL_F64, assert_literal, assert_value_equal, literal, strict

pytestmark = pytest.mark.gpu


def T():
    import torch
    return torch


def dev(a, dt=None):
    t = T().from_numpy(np.ascontiguousarray(a))
    if dt is not None:
        t = t.to(dt)
    return t.cuda()


# --- operator (test_operator.py) ----------------------------------------------

def test_mf_complex_golden_bitwise(sa, golden):
    out = sa.mf_complex(golden["mf_a"], golden["mf_b"])
    assert out.tobytes() == golden["mf_out"].tobytes()  # incl. signed zeros


def test_mf_complex_examples_and_errors(sa):
    assert sa.mf_complex(1 + 2j, 3 - 1j) == 7 + 3j
    assert sa.mf_complex(5 - 4j, 0j) == 0j
    assert sa.mf_complex(1 + 0j, 1j) == 2j
    assert sa.mf_real(3, 2) == 5.0 and sa.mf_real(-1.5, 2) == -3.5 and sa.mf_real(7, 0) == 0.0
    assert sa.mf_sign(-3, 2) == -1 and sa.mf_sign(0, 5) == 0
    assert sa.vector_product([1, -2, 3], [1, -2, 3]) == 12.0
    assert np.array_equal(sa.scalar_vector(2, [1, -1]), [3.0, -3.0])
    for bad in (float("nan"), float("inf")):
        with pytest.raises(sa.DomainError):
            sa.mf_complex(complex(bad, 0), 1 + 1j)
    a, b, c = 1 + 0j, 1 + 1j, 1 - 1j
    assert sa.mf_complex(sa.mf_complex(a, b), c) == 6 and sa.mf_complex(a, sa.mf_complex(b, c)) == 5


def test_mf_complex_fp32_device(sa):
    g = np.random.default_rng(1)
    a = (g.standard_normal(100001) + 1j * g.standard_normal(100001)).astype(np.complex64)
    b = (g.standard_normal(100001) + 1j * g.standard_normal(100001)).astype(np.complex64)
    a[::97] = 0
    b[5::89] = -0.0
    out = sa.mf_complex(dev(a), dev(b)).cpu().numpy()
    assert_value_equal(out, oracle.mf_complex(a, b, dtype="f32"))


def test_mf_complex_negation_and_commutativity(sa):
    g = np.random.default_rng(20240817)
    a = g.uniform(-10, 10, 1000) + 1j * g.uniform(-10, 10, 1000)
    b = g.uniform(-10, 10, 1000) + 1j * g.uniform(-10, 10, 1000)
    assert np.array_equal(sa.mf_complex(-a, b), -sa.mf_complex(a, b))  # test_operator.py:225-229
    assert np.array_equal(sa.mf_complex(a, b), sa.mf_complex(b, a))


# --- NDFT (test_transforms.py) -------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 16, 64, 128, 256])
def test_ndft_dropin_golden(sa, golden, n):
    s = sa.ndft(golden[f"ndft_x_{n}"])
    assert_value_equal(s.bins, golden[f"ndft_y_{n}"])
    assert s.op_counts.complex_mf_ops == n * n and s.transform_kind.value == "ndft"


def test_ndft_dropin_known_answers(sa, golden):
    assert np.array_equal(sa.ndft([1 + 0j, 0j]).bins, [2 + 0j, 2 + 0j])
    assert np.array_equal(sa.ndft(np.zeros(16, complex)).bins, np.zeros(16))
    tones = [sa.peak_index(sa.ndft(sa.unit_tone(k, 64))) for k in range(64)]
    assert tones == list(range(64))
    assert_value_equal(sa.ndft(golden["x_1024"]).bins, golden["ndft_y_1024"])
    assert_value_equal(sa.ndft(golden["nfft_edge_x"][:64]).bins, golden["ndft_edge_y"])
    with pytest.raises(sa.ContractError):
        sa.ndft(np.ones((2, 2), complex))
    with pytest.raises(sa.DomainError):
        sa.ndft([np.nan, 1.0])


def test_ndft_batch_c1(sa, golden):
    from paper_1402_0532_b200.workloads import c1_ndft64
    x = c1_ndft64(4096)
    ref = oracle.ndft(x, nthreads=8)
    # fp64 exact mode: value-identical to the oracle (and hence the reference)
    assert_value_equal(sa.ndft_batch(dev(x), mode="exact").cpu().numpy(), ref)
    # fp64 fast mode (regrouped accumulation)
    y = sa.ndft_batch(dev(x), mode="fast").cpu().numpy()
    assert_literal(y, ref, TOL_F64)
    assert int(np.argmax(np.abs(y[0]))) == 7
    assert abs(y[0, 7] - (162.8437409998975 + 0j)) < 1e-9 * 283.13656515590407
    # fp32 (complex64 input, compared against the fp64 oracle of the same values)
    x32 = x.astype(np.complex64)
    ref32 = oracle.ndft(x32.astype(np.complex128), nthreads=8)
    y32 = sa.ndft_batch(dev(x32), mode="fast").cpu().numpy()
    assert_literal(y32, ref32, TOL_F32)
    assert int(np.argmax(np.abs(y32[0]))) == 7
    # golden C1 rows
    assert_literal(sa.ndft_batch(dev(golden["c1_x"])).cpu().numpy(), golden["c1_y"], TOL_F64)


@pytest.mark.parametrize("n", [1, 2, 7, 100, 255, 256, 300, 1000, 1024, 2048, 5003, 16384])
def test_ndft_batch_sizes(sa, n):
    """Ragged batches, tiny / prime / large N (16384: twiddles read from global,
    the table no longer fits in smem), zeros; fast within tolerance, exact
    value-identical."""
    g = np.random.default_rng(n)
    rows = 33 if n <= 2048 else 5
    x = g.standard_normal((rows, n)) + 1j * g.standard_normal((rows, n))
    x[3] = 0
    x[4, ::3] = 0
    ref = oracle.ndft(x, nthreads=8)
    assert_literal(sa.ndft_batch(dev(x)).cpu().numpy(), ref, TOL_F64)
    assert_value_equal(sa.ndft_batch(dev(x), mode="exact").cpu().numpy(), ref)
    y32 = sa.ndft_batch(dev(x.astype(np.complex64))).cpu().numpy()
    assert_literal(y32, oracle.ndft(x.astype(np.complex64).astype(np.complex128), nthreads=8), TOL_F32)


def test_ndft_c2_subset(sa):
    """C2 (N=1024, 65536 vectors, 10% tones) on the GPU; oracle on every 256th row."""
    from paper_1402_0532_b200.workloads import c2_ndft
    x = c2_ndft()
    rows = np.arange(0, x.shape[0], 256)
    for dt, cdt, tol in ((T().complex128, np.complex128, TOL_F64), (T().complex64, np.complex64, TOL_F32)):
        xd = dev(x.astype(cdt))
        y = sa.ndft_batch(xd)
        ys = y[T().from_numpy(rows).cuda()].cpu().numpy()
        ref = oracle.ndft(x[rows].astype(cdt).astype(np.complex128), nthreads=8)
        e = assert_literal(ys, ref, tol)
        print(f"C2 {cdt.__name__}: literal max {e.max():.2e}, strict max {strict(ys, ref).max():.2e}")
        del xd, y


def test_ndft_gain(sa):
    g = np.random.default_rng(5)
    x = g.standard_normal((4, 64)) + 1j * g.standard_normal((4, 64))
    ref = oracle.ndft(16.0 * x)
    assert_value_equal(sa.ndft_batch(dev(x), mode="exact", gain=16.0).cpu().numpy(), ref)


# --- NL-FFT (test_transforms.py) ------------------------------------------------

@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256, 512, 2048, 4096])
def test_nfft_dropin_golden(sa, golden, n):
    s = sa.nfft(golden[f"nfft_x_{n}"])
    assert_value_equal(s.bins, golden[f"nfft_y_{n}"])
    assert s.op_counts.complex_mf_ops == n * (int(np.log2(n)) + 1)


def test_nfft_dropin_properties(sa, golden):
    assert np.array_equal(sa.nfft([1 + 0j, 0j]).bins, [2 + 0j, 2 + 0j])
    assert np.array_equal(sa.nfft(np.zeros(16, complex)).bins, np.zeros(16))
    assert [sa.peak_index(sa.nfft(sa.unit_tone(k, 64))) for k in range(64)] == list(range(64))
    tones = np.stack([sa.unit_tone(k, 64) for k in range(64)])
    assert_value_equal(sa.nfft_batch(dev(tones)).cpu().numpy(), golden["nfft_tones_64"])
    tones = np.stack([sa.unit_tone(k, 512) for k in range(0, 512, 37)])
    assert_value_equal(sa.nfft_batch(dev(tones)).cpu().numpy(), golden["nfft_tones_512"])
    assert_value_equal(sa.nfft(golden["nfft_edge_x"]).bins, golden["nfft_edge_y"])
    for n in (1, 3, 12, 100):
        with pytest.raises(sa.ContractError):
            sa.nfft(np.ones(n, complex))
    g = np.random.default_rng(61)
    for _ in range(20):
        x = g.standard_normal(2) + 1j * g.standard_normal(2)
        assert np.array_equal(sa.nfft(x).bins, sa.ndft(x).bins)


def test_nfft_65536_reference_hash(sa, golden):
    r = np.random.default_rng(14020534)
    x = r.standard_normal(65536) + 1j * r.standard_normal(65536)
    y = sa.nfft(x).bins
    assert_value_equal(y[::257], golden["nfft_65536_sample"])
    assert hashlib.sha256(y.tobytes()).hexdigest() == str(golden["nfft_65536_sha"])


@pytest.mark.parametrize("variant", ["dit", "dif"])
@pytest.mark.parametrize("logn", list(range(1, 19)) + [20, 22])
def test_nfft_batch_vs_oracle(sa, variant, logn):
    n = 1 << logn
    batch = max(1, min(64, (1 << 18) // n))
    g = np.random.default_rng(logn)
    x = g.standard_normal((batch, n)) + 1j * g.standard_normal((batch, n))
    x[0, ::5] = 0
    if batch > 1:
        x[1] = 0
    # fp64: value-identical to the oracle (= reference for DIT)
    y = sa.nfft_batch(dev(x), variant=variant).cpu().numpy()
    assert_value_equal(y, oracle.nfft(x, variant, nthreads=8))
    # fp32: value-identical to the fp32 restatement, and within 1e-4 of fp64
    x32 = x.astype(np.complex64)
    y32 = sa.nfft_batch(dev(x32), variant=variant).cpu().numpy()
    assert_value_equal(y32, oracle.nfft(x32, variant, dtype="f32", nthreads=8))
    assert_literal(y32, oracle.nfft(x32.astype(np.complex128), variant, nthreads=8), TOL_F32)


def test_nfft_c3_subset(sa):
    """C3 rows (CN + 1-4 off-grid tones), N=2^16: GPU vs oracle, both variants."""
    from paper_1402_0532_b200.workloads import c3_nlfft_rows
    x = c3_nlfft_rows(1 << 16, np.arange(0, 4096, 512))
    for variant in ("dit", "dif"):
        y = sa.nfft_batch(dev(x), variant=variant).cpu().numpy()
        assert_value_equal(y, oracle.nfft(x, variant, nthreads=8))
        y32 = sa.nfft_batch(dev(x.astype(np.complex64)), variant=variant).cpu().numpy()
        ref = oracle.nfft(x.astype(np.complex64).astype(np.complex128), variant, nthreads=8)
        e = assert_literal(y32, ref, TOL_F32)
        print(f"C3 {variant} fp32: literal max {e.max():.2e}; strict p50 "
              f"{np.median(strict(y32, ref)):.2e} max {strict(y32, ref).max():.2e}")


def test_nfft_gain_and_inplace(sa):
    g = np.random.default_rng(9)
    x = g.standard_normal((8, 256)) + 1j * g.standard_normal((8, 256))
    assert_value_equal(sa.nfft_batch(dev(x), gain=16.0).cpu().numpy(), oracle.nfft(16.0 * x))
    xd = dev(x)
    sa.nfft_batch(xd, out=xd)
    assert_value_equal(xd.cpu().numpy(), oracle.nfft(x))


# --- lag products and maps (test_ambiguity.py) -------------------------------------

def test_lag_product_golden(sa, golden):
    surv, ref = golden["lag_surv"], golden["lag_ref"]
    for i, l in enumerate(golden["lag_lags"]):
        assert_value_equal(sa.lag_product_mf(surv, ref, int(l), 64), golden["lag_conj"][i])
        assert_value_equal(sa.lag_product_mf(surv, ref, int(l), 64, conjugate_ref=False),
                           golden["lag_noconj"][i])
    assert_value_equal(sa.lag_product_mf(surv, ref, 5, 40), golden["lag_short_n"])
    assert np.array_equal(sa.lag_product_mf(np.full(4, 1 + 2j), np.full(4, 3 + 1j), 0), np.full(4, 7 + 3j))
    with pytest.raises(sa.ContractError):
        sa.lag_product_mf(np.ones(8, complex), np.ones(8, complex), 8)
    with pytest.raises(sa.ContractError):
        sa.lag_product_mf(np.ones(8, complex), np.ones(8, complex), -1)
    with pytest.raises(sa.ContractError):
        sa.lag_product_mf(np.ones(4, complex), np.ones(8, complex), 0, n=8)


def test_eq12a_golden(sa, golden):
    fs = 200_000.0
    S = sa.ComplexSignal
    surv, ref = S(golden["lag_surv"], fs), S(golden["lag_ref"], fs)
    a = sa.ambiguity_eq12a(surv, ref, 8, 64, transform_input_gain=16.0)
    assert_value_equal(a.values, golden["eq12a_g16"])
    assert a.lag_op_counts.complex_mf_ops == 8 * 64 and a.transform_op_counts.complex_mul_ops == 0
    assert_value_equal(sa.ambiguity_eq12a(surv, ref, 8, 64).values, golden["eq12a_g1"])
    assert_value_equal(sa.ambiguity_eq12a(surv, ref, 4, 64, conjugate_ref=False).values,
                       golden["eq12a_noconj"])
    s5 = sa.compute_ambiguity("eq12a", S(golden["eq12a_512_surv"], fs), S(golden["eq12a_512_ref"], fs),
                              16, 512, transform_input_gain=4.0)
    assert_value_equal(s5.values, golden["eq12a_512"])
    assert s5.doppler_bin_hz == fs / 512
    z = sa.ambiguity_eq12a(S(np.zeros(16), fs), S(np.ones(16), fs), 4, 16)
    assert np.array_equal(z.values, np.zeros((4, 16)))


def test_rows_independent_of_order(sa):
    # test_ambiguity.py:208-217: any row range gives bit-identical rows
    g = np.random.default_rng(988)
    surv = g.standard_normal(64) + 1j * g.standard_normal(64)
    ref = np.exp(2j * np.pi * g.random(64))
    full = sa.ambiguity_map(surv, ref, 8, 64, gain=16.0, mode="exact")
    for l in reversed(range(8)):
        row = sa.ambiguity_map(surv, ref, 1, 64, l0=l, gain=16.0, mode="exact")
        assert full[l].tobytes() == row[0].tobytes()
        y = sa.lag_product_mf(surv, ref, l, 64)
        assert_value_equal(row[0], sa.nfft(16.0 * y).bins)


def test_block_map_golden(sa, golden):
    rr, s = golden["map_surv"], golden["map_ref"]
    ex = sa.ambiguity_map(rr, s, 40, 64, mode="exact")
    assert_value_equal(ex, golden["map_ns4096_m64"])  # sequential sums: value-identical
    fa = sa.ambiguity_map(rr, s, 40, 64, mode="fast")
    assert_literal(fa, golden["map_ns4096_m64"], TOL_F64)
    nd = sa.ambiguity_map(rr, s, 8, 64, l0=100, gain=0.5, doppler="ndft", mode="exact")
    assert_literal(nd, golden["map_ns4096_m64_ndft_l100_g05"], TOL_F64)
    f32 = sa.ambiguity_map(dev(rr.astype(np.complex64)), dev(s.astype(np.complex64)), 40, 64).cpu().numpy()
    ref32 = oracle.ambiguity_map(rr.astype(np.complex64), s.astype(np.complex64), 0, 40, 64)
    assert_literal(f32, ref32, TOL_F32)


def test_map_c4_sampled_rows(sa):
    """C4: 2^20 samples, 1024 delay bins x 512 Doppler bins, c64 on the GPU; the fp64
    oracle (of the same complex64 inputs) on 16 sampled rows incl. the target rows."""
    from paper_1402_0532_b200.workloads import c4_scene
    sc = c4_scene()
    surv = sc.surv.astype(np.complex64)
    ref = sc.ref.astype(np.complex64)
    y = sa.ambiguity_map(dev(surv), dev(ref), 1024, 512).cpu().numpy()
    rows = sorted(set([0, 1, 511, 1023] + [int(t) for t in sc.delays] + list(range(100, 1000, 97))))
    for l in rows:
        ref_row = oracle.ambiguity_map(surv.astype(np.complex128), ref.astype(np.complex128), l, 1, 512)
        assert_literal(y[l:l + 1], ref_row, TOL_F32)
    # fp64 path on a few rows
    y64 = sa.ambiguity_map(dev(sc.surv), dev(sc.ref), 64, 512, l0=sc.delays[0] - 10).cpu().numpy()
    ref64 = oracle.ambiguity_map(sc.surv, sc.ref, int(sc.delays[0]) - 10, 64, 512, nthreads=8)
    assert_literal(y64, ref64, TOL_F64)


@pytest.mark.parametrize("dt", ["c64", "c128"])
def test_nfft64k_persistent_loop(sa, dt):
    """Fused single-pass 2^16 kernel with more signals than resident clusters
    (exercises the persistent loop, TMA double buffering and the cluster
    barriers), with gain and in place."""
    g = np.random.default_rng(164)
    b = 80
    x = g.standard_normal((b, 1 << 16)) + 1j * g.standard_normal((b, 1 << 16))
    x[7] = 0
    x[9, ::3] = 0
    cdt = np.complex64 if dt == "c64" else np.complex128
    xs = x.astype(cdt)
    od = "f32" if dt == "c64" else "f64"
    ref = oracle.nfft(2.5 * xs.astype(np.complex128) if dt == "c128" else (np.float32(2.5) * xs), "dit",
                      dtype=od, nthreads=8)
    y = sa.nfft_batch(dev(xs), gain=2.5).cpu().numpy()
    assert_value_equal(y, ref)
    xd = dev(xs)
    sa.nfft_batch(xd, out=xd)
    assert_value_equal(xd.cpu().numpy(), oracle.nfft(xs, "dit", dtype=od, nthreads=8))


@pytest.mark.parametrize("dt", ["c64", "c128"])
@pytest.mark.parametrize("variant", ["dit", "dif"])
def test_nfft64k_batch_edges(sa, variant, dt):
    """Fused 2^16 kernel, batch sizes around the number of resident clusters (33
    clusters of 4 CTAs for complex64, up to 18 of 8 for complex128 on a B200): 1, 2
    and 3+ signals per cluster and clusters with one signal fewer than others --
    every prologue / steady / drain case of the signal pipeline (the TMEM-parking
    schedule computes one tile of signal s + 2 before phase B of signal s + 1; the
    complex64 and complex128 kernels use different forms of that loop)."""
    g = np.random.default_rng(165)
    batches = (1, 2, 32, 33, 34, 66, 67, 100, 133) if dt == "c64" else (1, 2, 15, 16, 17, 18, 19, 35, 37, 55)
    bmax = batches[-1]
    cdt = np.complex64 if dt == "c64" else np.complex128
    xs = (g.standard_normal((bmax, 1 << 16)) + 1j * g.standard_normal((bmax, 1 << 16))).astype(cdt)
    ref = oracle.nfft(xs, variant, dtype="f32" if dt == "c64" else "f64", nthreads=8)
    xd = dev(xs)
    for b in batches:
        y = sa.nfft_batch(xd[:b], variant=variant).cpu().numpy()
        assert_value_equal(y, ref[:b])


def test_map_graph_replay_bit_identical(sa):
    """MapGraph: the captured map call replayed on new buffer contents equals the
    eager call bit for bit (complex64 int8 lag stage + Doppler NL-FFT, and a
    complex128 map), including after the inputs are replaced."""
    import torch
    g = np.random.default_rng(167)
    for dt, ns, L, M in ((np.complex64, 1 << 16, 64, 256), (np.complex128, 1 << 13, 24, 64)):
        tdt = torch.complex64 if dt == np.complex64 else torch.complex128
        mg = sa.MapGraph(ns, ns, L, M, dtype=tdt)
        for trial in range(3):
            s = np.exp(1j * 2 * np.pi * g.random(ns)).astype(dt)
            r = (s + 0.1 * (g.standard_normal(ns) + 1j * g.standard_normal(ns))).astype(dt)
            mg.load(r, s)
            y = mg.replay().clone()
            ref = sa.ambiguity_map(dev(r), dev(s), L, M)
            assert torch.equal(y.view(torch.uint8), ref.view(torch.uint8)), (dt, trial)
    with pytest.raises(sa.ContractError):
        sa.MapGraph(1024, 1024, 4, 16, out=None)


def test_nfft64k_concurrent_streams_and_tmem(sa):
    """The fused 2^16 kernels allocate TMEM (parking schedule). Calls on several
    streams at once -- complex64 DIT, complex128 DIF and an int8 tensor-core NDFT,
    which takes all 512 TMEM columns of an SM -- must give exactly the results of
    the same calls made one after the other, repeatedly (allocation and release
    of TMEM between co-scheduled kernels, no cross-call state)."""
    import torch
    g = np.random.default_rng(166)
    x64 = dev((g.standard_normal((70, 1 << 16)) + 1j * g.standard_normal((70, 1 << 16))).astype(np.complex64))
    x128 = dev(g.standard_normal((40, 1 << 16)) + 1j * g.standard_normal((40, 1 << 16)))
    xn = dev((g.standard_normal((3000, 1024)) + 1j * g.standard_normal((3000, 1024))).astype(np.complex64))
    calls = [lambda o: sa.nfft_batch(x64, out=o, variant="dit"),
             lambda o: sa.nfft_batch(x128, out=o, variant="dif"),
             lambda o: sa.ndft_batch(xn, out=o, mode="tc8")]
    ins = [x64, x128, xn]
    ref = [torch.empty_like(x) for x in ins]
    for c, r in zip(calls, ref):
        c(r)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in calls]
    outs = [torch.empty_like(x) for x in ins]
    for _ in range(5):
        for o in outs:
            o.zero_()
        for c, o, st in zip(calls, outs, streams):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                c(o)
                c(o)
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            assert torch.equal(o.view(torch.uint8), r.view(torch.uint8))


def test_map_c5_sampled_rows(sa):
    """C5 (2^22 samples, 8 targets), 4096 delay bins x 2048 Doppler bins, c64 on
    the GPU; the fp64 oracle of the same complex64 inputs on the target rows and
    the edge rows; a row range computed alone equals the same rows of the full map
    bit for bit (the delay-bin sharding invariant)."""
    from paper_1402_0532_b200.workloads import c5_scene
    sc = c5_scene()
    surv = sc.surv.astype(np.complex64)
    ref = sc.ref.astype(np.complex64)
    ds, dr = dev(surv), dev(ref)
    full = sa.ambiguity_map(ds, dr, 4096, 2048)
    assert full.shape == (4096, 2048)
    rows = sorted(set([0, 4095] + [int(t) for t in sc.delays[:3]]))
    y = full[T().tensor(rows, device=full.device)].cpu().numpy()
    s128, r128 = surv.astype(np.complex128), ref.astype(np.complex128)
    for i, l in enumerate(rows):
        assert_literal(y[i:i + 1], oracle.ambiguity_map(s128, r128, l, 1, 2048, nthreads=8), TOL_F32)
    part = sa.ambiguity_map(ds, dr, 512, 2048, l0=1536)
    assert T().equal(part, full[1536:2048])


def _sharded_worker(port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        import paper_1402_0532_b200 as sa
        from paper_1402_0532_b200.sharded import ambiguity_map_sharded, broadcast_inputs
        from paper_1402_0532_b200.workloads import radar_scene
        sc = radar_scene(1 << 16, 2, 4242)
        ds = torch.from_numpy(sc.surv.astype(np.complex64)).cuda()
        dr = torch.from_numpy(sc.ref.astype(np.complex64)).cuda()
        broadcast_inputs(ds, dr)
        full = ambiguity_map_sharded(ds, dr, 96, 128)
        direct = sa.ambiguity_map(ds, dr, 96, 128)
        q.put(bool(torch.equal(full, direct)))
    finally:
        dist.destroy_process_group()


def test_sharded_map_nccl_single_rank(sa):
    """The multi-GPU map path (NCCL broadcast, delay-bin shard, NCCL gather) on
    one GPU in a world of 1: the gathered map equals the single-call map."""
    import socket
    import torch.multiprocessing as mp
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_sharded_worker, args=(port, q))
    p.start()
    p.join(300)
    assert p.exitcode == 0
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("tb", [8, 16, 24, 48, 2048])
def test_map_c64_block_lengths(sa, tb):
    """complex64 fast lag integration for every kernel the block length T selects
    (T % 16 == 0: packed FFMA2 pairs i / i+T/2; T % 8 == 0: scalar tiles), with
    ragged lag counts (not a multiple of the 64-lag tile) and a nonzero l0, vs the
    oracle of the same complex64 inputs; exact mode is value-equal to the f32 oracle."""
    g = np.random.default_rng(500 + tb)
    m = 32
    ns = tb * m
    surv = (g.standard_normal(ns) + 1j * g.standard_normal(ns)).astype(np.complex64)
    ref = np.exp(2j * np.pi * g.random(ns)).astype(np.complex64)
    surv[5] = 0
    ref[9] = 0
    l0, L = 3, 70
    y = sa.ambiguity_map(dev(surv), dev(ref), L, m, l0=l0).cpu().numpy()
    assert_literal(y, oracle.ambiguity_map(surv.astype(np.complex128), ref.astype(np.complex128), l0, L, m,
                                           nthreads=8), TOL_F32)
    ye = sa.ambiguity_map(dev(surv), dev(ref), L, m, l0=l0, mode="exact").cpu().numpy()
    assert_value_equal(ye, oracle.ambiguity_map(surv, ref, l0, L, m, dtype="f32", nthreads=8))


@pytest.mark.parametrize("dt", ["c64", "c128"])
@pytest.mark.parametrize("lag", ["mf", "exact"])
@pytest.mark.parametrize("tb", [8, 33, 2048])
def test_map_exact_seq_tiles(sa, dt, lag, tb):
    """Exact (sequential) mode on the smem-tiled kernel (k_lag_integrate_seq, T >= 8):
    lag counts spanning several 256-lag tiles with a ragged tail, l0 > 0, zeros in
    both signals -- value-equal to the oracle's sequential composition."""
    g = np.random.default_rng(1300 + tb)
    m = {8: 128, 33: 32, 2048: 4}[tb]  # ns > l0 + L: every lag is below the reference length
    ns = tb * m
    cdt = np.complex64 if dt == "c64" else np.complex128
    surv = (g.standard_normal(ns) + 1j * g.standard_normal(ns)).astype(cdt)
    ref = np.exp(2j * np.pi * g.random(ns)).astype(cdt)
    surv[[0, 7, ns // 2]] = 0
    ref[[1, 3]] = 0
    l0, L = 5, 600
    y = sa.ambiguity_map(dev(surv), dev(ref), L, m, l0=l0, lag=lag, mode="exact").cpu().numpy()
    want = oracle.ambiguity_map(surv, ref, l0, L, m, lag=lag, dtype="f32" if dt == "c64" else "f64", nthreads=8)
    assert_value_equal(y, want)


@pytest.mark.parametrize("dt,tb", [("c64", 8192), ("c64", 6000), ("c128", 4096), ("c128", 16384)])
def test_map_large_block_lengths(sa, dt, tb):
    """Block lengths whose lag tiles exceed shared memory at some tiling: the
    launcher steps NT down, then to the scalar tiles, then to the sequential
    kernels -- fast mode stays within tolerance of the oracle, exact mode value-equal."""
    g = np.random.default_rng(1700 + tb)
    m = 4
    ns = tb * m
    cdt = np.complex64 if dt == "c64" else np.complex128
    surv = (g.standard_normal(ns) + 1j * g.standard_normal(ns)).astype(cdt)
    ref = np.exp(2j * np.pi * g.random(ns)).astype(cdt)
    l0, L = 2, 130
    f = "f32" if dt == "c64" else "f64"
    y = sa.ambiguity_map(dev(surv), dev(ref), L, m, l0=l0).cpu().numpy()
    assert_literal(y, oracle.ambiguity_map(surv.astype(np.complex128), ref.astype(np.complex128), l0, L, m,
                                           nthreads=8), TOL_F32 if dt == "c64" else TOL_F64)
    ye = sa.ambiguity_map(dev(surv), dev(ref), L, m, l0=l0, mode="exact").cpu().numpy()
    assert_value_equal(ye, oracle.ambiguity_map(surv, ref, l0, L, m, dtype=f, nthreads=8))


# --- exact-multiply variants --------------------------------------

@pytest.mark.parametrize("n", [2, 4, 8, 64, 512, 4096])
def test_fft_exact_dropin_golden(sa, golden, n):
    s = sa.fft_exact(golden[f"fftx_x_{n}"])
    assert s.transform_kind is sa.TransformKind.FFT_EXACT
    assert s.bins.tobytes() == golden[f"fftx_y_{n}"].tobytes()  # bitwise, signed zeros included
    assert s.op_counts.complex_mul_ops == (n // 2) * int(np.log2(n))


def test_fft_exact_signed_zero_golden(sa, golden):
    x = np.zeros(16, complex)
    x[3] = -0.0 - 0.0j
    assert sa.fft_exact(x).bins.tobytes() == golden["fftx_zero16"].tobytes()


@pytest.mark.parametrize("logn", [1, 5, 12, 13, 14, 16, 18])
@pytest.mark.parametrize("dt", ["c64", "c128"])
def test_fft_exact_batch_vs_oracle(sa, logn, dt):
    """Single-pass (n <= 2^13 / 2^12) and two-pass kernels, 2^16 included (the
    fused ⊙ kernel is not used for the exact FFT)."""
    n = 1 << logn
    b = max(1, min(64, (1 << 19) // n))
    g = np.random.default_rng(300 + logn)
    x = (g.standard_normal((b, n)) + 1j * g.standard_normal((b, n))).astype(np.complex64 if dt == "c64" else complex)
    y = sa.nfft_batch(dev(x), variant="exact").cpu().numpy()
    assert_value_equal(y, oracle.fft_exact(x, dtype="f32" if dt == "c64" else "f64", nthreads=8))


def test_lag_product_exact_golden(sa, golden):
    sv, rf = golden["vx_surv"], golden["vx_ref"]
    for l in (0, 1, 37, 255):
        assert sa.lag_product_exact(sv, rf, l, 256).tobytes() == golden[f"lagx_{l}"].tobytes()
    assert sa.lag_product_exact(sv, rf, 5, 256, conjugate_ref=False).tobytes() == golden["lagx_noconj_5"].tobytes()


@pytest.mark.parametrize("var", ["eq11", "eq12b", "eq12c"])
def test_exact_variant_surfaces_golden(sa, golden, var):
    S = sa.ComplexSignal
    sv, rf = golden["vx_surv"], golden["vx_ref"]
    sf = sa.compute_ambiguity(var, S(sv, 200_000.0), S(rf, 200_000.0), 12, 256, transform_input_gain=4.0)
    assert sf.variant.value == var
    assert_value_equal(sf.values, golden[f"amb_{var}"])
    c = golden[f"amb_{var}_counts"]
    got = [sf.lag_op_counts.sign_ops, sf.lag_op_counts.abs_ops, sf.lag_op_counts.add_ops,
           sf.lag_op_counts.complex_mf_ops, sf.lag_op_counts.complex_mul_ops,
           sf.transform_op_counts.sign_ops, sf.transform_op_counts.abs_ops, sf.transform_op_counts.add_ops,
           sf.transform_op_counts.complex_mf_ops, sf.transform_op_counts.complex_mul_ops]
    assert got == list(c)
    if var == "eq12c":
        v = sa.compute_ambiguity("eq12c", S(sv, 1.0), S(rf, 1.0), 6, 256, conjugate_ref=False).values
        assert_value_equal(v, golden["amb_eq12c_noconj_g1"])


@pytest.mark.parametrize("lag,doppler", [("exact", "fft"), ("mf", "fft"), ("exact", "nfft"), ("exact", "ndft")])
def test_block_map_exact_variants_vs_oracle(sa, golden, lag, doppler):
    """Block-integrated maps (T = 64) with every lag / Doppler combination:
    complex128 value-identical to the oracle composition, complex64 vs the f32 oracle."""
    rr, s = golden["map_surv"], golden["map_ref"]
    got = sa.ambiguity_map(rr, s, 20, 64, l0=30, gain=2.0, lag=lag, doppler=doppler, mode="exact")
    assert_value_equal(got, oracle.ambiguity_map(rr, s, 30, 20, 64, gain=2.0, lag=lag, doppler=doppler))
    r32, s32 = rr.astype(np.complex64), s.astype(np.complex64)
    got = sa.ambiguity_map(dev(r32), dev(s32), 20, 64, l0=30, lag=lag, doppler=doppler, mode="exact").cpu().numpy()
    assert_value_equal(got, oracle.ambiguity_map(r32, s32, 30, 20, 64, lag=lag, doppler=doppler, dtype="f32"))


def _p2p_worker(rank, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import paper_1402_0532_b200 as sa
        from paper_1402_0532_b200.sharded import PeerMap, ambiguity_map_sharded
        from paper_1402_0532_b200.workloads import radar_scene
        sc = radar_scene(1 << 16, 2, 4343)
        ds = torch.from_numpy(sc.surv.astype(np.complex64)).cuda()
        dr = torch.from_numpy(sc.ref.astype(np.complex64)).cuda()
        from paper_1402_0532_b200.sharded import blocks_shardable
        # c64, T = 512, 96 rows = 3 tiles of 16 per rank: block-sharded lag stage;
        # 101 rows (uneven): delay-row shards
        assert blocks_shardable(ds, 128, "fast", "mf", "nfft", 96, 2)
        assert not blocks_shardable(ds, 128, "fast", "mf", "nfft", 101, 2)
        ok = []
        for L in (96, 101):
            pm = PeerMap(L, 128, ds.dtype)
            for _ in range(2):  # the shared map is reused across calls
                full = ambiguity_map_sharded(ds, dr, L, 128, peer_map=pm)
            if rank == 0:
                ok.append(bool(torch.equal(full, sa.ambiguity_map(ds, dr, L, 128))))
            pm.close()
        if rank == 0:
            q.put(all(ok) and len(ok) == 2)
    finally:
        dist.destroy_process_group()


def test_sharded_map_p2p_two_ranks_one_gpu(sa):
    """Fused compute + delivery: two ranks (two processes sharing the GPU, gloo
    for the host handshake) integrate their Doppler blocks for all delay rows,
    the tensor-core lag kernel stores each z row into its owner's IPC-shared
    block, then each rank's Doppler NL-FFT stores its rows straight into rank
    0's IPC-shared map; the result equals the single-call map bit for bit."""
    import socket
    import torch.multiprocessing as mp
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_p2p_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    assert [p.exitcode for p in ps] == [0, 0]
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("rows", [1, 129, 5000])
def test_pinned_host_pipeline_matches_device_path(sa, rows):
    """ndft_batch / nfft_batch on pinned host tensors run chunked H2D / compute /
    D2H overlap; results equal the device-resident path bit for bit."""
    torch = T()
    g = torch.Generator().manual_seed(rows)
    n = 1024 if rows < 5000 else 4096
    x = torch.randn(rows, n, dtype=torch.complex64, generator=g).pin_memory()
    out = torch.empty_like(x).pin_memory()
    r = sa.ndft_batch(x, out=out)
    assert r.data_ptr() == out.data_ptr()
    assert torch.equal(out, sa.ndft_batch(x.cuda()).cpu())
    y = sa.nfft_batch(x)
    assert y.is_pinned() and torch.equal(y, sa.nfft_batch(x.cuda()).cpu())
    y = sa.nfft_batch(x, variant="dif")
    assert torch.equal(y, sa.nfft_batch(x.cuda(), variant="dif").cpu())


@pytest.mark.parametrize("tb", [8, 16, 48, 2048])
@pytest.mark.parametrize("dt", ["c64", "c128"])
def test_exact_lag_fast_tiles_vs_oracle(sa, tb, dt):
    """Exact-multiply lag product through the tiled fast kernels (4 FMA per
    product; packed FFMA2 for complex64 with T % 16 == 0), ragged lag counts,
    vs the oracle's exact-lag composition: within the fast-mode tolerances."""
    g = np.random.default_rng(900 + tb)
    m = 32
    ns = tb * m
    surv = g.standard_normal(ns) + 1j * g.standard_normal(ns)
    ref = np.exp(2j * np.pi * g.random(ns))
    cdt = np.complex64 if dt == "c64" else np.complex128
    s_, r_ = surv.astype(cdt), ref.astype(cdt)
    y = sa.ambiguity_map(dev(s_), dev(r_), 70, m, l0=3, lag="exact", doppler="fft").cpu().numpy()
    want = oracle.ambiguity_map(s_.astype(complex), r_.astype(complex), 3, 70, m, lag="exact", doppler="fft",
                                nthreads=8)
    assert_literal(y, want, TOL_F32 if dt == "c64" else TOL_F64)


@pytest.mark.parametrize("dt", ["c64", "c128"])
@pytest.mark.parametrize("variant", ["dit", "dif"])
def test_nfft_subnormal_and_signed_zero_inputs(sa, dt, variant):
    """sign(subnormal) = +-1 and sign(+-0) = 0 decide every butterfly (FTZ off):
    subnormal, signed-zero and mixed-magnitude samples through the fused 2^16
    cluster kernel and the single-pass kernel, value-identical to the oracle."""
    g = np.random.default_rng(77)
    cdt = np.complex64 if dt == "c64" else np.complex128
    tiny = np.float32(1e-42) if dt == "c64" else 1e-310  # subnormal in each dtype
    for n, b in ((1 << 16, 6), (1024, 8)):
        x = (g.standard_normal((b, n)) + 1j * g.standard_normal((b, n))).astype(cdt)
        x[0] = tiny * np.sign(g.standard_normal(n)) + 1j * tiny * np.sign(g.standard_normal(n))
        x[1, ::2] = -0.0
        x[1, 1::2] = 0.0 - 0.0j
        x[2, ::7] *= tiny
        x[3] = (g.integers(-3, 4, n) + 1j * g.integers(-3, 4, n)).astype(cdt)  # exact small integers: cancellations
        x[4, : n // 2] = 0
        od = "f32" if dt == "c64" else "f64"
        y = sa.nfft_batch(dev(x), variant=variant).cpu().numpy()
        assert_value_equal(y, oracle.nfft(x, variant, dtype=od, nthreads=8))


def test_ndft_and_map_subnormal_inputs(sa):
    """Subnormals and signed zeros through the NDFT fast/exact kernels and the lag
    kernels (signs staged once per sample): exact modes value-identical."""
    g = np.random.default_rng(78)
    x = g.standard_normal((5, 256)) + 1j * g.standard_normal((5, 256))
    x[0] = 1e-310 * (1 + 1j)
    x[1, ::3] = -0.0
    x[2, ::5] *= 1e-312
    assert_value_equal(sa.ndft_batch(dev(x), mode="exact").cpu().numpy(), oracle.ndft(x))
    assert_literal(sa.ndft_batch(dev(x)).cpu().numpy(), oracle.ndft(x), TOL_F64)
    s = np.exp(2j * np.pi * g.random(4096))
    r = s.copy()
    r[::11] *= 1e-310
    r[::13] = -0.0
    got = sa.ambiguity_map(r, s, 16, 64, mode="exact")
    assert_value_equal(got, oracle.ambiguity_map(r, s, 0, 16, 64))


@pytest.mark.parametrize("devs", [[0], [0, 0], [0, 0, 0]])
def test_map_multi_device_single_process(sa, devs):
    """sa_ambiguity_map_multi (single-process multi-GPU through the C ABI, no
    NCCL): shards listed on the same GPU run on separate streams and store their
    rows into the root's map; uneven row counts; equal to the single-call map."""
    from paper_1402_0532_b200.sharded import ambiguity_map_multi_device
    from paper_1402_0532_b200.workloads import radar_scene
    sc = radar_scene(1 << 16, 2, 4545)
    s = dev(sc.surv.astype(np.complex64))
    r = dev(sc.ref.astype(np.complex64))
    got = ambiguity_map_multi_device([s] * len(devs), [r] * len(devs), 101, 128, devs, l0=7)
    assert T().equal(got, sa.ambiguity_map(s, r, 101, 128, l0=7))
    got = ambiguity_map_multi_device([s] * len(devs), [r] * len(devs), 33, 128, devs, lag="exact", mode="exact",
                                     doppler="fft")
    assert T().equal(got, sa.ambiguity_map(s, r, 33, 128, lag="exact", mode="exact", doppler="fft"))


def test_empty_batches(sa):
    """Zero-row batches and zero-length elementwise inputs are no-ops, not errors."""
    torch = T()
    for dt in (torch.complex64, torch.complex128):
        for n in (64, 1000, 1 << 16):
            x = torch.empty((0, n), dtype=dt, device="cuda")
            assert sa.ndft_batch(x).shape == (0, n)
            if n & (n - 1) == 0:
                for v in ("dit", "dif", "exact"):
                    assert sa.nfft_batch(x, variant=v).shape == (0, n)
    assert sa.mf_complex(np.zeros(0, complex), np.zeros(0, complex)).size == 0


@pytest.mark.parametrize("n", [64, 255, 256, 1000, 1024])
def test_ndft_exact_tiled_value_identical(sa, n):
    """Exact mode on batches that fill the vector tile (the tiled EX kernels):
    value-identical to the sequential oracle in fp64 and fp32; zeros, a tone."""
    g = np.random.default_rng(600 + n)
    b = 300
    x = g.standard_normal((b, n)) + 1j * g.standard_normal((b, n))
    x[5] = 0
    x[6, ::4] = 0
    x[7] = np.conj(oracle.twiddle_table(n)[(3 * np.arange(n)) % n])
    assert_value_equal(sa.ndft_batch(dev(x), mode="exact").cpu().numpy(), oracle.ndft(x, nthreads=8))
    x32 = x.astype(np.complex64)
    assert_value_equal(sa.ndft_batch(dev(x32), mode="exact").cpu().numpy(),
                       oracle.ndft(x32, dtype="f32", nthreads=8))
    assert_value_equal(sa.ndft_batch(dev(x), mode="exact", gain=0.75).cpu().numpy(),
                       oracle.ndft(0.75 * x, nthreads=8))
