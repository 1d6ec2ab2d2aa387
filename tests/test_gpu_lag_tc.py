"""GPU parity of the tensor-core lag integration (fast mode, complex64,
T % 128 == 0; both kernels: sa_lag_i8.cu, int8 digits with exact int32 sums, the
default, and sa_lag_tc.cu, bf16x2 pieces with fp32 sums, selected by
sa_lag_kernel) through the C ABI sa_ambiguity_integrate, against an
fp64 numpy restatement of z_l[q] = Σ_t surv[qT+t] ⊙ conj(ref[qT+t-l])
(ambiguity.py:116-131,146-155 block-summed), at the fp32 bound
max_k |Δ_k| / ||z_row||_1 <= 1e-4 (tests/parity.py)."""

import ctypes

import numpy as np
import pytest

from parity import TOL_F32, assert_literal

pytestmark = pytest.mark.gpu
SA_LAGK_I8, SA_LAGK_BF16 = 0, 1


@pytest.fixture(params=["i8", "bf16"])
def lagk(request, sa):
    """Run the test with each lag kernel (process-wide switch, restored after)."""
    from paper_1402_0532_b200 import _native
    prev = _native.lib().sa_lag_kernel(SA_LAGK_I8 if request.param == "i8" else SA_LAGK_BF16)
    yield request.param
    _native.lib().sa_lag_kernel(prev)


def mf(a, b):
    return np.sign(a * b) * (np.abs(a) + np.abs(b))


def cmf(a, b):  # operator.py:128-131
    return (mf(a.real, b.real) - mf(a.imag, b.imag)) + 1j * (mf(a.imag, b.real) + mf(b.imag, a.real))


def z_ref(surv, ref, l0, L, m, conj=True):
    s = surv.astype(np.complex128)
    c = np.conj(ref.astype(np.complex128)) if conj else ref.astype(np.complex128)
    ns = s.size
    out = np.empty((L, m), np.complex128)
    for j in range(L):
        l = l0 + j
        sh = np.zeros(ns, np.complex128)
        sh[l:] = c[:ns - l]
        out[j] = cmf(s, sh).reshape(m, -1).sum(axis=1)
    return out


def integrate(sa, surv, ref, l0, L, m, conj=True):
    import torch
    from paper_1402_0532_b200 import _native
    ds = torch.from_numpy(surv).cuda()
    dr = torch.from_numpy(ref).cuda()
    z = torch.empty((L, m), dtype=torch.complex64, device="cuda")
    _native.check(_native.lib().sa_ambiguity_integrate(
        _native.SA_C64, _native.ptr(ds), _native.ptr(dr), ds.numel(), dr.numel(), l0, L, m, int(conj),
        _native.SA_NDFT_FAST, _native.ptr(z), _native.stream_ptr()))
    return z.cpu().numpy()


def signals(seed, ns):
    g = np.random.default_rng(seed)
    surv = ((g.standard_normal(ns) + 1j * g.standard_normal(ns)) / np.sqrt(2)).astype(np.complex64)
    ref = np.exp(2j * np.pi * g.random(ns)).astype(np.complex64)
    surv[5] = 0
    surv[77] = -0.0
    ref[9] = 0
    ref[300:340] = 0
    return surv, ref


@pytest.mark.parametrize("tb,m,l0,L,conj", [(128, 16, 0, 70, True), (256, 8, 3, 1024, True),
                                             (2048, 8, 0, 1030, True), (2048, 4, 1000, 300, False),
                                             (4096, 4, 17, 2100, True)])
def test_lag_tc_vs_fp64(sa, lagk, tb, m, l0, L, conj):
    surv, ref = signals(tb + L, tb * m)
    z = integrate(sa, surv, ref, l0, L, m, conj)
    r = z_ref(surv, ref, l0, L, m, conj)
    e = assert_literal(z.T, r.T, TOL_F32)   # per Doppler block (column of z), over its lags
    assert_literal(z, r, TOL_F32)           # and per lag row
    assert e.max() < 1e-5


def test_lag_tc_shard_offsets_bit_identical(sa, lagk):
    """Lag shards reproduce the single-call rows bit for bit, whatever lag they
    start at (groups are aligned to lag multiples of 16, so every product keeps
    its u alignment inside the MMA K steps): sharded maps equal the single-GPU map."""
    surv, ref = signals(7, 2048 * 8)
    full = integrate(sa, surv, ref, 0, 2048, 8)
    for a, b in ((0, 512), (512, 1024), (1024, 2048), (1536, 2048), (3, 101), (101, 1337), (1337, 2048)):
        assert np.array_equal(integrate(sa, surv, ref, a, b - a, 8), full[a:b]), (a, b)


def test_lag_tc_map_c4_rows(sa, lagk):
    """C4 map (lag stage on the tensor cores, Doppler NL-FFT) on target rows vs the oracle."""
    import oracle
    import torch
    from paper_1402_0532_b200.workloads import c4_scene
    sc = c4_scene()
    surv = sc.surv.astype(np.complex64)
    ref = sc.ref.astype(np.complex64)
    y = sa.ambiguity_map(torch.from_numpy(surv).cuda(), torch.from_numpy(ref).cuda(), 1024, 512).cpu().numpy()
    for l in [0, 1, 511, 1023] + [int(t) for t in sc.delays]:
        r = oracle.ambiguity_map(surv.astype(np.complex128), ref.astype(np.complex128), l, 1, 512, nthreads=8)
        assert_literal(y[l:l + 1], r, TOL_F32)


def test_map_ndft_doppler_tc_rows(sa):
    """C4 map with the NDFT along Doppler (fast mode, complex64, M = 512): both
    the lag stage and the Doppler NDFT run on the tensor cores; rows vs the oracle,
    and a row range alone equals the same rows of the full map bit for bit."""
    import oracle
    import torch
    from paper_1402_0532_b200.workloads import c4_scene
    sc = c4_scene()
    surv = sc.surv.astype(np.complex64)
    ref = sc.ref.astype(np.complex64)
    ds, dr = torch.from_numpy(surv).cuda(), torch.from_numpy(ref).cuda()
    y = sa.ambiguity_map(ds, dr, 1024, 512, doppler="ndft")
    for l in [0, 1023] + [int(t) for t in sc.delays]:
        r = oracle.ambiguity_map(surv.astype(np.complex128), ref.astype(np.complex128), l, 1, 512,
                                 doppler="ndft", nthreads=8)
        assert_literal(y[l:l + 1].cpu().numpy(), r, TOL_F32)
    part = sa.ambiguity_map(ds, dr, 200, 512, l0=300, doppler="ndft")
    assert torch.equal(part, y[300:500])


@pytest.mark.parametrize("l0", [3, 13])
def test_lag_tc_short_ref_never_read_past_end(sa, lagk, l0):
    """lag groups start at multiples of 16, so lags below l0 reach
    ref[ns - lalign - 1] > ref_len - 1 when ref is trimmed to ns - l0 (allowed by
    the lag_product_mf guards, ambiguity.py:121-128).  The words past ref_len are
    NaN here; the kept rows must stay finite and equal the restatement."""
    import torch
    from paper_1402_0532_b200 import _native
    ns, m = 2048 * 8, 8
    surv, ref = signals(21 + l0, ns)
    rl = ns - l0
    buf = np.full(ns + 64, np.nan + 1j * np.nan, np.complex64)
    buf[:rl] = ref[:rl]
    ds = torch.from_numpy(surv).cuda()
    db = torch.from_numpy(buf).cuda()
    L = 40
    z = torch.empty((L, m), dtype=torch.complex64, device="cuda")
    _native.check(_native.lib().sa_ambiguity_integrate(
        _native.SA_C64, _native.ptr(ds), _native.ptr(db), ns, rl, l0, L, m, 1, _native.SA_NDFT_FAST,
        _native.ptr(z), _native.stream_ptr()))
    got = z.cpu().numpy()
    assert np.isfinite(got).all()
    assert_literal(got, z_ref(surv, ref[:rl], l0, L, m), TOL_F32)


@pytest.mark.parametrize("ss,rs", [(1e-35, 1e30), (3e25, 2e-30), (1.0, 1.0)])
def test_lag_i8_extreme_scales(sa, ss, rs):
    """int8 digits: the exponents (per block for surv, one for the reference) take
    the fp64 digit path outside |e| < 100; results stay within the fp32 bound."""
    from paper_1402_0532_b200 import _native
    prev = _native.lib().sa_lag_kernel(SA_LAGK_I8)
    try:
        surv, ref = signals(99, 2048 * 4)
        surv = (surv * np.float32(ss)).astype(np.complex64)
        ref = (ref * np.float32(rs)).astype(np.complex64)
        z = integrate(sa, surv, ref, 5, 600, 4)
        assert np.isfinite(z).all()
        assert_literal(z, z_ref(surv, ref, 5, 600, 4), TOL_F32)
    finally:
        _native.lib().sa_lag_kernel(prev)


def test_lag_i8_nonfinite(sa):
    """A NaN in a surveillance block makes that block's column NaN (every lag of
    the block reads it); a non-finite reference value makes every row NaN (the
    reference shares one exponent)."""
    from paper_1402_0532_b200 import _native
    prev = _native.lib().sa_lag_kernel(SA_LAGK_I8)
    try:
        surv, ref = signals(5, 2048 * 4)
        s2 = surv.copy()
        s2[2048 + 7] = np.nan
        z = integrate(sa, s2, ref, 0, 64, 4)
        assert np.isnan(z[:, 1]).all() and np.isfinite(z[:, [0, 2, 3]]).all()
        r2 = ref.copy()
        r2[100] = np.inf
        assert np.isnan(integrate(sa, surv, r2, 0, 64, 4)).all()
    finally:
        _native.lib().sa_lag_kernel(prev)


def test_lag_i8_diagonal_bit_identical(sa):
    """Two T-lag groups (16 MR == T, the C5 shape): the rows equal, bit for
    bit, the same rows computed by single-group calls (exact int32 sums), and
    stay within the fp32 bound of the fp64 restatement."""
    from paper_1402_0532_b200 import _native
    prev = _native.lib().sa_lag_kernel(SA_LAGK_I8)
    try:
        surv, ref = signals(31, 2048 * 6)
        full = integrate(sa, surv, ref, 0, 4096, 6)
        for a, b in ((0, 2048), (2048, 4096), (100, 1100), (3000, 4096)):
            assert np.array_equal(integrate(sa, surv, ref, a, b - a, 6), full[a:b]), (a, b)
        part = integrate(sa, surv, ref, 7, 4000, 6)  # l0 % 16 != 0: still two groups
        assert np.array_equal(part, full[7:4007])
        assert_literal(full[::37], z_ref(surv, ref, 0, 4096, 6)[::37], TOL_F32)
    finally:
        _native.lib().sa_lag_kernel(prev)


def test_lag_i8_concurrent_streams(sa):
    """Two int8 lag stages on two streams at once (each call owns its reference
    planes and partials) equal the same calls made one after the other."""
    import torch
    from paper_1402_0532_b200 import _native
    prev = _native.lib().sa_lag_kernel(SA_LAGK_I8)
    try:
        cases = [signals(41, 2048 * 8), signals(42, 2048 * 8)]
        seq = [integrate(sa, s, r, 0, 1500, 8) for s, r in cases]
        dev_in = [(torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda()) for s, r in cases]
        zs = [torch.empty((1500, 8), dtype=torch.complex64, device="cuda") for _ in cases]
        streams = [torch.cuda.Stream() for _ in cases]
        torch.cuda.synchronize()
        for (ds, dr), z, st in zip(dev_in, zs, streams):
            with torch.cuda.stream(st):
                _native.check(_native.lib().sa_ambiguity_integrate(
                    _native.SA_C64, _native.ptr(ds), _native.ptr(dr), ds.numel(), dr.numel(), 0, 1500, 8, 1,
                    _native.SA_NDFT_FAST, _native.ptr(z), _native.stream_ptr()))
        torch.cuda.synchronize()
        for z, r in zip(zs, seq):
            assert np.array_equal(z.cpu().numpy(), r)
    finally:
        _native.lib().sa_lag_kernel(prev)


@pytest.mark.parametrize("ns,L,M", [(2048 * 64, 512, 64), (1024 * 128, 1000, 128), (2048 * 64, 64, 64)])
def test_map_host_pipelined_bit_identical(sa, ns, L, M):
    """Pinned host complex64 inputs take the upload-overlapped path (reference
    first, surveillance chunks each followed by its blocks' lag stage); the map
    equals the device-input map bit for bit (L = 1000: not whole 16-row tiles, the
    simple path)."""
    import torch
    surv, ref = signals(ns + L, ns)
    hs = torch.from_numpy(surv).pin_memory()
    hr = torch.from_numpy(ref).pin_memory()
    hout = torch.empty((L, M), dtype=torch.complex64).pin_memory()
    got = sa.ambiguity_map(hs, hr, L, M, out=hout, gain=3.0)
    dev = sa.ambiguity_map(hs.cuda(), hr.cuda(), L, M, gain=3.0).cpu()
    assert torch.equal(got, dev)
    assert np.array_equal(sa.ambiguity_map(hs, hr, L, M, gain=3.0), dev.numpy())
