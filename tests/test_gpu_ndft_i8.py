"""GPU parity of the complex128 tensor-core NDFT (mode "tc", sa_ndft_i8.cu:
exact int8-digit products, int32 accumulation, fp64 epilogue) against the fp64
oracle (oracle.ndft = transforms.py:223-251 restated), at the north-star fp64
tolerance: per vector max_k |Δ_k| / ||y_ref||_1 <= 1e-9 (tests/parity.py).
The only approximation is the 26-bit digit split of Wv and of each vector
scaled by its power-of-two exponent, so the measured error is ~1e-12.
"""

import numpy as np
import pytest

import oracle
from parity import TOL_F64, assert_literal, literal, strict

pytestmark = pytest.mark.gpu


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n,rows", [(128, 1), (128, 300), (192, 255), (256, 257), (1024, 129), (2048, 5)])
def test_ndft_i8_sizes(sa, n, rows):
    g = np.random.default_rng(3000 + n + rows)
    x = (g.standard_normal((rows, n)) + 1j * g.standard_normal((rows, n))) / np.sqrt(2)
    if rows > 4:
        x[3] = 0                      # zero vector -> exact zero spectrum
        x[4, ::3] = 0
        x[2, 1::2] = -0.0
    y = sa.ndft_batch(dev(x), mode="tc").cpu().numpy()
    r = oracle.ndft(x, nthreads=8)
    e = assert_literal(y, r, TOL_F64)
    assert e.max() < 4e-10, e.max()  # error model (sa_ndft_i8.cu): ~sqrt(2n) 2^-28 / n sqrt(2n)
    print(f"n={n} rows={rows}: literal max {e.max():.2e}, strict max {strict(y, r).max():.2e}")
    if rows > 4:
        assert np.all(y[3] == 0)


def test_ndft_i8_dynamic_range_and_gain(sa):
    """Per-vector exponents: tiny, huge, subnormal-laden and mixed-magnitude rows, with a gain."""
    g = np.random.default_rng(11)
    n = 256
    x = g.standard_normal((140, n)) + 1j * g.standard_normal((140, n))
    x[5] *= 1e-200
    x[6] *= 1e200
    x[7, ::2] *= 1e-12            # mixed magnitudes inside one row
    x[8] = 0
    x[8, 17] = 3.0 - 1e-300j      # a single nonzero (sparse: small ||y||_1)
    x[9, ::5] = 5e-324            # subnormals: sign +1, magnitude below every digit
    for gain in (1.0, 16.0, 0.37):
        y = sa.ndft_batch(dev(x), mode="tc", gain=gain).cpu().numpy()
        r = oracle.ndft(gain * x, nthreads=8)
        e = assert_literal(y, r, TOL_F64)
        assert e.max() < 5e-10, (gain, e.max(), int(np.argmax(e)))


def test_ndft_i8_tones_and_fallback(sa):
    """C2 tone rows keep their peak; n % 64 != 0 and n < 128 run the DFMA fast kernel under mode "tc"."""
    from paper_1402_0532_b200.transforms import unit_tone
    n = 1024
    ks = [0, 1, 7, 300, 511, 512, 1023]
    x = np.stack([unit_tone(k, n) for k in ks])
    y = sa.ndft_batch(dev(x), mode="tc").cpu().numpy()
    assert_literal(y, oracle.ndft(x, nthreads=8), TOL_F64)
    assert [int(np.argmax(np.abs(r))) for r in y] == ks
    g = np.random.default_rng(5)
    for n in (96, 64, 160):
        x = g.standard_normal((9, n)) + 1j * g.standard_normal((9, n))
        yt = sa.ndft_batch(dev(x), mode="tc").cpu().numpy()
        yf = sa.ndft_batch(dev(x), mode="fast").cpu().numpy()
        assert np.array_equal(yt, yf)


def test_ndft_i8_c2_sampled_rows(sa):
    """Full C2 batch (65536 x 1024, complex128): every 256th row (tone rows
    included) against the oracle at the fp64 bound."""
    import torch
    from paper_1402_0532_b200.workloads import c2_ndft
    x = c2_ndft(1024, 65536)
    y = sa.ndft_batch(torch.from_numpy(x).cuda(), mode="tc")
    idx = np.arange(0, 65536, 256)
    ys = y[torch.from_numpy(idx).cuda()].cpu().numpy()
    r = oracle.ndft(x[idx], nthreads=16)
    e = assert_literal(ys, r, TOL_F64)
    print(f"C2 c128 tc: literal max {e.max():.2e}, strict max {strict(ys, r).max():.2e}")


def test_ndft_i8_non_finite_rows_are_nan(sa):
    """A row holding NaN / Inf comes out NaN (as the DFMA kernel's would), other rows unaffected."""
    g = np.random.default_rng(17)
    x = g.standard_normal((6, 256)) + 1j * g.standard_normal((6, 256))
    x[1, 7] = np.nan
    x[3, 0] = np.inf
    y = sa.ndft_batch(dev(x), mode="tc").cpu().numpy()
    assert np.isnan(y[1]).all() and np.isnan(y[3]).all()
    keep = [0, 2, 4, 5]
    assert_literal(y[keep], oracle.ndft(x[keep], nthreads=8), TOL_F64)


# ---- complex64 on the int8 path (mode "tc8", sa_ndft_i8.cu ND=1) -------------
# One digit pair per operand (radix 127 x 127, residual <= 2^e / 32258, ~15 bits):
# the same exact int32 products, half the MMAs of complex128.  Error model
# ~sqrt(2n) 2^-15 2^e / (n sqrt(2n)): a few 1e-6 relative to ||y||_1, inside the
# 1e-4 fp32 bound.  For n <= 1024 the digit prep runs inside the tensor-core
# kernel (prep warps + per-block ready counters), so every case here with
# n <= 1024 also covers that path (tiny, ragged and 256-multiple batches).

def _ref32(x):
    return oracle.ndft(np.asarray(x, np.complex64).astype(np.complex128), nthreads=8)


@pytest.mark.parametrize("n,rows", [(128, 1), (128, 300), (256, 257), (512, 7), (1024, 129), (2048, 5)])
def test_ndft_i8_c64_sizes(sa, n, rows):
    from parity import TOL_F32
    g = np.random.default_rng(4000 + n + rows)
    x = ((g.standard_normal((rows, n)) + 1j * g.standard_normal((rows, n))) / np.sqrt(2)).astype(np.complex64)
    if rows > 4:
        x[3] = 0
        x[4, ::3] = 0
        x[2, 1::2] = -0.0
    y = sa.ndft_batch(dev(x), mode="tc8").cpu().numpy()
    assert y.dtype == np.complex64
    r = _ref32(x)
    e = assert_literal(y, r, TOL_F32)
    assert e.max() < 2e-5, e.max()
    print(f"c64 n={n} rows={rows}: literal max {e.max():.2e}")
    if rows > 4:
        assert np.all(y[3] == 0)


def test_ndft_i8_c64_range_gain_nonfinite_fallback(sa):
    from parity import TOL_F32
    g = np.random.default_rng(21)
    x = (g.standard_normal((140, 256)) + 1j * g.standard_normal((140, 256))).astype(np.complex64)
    x[5] *= 1e-30
    x[6] *= 1e30
    x[7, ::2] *= 1e-6
    x[9, ::5] = 1e-45             # fp32 subnormals
    for gain in (1.0, 16.0, 0.37):
        y = sa.ndft_batch(dev(x), mode="tc8", gain=gain).cpu().numpy()
        assert_literal(y, _ref32(gain * x.astype(np.complex128)), TOL_F32)
    z = x[:6].copy()
    z[1, 7] = np.nan
    z[3, 0] = np.inf
    y = sa.ndft_batch(dev(z), mode="tc8").cpu().numpy()
    assert np.isnan(y[1]).all() and np.isnan(y[3]).all()
    assert_literal(y[[0, 2, 4, 5]], _ref32(z[[0, 2, 4, 5]]), TOL_F32)
    for n in (96, 64, 4096):      # outside the int8 shapes: the fast kernel
        w = (g.standard_normal((9, n)) + 1j * g.standard_normal((9, n))).astype(np.complex64)
        assert np.array_equal(sa.ndft_batch(dev(w), mode="tc8").cpu().numpy(),
                              sa.ndft_batch(dev(w), mode="fast").cpu().numpy())


def test_ndft_i8_c64_c2_subset(sa):
    import torch
    from parity import TOL_F32
    from paper_1402_0532_b200.workloads import c2_ndft
    x = c2_ndft().astype(np.complex64)
    y = sa.ndft_batch(dev(x), mode="tc8")
    rows = np.arange(0, x.shape[0], 512)
    ys = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    e = assert_literal(ys, _ref32(x[rows]), TOL_F32)
    print(f"C2 c64 tc8: literal max {e.max():.2e}")


def test_ndft_i8_c64_concurrent_streams(sa):
    """The fused prep's ready counters and row ticket are per call: two tc8 calls
    on two streams at once (their persistent grids sharing the SMs) give exactly
    the results of the same calls made one after the other."""
    import torch
    g = np.random.default_rng(77)
    xs = [dev(((g.standard_normal((1000 + 300 * i, 1024)) + 1j * g.standard_normal((1000 + 300 * i, 1024))) /
               np.sqrt(2)).astype(np.complex64)) for i in range(2)]
    ref = [sa.ndft_batch(x, mode="tc8") for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in xs]
    outs = [torch.empty_like(x) for x in xs]
    for _ in range(3):
        for x, o, st in zip(xs, outs, streams):
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                sa.ndft_batch(x, out=o, mode="tc8")
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            assert torch.equal(o, r)
