"""CPU model of the tensor-core formulations (sa_ndft_tc.cu, sa_lag_tc.cu): the
sign-split sums with the non-sign operands split into two bf16 pieces, summed in
fp64 (the kernels sum in fp32 TMEM).  Pins the split's error budget against the
oracle (transforms.py:223-251 restated in oracle/) on CPU: the GPU tests then
only add fp32 accumulation on top (tests/test_gpu_ndft_tc.py, test_gpu_lag_tc.py)."""

import numpy as np

import oracle
from parity import literal, strict


def bf16(a):
    """Round-to-nearest-even to bfloat16 (as cvt.rn.bf16x2.f32), returned as float64."""
    a = np.asarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def split2(a):
    hi = bf16(a)
    lo = bf16(np.asarray(a, np.float32).astype(np.float64) - hi)  # residual exact in fp32
    return hi, lo


def test_ndft_two_piece_split_error_budget():
    g = np.random.default_rng(11)
    n, rows = 256, 6
    x = ((g.standard_normal((rows, n)) + 1j * g.standard_normal((rows, n))) / np.sqrt(2)).astype(np.complex64)
    x[2] = 0
    tw = np.asarray(__import__("paper_1402_0532_b200").twiddle.twiddle_table(n).entries).astype(np.complex64)
    W = tw[(np.arange(n)[:, None] * np.arange(n)[None, :]) % n]
    Wr, Wi = W.real.astype(np.float64), W.imag.astype(np.float64)
    xr, xi = x.real.astype(np.float64), x.imag.astype(np.float64)
    sg = np.sign
    Wr0, Wr1 = split2(Wr); Wi0, Wi1 = split2(Wi)
    xr0, xr1 = split2(xr); xi0, xi1 = split2(xi)
    re = sg(xr) @ (Wr0 + Wr1).T + (xr0 + xr1) @ sg(Wr).T - sg(xi) @ (Wi0 + Wi1).T - (xi0 + xi1) @ sg(Wi).T
    im = sg(xr) @ (Wi0 + Wi1).T + (xr0 + xr1) @ sg(Wi).T + sg(xi) @ (Wr0 + Wr1).T + (xi0 + xi1) @ sg(Wr).T
    y = re + 1j * im
    ref = oracle.ndft(x.astype(np.complex128))
    assert literal(y, ref).max() < 1e-7
    assert strict(y, ref).max() < 1e-4
    assert np.all(y[2] == 0)


def test_lag_hankel_decomposition_model():
    """z_l[q] via the kernel's Hankel/Toeplitz decomposition (l = lbase + 8 l1 + l0,
    u = t - 8 l1, groups aligned to 16) equals the direct block-summed lag products."""
    g = np.random.default_rng(5)
    T, m, L, l0g = 64, 4, 40, 3
    ns = T * m
    s = g.standard_normal(ns) + 1j * g.standard_normal(ns)
    c = np.conj(g.standard_normal(ns) + 1j * g.standard_normal(ns))

    def mf(a, b):
        return np.sign(a * b) * (np.abs(a) + np.abs(b))

    def cmf(a, b):
        return (mf(a.real, b.real) - mf(a.imag, b.imag)) + 1j * (mf(a.imag, b.real) + mf(b.imag, a.real))

    direct = np.zeros((L, m), complex)
    for j in range(L):
        lag = l0g + j
        sh = np.zeros(ns, complex)
        sh[lag:] = c[:ns - lag]
        direct[j] = cmf(s, sh).reshape(m, T).sum(axis=1)
    lalign = l0g - (l0g & 15)
    M1 = (l0g - lalign + L + 7) // 8
    hank = np.zeros((L, m), complex)
    for q in range(m):
        a = s[q * T:(q + 1) * T]
        for l1 in range(M1):
            for l0 in range(8):
                lag = lalign + 8 * l1 + l0
                if not (l0g <= lag < l0g + L):
                    continue
                acc = 0j
                for u in range(-8 * (M1 - 1), T):
                    t = u + 8 * l1
                    if not 0 <= t < T:
                        continue
                    ci = q * T + t - lag  # = q T - lalign + u - l0
                    acc += cmf(a[t], c[ci] if ci >= 0 else 0)
                hank[lag - l0g, q] = acc
    assert np.allclose(hank, direct, rtol=0, atol=1e-12 * np.abs(direct).max())
