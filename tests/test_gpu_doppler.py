"""The map's Doppler NL-FFT stage (sa_doppler.cu) and the blocked z layout the
tensor-core lag kernel writes for it (sa_lag_tc.cu).

* sa_doppler_nlfft_blocked on a z laid out in 16-row tiles equals nfft of
  gain * z row by row (transforms.py:254-298), value-identical (fp64) and
  equal to the fp32 restatement (fp32);
* maps whose Doppler stage runs it -- row-major z from the CUDA-core lag
  kernels (exact modes, complex128) and blocked z from the tensor-core lag
  kernel at unaligned l0 -- against the oracle composition.
"""

import ctypes

import numpy as np
import pytest

import oracle
from parity import TOL_F32, assert_literal

pytestmark = pytest.mark.gpu


def T():
    import torch
    return torch


def blocked(z):
    """(L x M) rows -> the blocked layout zb[(k*M + q)*16 + j] = z[16k + j][q] (L % 16 == 0)."""
    L, M = z.shape
    return np.ascontiguousarray(z.reshape(L // 16, 16, M).transpose(0, 2, 1)).reshape(-1)


@pytest.mark.parametrize("m", [64, 128, 256, 512, 1024, 2048])
@pytest.mark.parametrize("dt", ["c64", "c128"])
def test_doppler_blocked_equals_nfft(sa, m, dt):
    torch = T()
    from paper_1402_0532_b200 import _native
    from paper_1402_0532_b200.twiddle import device_twiddles
    g = np.random.default_rng(m)
    L = 48
    cdt = np.complex64 if dt == "c64" else np.complex128
    z = (g.standard_normal((L, m)) + 1j * g.standard_normal((L, m))).astype(cdt)
    z[3, ::5] = 0
    zb = torch.from_numpy(blocked(z)).cuda()
    out = torch.empty((L, m), dtype=zb.dtype, device="cuda")
    d = _native.SA_C64 if dt == "c64" else _native.SA_C128
    gain = 2.0
    _native.check(_native.lib().sa_doppler_nlfft_blocked(
        d, _native.ptr(zb), _native.ptr(out), L, m, ctypes.c_void_p(device_twiddles(m, d, 0)), gain,
        _native.stream_ptr()))
    want = oracle.nfft((gain * z).astype(cdt), "dit", dtype="f32" if dt == "c64" else "f64")
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("m,l0,L", [(64, 5, 37), (512, 13, 70), (2048, 3, 21)])
def test_map_tc_blocked_doppler_vs_oracle(sa, m, l0, L):
    """complex64 fast maps: tensor-core lag stage writing blocked z at an
    unaligned first row, then the blocked Doppler stage, vs the fp64 oracle."""
    torch = T()
    from paper_1402_0532_b200.workloads import radar_scene
    sc = radar_scene(128 * m, 2, 900 + m)
    s = sc.surv.astype(np.complex64)
    r = sc.ref.astype(np.complex64)
    got = sa.ambiguity_map(torch.from_numpy(s).cuda(), torch.from_numpy(r).cuda(), L, m, l0=l0,
                           gain=1.5).cpu().numpy()
    want = oracle.ambiguity_map(s.astype(complex), r.astype(complex), l0, L, m, gain=1.5, nthreads=8)
    assert_literal(got, want, TOL_F32)


def test_map_row_ranges_bit_identical_with_blocked_z(sa):
    """Any delay-row range of a map equals the same rows of the full call bit for
    bit (lag groups start at lag multiples of 16, tiles are absolute)."""
    torch = T()
    from paper_1402_0532_b200.workloads import radar_scene
    sc = radar_scene(1 << 17, 3, 4242)
    s = torch.from_numpy(sc.surv.astype(np.complex64)).cuda()
    r = torch.from_numpy(sc.ref.astype(np.complex64)).cuda()
    full = sa.ambiguity_map(s, r, 1100, 256)
    for l0, L in ((0, 16), (7, 1), (33, 100), (1000, 100), (1023, 77)):
        part = sa.ambiguity_map(s, r, L, 256, l0=l0)
        assert torch.equal(part, full[l0:l0 + L]), (l0, L)
