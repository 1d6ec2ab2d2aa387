"""GPU parity of the tensor-core NDFT (mode "tc", sa_ndft_tc.cu) against the
oracle (oracle.ndft = transforms.py:223-251 restated), at the north-star fp32
tolerance: per vector max_k |Δ_k| / ||y_ref||_1 <= 1e-4 (tests/parity.py).
The tc path computes the same regrouped sum as fast mode; its products are
sign x bf16 pieces (two-term splits of x and W), accumulated in fp32.
"""

import numpy as np
import pytest

import oracle
from parity import TOL_F32, assert_literal, literal, strict

pytestmark = pytest.mark.gpu


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def ref32(x):
    return oracle.ndft(np.asarray(x, np.complex64).astype(np.complex128), nthreads=8)


@pytest.mark.parametrize("n,rows", [(128, 1), (128, 200), (256, 129), (512, 7), (1024, 300), (2048, 3), (4096, 2)])
def test_ndft_tc_sizes(sa, n, rows):
    g = np.random.default_rng(1000 + n + rows)
    x = ((g.standard_normal((rows, n)) + 1j * g.standard_normal((rows, n))) / np.sqrt(2)).astype(np.complex64)
    if rows > 4:
        x[3] = 0                      # zero vector -> exact zero spectrum
        x[4, ::3] = 0
        x[2, 1::2] = -0.0
    y = sa.ndft_batch(dev(x), mode="tc").cpu().numpy()
    r = ref32(x)
    e = assert_literal(y, r, TOL_F32)
    assert e.max() < 1e-6, e.max()   # measured ~3e-8: far inside the bound
    if rows > 4:
        assert np.all(y[3] == 0)
    yf = sa.ndft_batch(dev(x), mode="fast").cpu().numpy()
    assert literal(y, yf).max() < 1e-6


def test_ndft_tc_tones_peak(sa):
    """Tone rows (C2 model): the peak stays on the tone bin."""
    from paper_1402_0532_b200.transforms import unit_tone
    n = 1024
    ks = [0, 1, 7, 300, 511, 512, 1023]
    x = np.stack([unit_tone(k, n) for k in ks]).astype(np.complex64)
    y = sa.ndft_batch(dev(x), mode="tc").cpu().numpy()
    assert_literal(y, ref32(x), TOL_F32)
    assert [int(np.argmax(np.abs(r))) for r in y] == ks


def test_ndft_tc_gain_and_scale(sa):
    g = np.random.default_rng(7)
    x = (g.standard_normal((130, 256)) + 1j * g.standard_normal((130, 256))).astype(np.complex64)
    x[5] *= 1e-30                      # tiny (still normal in fp32) and large rows
    x[6] *= 1e30
    y = sa.ndft_batch(dev(x), mode="tc", gain=16.0).cpu().numpy()
    assert_literal(y, ref32(16.0 * x.astype(np.complex128)), TOL_F32)


def test_ndft_tc_c2_subset(sa):
    """C2 (N=1024 x 65536, 10% tones) through the tc kernel; oracle on every 512th row."""
    import torch
    from paper_1402_0532_b200.workloads import c2_ndft
    x = c2_ndft().astype(np.complex64)
    y = sa.ndft_batch(dev(x), mode="tc")
    rows = np.arange(0, x.shape[0], 512)
    ys = y[torch.from_numpy(rows).cuda()].cpu().numpy()
    r = ref32(x[rows])
    e = assert_literal(ys, r, TOL_F32)
    print(f"C2 tc: literal max {e.max():.2e}, strict max {strict(ys, r).max():.2e}")


def test_ndft_tc_unsupported_shapes_run_fast(sa):
    """n % 128 != 0 runs the fast (FFMA2 / DFMA) kernels under mode "tc";
    complex128 with n % 64 == 0 runs the int8 tensor-core path (sa_ndft_i8.cu,
    tests/test_gpu_ndft_i8.py): within the fp64 bound of the DFMA kernel."""
    from parity import TOL_F64
    g = np.random.default_rng(3)
    for dt in (np.complex64, np.complex128):
        x = (g.standard_normal((9, 100)) + 1j * g.standard_normal((9, 100))).astype(dt)
        y = sa.ndft_batch(dev(x), mode="tc").cpu().numpy()
        assert np.array_equal(y, sa.ndft_batch(dev(x), mode="fast").cpu().numpy())
    x2 = g.standard_normal((9, 256)) + 1j * g.standard_normal((9, 256))   # c128
    assert_literal(sa.ndft_batch(dev(x2), mode="tc").cpu().numpy(),
                   sa.ndft_batch(dev(x2), mode="fast").cpu().numpy(), TOL_F64)


def test_ndft_tc_empty_batch(sa):
    import torch
    x = torch.zeros((0, 256), dtype=torch.complex64, device="cuda")
    assert sa.ndft_batch(x, mode="tc").shape == (0, 256)
