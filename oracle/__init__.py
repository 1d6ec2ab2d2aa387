"""CPU oracle for the signadd hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline -- never as the thing measured or shipped.
The product package ``paper_1402_0532_b200`` does not import it.

It wraps ``liboracle.so`` (``signadd_oracle.c``, a C restatement of the
reference, op-for-op, file:line cited there) and restates the reference
twiddle table (``transforms.py:108-146``) in numpy so that the oracle does not
depend on the product package.

Pinning: ``tests/test_oracle_golden.py`` checks every routine here against
golden vectors produced by the unmodified reference (``tests/golden/
make_golden.py``), value-for-value for fp64.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

__all__ = [
    "build",
    "twiddle_table",
    "unit_tone",
    "mf_complex",
    "ndft",
    "nfft",
    "lag_product_mf",
    "ambiguity_map",
    "fft_exact",
    "lag_product_exact",
    "abs_np",
    "scene_stereo_fm",
    "scene_surveillance",
    "find_peaks",
    "map_floor",
]


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    src = os.path.join(_HERE, "signadd_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB_PATH)
    p = ctypes.c_void_p
    i64 = ctypes.c_int64
    ci = ctypes.c_int
    for sfx in ("f64", "f32"):
        getattr(lib, f"or_mf_complex_{sfx}").argtypes = [i64, p, p, p]
        getattr(lib, f"or_ndft_{sfx}").argtypes = [i64, i64, p, p, p, ci]
        getattr(lib, f"or_nfft_{sfx}").argtypes = [i64, i64, ci, p, p, p, ci]
        getattr(lib, f"or_lag_product_mf_{sfx}").argtypes = [i64, p, p, i64, ci, p]
        getattr(lib, f"or_ambiguity_map_{sfx}").argtypes = [
            i64, p, p, i64, i64, i64, ctypes.c_double, ci, ci, p, p, ci]
        getattr(lib, f"or_ambiguity_map_v_{sfx}").argtypes = [
            i64, p, p, i64, i64, i64, ctypes.c_double, ci, ci, ci, p, p, ci]
        getattr(lib, f"or_ambiguity_map_v_{sfx}").restype = ci
        getattr(lib, f"or_fft_exact_{sfx}").argtypes = [i64, i64, p, p, p, ci]
        getattr(lib, f"or_fft_exact_{sfx}").restype = ci
        getattr(lib, f"or_lag_product_exact_{sfx}").argtypes = [i64, p, p, i64, ci, p]
        for name in ("ndft", "nfft", "lag_product_mf", "ambiguity_map"):
            getattr(lib, f"or_{name}_{sfx}").restype = ci
        getattr(lib, f"or_abs_np_{sfx}").argtypes = [i64, p, p]
        getattr(lib, f"or_find_peaks_{sfx}").argtypes = [i64, i64, p, i64, p, p]
        getattr(lib, f"or_find_peaks_{sfx}").restype = i64
        getattr(lib, f"or_map_floor_{sfx}").argtypes = [i64, i64, p, p, ci, ci, ci, p]
    _lib = lib
    return lib


# --- twiddles: restates transforms.py:108-146 -------------------------------

_QUADRANT = np.array([1.0 + 0.0j, 0.0 - 1.0j, -1.0 + 0.0j, 0.0 + 1.0j])
_TW_CACHE: dict[int, np.ndarray] = {}


def twiddle_table(n: int) -> np.ndarray:
    """exp(-2j*pi*m/n), m=0..n-1, quadrant entries exact (transforms.py:122-133)."""
    t = _TW_CACHE.get(n)
    if t is None:
        m = np.arange(n)
        ang = (-2.0 * np.pi) * m / n
        t = np.cos(ang) + 1j * np.sin(ang)
        quad, rem = np.divmod(4 * m, n)
        exact = rem == 0
        t[exact] = _QUADRANT[quad[exact] % 4]
        t.setflags(write=False)
        _TW_CACHE[n] = t
    return t


def unit_tone(k0: int, n: int) -> np.ndarray:
    """transforms.py:149-152."""
    return np.conj(twiddle_table(n)[(k0 * np.arange(n)) % n])


def _prep(x, dtype):
    ct = np.complex128 if dtype == "f64" else np.complex64
    return np.ascontiguousarray(np.asarray(x).astype(ct, copy=False))


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _table(n, dtype):
    t = twiddle_table(n)
    return np.ascontiguousarray(t if dtype == "f64" else t.astype(np.complex64))


def mf_complex(a, b, dtype: str = "f64") -> np.ndarray:
    lib = _load()
    a = _prep(a, dtype)
    b = _prep(b, dtype)
    a, b = np.broadcast_arrays(a, b)
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    out = np.empty_like(a)
    getattr(lib, f"or_mf_complex_{dtype}")(a.size, _ptr(a), _ptr(b), _ptr(out))
    return out


def ndft(x, dtype: str = "f64", nthreads: int = 1) -> np.ndarray:
    """Batched NDFT over the last axis (transforms.py:223-251)."""
    lib = _load()
    x = _prep(x, dtype)
    n = x.shape[-1]
    y = np.empty_like(x)
    tw = _table(n, dtype)
    rc = getattr(lib, f"or_ndft_{dtype}")(x.size // max(n, 1), n, _ptr(x), _ptr(tw), _ptr(y), nthreads)
    if rc:
        raise ValueError("oracle ndft: bad size")
    return y


def nfft(x, variant: str = "dit", dtype: str = "f64", nthreads: int = 1) -> np.ndarray:
    """Batched NL-FFT over the last axis (DIT: transforms.py:254-298; DIF: DESIGN.md)."""
    lib = _load()
    x = _prep(x, dtype)
    n = x.shape[-1]
    y = np.empty_like(x)
    tw = _table(n, dtype)
    v = 1 if variant == "dif" else 0
    rc = getattr(lib, f"or_nfft_{dtype}")(x.size // max(n, 1), n, v, _ptr(x), _ptr(tw), _ptr(y), nthreads)
    if rc:
        raise ValueError("oracle nfft: size must be a power of two >= 2")
    return y


def lag_product_mf(surv, ref, lag: int, n: int | None = None, conj: bool = True,
                   dtype: str = "f64") -> np.ndarray:
    """ambiguity.py:146-155 (guards are the caller's; see ambiguity.py:116-131)."""
    lib = _load()
    surv = _prep(surv, dtype)
    ref = _prep(ref, dtype)
    if n is None:
        n = surv.size
    assert surv.size >= n and ref.size >= n - lag and 0 <= lag
    out = np.empty(n, dtype=surv.dtype)
    getattr(lib, f"or_lag_product_mf_{dtype}")(n, _ptr(surv), _ptr(ref), lag, int(conj), _ptr(out))
    return out


def fft_exact(x, dtype: str = "f64", nthreads: int = 1) -> np.ndarray:
    """Batched exact radix-2 DIT FFT over the last axis (transforms.py:200-220)."""
    lib = _load()
    x = _prep(x, dtype)
    n = x.shape[-1]
    y = np.empty_like(x)
    tw = _table(n, dtype)
    rc = getattr(lib, f"or_fft_exact_{dtype}")(x.size // max(n, 1), n, _ptr(x), _ptr(tw), _ptr(y), nthreads)
    if rc:
        raise ValueError("oracle fft_exact: size must be a power of two")
    return y


def lag_product_exact(surv, ref, lag: int, n: int | None = None, conj: bool = True,
                      dtype: str = "f64") -> np.ndarray:
    """ambiguity.py:134-143 (numpy complex multiply, guards are the caller's)."""
    lib = _load()
    surv = _prep(surv, dtype)
    ref = _prep(ref, dtype)
    if n is None:
        n = surv.size
    assert surv.size >= n and ref.size >= n - lag and 0 <= lag
    out = np.empty(n, dtype=surv.dtype)
    getattr(lib, f"or_lag_product_exact_{dtype}")(n, _ptr(surv), _ptr(ref), lag, int(conj), _ptr(out))
    return out


_DOPPLER = {"nfft": 0, "ndft": 1, "fft": 2}


def ambiguity_map(surv, ref, l0: int, l_count: int, m: int, gain: float = 1.0,
                  conj: bool = True, doppler: str = "nfft", dtype: str = "f64",
                  nthreads: int = 1, lag: str = "mf") -> np.ndarray:
    """Rows l0..l0+l_count-1 of the block-integrated map: lag "mf"
    (eq12a/eq12b) or "exact" (eq11/eq12c); doppler "nfft", "ndft" or "fft"
    (fft_exact).  With m == len(surv) (T = 1) these are the reference variants."""
    lib = _load()
    surv = _prep(surv, dtype)
    ref = _prep(ref, dtype)
    ns = surv.size
    assert ref.size >= ns
    out = np.empty((l_count, m), dtype=surv.dtype)
    tw = _table(m, dtype)
    rc = getattr(lib, f"or_ambiguity_map_v_{dtype}")(
        ns, _ptr(surv), _ptr(ref), l0, l_count, m, float(gain), int(conj), 0 if lag == "mf" else 1,
        _DOPPLER[doppler], _ptr(tw), _ptr(out), nthreads)
    if rc:
        raise ValueError("oracle ambiguity_map: bad sizes")
    return out


# --- detection: restates detection.py:85-171 ----------------

def _prep2d(values, dtype: str) -> np.ndarray:
    v = np.asarray(values)
    if v.ndim != 2:
        raise ValueError("surface values must be 2-D")
    return np.ascontiguousarray(v, dtype=np.complex128 if dtype == "f64" else np.complex64)


def abs_np(z, dtype: str = "f64") -> np.ndarray:
    """numpy's complex magnitude as the reference host computes it (C restatement)."""
    zz = np.ascontiguousarray(np.asarray(z).ravel(), dtype=np.complex128 if dtype == "f64" else np.complex64)
    out = np.empty(zz.size, dtype=np.float64 if dtype == "f64" else np.float32)
    getattr(_load(), f"or_abs_np_{dtype}")(
        zz.size, zz.ctypes.data, out.ctypes.data)
    return out


def find_peaks(values, k: int, dtype: str = "f64") -> np.ndarray:
    """detection.find_peaks (detection.py:85-108): rows (l, p, magnitude), strongest first."""
    v = _prep2d(values, dtype)
    idx = np.empty(max(k, 1), dtype=np.int64)
    mag = np.empty(max(k, 1), dtype=np.float64)
    n = getattr(_load(), f"or_find_peaks_{dtype}")(v.shape[0], v.shape[1], v.ctypes.data, k,
                                                    idx.ctypes.data, mag.ctypes.data)
    if n < 0:
        raise ValueError("find_peaks: bad arguments")
    out = np.empty((n, 3))
    out[:, 0], out[:, 1], out[:, 2] = idx[:n] // v.shape[1], idx[:n] % v.shape[1], mag[:n]
    return out


def map_floor(values, centers, guard, dtype: str = "f64") -> tuple[float, float, int]:
    """(max |v|, max |v| outside every guard box, outside cells) -- the inputs of
    detection.sidelobe_floor_db (detection.py:148-171; boxes as _guard_mask :137-145)."""
    v = _prep2d(values, dtype)
    c = np.ascontiguousarray(np.asarray(centers, dtype=np.int32).reshape(-1, 2))
    out = np.empty(3)
    getattr(_load(), f"or_map_floor_{dtype}")(v.shape[0], v.shape[1], v.ctypes.data, c.ctypes.data,
                                               c.shape[0], int(guard[0]), int(guard[1]), out.ctypes.data)
    return float(out[0]), float(out[1]), int(out[2])


# --- scene synthesis: restates radar.py:179-275 ------------
# numpy, written in the evaluation order the device kernels follow
# (csrc/sa_scene.cu); pinned bit-for-bit against the reference's own outputs
# in tests/test_oracle_golden.py, which is what licenses that order.

def scene_stereo_fm(n: int, f_s: float, k_f: float, f_p: float, seed: int) -> np.ndarray:
    """gen_stereo_fm (radar.py:179-192)."""
    x1, x2 = np.random.default_rng(seed).uniform(-1.0, 1.0, size=(2, n))
    t = np.arange(n) / f_s
    ca, cb, cc, ck = 2.0 * np.pi * 2.0 * f_p, 2.0 * np.pi * 3.0 * f_p, 2.0 * np.pi * f_p, 2.0 * np.pi * k_f
    m = 0.9 * (x1 + x2)
    m = m + (0.5 * (x1 - x2)) * np.cos(ca * t)
    m = m + 0.25 * np.cos(cb * t)
    m = m + 0.1 * np.cos(cc * t)
    ph = ck * m
    out = np.empty(n, dtype=complex)
    out.real, out.imag = np.cos(ph), np.sin(ph)
    return out


def scene_surveillance(ref, delays, amps, dopplers, f_s: float, noise: dict, gain: float) -> np.ndarray:
    """synth_surveillance + apply_noise (radar.py:215-275): per obstacle
    amplitude * shifted (* exp(j ((2 pi f) i) (1/f_s)) when f != 0), summed
    from +0; noise from the reference's numpy streams; times the gain."""
    ref = np.asarray(ref, dtype=complex)
    d = ref.size
    i = np.arange(d)
    acc = np.zeros(d, dtype=complex)
    for l, a, f in zip(delays, amps, dopplers):
        sh = np.zeros(d, dtype=complex)
        sh[l:] = ref[: d - l]
        term = complex(a) * sh
        if f != 0.0:
            ph = ((2j * np.pi * f).imag * i) * (1.0 / f_s)
            e = np.empty(d, dtype=complex)
            e.real, e.imag = np.cos(ph), np.sin(ph)
            term = term * e
        acc = acc + term
    kind = noise.get("kind", "none")
    if kind == "awgn":
        p_sig = float(np.mean(np.abs(acc) ** 2))
        scale = np.sqrt(p_sig / 10.0 ** (noise["snr_db"] / 10.0) / 2.0)
        z = np.random.default_rng(noise["seed"]).standard_normal((2, d)) * scale
        acc = (acc.real + z[0]) + 1j * (acc.imag + z[1])
    elif kind == "eps_contaminated":
        rng = np.random.default_rng(noise["seed"])
        sig = np.where(rng.random((2, d)) < noise["eps"], noise["sigma1"], noise["sigma2"])
        z = rng.standard_normal((2, d)) * sig
        acc = (acc.real + z[0]) + 1j * (acc.imag + z[1])
    out = np.empty(d, dtype=complex)
    out.real, out.imag = acc.real * gain, acc.imag * gain
    return out
