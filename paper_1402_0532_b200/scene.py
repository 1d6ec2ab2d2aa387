"""Scene synthesis on the device (mirrors radar.py of signadd 0.1.0).

The reference builds its inputs with numpy: a stereo-FM illuminator
(``gen_stereo_fm``, radar.py:179-192) and a surveillance signal that sums
delayed, Doppler-shifted echoes, adds noise and applies the receiver gain
(``synth_surveillance`` / ``apply_noise``, radar.py:215-275).  For CPI-scale
scenes (2^20 - 2^22 samples) these run here as CUDA kernels
(``libsignadd_b200.so``, ``sa_scene_*``) and the signals land in HBM, ready
for ``ambiguity_map``.

Reproducibility: the random draws are numpy's own streams, drawn on the host
exactly as the reference draws them and uploaded; the arithmetic follows
numpy's evaluation order step by step.  The device sin/cos differ from the
host libm by an ulp or two and the AWGN power is a device reduction, so the
signals agree with the reference to ~1e-15 relative, not bitwise
(tests/test_gpu_scene.py pins them against the reference's own outputs).

Entry points take the reference's own dataclasses (``Scenario``,
``StereoFmConfig``, duck-typed) or the light specs below, which need no
reference install:

  * ``gen_stereo_fm(cfg)``              radar.py:179-192
  * ``synth_surveillance(scn, s_ref)``  radar.py:215-243 (+ apply_noise :270-275)
  * ``build_signals(scn)``              radar.py:278-282
  * ``bistatic_delay_bins``             radar.py:195-199
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._device import require_cuda, torch
from .errors import ContractError

__all__ = ["FmSpec", "Echo", "NoiseSpec", "SceneSpec", "DeviceSignal", "bistatic_delay_bins",
           "gen_stereo_fm", "synth_surveillance", "build_signals", "MAX_ECHOES"]

SPEED_OF_LIGHT = 299_792_458.0
PILOT_HZ = 19_000.0
MAX_ECHOES = 64


@dataclass(frozen=True)
class FmSpec:
    """StereoFmConfig's fields (radar.py:64-85)."""
    f_s: float = 200_000.0
    duration_samples: int = 4160
    k_f: float = 0.25
    f_p: float = PILOT_HZ
    seed: int = 0


@dataclass(frozen=True)
class Echo:
    """One obstacle by its integer delay (the reference derives it from geometry)."""
    delay: int
    amplitude: complex = 1.0 + 0.0j
    doppler_hz: float = 0.0


@dataclass(frozen=True)
class NoiseSpec:
    """NoiseModel's fields (radar.py:108-121); kind "none" | "awgn" | "eps_contaminated"."""
    kind: str = "none"
    snr_db: float = 0.0
    eps: float = 0.9
    sigma1: float = 0.25
    sigma2: float = 10.0
    seed: int = 0


@dataclass(frozen=True)
class SceneSpec:
    """The parts of a Scenario the signal builders read (radar.py:132-176)."""
    echoes: tuple
    fm: FmSpec = field(default_factory=FmSpec)
    noise: NoiseSpec = field(default_factory=NoiseSpec)
    n: int = 4096
    surv_gain: float = 64.0

    @property
    def obstacles(self) -> tuple:
        return tuple(self.echoes)

    def delay_bins(self) -> list[int]:
        return [int(e.delay) for e in self.echoes]


@dataclass(frozen=True)
class DeviceSignal:
    """Samples in HBM (complex CUDA tensor) and the sample rate; ``.samples``
    is what ``ambiguity_map`` / ``ambiguity_peaks`` accept."""
    samples: object
    f_s: float

    def __len__(self) -> int:
        return int(self.samples.numel())


def bistatic_delay_bins(tx_km, rx_km, obstacle, f_s: float) -> int:
    """Integer transmitter -> obstacle -> receiver delay in samples (radar.py:195-199)."""
    d1 = math.hypot(obstacle.x_km - tx_km[0], obstacle.y_km - tx_km[1])
    d2 = math.hypot(obstacle.x_km - rx_km[0], obstacle.y_km - rx_km[1])
    return round((d1 + d2) * 1000.0 / SPEED_OF_LIGHT * f_s)


def _upload(a: np.ndarray):
    T = torch()
    return T.from_numpy(np.ascontiguousarray(a)).pin_memory().to("cuda", non_blocking=True)


def _out_dtype(dtype) -> int:
    T = torch()
    if dtype == T.complex128:
        return _native.SA_C128
    if dtype == T.complex64:
        return _native.SA_C64
    raise ContractError(f"scene synthesis writes complex64 or complex128, not {dtype}")


def gen_stereo_fm(cfg, dtype=None) -> DeviceSignal:
    """The unit-modulus FM baseband signal, deterministic per seed (radar.py:179-192)."""
    T = torch()
    require_cuda()
    dtype = dtype or T.complex128
    n = int(cfg.duration_samples)
    if n < 1:
        raise ContractError("StereoFmConfig: duration_samples must be >= 1")
    f_s, f_p, k_f = float(cfg.f_s), float(cfg.f_p), float(cfg.k_f)
    rng = np.random.default_rng(cfg.seed)
    u = _upload(rng.uniform(-1.0, 1.0, size=(2, n)))  # the reference's draws
    out = T.empty(n, dtype=dtype, device="cuda")
    # the constant factors exactly as the reference's Python scalars form them
    ca = 2.0 * np.pi * 2.0 * f_p
    cb = 2.0 * np.pi * 3.0 * f_p
    cc = 2.0 * np.pi * f_p
    ck = 2.0 * np.pi * k_f
    _native.check(_native.lib().sa_scene_stereo_fm(_out_dtype(dtype), _native.ptr(u), n, f_s, ca, cb, cc, ck,
                                                   _native.ptr(out), _native.stream_ptr()))
    return DeviceSignal(out, f_s)


def _noise_kind(noise) -> str:
    k = getattr(noise.kind, "value", noise.kind)
    if k not in ("none", "awgn", "eps_contaminated"):
        raise ContractError(f"unknown noise kind {k!r}")
    return k


def synth_surveillance(scn, s_ref, dtype=None) -> DeviceSignal:
    """Sum of delayed Doppler-shifted echoes, plus noise, times the gain
    (radar.py:215-243 with apply_noise, radar.py:245-275)."""
    T = torch()
    require_cuda()
    dtype = dtype or T.complex128
    f_s = float(scn.fm.f_s)
    ref = getattr(s_ref, "samples", s_ref)
    if not (isinstance(ref, T.Tensor) and ref.is_cuda):
        ref = T.as_tensor(np.asarray(ref, dtype=complex)).to("cuda")
    if ref.dtype != T.complex128:
        raise ContractError("synth_surveillance: the reference signal must be complex128 (as the reference)")
    ref = ref.contiguous()
    d = int(ref.numel())
    delays = [int(v) for v in scn.delay_bins()]
    obs = list(scn.obstacles)
    if len(obs) < 1:
        raise ContractError("Scenario: need at least one obstacle")
    if len(obs) > MAX_ECHOES:
        raise ContractError(f"synth_surveillance: at most {MAX_ECHOES} obstacles on the device")
    need = int(scn.n) + max(delays)
    if d < need:
        raise ContractError(f"synth_surveillance: reference length {d} is below n + max delay = {need}")

    dl = (ctypes.c_int64 * len(obs))(*delays)
    amps = (ctypes.c_double * (2 * len(obs)))()
    w = (ctypes.c_double * len(obs))()
    for k, ob in enumerate(obs):
        a = complex(ob.amplitude)
        amps[2 * k], amps[2 * k + 1] = a.real, a.imag
        f = float(ob.doppler_hz)
        w[k] = 0.0 if f == 0.0 else (2j * np.pi * f).imag  # the reference's 2j*pi*f
    lib = _native.lib()
    x = T.empty(d, dtype=T.complex128, device="cuda")
    _native.check(lib.sa_scene_echoes(_native.ptr(ref), d, len(obs), dl, amps, w, 1.0 / f_s, _native.ptr(x),
                                      _native.stream_ptr()))

    noise = scn.noise
    kind = _noise_kind(noise)
    z = u = None
    scale = 0.0
    if kind == "awgn":
        rng = np.random.default_rng(noise.seed)
        zh = rng.standard_normal((2, d))  # drawn while the echoes run
        need_ws = ctypes.c_int64()
        _native.check(lib.sa_scene_power_workspace_bytes(d, ctypes.byref(need_ws)))
        ws = T.empty(max(1, need_ws.value), dtype=T.uint8, device="cuda")
        psum = T.empty(1, dtype=T.float64, device="cuda")
        _native.check(lib.sa_scene_power(_native.ptr(x), d, _native.ptr(psum), _native.ptr(ws), need_ws.value,
                                         _native.stream_ptr()))
        p_sig = float(psum.item()) / d
        if p_sig <= 0.0:
            raise ContractError("add_awgn: zero-power input with finite SNR target")
        p_noise = p_sig / 10.0 ** (noise.snr_db / 10.0)
        scale = math.sqrt(p_noise / 2.0)
        z = _upload(zh)
    elif kind == "eps_contaminated":
        rng = np.random.default_rng(noise.seed)
        u = _upload(rng.random((2, d)))
        z = _upload(rng.standard_normal((2, d)))
    out = T.empty(d, dtype=dtype, device="cuda")
    code = {"none": _native.SA_NOISE_NONE, "awgn": _native.SA_NOISE_AWGN,
            "eps_contaminated": _native.SA_NOISE_EPS}[kind]
    _native.check(lib.sa_scene_noise_gain(_out_dtype(dtype), _native.ptr(x), d, code,
                                          _native.ptr(z) if z is not None else None,
                                          _native.ptr(u) if u is not None else None, scale,
                                          float(noise.eps), float(noise.sigma1), float(noise.sigma2),
                                          float(scn.surv_gain), _native.ptr(out), _native.stream_ptr()))
    return DeviceSignal(out, f_s)


def build_signals(scn, dtype=None) -> tuple[DeviceSignal, DeviceSignal]:
    """(reference, surveillance) pair for a scenario (radar.py:278-282).  The
    echoes are built from the complex128 reference; ``dtype`` applies to both
    returned signals."""
    T = torch()
    dtype = dtype or T.complex128
    s_ref = gen_stereo_fm(scn.fm, T.complex128)
    s_surv = synth_surveillance(scn, s_ref, dtype)
    if dtype != T.complex128:
        s_ref = DeviceSignal(s_ref.samples.to(dtype), s_ref.f_s)
    return s_ref, s_surv
