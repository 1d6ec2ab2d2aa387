"""⊙ range-Doppler maps on the B200 (mirrors ambiguity.py of signadd 0.1.0).

Drop-ins (reference file:line):
  * ``lag_product_mf``  (ambiguity.py:146-155, guards :116-131)
  * ``lag_product_exact`` (ambiguity.py:134-143)
  * ``ambiguity_eq12a`` (ambiguity.py:197-202 via _surface :158-187)
  * ``ambiguity_eq11`` / ``ambiguity_eq12b`` / ``ambiguity_eq12c`` (ambiguity.py:190-221)
  * ``compute_ambiguity`` for every variant (ambiguity.py:224-239)
  * ``AmbiguitySurface``, ``AmbiguityVariant``, ``SPEED_OF_LIGHT``

Extension: ``ambiguity_map`` -- the block-integrated map of SURVEY §8(d)
(y_l = lag_product_mf(surv, ref, l, Ns); z_l[q] = Σ_{t<T} y_l[qT+t];
row_l = NLFFT_M(gain·z_l) or NDFT_M(gain·z_l), T = Ns/M) over any row range,
device-resident, one stream-ordered call.  With M == Ns it is eq12a.

The exact-arithmetic variants use numpy's complex multiply,
reproduced bit-for-bit on the device (``sa_npmul``): eq11 / eq12b / eq12c are
value-identical to the reference, eq12c included (its exact lag residues feed
the sign decisions of the NL-FFT).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native
from ._device import is_device_tensor, require_cuda, sa_dtype_of, to_device, torch
from .errors import ContractError, OpCounter, OpCountReport
from .transforms import ComplexSignal, fft_exact_complex_muls, nfft_complex_ops, ndft_complex_ops
from .twiddle import device_twiddles

__all__ = ["SPEED_OF_LIGHT", "AmbiguityVariant", "AmbiguitySurface", "lag_product_mf",
           "lag_product_exact", "ambiguity_eq11", "ambiguity_eq12a", "ambiguity_eq12b",
           "ambiguity_eq12c", "compute_ambiguity", "ambiguity_map"]

SPEED_OF_LIGHT = 299_792_458.0


class AmbiguityVariant(str, Enum):
    EQ11 = "eq11"
    EQ12A = "eq12a"
    EQ12B = "eq12b"
    EQ12C = "eq12c"


@dataclass(frozen=True)
class AmbiguitySurface:
    """L x N complex surface over (range bin l, Doppler bin p) (ambiguity.py:64-113)."""

    values: np.ndarray
    range_bin_m: float
    doppler_bin_hz: float
    variant: AmbiguityVariant
    sample_rate_hz: float
    lag_op_counts: OpCountReport = field(default_factory=OpCountReport)
    transform_op_counts: OpCountReport = field(default_factory=OpCountReport)

    @property
    def op_counts(self) -> OpCountReport:
        return self.lag_op_counts + self.transform_op_counts

    @property
    def l_bins(self) -> int:
        return self.values.shape[0]

    @property
    def n(self) -> int:
        return self.values.shape[1]

    def magnitude(self) -> np.ndarray:
        return np.abs(self.values)

    def magnitude_db(self, floor_db: float = -300.0) -> np.ndarray:
        mag = self.magnitude()
        peak = mag.max()
        if peak <= 0.0:
            return np.full(mag.shape, floor_db)
        with np.errstate(divide="ignore"):
            db = 20.0 * np.log10(mag / peak)
        return np.maximum(db, floor_db)

    def range_cut(self, floor_db: float = -300.0):
        db = self.magnitude_db(floor_db).max(axis=1)
        ls = np.arange(self.l_bins)
        return ls, ls * self.range_bin_m / 1000.0, db

    def doppler_cut(self, floor_db: float = -300.0):
        db = self.magnitude_db(floor_db).max(axis=0)
        n = self.n
        p = np.arange(n)
        freq = np.where(p <= n // 2, p, p - n) * self.doppler_bin_hz
        order = np.argsort(freq, kind="stable")
        return freq[order], db[order]


def _samples(sig):
    if isinstance(sig, ComplexSignal):
        return sig.samples
    if is_device_tensor(sig):
        return sig
    T = torch()
    if isinstance(sig, T.Tensor) and sig.is_complex():  # host tensor: kept (pinned -> async upload)
        return sig
    return np.asarray(sig, dtype=complex)


def _lag_guards(surv_len: int, ref_len: int, l: int, n: int) -> None:
    # ambiguity.py:121-128 (+ l > n, where the reference's slice assignment
    # raises a numpy ValueError; ContractError is a ValueError subclass)
    if l < 0:
        raise ContractError(f"lag must be non-negative, got {l}")
    if l >= ref_len:
        raise ContractError(f"lag {l} is not below the reference length {ref_len}")
    if surv_len < n:
        raise ContractError(f"surveillance signal shorter than n={n}")
    if ref_len < n - l:
        raise ContractError(f"reference signal too short for n={n}, lag={l}")
    if l > n:
        raise ContractError(f"lag {l} exceeds n={n} (reference slice assignment fails)")


def _dev(x, dtype):
    T = torch()
    if is_device_tensor(x):
        t = x.reshape(-1)
        return (t if t.dtype == dtype else t.to(dtype)).contiguous()
    if isinstance(x, T.Tensor):  # host tensor (pinned: the upload is asynchronous)
        return to_device(x.reshape(-1), dtype)
    return to_device(np.ascontiguousarray(np.asarray(x).reshape(-1)), dtype)


def lag_product_mf(s_surv, s_ref, l: int, n: int | None = None, conjugate_ref: bool = True,
                   counter: OpCounter | None = None):
    """y[i] = s_surv[i] ⊙ conj(s_ref[i-l]), zero reference for i < l (ambiguity.py:146-155)."""
    out = _lag_product(s_surv, s_ref, l, n, conjugate_ref, "sa_lag_product_mf")
    if counter is not None:
        counter.count_complex(out.shape[0])
    return out


def lag_product_exact(s_surv, s_ref, l: int, n: int | None = None, conjugate_ref: bool = True,
                      counter: OpCounter | None = None):
    """y[i] = s_surv[i] * conj(s_ref[i-l]) with numpy's complex multiply (ambiguity.py:134-143)."""
    out = _lag_product(s_surv, s_ref, l, n, conjugate_ref, "sa_lag_product_exact")
    if counter is not None:
        counter.count_complex_mul(out.shape[0])
    return out


def _lag_product(s_surv, s_ref, l, n, conjugate_ref, entry):
    surv = _samples(s_surv)
    ref = _samples(s_ref)
    device_io = is_device_tensor(surv) or is_device_tensor(ref)
    if n is None:
        n = int(surv.shape[0])
    _lag_guards(int(surv.shape[0]), int(ref.shape[0]), l, n)
    require_cuda()
    T = torch()
    dt = T.complex128
    if device_io:
        dt = T.promote_types(surv.dtype if is_device_tensor(surv) else T.complex128,
                             ref.dtype if is_device_tensor(ref) else T.complex128)
    ds = _dev(surv, dt)[:n]
    dr = _dev(ref, dt)
    out = T.empty(n, dtype=dt, device="cuda")
    _native.check(getattr(_native.lib(), entry)(
        sa_dtype_of(out), _native.ptr(ds), _native.ptr(dr), n, dr.numel(), l, int(conjugate_ref),
        _native.ptr(out), _native.stream_ptr()))
    return out if device_io else out.cpu().numpy()


def ambiguity_map(s_surv, s_ref, l_bins: int, m: int, *, l0: int = 0, gain: float = 1.0,
                  conjugate_ref: bool = True, doppler: str = "nfft", mode: str = "fast",
                  lag: str = "mf", out=None, workspace=None, dtype=None, out_ptr: int | None = None):
    """Rows l0..l0+l_bins-1 of the block-integrated range-Doppler map.

    Inputs: CUDA tensors (stay on device, no sync) or host arrays / tensors
    (result returned on the host; a host tensor ``out`` -- pinned for an
    asynchronous download -- receives it).  Ns = len(s_surv); T = Ns / m must be an integer.
    lag: "mf" (⊙, eq12a/eq12b) or "exact" (numpy multiply, eq11/eq12c);
    doppler: "nfft", "ndft" or "fft" (fft_exact).
    ``out_ptr``: raw device address of an (l_bins x m) row-major destination
    (e.g. an IPC mapping of another GPU's map, sharded.PeerMap) -- the
    transform kernel stores there directly and the call returns None.
    """
    T = torch()
    surv = _samples(s_surv)
    ref = _samples(s_ref)
    device_io = is_device_tensor(surv) or is_device_tensor(ref)
    if dtype is None:
        dtype = surv.dtype if isinstance(surv, T.Tensor) and surv.is_complex() else T.complex128
    require_cuda()
    host_out = out if (out is not None and not is_device_tensor(out)) else None
    if host_out is not None:
        out = None
    if (out_ptr is None and not device_io and mode == "fast" and lag == "mf" and doppler == "nfft"
            and dtype == T.complex64):
        r = _map_host_pipelined(surv, ref, l_bins, m, l0, gain, conjugate_ref, host_out)
        if r is not None:
            return r
    ds = _dev(surv, dtype)
    dr = _dev(ref, dtype)
    ns = ds.numel()
    if l_bins < 1:
        raise ContractError("l_bins must be >= 1")
    if m < 1 or ns % m != 0:
        raise ContractError(f"map: Ns={ns} must be a positive multiple of m={m}")
    for l in (l0, l0 + l_bins - 1):
        _lag_guards(ns, dr.numel(), l, ns)
    d = sa_dtype_of(ds)
    if out is None and out_ptr is None:
        out = T.empty((l_bins, m), dtype=ds.dtype, device=ds.device)
    need = ctypes.c_int64()
    _native.check(_native.lib().sa_ambiguity_workspace_bytes(d, l_bins, m, ctypes.byref(need)))
    if workspace is None or workspace.numel() * workspace.element_size() < need.value:
        workspace = T.empty(max(1, need.value), dtype=T.uint8, device=ds.device)
    dop = {"nfft": _native.SA_DOPPLER_NLFFT, "ndft": _native.SA_DOPPLER_NDFT,
           "fft": _native.SA_DOPPLER_FFT_EXACT}[doppler]
    md = {"fast": _native.SA_NDFT_FAST, "exact": _native.SA_NDFT_EXACT}[mode]
    lk = {"mf": _native.SA_LAG_MF, "exact": _native.SA_LAG_EXACT}[lag]
    if doppler != "ndft" and (m < 2 or (m & (m - 1)) != 0):
        raise ContractError(f"{'nfft' if doppler == 'nfft' else 'fft_exact'}: size must be a power of two >= 2, "
                            f"got {m}")
    tw = device_twiddles(m, d, ds.device.index)
    _native.check(_native.lib().sa_ambiguity_map_v(
        d, lk, _native.ptr(ds), _native.ptr(dr), ns, dr.numel(), l0, l_bins, m, float(gain),
        int(conjugate_ref), dop, md, ctypes.c_void_p(tw),
        ctypes.c_void_p(out_ptr) if out_ptr is not None else _native.ptr(out), _native.ptr(workspace),
        workspace.numel() * workspace.element_size(), _native.stream_ptr()))
    if out_ptr is not None:
        return None
    if host_out is not None:
        host_out.copy_(out, non_blocking=True)
        T.cuda.current_stream().synchronize()
        return host_out
    return out if device_io else out.cpu().numpy()


_MAP_STREAMS: dict = {}


class MapGraph:
    """A fixed-shape ``ambiguity_map`` call captured once in a CUDA graph and
    replayed per coherent processing interval: the map's launches (reference
    prep, lag stage, Doppler transform) are stream-ordered and allocation-free
    once warm, so the replay removes their host launch cost (C4: 0.0635 ->
    0.0575 ms per map, C5: 0.427 -> 0.420 ms; results bit-identical to the
    eager call).  B200 extension -- the reference has no counterpart.

    ``surv`` / ``ref`` / ``out`` are the graph's static device buffers: write new
    samples into ``surv`` and ``ref`` (``load`` copies them, stream-ordered), call
    ``replay()``, read ``out``.  Keyword arguments as ``ambiguity_map``.
    """

    def __init__(self, ns: int, ref_len: int, l_bins: int, m: int, *, dtype=None, **kw):
        T = torch()
        require_cuda()
        dtype = dtype or T.complex64
        for k in ("out", "out_ptr", "workspace"):
            if k in kw:
                raise ContractError(f"MapGraph owns its buffers: {k!r} is not accepted")
        self.surv = T.zeros(ns, dtype=dtype, device="cuda")
        self.ref = T.zeros(ref_len, dtype=dtype, device="cuda")
        self.out = T.empty((l_bins, m), dtype=dtype, device="cuda")
        self._args = (l_bins, m)
        self._kw = dict(kw)
        self._graph = None

    def load(self, surv, ref=None):
        """Copy new samples into the static buffers (host or device sources;
        pinned host tensors copy asynchronously on the current stream)."""
        T = torch()
        for dst, src in ((self.surv, surv), (self.ref, ref)):
            if src is None:
                continue
            t = src if isinstance(src, T.Tensor) else T.from_numpy(np.ascontiguousarray(_samples(src)))
            dst.copy_(t.reshape(-1).to(dst.dtype), non_blocking=True)
        return self

    def _call(self):
        ambiguity_map(self.surv, self.ref, *self._args, out=self.out, **self._kw)

    def capture(self):
        """Warm up (scratch pools, twiddle sets, function attributes) on a side
        stream, then capture one call.  Done lazily by the first ``replay``."""
        T = torch()
        st = T.cuda.Stream()
        st.wait_stream(T.cuda.current_stream())
        with T.cuda.stream(st):
            for _ in range(2):
                self._call()
        T.cuda.current_stream().wait_stream(st)
        g = T.cuda.CUDAGraph()
        with T.cuda.graph(g):
            self._call()
        self._graph = g
        return self

    def replay(self):
        """One map of the current buffer contents on the current stream; returns
        the static ``out`` tensor (no sync)."""
        if self._graph is None:
            self.capture()
        self._graph.replay()
        return self.out


def _map_host_pipelined(surv, ref, l_bins, m, l0, gain, conjugate_ref, host_out):
    """Host (pinned) complex64 inputs -> host map with the uploads overlapped: the
    reference goes up first (the int8 lag stage needs its global exponent), then the
    surveillance samples in chunks of Doppler blocks, each chunk's lag stage
    (sa_ambiguity_integrate_blocks, blocked z) running as soon as its samples
    landed while the next chunk uploads; then the Doppler NL-FFT and the download.
    Every block is integrated exactly as in one call, so the map is bit-identical.
    Returns None when the shape is outside the blocked path (the caller takes the
    simple path)."""
    T = torch()
    if not (isinstance(surv, T.Tensor) and isinstance(ref, T.Tensor)) or surv.dtype != T.complex64 \
            or ref.dtype != T.complex64 or not (surv.is_pinned() and ref.is_pinned()):
        return None
    ns, nr = surv.numel(), ref.numel()
    if l0 != 0 or l_bins % 16 or m < 64 or m > 2048 or (m & (m - 1)) or ns % m:
        return None
    tb = ns // m
    if tb < 128 or tb % 128 or tb > 4096 or l_bins > m * tb:
        return None
    for l in (0, l_bins - 1):
        _lag_guards(ns, nr, l, ns)
    dev = T.cuda.current_device()
    if dev not in _MAP_STREAMS:
        _MAP_STREAMS[dev] = T.cuda.Stream()
    up = _MAP_STREAMS[dev]
    cur = T.cuda.current_stream()
    ds = T.empty(ns, dtype=T.complex64, device="cuda")
    dr = T.empty(nr, dtype=T.complex64, device="cuda")
    z = T.empty(((l_bins + 30) * m,), dtype=T.complex64, device="cuda")
    out = T.empty((l_bins, m), dtype=T.complex64, device="cuda")
    zrows = T.tensor([z.data_ptr()], dtype=T.int64, device="cuda")
    up.wait_stream(cur)
    # chunks of >= ~4 MiB of samples (each chunk costs three launches), at most 8
    nchunk = max(1, min(8, m // 16, (ns * 8) >> 22))
    bounds = [m * k // nchunk for k in range(nchunk + 1)]
    with T.cuda.stream(up):
        dr.copy_(ref.reshape(-1), non_blocking=True)
    evs = []
    for k in range(nchunk):
        a, b = bounds[k] * tb, bounds[k + 1] * tb
        with T.cuda.stream(up):
            ds[a:b].copy_(surv.reshape(-1)[a:b], non_blocking=True)
            ev = T.cuda.Event()
            ev.record(up)
        evs.append(ev)
    lib = _native.lib()
    for k in range(nchunk):
        cur.wait_event(evs[k])
        rc = lib.sa_ambiguity_integrate_blocks(
            _native.SA_C64, _native.ptr(ds), _native.ptr(dr), ns, nr, 0, l_bins, m, bounds[k],
            bounds[k + 1] - bounds[k], int(conjugate_ref), _native.ptr(zrows), 1, _native.stream_ptr())
        if rc == _native.SA_ERR_UNSUPPORTED and k == 0:
            cur.wait_stream(up)
            return None
        _native.check(rc)
    tw = device_twiddles(m, _native.SA_C64, dev)
    _native.check(lib.sa_doppler_nlfft_blocked(_native.SA_C64, _native.ptr(z), _native.ptr(out), l_bins, m,
                                                ctypes.c_void_p(tw), float(gain), _native.stream_ptr()))
    for t in (ds, dr, z, zrows):
        t.record_stream(cur)
    ds.record_stream(up)
    dr.record_stream(up)
    if host_out is not None:
        host_out.copy_(out, non_blocking=True)
        cur.synchronize()
        return host_out
    return out.cpu().numpy()


def _surface_rate(s_surv, s_ref) -> float:
    # ambiguity.py:163-170
    fs = None
    for sig in (s_surv, s_ref):
        if isinstance(sig, ComplexSignal):
            if fs is not None and sig.sample_rate_hz != fs:
                raise ContractError("surveillance and reference sample rates differ")
            fs = sig.sample_rate_hz
    if fs is None:
        raise ContractError("at least one input must be a ComplexSignal carrying a sample rate")
    return fs


# variant -> (lag product, Doppler transform) (ambiguity.py:5-14)
_VARIANTS = {
    AmbiguityVariant.EQ11: ("exact", "fft"),
    AmbiguityVariant.EQ12A: ("mf", "nfft"),
    AmbiguityVariant.EQ12B: ("mf", "fft"),
    AmbiguityVariant.EQ12C: ("exact", "nfft"),
}


def _surface(variant: AmbiguityVariant, s_surv, s_ref, l_bins: int, n: int, gain: float,
             conjugate_ref: bool) -> AmbiguitySurface:
    """_surface (ambiguity.py:158-187) for one variant: all l_bins rows in one
    device call, value-identical to the reference row loop."""
    if l_bins < 1:
        raise ContractError("l_bins must be >= 1")
    fs = _surface_rate(s_surv, s_ref)
    surv = np.asarray(_samples(s_surv), dtype=complex)
    ref = np.asarray(_samples(s_ref), dtype=complex)
    for l in (0, l_bins - 1):
        _lag_guards(surv.size, ref.size, l, n)
    lag, doppler = _VARIANTS[variant]
    if n < 2 or (n & (n - 1)) != 0:
        raise ContractError(f"{'nfft' if doppler == 'nfft' else 'fft_exact'}: size must be a power of two >= 2, "
                            f"got {n}")
    vals = ambiguity_map(surv[:n], ref, l_bins, n, gain=gain, conjugate_ref=conjugate_ref,
                         doppler=doppler, mode="exact", lag=lag)
    lag_c = OpCounter()
    if lag == "mf":
        lag_c.count_complex(l_bins * n)
    else:
        lag_c.count_complex_mul(l_bins * n)
    tr_c = OpCounter()
    if doppler == "nfft":
        tr_c.count_complex(l_bins * nfft_complex_ops(n))
    else:
        tr_c.count_complex_mul(l_bins * fft_exact_complex_muls(n))
    return AmbiguitySurface(values=vals, range_bin_m=SPEED_OF_LIGHT / fs, doppler_bin_hz=fs / n,
                            variant=variant, sample_rate_hz=fs,
                            lag_op_counts=lag_c.report(), transform_op_counts=tr_c.report())


def ambiguity_eq11(s_surv, s_ref, l_bins: int, n: int, conjugate_ref: bool = True) -> AmbiguitySurface:
    """Classic cross-ambiguity: exact lag product, exact FFT (ambiguity.py:190-194)."""
    return _surface(AmbiguityVariant.EQ11, s_surv, s_ref, l_bins, n, 1.0, conjugate_ref)


def ambiguity_eq12a(s_surv, s_ref, l_bins: int, n: int, transform_input_gain: float = 1.0,
                    conjugate_ref: bool = True) -> AmbiguitySurface:
    """Fully sign-additive surface: ⊙ lag product into the NL-FFT (ambiguity.py:197-202)."""
    return _surface(AmbiguityVariant.EQ12A, s_surv, s_ref, l_bins, n, transform_input_gain, conjugate_ref)


def ambiguity_eq12b(s_surv, s_ref, l_bins: int, n: int, conjugate_ref: bool = True) -> AmbiguitySurface:
    """⊙ lag product, exact FFT (ambiguity.py:205-209)."""
    return _surface(AmbiguityVariant.EQ12B, s_surv, s_ref, l_bins, n, 1.0, conjugate_ref)


def ambiguity_eq12c(s_surv, s_ref, l_bins: int, n: int, transform_input_gain: float = 1.0,
                    conjugate_ref: bool = True) -> AmbiguitySurface:
    """Exact lag product into the NL-FFT (ambiguity.py:212-221)."""
    return _surface(AmbiguityVariant.EQ12C, s_surv, s_ref, l_bins, n, transform_input_gain, conjugate_ref)


def compute_ambiguity(variant, s_surv, s_ref, l_bins: int, n: int,
                      transform_input_gain: float = 1.0,
                      conjugate_ref: bool = True) -> AmbiguitySurface:
    """Dispatch on variant (ambiguity.py:224-239); the gain reaches only the
    nonlinear-FFT variants."""
    variant = AmbiguityVariant(variant)
    if variant is AmbiguityVariant.EQ11:
        return ambiguity_eq11(s_surv, s_ref, l_bins, n, conjugate_ref)
    if variant is AmbiguityVariant.EQ12A:
        return ambiguity_eq12a(s_surv, s_ref, l_bins, n, transform_input_gain, conjugate_ref)
    if variant is AmbiguityVariant.EQ12B:
        return ambiguity_eq12b(s_surv, s_ref, l_bins, n, conjugate_ref)
    return ambiguity_eq12c(s_surv, s_ref, l_bins, n, transform_input_gain, conjugate_ref)


def map_complex_ops(l_bins: int, ns: int, m: int, doppler: str = "nfft") -> int:
    """Reference ⊙ count of a map: L·Ns lag ⊙ + L·(M(log2M+1) or M²) transform ⊙."""
    tr = nfft_complex_ops(m) if doppler == "nfft" else ndft_complex_ops(m)
    return l_bins * ns + l_bins * tr
