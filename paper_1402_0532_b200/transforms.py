"""Sign-additive transforms on the B200: drop-in ``ndft``/``nfft`` + batched API.

Reference interface (signadd 0.1.0, transforms.py):
  * ``ndft(x, counter=None) -> Spectrum``   (transforms.py:223-251)
  * ``nfft(x, counter=None) -> Spectrum``   (transforms.py:254-298)
  * ``ComplexSignal``, ``TransformKind``, ``Spectrum``, ``unit_tone``,
    ``peak_index`` and the count formulas (:68-105, :149-152, :301-327).

The 1-D drop-ins keep the reference contract exactly: 1-d input of length
>= 1, finite (``DomainError``), power of two >= 2 for nfft (``ContractError``),
numpy complex128 ``bins``, analytic op counts merged into ``counter``.  They run
the value-identical kernels (EXACT NDFT; the NL-FFT is always value-identical).

The batched extension (``ndft_batch``/``nfft_batch``) takes a (B, N)
complex64/complex128 tensor; CUDA tensors stay on the device (no sync), host
arrays/tensors are staged through the device and returned on the host (the
end-to-end path timed by bench.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native
from ._device import check_finite_device, is_device_tensor, require_cuda, sa_dtype_of, to_device, torch
from .errors import ContractError, DomainError, OpCounter, OpCountReport
from .twiddle import TwiddleTable, device_twiddles, twiddle_table

__all__ = [
    "ComplexSignal", "TransformKind", "Spectrum", "TwiddleTable", "twiddle_table", "unit_tone",
    "ndft", "nfft", "fft_exact", "ndft_batch", "nfft_batch", "peak_index", "ndft_complex_ops",
    "nfft_complex_ops", "nfft_butterflies", "nfft_dif_complex_ops", "fft_exact_complex_muls",
    "pipeline_chunks",
]


@dataclass(frozen=True)
class ComplexSignal:
    """A finite sequence of complex samples with its sample rate (transforms.py:68-86)."""

    samples: np.ndarray
    sample_rate_hz: float

    def __post_init__(self):
        s = np.asarray(self.samples, dtype=complex)
        if s.ndim != 1 or s.size < 1:
            raise ContractError("ComplexSignal: need a 1-d sequence of length >= 1")
        if not np.all(np.isfinite(s.real)) or not np.all(np.isfinite(s.imag)):
            raise DomainError("ComplexSignal: samples must be finite")
        if not (self.sample_rate_hz > 0):
            raise ContractError("ComplexSignal: sample_rate_hz must be positive")
        object.__setattr__(self, "samples", s)

    def __len__(self) -> int:
        return self.samples.size


class TransformKind(str, Enum):
    DFT_EXACT = "dft"
    FFT_EXACT = "fft"
    NDFT = "ndft"
    NFFT = "nfft"


@dataclass(frozen=True)
class Spectrum:
    """Transform output: one complex bin per input sample (transforms.py:89-105)."""

    bins: np.ndarray
    transform_kind: TransformKind
    op_counts: OpCountReport = field(default_factory=OpCountReport)

    def magnitude(self) -> np.ndarray:
        return np.abs(self.bins)


def unit_tone(k0: int, n: int) -> np.ndarray:
    """exp(+2j*pi*k0*m/n) on the exact twiddle grid (transforms.py:149-152)."""
    tbl = twiddle_table(n)
    return np.conj(tbl.entries[(k0 * np.arange(n)) % n])


def _as_samples(x) -> np.ndarray:
    # transforms.py:155-163
    if isinstance(x, ComplexSignal):
        return x.samples
    if is_device_tensor(x):
        x = x.detach().cpu().numpy()
    s = np.asarray(x, dtype=complex)
    if s.ndim != 1 or s.size < 1:
        raise ContractError("transform input must be a 1-d sequence of length >= 1")
    if not np.all(np.isfinite(s.real)) or not np.all(np.isfinite(s.imag)):
        raise DomainError("transform input must be finite")
    return s


def _require_pow2(n: int, what: str) -> int:
    # transforms.py:166-169
    if n < 2 or (n & (n - 1)) != 0:
        raise ContractError(f"{what}: size must be a power of two >= 2, got {n}")
    return int(np.log2(n))


# --- raw launchers (device tensors in, device tensors out, stream-ordered) ---

def _launch_ndft(x, y, mode: int, gain: float) -> None:
    batch, n = x.shape
    d = sa_dtype_of(x)
    tw = device_twiddles(n, d, x.device.index)
    _native.check(_native.lib().sa_ndft(d, _native.ptr(x), _native.ptr(y), batch, n,
                                        ctypes.c_void_p(tw), mode, float(gain),
                                        _native.stream_ptr()))


def _launch_nlfft(x, y, variant: int, gain: float) -> None:
    batch, n = x.shape
    d = sa_dtype_of(x)
    tw = device_twiddles(n, d, x.device.index)
    _native.check(_native.lib().sa_nlfft(d, variant, _native.ptr(x), _native.ptr(y), batch, n,
                                         ctypes.c_void_p(tw), float(gain), _native.stream_ptr()))


# --- reference drop-ins --------------------------------------------------------

def ndft(x, counter: OpCounter | None = None) -> Spectrum:
    """Nonlinear DFT, value-identical to transforms.py:223-251 (EXACT kernel)."""
    v = _as_samples(x)
    n = v.size
    require_cuda()
    d = to_device(v, torch().complex128).view(1, n)
    y = torch().empty_like(d)
    _launch_ndft(d, y, _native.SA_NDFT_EXACT, 1.0)
    local = OpCounter()
    local.count_complex(n * n)
    bins = y.view(n).cpu().numpy()
    if counter is not None:
        counter.merge(local)
    return Spectrum(bins, TransformKind.NDFT, local.report())


def nfft(x, counter: OpCounter | None = None) -> Spectrum:
    """Nonlinear FFT (DIT), value-identical to transforms.py:254-298."""
    v = _as_samples(x)
    n = v.size
    _require_pow2(n, "nfft")
    require_cuda()
    d = to_device(v, torch().complex128).view(1, n)
    y = torch().empty_like(d)
    _launch_nlfft(d, y, _native.SA_DIT, 1.0)
    local = OpCounter()
    local.count_complex(nfft_complex_ops(n))
    bins = y.view(n).cpu().numpy()
    if counter is not None:
        counter.merge(local)
    return Spectrum(bins, TransformKind.NFFT, local.report())


def fft_exact(x, counter: OpCounter | None = None) -> Spectrum:
    """Exact radix-2 DIT FFT, bit-identical to transforms.py:200-220 (numpy's
    complex multiply of every twiddle product reproduced on the device)."""
    v = _as_samples(x)
    n = v.size
    logn = _require_pow2(n, "fft_exact")
    require_cuda()
    d = to_device(v, torch().complex128).view(1, n)
    y = torch().empty_like(d)
    _launch_nlfft(d, y, _native.SA_FFT_EXACT, 1.0)
    local = OpCounter()
    local.count_complex_mul((n // 2) * logn)
    bins = y.view(n).cpu().numpy()
    if counter is not None:
        counter.merge(local)
    return Spectrum(bins, TransformKind.FFT_EXACT, local.report())


# --- batched extension -------------------------------------------------------------

def _batched(x, out, check_finite: bool, dtype):
    """Normalise a batched call: returns (device_in, device_out, host_out_or_None)."""
    T = torch()
    require_cuda()
    host_result = None
    if is_device_tensor(x):
        xd = x if x.dim() == 2 else x.reshape(1, -1)
        if not xd.is_contiguous():
            xd = xd.contiguous()
        if dtype is not None and xd.dtype != dtype:
            xd = xd.to(dtype)
        sa_dtype_of(xd)
    else:
        if isinstance(x, T.Tensor):
            h = x
            if h.dim() == 1:
                h = h.reshape(1, -1)
        else:
            a = np.asarray(x)
            if a.ndim == 1:
                a = a.reshape(1, -1)
            if not np.iscomplexobj(a):
                a = a.astype(np.complex128)
            h = T.from_numpy(np.ascontiguousarray(a))
        if dtype is not None and h.dtype != dtype:
            h = h.to(dtype)
        sa_dtype_of(h)
        xd = h.to("cuda", non_blocking=True)
        host_result = h if out is None else out
    if xd.dim() != 2 or xd.shape[1] < 1:
        raise ContractError("batched transform input must be (batch, n) with n >= 1")
    if check_finite:
        check_finite_device(xd)
    if out is not None and is_device_tensor(out):
        yd = out
    else:
        yd = T.empty_like(xd)
    return xd, yd, host_result


def _finish(yd, host_result, out, x):
    if host_result is None:
        return yd
    T = torch()
    if out is not None:
        out.copy_(yd.view_as(out), non_blocking=True)
        T.cuda.current_stream().synchronize()
        return out
    res = yd.cpu()
    if isinstance(x, T.Tensor):
        return res.view(x.shape) if x.dim() == 1 else res
    r = res.numpy()
    return r.reshape(-1) if np.asarray(x).ndim == 1 else r


_SIDE_STREAMS: dict = {}


def _pinned_host(t) -> bool:
    T = torch()
    return isinstance(t, T.Tensor) and not t.is_cuda and t.is_pinned()


def pipeline_chunks(nbytes: int) -> int:
    """Steady-state row chunks of a pinned-host batched call: 32 MiB each, at
    most 64 -- measured best on C2 (512 MiB each way)."""
    return int(max(1, min(64, nbytes // (PIPELINE_MIB << 20))))


PIPELINE_MIB = int(__import__("os").environ.get("SA_PIPELINE_MIB", "32"))
PIPELINE_RAMP = int(__import__("os").environ.get("SA_PIPELINE_RAMP", "1"))


def pipeline_plan(rows: int, row_bytes: int, row_align: int) -> list[tuple[int, int]]:
    """Row ranges of a pinned-host batched call.  Steady chunks of
    ``pipeline_chunks``' size; the first and last PIPELINE_RAMP chunks halve
    towards the ends (32 -> 16 -> 8 MiB), so the pipeline fills after a
    small upload and drains after a small download.  One transform launch per
    chunk."""
    total = rows * row_bytes
    step = -(-rows // pipeline_chunks(total))
    step = -(-step // row_align) * row_align
    ramp = []
    for k in range(1, PIPELINE_RAMP + 1):
        r = (step >> k) // row_align * row_align
        if r < row_align or 2 * sum(ramp) + 2 * r > rows // 2:
            break
        ramp.append(r)
    sizes_head = ramp[::-1]
    head = sum(sizes_head)
    tail = head
    mid_rows = rows - head - tail
    out, r0 = [], 0
    for sz in sizes_head:
        out.append((r0, r0 + sz))
        r0 += sz
    mid_end = r0 + mid_rows
    nmid = max(1, -(-mid_rows // step))
    even = -(-(-(-mid_rows // nmid)) // row_align) * row_align  # equal chunks, aligned
    while r0 < mid_end:
        r1 = min(mid_end, r0 + even)
        out.append((r0, r1))
        r0 = r1
    for sz in ramp:
        out.append((r0, r0 + sz))
        r0 += sz
    assert r0 == rows
    return out


def _host_pipelined(x, out, launch_rows, row_align: int, dtype):
    """Pinned host (B, N) in -> pinned host out, with H2D / compute / D2H
    overlapped over row chunks: chunk i uploads on one side stream, runs once
    uploaded (alternating between the current stream and a second compute
    stream, so consecutive chunks' waves overlap), downloads on another side
    stream once computed.  PCIe is full duplex, so the transform of chunk i
    overlaps the copies of chunks i+-1.  Returns the host output (synchronised)."""
    T = torch()
    xh = x if x.dim() == 2 else x.reshape(1, -1)
    if dtype is not None and xh.dtype != dtype:
        return None  # would need a host-side conversion: take the simple path
    sa_dtype_of(xh)
    if out is None:
        out = T.empty(xh.shape, dtype=xh.dtype, pin_memory=True)
    oh = out if out.dim() == 2 else out.view(xh.shape)
    rows, n = xh.shape
    plan = pipeline_plan(rows, n * xh.element_size(), row_align)
    dev = T.cuda.current_device()
    if dev not in _SIDE_STREAMS:
        _SIDE_STREAMS[dev] = (T.cuda.Stream(), T.cuda.Stream(), T.cuda.Stream())
    up, down, alt = _SIDE_STREAMS[dev]
    cur = T.cuda.current_stream()
    alt.wait_stream(cur)
    xd = T.empty(xh.shape, dtype=xh.dtype, device="cuda")
    yd = T.empty_like(xd)
    up.wait_stream(cur)  # device buffers are fresh allocations on `cur`
    for ci, (r0, r1) in enumerate(plan):
        with T.cuda.stream(up):
            xd[r0:r1].copy_(xh[r0:r1], non_blocking=True)
            ev_in = T.cuda.Event()
            ev_in.record(up)
        # consecutive chunks alternate between two compute streams, so one
        # chunk's last wave overlaps the next chunk's first
        ks = alt if ci % 2 else cur
        ks.wait_event(ev_in)
        with T.cuda.stream(ks):
            launch_rows(xd[r0:r1], yd[r0:r1])
        ev_k = T.cuda.Event()
        ev_k.record(ks)
        down.wait_event(ev_k)
        with T.cuda.stream(down):
            oh[r0:r1].copy_(yd[r0:r1], non_blocking=True)
    cur.wait_stream(down)
    xd.record_stream(up)
    yd.record_stream(down)
    xd.record_stream(alt)
    yd.record_stream(alt)
    cur.synchronize()
    return out.view(x.shape) if x.dim() == 1 else out


def ndft_batch(x, *, mode: str = "fast", gain: float = 1.0, out=None, check_finite: bool = False,
               dtype=None):
    """Batched NDFT over the last axis of a (B, N) complex64/complex128 input.

    mode "fast": sign-split regrouped accumulation (8 FMA per ⊙); "exact":
    value-identical to the reference per vector; "tc": the fast-mode sum on the
    tcgen05 tensor cores -- complex64 as a sign-split bf16 GEMM (n % 128 == 0,
    n <= 4096), complex128 with exact int8 digits (n % 64 == 0, 128 <= n <= 2048,
    within the fp64 bound); "tc8": exact int8 digits for complex64 too (one digit
    pair, n % 128 == 0, 128 <= n <= 2048).  Other shapes run "fast".  ``gain`` scales the input first
    (as ``transform_gain * y`` in ambiguity.py:176-177).
    """
    m = {"fast": _native.SA_NDFT_FAST, "exact": _native.SA_NDFT_EXACT, "tc": _native.SA_NDFT_TC,
         "tc8": _native.SA_NDFT_TC_I8}[mode]
    if _pinned_host(x) and (out is None or _pinned_host(out)) and not check_finite:
        r = _host_pipelined(x, out, lambda a, b: _launch_ndft(a, b, m, gain), 128, dtype)
        if r is not None:
            return r
    xd, yd, host = _batched(x, out, check_finite, dtype)
    _launch_ndft(xd, yd, m, gain)
    return _finish(yd, host, out, x)


def nfft_batch(x, *, variant: str = "dit", gain: float = 1.0, out=None, check_finite: bool = False,
               dtype=None):
    """Batched NL-FFT (DIT = reference nfft; DIF = DESIGN.md convention);
    variant "exact" is the exact-multiply fft_exact (transforms.py:200-220)."""
    v = {"dit": _native.SA_DIT, "dif": _native.SA_DIF, "exact": _native.SA_FFT_EXACT}[variant]
    if _pinned_host(x) and (out is None or _pinned_host(out)) and not check_finite:
        _require_pow2(x.shape[-1], "nfft")
        r = _host_pipelined(x, out, lambda a, b: _launch_nlfft(a, b, v, gain), 1, dtype)
        if r is not None:
            return r
    xd, yd, host = _batched(x, out, check_finite, dtype)
    _require_pow2(xd.shape[1], "nfft")
    _launch_nlfft(xd, yd, v, gain)
    return _finish(yd, host, out, x)


def peak_index(s) -> int:
    """Index of the largest-magnitude bin; ties go to the smallest (transforms.py:301-306)."""
    bins = s.bins if isinstance(s, Spectrum) else np.asarray(s)
    if bins.size < 1:
        raise ContractError("peak_index: spectrum must be non-empty")
    return int(np.argmax(np.abs(bins)))


def ndft_complex_ops(n: int) -> int:
    return n * n


def nfft_complex_ops(n: int) -> int:
    """N*(log2(N)+1): 4 per bottom-stage pair, 2 per butterfly above (transforms.py:313-315)."""
    return n * (_require_pow2(n, "nfft_complex_ops") + 1)


def nfft_butterflies(n: int) -> int:
    return (n // 2) * _require_pow2(n, "nfft_butterflies")


def fft_exact_complex_muls(n: int) -> int:
    """(N/2)*log2(N) twiddle products (transforms.py:213)."""
    return (n // 2) * _require_pow2(n, "fft_exact_complex_muls")


def nfft_dif_complex_ops(n: int) -> int:
    """DIF convention: (N/2)(log2N-1) stage ⊙ + 2N in the final 2-point stage."""
    return (n // 2) * (_require_pow2(n, "nfft_dif_complex_ops") - 1) + 2 * n
