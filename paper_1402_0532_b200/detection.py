"""Detection on the device-resident map (mirrors detection.py of signadd 0.1.0).

SURVEY §8(f)-1: the map's direct consumer.  The peak search and the side-lobe
maxima run in ``libsignadd_b200.so`` (``sa_map_peaks``, ``sa_map_floor``), so a
4096 x 2048 map never leaves the GPU -- only k peaks and three scalars do.

Drop-ins (reference file:line):
  * ``find_peaks(surface, k)``       detection.py:85-108
  * ``classify_bins``                the guard-box logic of ``classify`` (:115-134)
  * ``sidelobe_floor_db``            detection.py:148-171 (boxes as _guard_mask :137-145)
  * ``Peak``                         detection.py:53-57

Extension: ``map_peaks(values, k)`` on any complex CUDA tensor or host array,
and ``ambiguity_peaks`` = ``ambiguity_map`` + ``map_peaks`` device to device.

Magnitudes are numpy's complex absolute value exactly as the reference host
computes it (``max * sqrt(fma(r, r, 1))``, r = min/max), so strict-maximum
decisions, ties (row-major order) and the floor values match the reference
bit for bit.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from ._device import is_device_tensor, require_cuda, sa_dtype_of, to_device, torch
from .errors import ContractError

__all__ = ["Peak", "DEFAULT_GUARD", "DB_FLOOR_CAP", "map_peaks", "find_peaks", "floor_maxima",
           "sidelobe_floor_db", "classify_bins", "ambiguity_peaks"]

DEFAULT_GUARD = (2, 2)
DB_FLOOR_CAP = -300.0
MAX_K = 1024


@dataclass(frozen=True)
class Peak:
    l: int
    p: int
    magnitude: float


def _values(x):
    """Complex 2-D CUDA tensor for a surface / tensor / host array (host data is uploaded)."""
    v = x if isinstance(x, (np.ndarray, torch().Tensor)) else getattr(x, "values", x)
    if is_device_tensor(v):
        t = v if v.is_complex() else v.to(torch().complex128)
    else:
        a = np.asarray(v)
        t = to_device(a if np.iscomplexobj(a) else a.astype(np.complex128))
    if t.dim() != 2:
        raise ContractError("surface values must be 2-D (range bins x Doppler bins)")
    return t.contiguous()


def map_peaks(values, k: int) -> list[Peak]:
    """Top-k strict 8-neighbour local maxima of |values|, strongest first."""
    if k < 1:
        raise ContractError("find_peaks: k must be >= 1")
    if k > MAX_K:
        raise ContractError(f"find_peaks: k = {k} exceeds the device limit {MAX_K}")
    T = torch()
    require_cuda()
    v = _values(values)
    rows, cols = v.shape
    need = ctypes.c_int64()
    _native.check(_native.lib().sa_peaks_workspace_bytes(rows, cols, k, ctypes.byref(need)))
    ws = T.empty(max(1, need.value), dtype=T.uint8, device=v.device)
    idx = T.empty(k, dtype=T.int64, device=v.device)
    mag = T.empty(k, dtype=T.float64, device=v.device)
    cnt = T.empty(1, dtype=T.int32, device=v.device)
    _native.check(_native.lib().sa_map_peaks(sa_dtype_of(v), _native.ptr(v), rows, cols, k, _native.ptr(idx),
                                             _native.ptr(mag), _native.ptr(cnt), _native.ptr(ws), need.value,
                                             _native.stream_ptr()))
    n = int(cnt.item())
    ih, mh = idx[:n].cpu().numpy(), mag[:n].cpu().numpy()
    return [Peak(int(i // cols), int(i % cols), float(m)) for i, m in zip(ih, mh)]


def find_peaks(surface, k: int) -> list[Peak]:
    """detection.find_peaks (detection.py:85-108) on the GPU."""
    return map_peaks(surface, k)


def floor_maxima(values, centers: Sequence[tuple[int, int]], guard=DEFAULT_GUARD) -> tuple[float, float, int]:
    """(max |v|, max |v| outside every guard box, number of outside cells)."""
    T = torch()
    require_cuda()
    v = _values(values)
    rows, cols = v.shape
    c = T.tensor(np.asarray(list(centers), dtype=np.int32).reshape(-1, 2), device=v.device)
    out = T.empty(3, dtype=T.int64, device=v.device)
    _native.check(_native.lib().sa_map_floor(sa_dtype_of(v), _native.ptr(v), rows, cols, _native.ptr(c),
                                             c.shape[0], int(guard[0]), int(guard[1]), _native.ptr(out),
                                             _native.stream_ptr()))
    o = out.cpu().numpy()
    bits = o[:2].view(np.float64)
    return float(bits[0]), float(bits[1]), int(o[2])


def sidelobe_floor_db(values, centers: Sequence[tuple[int, int]], guard=DEFAULT_GUARD) -> float:
    """Largest magnitude outside every guard box, dB re the global peak
    (detection.py:148-171): never above 0, capped at DB_FLOOR_CAP."""
    gmax, outside, n_out = floor_maxima(values, centers, guard)
    if n_out == 0:
        raise ContractError("sidelobe_floor_db: guard regions cover the whole surface")
    if gmax <= 0.0 or outside <= 0.0:
        return DB_FLOOR_CAP
    return max(20.0 * np.log10(outside / gmax), DB_FLOOR_CAP)


def _circular_distance(a: int, b: int, n: int) -> int:
    d = abs(a - b) % n
    return min(d, n - d)


def classify_bins(values, true_bins: Sequence[tuple[int, int]], guard=DEFAULT_GUARD):
    """classify's decision (detection.py:115-134) for explicit true bins:
    returns (statuses, overall, floor_db, peaks)."""
    if guard[0] < 1 or guard[1] < 1:
        raise ContractError("classify: guard must be at least (1, 1)")
    v = _values(values)
    n = v.shape[1]
    peaks = map_peaks(v, len(true_bins))
    statuses = []
    for l0, p0 in true_bins:
        hit = any(abs(pk.l - l0) <= guard[0] and _circular_distance(pk.p, p0, n) <= guard[1] for pk in peaks)
        statuses.append("detected" if hit else "masked")
    n_det = statuses.count("detected")
    overall = "detected" if n_det == len(statuses) else ("no detection" if n_det == 0 else "partial")
    return tuple(statuses), overall, sidelobe_floor_db(v, true_bins, guard), tuple(peaks)


def ambiguity_peaks(s_surv, s_ref, l_bins: int, m: int, k: int, **map_kw) -> list[Peak]:
    """``ambiguity_map`` + ``map_peaks`` without leaving the device (rows are l0-relative)."""
    from .ambiguity import ambiguity_map
    T = torch()
    surv = getattr(s_surv, "samples", s_surv)
    ref = getattr(s_ref, "samples", s_ref)
    if not is_device_tensor(surv):
        surv = to_device(np.asarray(surv), map_kw.pop("dtype", None) or T.complex128)
    if not is_device_tensor(ref):
        ref = to_device(np.asarray(ref), surv.dtype)
    return map_peaks(ambiguity_map(surv, ref, l_bins, m, **map_kw), k)

