"""Host twiddle tables and their device-resident copies.

``TwiddleTable`` restates transforms.py:115-133: entries exp(-2j*pi*m/N) from
``np.cos/np.sin`` of ``(-2*pi)*m/N`` with quarter-turn entries forced exact.
The GPU consumes exactly this host table (uploaded once per (device, N,
dtype)); device ``sincos`` is never used because ⊙ is discontinuous at 0 and a
1-ulp twiddle difference can flip a sign decision (SURVEY §7 hard part 1).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from .errors import ContractError

__all__ = ["TwiddleTable", "twiddle_table", "device_twiddles"]


class TwiddleTable:
    """Precomputed roots of unity ``exp(-2j*pi*m/N)`` for m = 0..N-1."""

    _QUADRANT = (complex(1.0, 0.0), complex(0.0, -1.0), complex(-1.0, 0.0), complex(0.0, 1.0))

    def __init__(self, n: int):
        if n < 1:
            raise ContractError("TwiddleTable: size must be >= 1")
        m = np.arange(n)
        ang = (-2.0 * np.pi) * m / n
        entries = np.cos(ang) + 1j * np.sin(ang)
        quad, rem = np.divmod(4 * m, n)
        exact = rem == 0
        entries[exact] = np.asarray(self._QUADRANT)[quad[exact] % 4]
        self.n = n
        self.entries = entries
        self.entries.setflags(write=False)


_TABLE_CACHE: dict[int, TwiddleTable] = {}


def twiddle_table(n: int) -> TwiddleTable:
    tbl = _TABLE_CACHE.get(n)
    if tbl is None:
        tbl = TwiddleTable(n)
        if len(_TABLE_CACHE) > 32:
            _TABLE_CACHE.clear()
        _TABLE_CACHE[n] = tbl
    return tbl


_DEV_CACHE: dict[tuple[int, int, int], int] = {}
_DEV_LOCK = threading.Lock()


def device_twiddles(n: int, sa_dtype: int, device: int) -> int:
    """Opaque handle of the device twiddle set for (device, n, dtype), cached."""
    from . import _native
    key = (device, n, sa_dtype)
    h = _DEV_CACHE.get(key)
    if h is not None:
        return h
    with _DEV_LOCK:
        h = _DEV_CACHE.get(key)
        if h is not None:
            return h
        import torch
        tab = np.ascontiguousarray(twiddle_table(n).entries, dtype=np.complex128)
        out = ctypes.c_void_p()
        with torch.cuda.device(device):
            stream = _native.stream_ptr()
            _native.check(_native.lib().sa_twiddle_create(
                device, sa_dtype, n, tab.ctypes.data_as(ctypes.c_void_p), stream, ctypes.byref(out)))
        _DEV_CACHE[key] = out.value
        return out.value
