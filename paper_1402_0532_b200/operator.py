"""Sign-additive product API on the B200 (mirrors operator.py:134-207).

``mf_complex`` is the elementwise ⊙ kernel (sa_mf_complex, bit-for-bit the
reference's ``_mf_complex_raw`` evaluation incl. signed zeros).  The real-valued
helpers route through the same kernel with zero imaginary parts:
(a+0j)⊙(b+0j) = (a⊗b − 0⊗0) + j(0⊗b + 0⊗a) = a⊗b exactly.
"""

from __future__ import annotations

import numpy as np

from . import _native
from ._device import check_finite_device, is_device_tensor, require_cuda, sa_dtype_of, to_device, torch
from .errors import ContractError, DomainError, OpCounter, OpCountReport

__all__ = ["ContractError", "DomainError", "OpCountReport", "OpCounter", "mf_sign", "mf_real",
           "mf_complex", "vector_product", "scalar_vector"]


def _require_finite(name: str, *values) -> None:
    # operator.py:112-115
    for v in values:
        if not np.all(np.isfinite(v)):
            raise DomainError(f"{name}: operands must be finite (no NaN/Inf)")


def _mf_device(a, b):
    """Elementwise ⊙ of two same-shape complex CUDA tensors."""
    T = torch()
    out = T.empty_like(a)
    _native.check(_native.lib().sa_mf_complex(sa_dtype_of(a), _native.ptr(a), _native.ptr(b),
                                              _native.ptr(out), a.numel(), _native.stream_ptr()))
    return out


def mf_complex(a, b, counter: OpCounter | None = None):
    """Complex sign-additive product, broadcasting (operator.py:159-176).

    Host inputs return host results (complex scalar for 0-d, else ndarray);
    CUDA tensors stay on the device.
    """
    T = torch()
    if is_device_tensor(a) or is_device_tensor(b):
        require_cuda()
        ta = a if is_device_tensor(a) else to_device(a)
        tb = b if is_device_tensor(b) else to_device(b)
        dt = T.promote_types(ta.dtype, tb.dtype)
        ta, tb = T.broadcast_tensors(ta.to(dt), tb.to(dt))
        ta, tb = ta.contiguous(), tb.contiguous()
        check_finite_device(ta)
        check_finite_device(tb)
        out = _mf_device(ta, tb)
        if counter is not None:
            counter.count_complex(out.numel())
        return out
    a = np.asarray(a, dtype=complex)
    b = np.asarray(b, dtype=complex)
    _require_finite("mf_complex", a.real, a.imag, b.real, b.imag)
    ab, bb = np.broadcast_arrays(a, b)
    shape = ab.shape
    if ab.size == 0:
        out = np.empty(shape, dtype=complex)
    else:
        da = to_device(np.ascontiguousarray(ab).reshape(-1))
        db = to_device(np.ascontiguousarray(bb).reshape(-1))
        out = _mf_device(da, db).cpu().numpy().reshape(shape)
    if counter is not None:
        counter.count_complex(np.broadcast(a, b).size)
    if out.ndim == 0:
        return complex(out)
    return out


def mf_real(a, b, counter: OpCounter | None = None):
    """sign(a*b) * (|a| + |b|) for reals (operator.py:146-156)."""
    _require_finite("mf_real", a, b)
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    out = np.real(mf_complex(a.astype(complex), b.astype(complex)))
    out = np.asarray(out, dtype=float)
    if counter is not None:
        counter.count_real(out.size)
    if out.ndim == 0:
        return float(out)
    return out


def mf_sign(a, b):
    """Three-valued sign of a*b from operand signs (operator.py:134-143)."""
    _require_finite("mf_sign", a, b)
    s = np.sign(mf_real(np.asarray(a, dtype=float), np.asarray(b, dtype=float)))
    s = np.asarray(s)
    if s.ndim == 0:
        return int(s)
    return s.astype(int)


def vector_product(x, y, counter: OpCounter | None = None) -> float:
    """Σ x_i ⊗ y_i (operator.py:179-197)."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    if x.shape != y.shape or x.ndim != 1:
        raise ContractError(
            f"vector_product: need two 1-d vectors of equal length, got shapes {x.shape} and {y.shape}")
    if x.size < 1:
        raise ContractError("vector_product: vectors must have length >= 1")
    _require_finite("vector_product", x, y)
    terms = mf_real(x, y)
    if counter is not None:
        counter.count_real(x.size)
    return float(np.sum(terms))


def scalar_vector(a, x, counter: OpCounter | None = None) -> np.ndarray:
    """a ⊗ x_i for each element (operator.py:200-207)."""
    _require_finite("scalar_vector", a, x)
    x = np.asarray(x, dtype=float)
    out = np.asarray(mf_real(float(a), x), dtype=float)
    if counter is not None:
        counter.count_real(x.size)
    return out
