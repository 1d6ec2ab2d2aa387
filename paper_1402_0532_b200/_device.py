"""Device plumbing: tensor conversion, dtype mapping, host<->device staging.

PyTorch is used only for device memory, streams and copies; all arithmetic on
the hot path runs in libsignadd_b200.so.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ContractError, DomainError


def torch():
    import torch as _t
    return _t


def require_cuda() -> None:
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_1402_0532_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _native.lib()


def sa_dtype_of(t) -> int:
    T = torch()
    if t.dtype == T.complex64:
        return _native.SA_C64
    if t.dtype == T.complex128:
        return _native.SA_C128
    raise ContractError(f"expected complex64 or complex128, got {t.dtype}")


def is_device_tensor(x) -> bool:
    T = torch()
    return isinstance(x, T.Tensor) and x.is_cuda


def to_device(x, complex_dtype=None):
    """Host array/list/tensor -> contiguous complex CUDA tensor (copy)."""
    T = torch()
    require_cuda()
    if isinstance(x, T.Tensor):
        t = x
        if not t.is_complex():
            t = t.to(T.complex128)
    else:
        a = np.asarray(x)
        if not np.iscomplexobj(a):
            a = a.astype(np.complex128)
        t = T.from_numpy(np.ascontiguousarray(a))
    if complex_dtype is not None and t.dtype != complex_dtype:
        t = t.to(complex_dtype)
    return t.to("cuda", non_blocking=True).contiguous()


def check_finite_device(t) -> None:
    """Raise DomainError if a complex CUDA tensor holds NaN/Inf (one sync)."""
    T = torch()
    flag = T.zeros(1, dtype=T.int32, device=t.device)
    _native.check(_native.lib().sa_check_finite(sa_dtype_of(t), _native.ptr(t), t.numel(),
                                                _native.ptr(flag), _native.stream_ptr()))
    if int(flag.item()):
        raise DomainError("transform input must be finite")
