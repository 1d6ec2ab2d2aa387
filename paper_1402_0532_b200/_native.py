"""ctypes binding of ``libsignadd_b200.so`` (include/signadd_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every compute call raises.  Status codes map onto the reference's
exception classes (operator.py:39-44).
"""

from __future__ import annotations

import ctypes
import os

from .errors import ContractError, DomainError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsignadd_b200.so")
if os.environ.get("SA_LIB_PATH"):  # development: time an alternative build of the library
    LIB_PATH = os.environ["SA_LIB_PATH"]

SA_C64, SA_C128 = 0, 1
SA_NDFT_FAST, SA_NDFT_EXACT, SA_NDFT_TC, SA_NDFT_TC_I8 = 0, 1, 2, 3
SA_DIT, SA_DIF, SA_FFT_EXACT = 0, 1, 2
SA_LAG_MF, SA_LAG_EXACT = 0, 1
SA_DOPPLER_NLFFT, SA_DOPPLER_NDFT, SA_DOPPLER_FFT_EXACT = 0, 1, 2
SA_NOISE_NONE, SA_NOISE_AWGN, SA_NOISE_EPS = 0, 1, 2

SA_OK, SA_ERR_ARG, SA_ERR_CONTRACT, SA_ERR_DOMAIN, SA_ERR_CUDA, SA_ERR_UNSUPPORTED = 0, -1, -2, -3, -4, -5

# every symbol include/signadd_b200.h declares: (name, restype, argtypes)
_P, _I64, _I, _D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
SIGNATURES = {
    "sa_version": (_I, []),
    "sa_last_error": (ctypes.c_char_p, []),
    "sa_twiddle_create": (_I, [_I, _I, _I64, _P, _P, ctypes.POINTER(_P)]),
    "sa_twiddle_destroy": (_I, [_P]),
    "sa_mf_complex": (_I, [_I, _P, _P, _P, _I64, _P]),
    "sa_check_finite": (_I, [_I, _P, _I64, _P, _P]),
    "sa_ndft": (_I, [_I, _P, _P, _I64, _I64, _P, _I, _D, _P]),
    "sa_nlfft": (_I, [_I, _I, _P, _P, _I64, _I64, _P, _D, _P]),
    "sa_lag_product_mf": (_I, [_I, _P, _P, _I64, _I64, _I64, _I, _P, _P]),
    "sa_ambiguity_workspace_bytes": (_I, [_I, _I64, _I64, ctypes.POINTER(_I64)]),
    "sa_ambiguity_map": (_I, [_I, _P, _P, _I64, _I64, _I64, _I64, _I64, _D, _I, _I, _I, _P, _P,
                             _P, _I64, _P]),
    "sa_ambiguity_integrate": (_I, [_I, _P, _P, _I64, _I64, _I64, _I64, _I64, _I, _I, _P, _P]),
    "sa_lag_product_exact": (_I, [_I, _P, _P, _I64, _I64, _I64, _I, _P, _P]),
    "sa_ambiguity_map_v": (_I, [_I, _I, _P, _P, _I64, _I64, _I64, _I64, _I64, ctypes.c_double, _I, _I, _I, _P,
                                _P, _P, _I64, _P]),
    "sa_ambiguity_integrate_v": (_I, [_I, _I, _P, _P, _I64, _I64, _I64, _I64, _I64, _I, _I, _P, _P]),
    "sa_ambiguity_integrate_blocks": (_I, [_I, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I, _P, _I64, _P]),
    "sa_doppler_nlfft_blocked": (_I, [_I, _P, _P, _I64, _I64, _P, ctypes.c_double, _P]),
    "sa_format_surface_csv": (_I, [_P, _I64, _I64, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                   ctypes.POINTER(ctypes.c_int64), _I]),
    "sa_format_float_repr": (_I, [ctypes.c_double, ctypes.c_char_p, _I]),
    "sa_free_host": (None, [_P]),
    "sa_peaks_workspace_bytes": (_I, [_I64, _I64, _I, ctypes.POINTER(_I64)]),
    "sa_map_peaks": (_I, [_I, _P, _I64, _I64, _I, _P, _P, _P, _P, _I64, _P]),
    "sa_map_floor": (_I, [_I, _P, _I64, _I64, _P, _I, _I, _I, _P, _P]),
    "sa_ambiguity_map_multi": (_I, [_I, _P, _I, _I, _P, _P, _I64, _I64, _I64, _I64, _I64, ctypes.c_double, _I, _I,
                                    _I, _P, _P, _P, _P, _P]),
    "sa_enable_peer_access": (_I, [_I]),
    "sa_lag_kernel": (_I, [_I]),
    "sa_ipc_open": (_I, [_P, ctypes.POINTER(_P)]),
    "sa_ipc_close": (_I, [_P]),
    "sa_scene_stereo_fm": (_I, [_I, _P, _I64, _D, _D, _D, _D, _D, _P, _P]),
    "sa_scene_echoes": (_I, [_P, _I64, _I, _P, _P, _P, _D, _P, _P]),
    "sa_scene_power_workspace_bytes": (_I, [_I64, ctypes.POINTER(_I64)]),
    "sa_scene_power": (_I, [_P, _I64, _P, _P, _I64, _P]),
    "sa_scene_noise_gain": (_I, [_I, _P, _I64, _I, _P, _P, _D, _D, _D, _D, _D, _P, _P]),
    "sa_fma_peak": (_I, [_I, _I64, _P, _I, _P]),
}

_lib = None


class NativeMissing(ImportError):
    """libsignadd_b200.so is not built (run __graft_entry__.build())."""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeMissing(f"{LIB_PATH} not found: build the CUDA library first (python -c "
                            "'import __graft_entry__ as g; g.build()')")
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.sa_version() != 1:
        raise NativeMissing(f"ABI version mismatch: {L.sa_version()}")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == SA_OK:
        return
    msg = (lib().sa_last_error() or b"").decode(errors="replace")
    if rc == SA_ERR_CONTRACT:
        raise ContractError(msg)
    if rc == SA_ERR_DOMAIN:
        raise DomainError(msg)
    raise RuntimeError(f"signadd_b200 native error {rc}: {msg}")


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None) -> ctypes.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
