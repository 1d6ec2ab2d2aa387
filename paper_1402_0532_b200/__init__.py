"""paper_1402_0532_b200 -- B200-native hot path of signadd (arXiv 1402.0532).

The sign-additive operator a⊗b = sign(a·b)(|a|+|b|), its complex extension, and
the three things built on it -- the N²-point NDFT, the radix-2 NL-FFT (DIT and
DIF) and the ⊙ passive-radar range-Doppler map -- as hand-written sm_100a CUDA
kernels behind a C ABI (include/signadd_b200.h), exposed through the reference
package's own Python entry points (drop-in) plus batched device APIs.

There is no CPU fallback: without libsignadd_b200.so or a CUDA device every
compute call raises.
"""

__version__ = "0.1.0"

from .errors import ContractError, DomainError, OpCounter, OpCountReport
from .operator import mf_complex, mf_real, mf_sign, scalar_vector, vector_product
from .twiddle import TwiddleTable, twiddle_table
from .transforms import (
    ComplexSignal,
    Spectrum,
    TransformKind,
    fft_exact,
    fft_exact_complex_muls,
    ndft,
    ndft_batch,
    ndft_complex_ops,
    nfft,
    nfft_batch,
    nfft_butterflies,
    nfft_complex_ops,
    nfft_dif_complex_ops,
    peak_index,
    unit_tone,
)
from .ambiguity import (
    SPEED_OF_LIGHT,
    AmbiguitySurface,
    AmbiguityVariant,
    MapGraph,
    ambiguity_eq11,
    ambiguity_eq12a,
    ambiguity_eq12b,
    ambiguity_eq12c,
    ambiguity_map,
    compute_ambiguity,
    lag_product_exact,
    lag_product_mf,
    map_complex_ops,
)
from . import scene
from .detection import Peak, ambiguity_peaks, classify_bins, find_peaks, map_peaks, sidelobe_floor_db


def require_native():
    """Load libsignadd_b200.so and check a CUDA device is present (raises otherwise)."""
    from ._device import require_cuda
    require_cuda()
    from . import _native
    return _native.lib()


__all__ = [name for name in dir() if not name.startswith("_")]
