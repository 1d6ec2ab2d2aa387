"""Install the B200 hot path into an imported reference ``signadd`` package.

    import signadd
    from paper_1402_0532_b200 import dropin
    dropin.install(signadd)          # patches every name binding of the path

Names patched: ``signadd.{ndft, nfft, fft_exact,
lag_product_mf, lag_product_exact, ambiguity_eq11/12a/12b/12c,
compute_ambiguity}``, ``signadd.transforms.{ndft, nfft, fft_exact}``,
``signadd.ambiguity.{nfft, fft_exact, lag_product_mf, lag_product_exact,
ambiguity_eq11/12a/12b/12c, compute_ambiguity}`` (module globals looked up at
call time, ambiguity.py:39,190-221),
``signadd.detection.{compute_ambiguity, find_peaks, sidelobe_floor_db}``
(detection.py:24,85,148,187; ``classify`` looks both up at call time),
``signadd.cli.{ndft, nfft, fft_exact}`` and ``cli._TRANSFORMS`` (captured at
import, cli.py:51-71).  ``mf_complex`` is optional (``mf_complex=True``): the reference
test oracles (tests/oracles.py:10) call it and are meant to stay on the CPU.

The wrappers return the reference's own types (``Spectrum``,
``AmbiguitySurface``, ``OpCountReport``) and raise the reference's own
exception classes, so callers cannot tell the difference except by speed.
All four surface variants run on the GPU (the exact-multiply ones with numpy's
complex multiply reproduced bit-for-bit).
"""

from __future__ import annotations

import functools

from . import ambiguity as _amb
from . import operator as _op
from . import transforms as _tr
from .errors import ContractError, DomainError

_ORIG: dict = {}


def _translate(ref):
    """Decorator factory: map our exceptions to the reference's classes."""
    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*a, **kw):
            try:
                return fn(*a, **kw)
            except ContractError as e:
                raise ref.ContractError(str(e)) from None
            except DomainError as e:
                raise ref.DomainError(str(e)) from None
        return wrapper
    return deco


def _to_ref_counts(ref, r):
    return ref.OpCountReport(r.sign_ops, r.abs_ops, r.add_ops, r.complex_mf_ops, r.complex_mul_ops)


def _unwrap_signal(ref, x):
    return x.samples if isinstance(x, ref.ComplexSignal) else x


def install(ref, *, mf_complex: bool = False) -> None:
    """Patch the reference module ``ref`` (the imported ``signadd`` package)."""
    import importlib
    tmod = importlib.import_module(ref.__name__ + ".transforms")
    amod = importlib.import_module(ref.__name__ + ".ambiguity")
    dmod = importlib.import_module(ref.__name__ + ".detection")
    cmod = importlib.import_module(ref.__name__ + ".cli")
    tr = _translate(ref)

    @tr
    def ndft(x, counter=None):
        s = _tr.ndft(_unwrap_signal(ref, x), counter)
        return ref.Spectrum(s.bins, ref.TransformKind.NDFT, _to_ref_counts(ref, s.op_counts))

    @tr
    def nfft(x, counter=None):
        s = _tr.nfft(_unwrap_signal(ref, x), counter)
        return ref.Spectrum(s.bins, ref.TransformKind.NFFT, _to_ref_counts(ref, s.op_counts))

    @tr
    def fft_exact(x, counter=None):
        s = _tr.fft_exact(_unwrap_signal(ref, x), counter)
        return ref.Spectrum(s.bins, ref.TransformKind.FFT_EXACT, _to_ref_counts(ref, s.op_counts))

    @tr
    def lag_product_mf(s_surv, s_ref, l, n=None, conjugate_ref=True, counter=None):
        return _amb.lag_product_mf(_unwrap_signal(ref, s_surv), _unwrap_signal(ref, s_ref), l, n,
                                   conjugate_ref, counter)

    @tr
    def lag_product_exact(s_surv, s_ref, l, n=None, conjugate_ref=True, counter=None):
        return _amb.lag_product_exact(_unwrap_signal(ref, s_surv), _unwrap_signal(ref, s_ref), l, n,
                                      conjugate_ref, counter)

    def surface_fn(name):
        """A reference-typed surface entry point (ambiguity.py:190-221) on the GPU."""
        ours_fn = getattr(_amb, f"ambiguity_{name}")
        with_gain = name in ("eq12a", "eq12c")

        @tr
        def fn(s_surv, s_ref, l_bins, n, *args, **kw):
            # ambiguity.py:158-170 checks (sample rates) on the reference's own types
            if l_bins < 1:
                raise ContractError("l_bins must be >= 1")
            fs = None
            for sig in (s_surv, s_ref):
                if isinstance(sig, ref.ComplexSignal):
                    if fs is not None and sig.sample_rate_hz != fs:
                        raise ContractError("surveillance and reference sample rates differ")
                    fs = sig.sample_rate_hz
            if fs is None:
                raise ContractError("at least one input must be a ComplexSignal carrying a sample rate")
            ours = ours_fn(_tr.ComplexSignal(_unwrap_signal(ref, s_surv), fs),
                           _tr.ComplexSignal(_unwrap_signal(ref, s_ref), fs), l_bins, n, *args, **kw)
            return ref.AmbiguitySurface(values=ours.values, range_bin_m=ours.range_bin_m,
                                        doppler_bin_hz=ours.doppler_bin_hz,
                                        variant=ref.AmbiguityVariant(ours.variant.value), sample_rate_hz=fs,
                                        lag_op_counts=_to_ref_counts(ref, ours.lag_op_counts),
                                        transform_op_counts=_to_ref_counts(ref, ours.transform_op_counts))
        fn.__name__ = f"ambiguity_{name}"
        fn.with_gain = with_gain
        return fn

    surfaces = {name: surface_fn(name) for name in ("eq11", "eq12a", "eq12b", "eq12c")}
    ambiguity_eq12a = surfaces["eq12a"]

    def compute_ambiguity(variant, s_surv, s_ref, l_bins, n, transform_input_gain=1.0,
                          conjugate_ref=True):
        # ambiguity.py:224-239: the gain reaches only the nonlinear-FFT variants
        v = ref.AmbiguityVariant(variant).value
        if surfaces[v].with_gain:
            return surfaces[v](s_surv, s_ref, l_bins, n, transform_input_gain, conjugate_ref)
        return surfaces[v](s_surv, s_ref, l_bins, n, conjugate_ref)

    from . import detection as _det
    rmod = importlib.import_module(ref.__name__ + ".radar")

    @tr
    def find_peaks(surface, k):
        return [dmod.Peak(pk.l, pk.p, pk.magnitude) for pk in _det.find_peaks(surface, k)]

    @tr
    def sidelobe_floor_db(surface, scenario, guard=_det.DEFAULT_GUARD):
        return _det.sidelobe_floor_db(surface, rmod.true_bins(scenario), guard)

    patches = [
        (ref, "ndft", ndft), (ref, "nfft", nfft), (ref, "fft_exact", fft_exact),
        (ref, "lag_product_mf", lag_product_mf), (ref, "lag_product_exact", lag_product_exact),
        (ref, "compute_ambiguity", compute_ambiguity),
        (tmod, "ndft", ndft), (tmod, "nfft", nfft), (tmod, "fft_exact", fft_exact),
        (amod, "nfft", nfft), (amod, "fft_exact", fft_exact), (amod, "lag_product_mf", lag_product_mf),
        (amod, "lag_product_exact", lag_product_exact), (amod, "compute_ambiguity", compute_ambiguity),
        (dmod, "compute_ambiguity", compute_ambiguity),
        (dmod, "find_peaks", find_peaks), (dmod, "sidelobe_floor_db", sidelobe_floor_db),
        (cmod, "ndft", ndft), (cmod, "nfft", nfft), (cmod, "fft_exact", fft_exact),
    ]
    for name, fn in surfaces.items():
        patches += [(ref, f"ambiguity_{name}", fn), (amod, f"ambiguity_{name}", fn)]
    if mf_complex:
        patches.append((ref, "mf_complex", tr(_op.mf_complex)))
    for mod, name, fn in patches:
        _ORIG.setdefault((mod.__name__, name), getattr(mod, name))
        setattr(mod, name, fn)
    cmod._TRANSFORMS["ndft"] = ndft
    cmod._TRANSFORMS["nfft"] = nfft
    cmod._TRANSFORMS["fft"] = fft_exact


def uninstall(ref) -> None:
    """Restore the reference bindings saved by install()."""
    import importlib
    for (modname, name), fn in _ORIG.items():
        setattr(importlib.import_module(modname), name, fn)
    cmod = importlib.import_module(ref.__name__ + ".cli")
    cmod._TRANSFORMS["ndft"] = _ORIG.get((cmod.__name__, "ndft"), cmod._TRANSFORMS["ndft"])
    cmod._TRANSFORMS["nfft"] = _ORIG.get((cmod.__name__, "nfft"), cmod._TRANSFORMS["nfft"])
    cmod._TRANSFORMS["fft"] = _ORIG.get((cmod.__name__, "fft_exact"), cmod._TRANSFORMS["fft"])
    _ORIG.clear()
