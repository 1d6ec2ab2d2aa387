"""Parity metrics.

literal: per output vector, max_k |Δ_k| / ||y_ref||_1   (the north-star tolerance;
         fp64 <= 1e-9, fp32 <= 1e-4; exact zero required when ||y_ref||_1 == 0)
strict:  per output vector, ||Δ||_1 / ||y_ref||_1        (reported, distribution)
"""

import numpy as np

TOL_F64 = 1e-9
TOL_F32 = 1e-4


def _2d(a):
    a = np.asarray(a)
    return a.reshape(1, -1) if a.ndim == 1 else a.reshape(-1, a.shape[-1])


def literal(y, ref):
    y, ref = _2d(y).astype(np.complex128), _2d(ref).astype(np.complex128)
    l1 = np.sum(np.abs(ref), axis=1)
    d = np.max(np.abs(y - ref), axis=1)
    out = np.where(l1 > 0, d / np.where(l1 > 0, l1, 1.0), np.where(d == 0, 0.0, np.inf))
    return out


def strict(y, ref):
    y, ref = _2d(y).astype(np.complex128), _2d(ref).astype(np.complex128)
    l1 = np.sum(np.abs(ref), axis=1)
    d = np.sum(np.abs(y - ref), axis=1)
    return np.where(l1 > 0, d / np.where(l1 > 0, l1, 1.0), np.where(d == 0, 0.0, np.inf))


def assert_literal(y, ref, tol):
    e = literal(y, ref)
    worst = int(np.argmax(e))
    assert np.all(e <= tol), f"literal error {e[worst]:.3e} > {tol} at vector {worst} (of {e.size})"
    return e


def assert_value_equal(y, ref):
    y, ref = np.asarray(y), np.asarray(ref)
    assert y.shape == ref.shape, (y.shape, ref.shape)
    bad = np.flatnonzero(~(y == ref))
    assert bad.size == 0, f"{bad.size}/{y.size} values differ; first {bad[:4]}: {y.ravel()[bad[:2]]} vs {ref.ravel()[bad[:2]]}"
