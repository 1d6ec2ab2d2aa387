"""CSV / manifest writers of the reference CLI for CPI-scale maps.

The reference writes an ambiguity run as a JSON manifest plus three CSVs
(cli.py:74-116 ``_write_csv`` / ``_write_manifest``, cli.py:173-209
``_cmd_ambiguity``): the surface in dB, one ``l,p,magnitude_db`` row per cell,
floats as Python ``repr()``, and the range / Doppler cuts.  For a 4096 x 2048
map the surface file is 8.4 M rows, and the per-row Python csv/repr loop takes
~10 s.  Here the dB map is formed exactly as ``AmbiguitySurface.magnitude_db``
does (numpy on the host: the reference's own arithmetic), and the surface rows
are formatted by ``sa_format_surface_csv`` in parallel host threads with the
shortest round-trip digits laid out as repr() -- the file is byte-identical
(tests/test_writers.py).  The cuts and the manifest are small and are written
with the same Python code paths as the reference.
"""

from __future__ import annotations

import csv
import ctypes
import hashlib
import io
import json
import os
from datetime import datetime, timezone

import numpy as np

from . import _native


def format_float_repr(x: float) -> str:
    """repr(float(x)) from the native formatter (test hook)."""
    buf = ctypes.create_string_buffer(64)
    n = _native.lib().sa_format_float_repr(float(x), buf, 64)
    if n < 0:
        _native.check(n)
    return buf.raw[:n].decode()


def magnitude_db(values, floor_db: float = -300.0) -> np.ndarray:
    """AmbiguitySurface.magnitude_db (ambiguity.py:92-99) on a host copy of the map."""
    if not isinstance(values, np.ndarray):
        values = values.detach().cpu().numpy()
    mag = np.abs(np.asarray(values, dtype=complex))
    peak = mag.max()
    if peak <= 0.0:
        return np.full(mag.shape, floor_db)
    with np.errstate(divide="ignore"):
        db = 20.0 * np.log10(mag / peak)
    return np.maximum(db, floor_db)


def surface_csv_bytes(db: np.ndarray, manifest_name: str, nthreads: int = 0) -> bytes:
    """The reference's surface CSV (cli.py:184-191) for a dB map, byte for byte."""
    db = np.ascontiguousarray(db, dtype=np.float64)
    if db.ndim != 2:
        raise ValueError("db must be a 2-d (l_bins x n) array")
    out = ctypes.c_void_p()
    n = ctypes.c_int64()
    _native.check(_native.lib().sa_format_surface_csv(
        db.ctypes.data_as(ctypes.c_void_p), db.shape[0], db.shape[1], manifest_name.encode(), ctypes.byref(out),
        ctypes.byref(n), int(nthreads)))
    try:
        return ctypes.string_at(out.value, n.value)
    finally:
        _native.lib().sa_free_host(out)


def _atomic_write(path: str, data: bytes) -> None:
    # cli.py:74-81
    tmp = path + ".tmp"
    try:
        with open(tmp, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.remove(tmp)
        raise


def _small_csv(path: str, header, rows, manifest_name: str) -> None:
    # cli.py:83-90, for the short cut files
    buf = io.StringIO()
    buf.write(f"# manifest={manifest_name}\n")
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(header)
    for row in rows:
        w.writerow([repr(float(v)) if isinstance(v, float) else v for v in row])
    _atomic_write(path, buf.getvalue().encode())


def write_manifest(prefix: str, command: str, args_desc: dict, counts=None, tool: str = "signadd 0.1.0") -> str:
    """cli.py:93-116: <prefix>.manifest.json; returns its basename."""
    path = prefix + ".manifest.json"
    doc = {"tool": tool, "created_utc": datetime.now(timezone.utc).isoformat(), "command": command,
           "args": args_desc,
           "args_sha256": hashlib.sha256(json.dumps(args_desc, sort_keys=True).encode()).hexdigest()}
    if counts is not None:
        doc["op_counts"] = {k: getattr(counts, k) for k in
                            ("sign_ops", "abs_ops", "add_ops", "complex_mf_ops", "complex_mul_ops")}
    _atomic_write(path, (json.dumps(doc, indent=2, sort_keys=True) + "\n").encode())
    return os.path.basename(path)


def write_ambiguity_outputs(prefix: str, surface, args_desc: dict, floor_db: float = -300.0,
                            nthreads: int = 0) -> dict:
    """The output set of ``signadd ambiguity`` (cli.py:173-209) for a surface
    (ours or the reference's AmbiguitySurface; ``values`` may live on the GPU):
    manifest, surface / range-cut / Doppler-cut CSVs.  Returns the paths."""
    counts = getattr(surface, "op_counts", None)
    manifest = write_manifest(prefix, "ambiguity", args_desc, counts)
    db = magnitude_db(surface.values, floor_db)
    _atomic_write(prefix + ".surface.csv", surface_csv_bytes(db, manifest, nthreads))
    lb, n = db.shape
    # AmbiguitySurface.range_cut / doppler_cut (ambiguity.py:101-113)
    ls = np.arange(lb)
    row_db = db.max(axis=1)
    range_km = ls * surface.range_bin_m / 1000.0
    _small_csv(prefix + ".range_cut.csv", ["l", "bistatic_range_km", "magnitude_db"],
               [(int(l), float(r), float(v)) for l, r, v in zip(ls, range_km, row_db)], manifest)
    p = np.arange(n)
    freq = np.where(p <= n // 2, p, p - n) * surface.doppler_bin_hz
    order = np.argsort(freq, kind="stable")
    col_db = db.max(axis=0)
    _small_csv(prefix + ".doppler_cut.csv", ["doppler_hz", "magnitude_db"],
               [(float(f), float(v)) for f, v in zip(freq[order], col_db[order])], manifest)
    return {k: prefix + s for k, s in (("manifest", ".manifest.json"), ("surface", ".surface.csv"),
                                      ("range_cut", ".range_cut.csv"), ("doppler_cut", ".doppler_cut.csv"))}
