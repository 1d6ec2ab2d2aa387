"""The UNMODIFIED numpy reference (signadd 0.1.0 from baseline/_ref) timed on the
host cores, as BASELINE.md §3 asks: ``multiprocessing.Pool(P)`` with
P = len(os.sched_getaffinity(0)), BLAS/OMP threads 1, a fixed deterministic
sample per worker, the measured RATE reported (not extrapolated wall time),
plus a 1-core figure and the CPU model string.

bench.py attaches the result to each workload's ``cpu_baseline`` as
``reference_numpy``.  It is a reported baseline next to the oracle C port
(``kind: port``), never a checker and never on the product path.

Work per task (reference call sites):
  ndft rows   -> signadd.ndft(row)                  (transforms.py:223-251)
  nfft rows   -> signadd.nfft(row)                  (transforms.py:254-298)
  map rows    -> lag_product_mf(r, s, l, n=Ns)      (ambiguity.py:146-155)
                 -> T-sample block sums -> nfft(z)   (SURVEY §8(d) composition, gain 1.0)
Inputs are handed to the workers as .npy files memory-mapped read-only.
"""

from __future__ import annotations

import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

_G: dict = {}


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "signadd"))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _init(paths):
    for k in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[k] = "1"
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import signadd  # noqa: F401  (the unmodified reference)
    _G["signadd"] = signadd
    _G["arrays"] = {k: np.load(p, mmap_mode="r") for k, p in paths.items()}


def _task(spec):
    """One worker task; returns (⊙ count by the reference's own formulas, seconds)."""
    sg = _G["signadd"]
    a = _G["arrays"]
    kind = spec[0]
    t = time.perf_counter()
    if kind == "ndft":
        rows = a["x"][spec[1]:spec[2]]
        ops = 0
        for r in rows:
            sg.ndft(np.array(r))
            ops += r.size * r.size
    elif kind == "nfft":
        rows = a["x"][spec[1]:spec[2]]
        ops = 0
        for r in rows:
            sg.nfft(np.array(r))
            n = r.size
            ops += n * (n.bit_length())  # N (log2 N + 1)
    else:  # map rows
        _, lags, m = spec
        surv, ref = np.array(a["surv"]), np.array(a["ref"])
        ns = surv.size
        ops = 0
        for l in lags:
            y = sg.lag_product_mf(surv, ref, int(l), n=ns)
            z = y.reshape(m, -1).sum(axis=1)
            sg.nfft(1.0 * z)
            ops += ns + m * (m.bit_length())
    return ops, time.perf_counter() - t


def measure(kind: str, arrays: dict, tasks_per_worker, P: int | None = None) -> dict:
    """Run ``tasks_per_worker(P)`` (a list of task specs) on Pool(P) and on one core.

    Returns {"value", "unit", "cores", "one_core_value", "cpu_model", "sample", ...}
    or {"unavailable": why}."""
    if not available():
        return {"unavailable": "baseline/_ref not installed (tools/install_ref.sh)"}
    import multiprocessing as mp
    P = P or len(os.sched_getaffinity(0))
    tmp = tempfile.mkdtemp(prefix="refcpu")
    paths = {}
    for k, v in arrays.items():
        paths[k] = os.path.join(tmp, k + ".npy")
        np.save(paths[k], np.ascontiguousarray(v).astype(np.complex128))  # the reference is complex128-only
    env_pp = os.environ.get("PYTHONPATH", "")
    os.environ["PYTHONPATH"] = os.pathsep.join([ROOT, env_pp]) if env_pp else ROOT
    ctx = mp.get_context("spawn")  # the parent holds a CUDA context: never fork it
    try:
        tasks = tasks_per_worker(P)
        with ctx.Pool(1, initializer=_init, initargs=(paths,)) as p1:
            p1.apply(_task, (tasks[0],))  # warm (imports, page-in)
            o1, s1 = p1.apply(_task, (tasks[0],))
        with ctx.Pool(P, initializer=_init, initargs=(paths,)) as pool:
            pool.map(_task, tasks[:P], chunksize=1)  # warm every worker
            t = time.perf_counter()
            res = pool.map(_task, tasks, chunksize=1)
            wall = time.perf_counter() - t
    finally:
        os.environ["PYTHONPATH"] = env_pp
        for p in paths.values():
            os.unlink(p)
        os.rmdir(tmp)
    ops = sum(r[0] for r in res)
    unit = "cells/s" if kind == "map" else "⊙/s"
    out = {"value": ops / wall, "unit": "⊙/s", "cores": P, "one_core_value": o1 / s1,
           "cpu_model": cpu_model(), "kind": "reference (unmodified numpy, baseline/_ref)",
           "tasks": len(tasks), "wall_s": round(wall, 3),
           "threads_env": "OMP/MKL/OPENBLAS_NUM_THREADS=1", "pool": f"multiprocessing spawn Pool({P})"}
    if kind == "map":
        cells = sum(len(t[1]) * t[2] for t in tasks)
        out["cells_per_s"] = cells / wall
        out["one_core_cells_per_s"] = len(tasks[0][1]) * tasks[0][2] / s1
        out["unit_note"] = f"value in ⊙/s (lag + Doppler counts); {unit} alongside"
    return out
