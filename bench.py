"""bench.py -- driver contract benchmark for the B200 ⊙ hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload ndft|nlfft|map|map5]
                    [--impl ours|reference] [--dtype c64|c128] [--no-extras]

Headline (N=1): BASELINE.json configs[1] = C2, batched NDFT N=1024 x 65536
vectors, complex64, fast (regrouped) mode.  One step = one pass of the NDFT over
the whole batch (512 MiB in, 512 MiB out: larger than the 126 MB L2, so no flush
is needed between steps).  value = complex ⊙-ops/s (reference count B*N^2,
transforms.py:247) summed over ranks; ms_per_step is the max over ranks.

Extras (N=1, rank 0): C3 NL-FFT 2^16 x 4096 (DIT and DIF) and C4 ⊙ map
(1024 x 512 from 2^20) with their own rooflines, reported under "workloads".

N>1 (torchrun, one process per GPU, NCCL): NDFT is weak-scaled (each rank its
own C2 batch, no collective).  --workload map5 runs C5 (4096 x 2048 from 2^22)
strong-scaled: delay bins sharded contiguously, map gathered to rank 0 with
NCCL inside the timed region.

--impl reference: the reference's CPU algorithm (oracle/ C port, all host
threads) on the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "complex ⊙-ops/s (NDFT, NL-FFT); range-Doppler cells/s at 1/2/4/8 B200"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(prefix="clk", suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "-i", str(self.dev),
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except Exception as e:  # pragma: no cover
            log("clock sampler unavailable:", e)
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["sampler_unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        rows = []
        for line in open(self.path):
            p = [s.strip() for s in line.split(",")]
            if len(p) < 9:
                continue
            try:
                rows.append((float(p[1]), float(p[2]), float(p[3]), p[5], p[6], p[7], p[8]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no_samples"]}
        maxclk = max(r[1] for r in rows)
        pmax = max(r[2] for r in rows)
        load = [r for r in rows if r[2] >= 0.5 * pmax] or rows
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in load:
            for nm, v in zip(names, r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": maxclk,
                "power_w_max": pmax, "samples": len(rows), "reasons": sorted(reasons)}


# --------------------------------------------------------------------------- dist
def dist_init(backend="nccl", share_gpu=False):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if share_gpu:  # test mode: every rank on cuda:0 (NCCL refuses duplicate GPUs: gloo)
        local = 0
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, v: float) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(fn, steps, warmup, ws, sampler=None, flush=None):
    """W untimed steps, then K steps between barrier+sync; CUDA events on the
    launching stream (``flush`` makes it wait for any side stream the steps use
    before the end event); returns (ms_per_step max over ranks, clocks)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(ws)
    if sampler:
        sampler.start()
    torch.cuda.synchronize()
    barrier(ws)
    s = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        fn()
    if flush:
        flush()
    e1.record(s)
    torch.cuda.synchronize()
    barrier(ws)
    ms = e0.elapsed_time(e1) / steps
    clocks = sampler.stop() if sampler else None
    return max_over_ranks(ws, ms), clocks


# --------------------------------------------------------------------------- peaks
def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


def fma_peak_tflops(dtype: str) -> float:
    """Measured FMA-pipe peak in TFLOP/s, live on this GPU: fp32 = max of scalar
    FFMA and packed FFMA2 (the kernels issue FFMA2), fp64 = DFMA."""
    if dtype == "c64":
        return max(_fma_peak(0), _fma_peak(2))
    return _fma_peak(1)


def _fma_peak(code: int) -> float:
    import ctypes
    import torch
    from paper_1402_0532_b200 import _native
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks = sms * 8
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    d = code
    lanes = 2 if code == 2 else 1
    iters = 1024 if code == 1 else 4096
    best = 0.0
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(_native.lib().sa_fma_peak(d, iters, _native.ptr(sink), blocks, _native.stream_ptr()))
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        fmas = blocks * 256 * iters * 16 * 8 * lanes
        best = max(best, 2 * fmas / t / 1e12)
    return best


# --------------------------------------------------------------------------- workloads
def complex_dtype(name):
    import torch
    return torch.complex64 if name == "c64" else torch.complex128


def wl_ndft(args, ws, rank, mode=None, e2e=True, dtype=None):
    """C2: batched NDFT N=1024 x 65536.  mode "tc" (complex64 default): the
    fast-mode sum as a sign-split bf16 GEMM on tcgen05 (sa_ndft_tc.cu); "fast":
    the FFMA2 / DFMA CUDA-core kernel (sa_ndft.cu)."""
    import torch
    import paper_1402_0532_b200 as sa
    from paper_1402_0532_b200.workloads import c2_ndft
    n, batch = 1024, 65536
    dtype = dtype or args.dtype
    cdt = complex_dtype(dtype)
    mode = mode or (args.ndft_mode if dtype == "c64" else "fast")
    t0 = time.time()
    xh = torch.from_numpy(c2_ndft(n, batch)).to(cdt)
    log(f"[rank {rank}] C2 input generated in {time.time() - t0:.1f}s")
    xd = xh.cuda()
    yd = torch.empty_like(xd)
    ops = batch * n * n
    step = lambda: sa.ndft_batch(xd, out=yd, mode=mode)  # noqa: E731
    desc = {"tc": "tc (fast-mode sum as a sign-split GEMM on tcgen05 tensor cores: bf16x2-split operands, "
                  "fp32 accumulate)",
            "tc8": "tc8 (fast-mode sum as a sign-split GEMM on tcgen05 kind::i8: exact int8 digit pairs of Wv "
                   "and of x / 2^e_v, exact int32 accumulation, fp32 epilogue)",
            "fast": "fast (sign-split regrouped accumulation, " + ("FFMA2)" if dtype == "c64" else "DFMA)")}[mode]
    res = {"ops": ops, "step": step, "launches_per_step": 1,
           "config": {"workload": "C2 batched NDFT (BASELINE.json configs[1])", "n": n,
                      "batch": batch, "mode": desc,
                      "dtype": "complex64" if dtype == "c64" else "complex128",
                      "l2_policy": f"inputs ({2 * n * batch * xh.element_size() >> 21} MiB in + out) larger "
                                   "than L2; no flush",
                      "parallelism": f"dp{ws} (independent vectors, weak scaling)"}}
    if e2e and not args.no_e2e:
        hin = xh.pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        res["e2e_step"] = lambda: sa.ndft_batch(hin, out=hout, mode=mode)
        res["e2e_rows"], res["e2e_row_bytes"] = hin.shape[0], hin.shape[1] * hin.element_size()
        res["h2d"] = hin.numel() * hin.element_size()
        res["d2h"] = hout.numel() * hout.element_size()
        res["e2e_api"] = f"paper_1402_0532_b200.ndft_batch(pinned host tensor, out=pinned host tensor, mode={mode!r})"
        res["e2e_launches"] = len(_pipeline_plan(res["e2e_rows"], res["e2e_row_bytes"]))
    if mode == "tc8" and dtype == "c64":
        res["roofline"] = lambda ms: roof_i8(ops * 32 / (ms * 1e-3) / 1e12, "c64")
        res["dtype"] = "int8 digits x sign, exact int32 accumulate, f32 epilogue"
    elif mode == "tc" and dtype == "c128":
        res["roofline"] = lambda ms: roof_i8(ops * 64 / (ms * 1e-3) / 1e12)
        res["dtype"] = "int8 digits x sign, exact int32 accumulate, f64 epilogue"
        res["config"]["mode"] = ("tc (complex128: Ozaki-style int8 digits of Wv and of x / 2^e_v on tcgen05 kind::i8, "
                                 "exact int32 accumulation, fp64 epilogue; max|d|/|y|1 ~1.5e-10)")
    elif mode == "tc":
        res["roofline"] = lambda ms: roof_tensor(ops * 32 / (ms * 1e-3) / 1e12)
        res["dtype"] = "bf16x2-split x sign, f32 accumulate"
    else:
        res["roofline"] = lambda ms: roof_alu(dtype, ops * 16 / (ms * 1e-3) / 1e12, "ndft")
        res["dtype"] = "f32" if dtype == "c64" else "f64"
    res["cpu"] = lambda P: cpu_ndft(xh.numpy(), P)
    res["cpu_numpy"] = lambda P: numpy_ref_rows("ndft", xh.numpy(), P, per_task=2, tasks_per_worker=4)
    return res


def wl_ndft64(args):
    """C1: NDFT N=64 complex128, the exact-grid tone exp(j2π·7n/64) + 4096 CN(0,1)
    vectors (BASELINE.json configs[0]); fast mode (DFMA kernel).  Launch-bound at
    this size: reported, not a roofline target."""
    import torch
    import paper_1402_0532_b200 as sa
    from paper_1402_0532_b200.workloads import c1_ndft64
    xh = torch.from_numpy(c1_ndft64())
    xd = xh.cuda()
    yd = torch.empty_like(xd)
    b, n = xd.shape
    ops = b * n * n
    res = {"ops": ops, "step": lambda: sa.ndft_batch(xd, out=yd, mode="fast"), "launches_per_step": 1,
           "config": {"workload": "C1 NDFT N=64 (BASELINE.json configs[0])", "n": n, "batch": b,
                      "dtype": "complex128", "mode": "fast (DFMA)", "rows": "row 0 = unit_tone(7, 64), then 4096 CN(0,1)"},
           "dtype": "f64"}
    res["roofline"] = lambda ms: roof_alu("c128", ops * 16 / (ms * 1e-3) / 1e12, "ndft")
    res["cpu"] = lambda P: cpu_ndft(xh.numpy(), P, rows=b)
    res["cpu_numpy"] = lambda P: numpy_ref_rows("ndft", xh.numpy(), P, per_task=max(1, b // (4 * P)),
                                                tasks_per_worker=4, all_rows=True)
    hin = xh.pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    res["e2e_step"] = lambda: sa.ndft_batch(hin, out=hout, mode="fast")
    res["h2d"] = res["d2h"] = hin.numel() * hin.element_size()
    res["e2e_api"] = "paper_1402_0532_b200.ndft_batch(pinned host tensor, out=pinned host tensor, mode='fast')"
    res["e2e_launches"] = len(_pipeline_plan(b, n * 16))
    return res


def _pipeline_plan(rows, row_bytes):
    from paper_1402_0532_b200.transforms import pipeline_plan
    return pipeline_plan(rows, row_bytes, 128)


def roof_tensor(achieved_tflops):
    """tcgen05 NDFT against the measured dense bf16 peak (MEASURED_PEAKS.json,
    burst figure: one C2 step is a ~2 ms kernel timed alone)."""
    peaks, src = measured_peaks()
    peak = peaks.get("bf16_tflops", 1590.0)
    tr = ncu_traffic("k_ndft_tc")
    return {"bound": "tensor", "achieved": round(achieved_tflops, 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved_tflops / peak, 4),
            "traffic": tr["bytes_per_launch"] if tr else None, "traffic_unit": "bytes/launch",
            "traffic_source": tr["source"] if tr else None,
            "algorithmic_bytes": 2 * 65536 * 1024 * 8, "kernel": "k_ndft_tc",
            "peak_source": f"{src} bf16_tflops (burst, cuBLAS 8192^3; sustained {peaks.get('bf16_tflops_sustained')})",
            "nominal_peak": 2250.0, "frac_nominal": round(achieved_tflops / 2250.0, 4),
            "algorithmic": "32 bf16 tensor flop per complex ⊙: re/im outputs x re/im inputs x "
                           "{sgn(x)·W0, sgn(x)·W1, X0·sgn(W), X1·sgn(W)} MACs (two-term bf16 splits)",
            **({"ncu_utilisation_pct": tr["ncu"]} if tr and tr.get("ncu") else {})}


def roof_i8(achieved_tops, dtype="c128"):
    """NDFT on tcgen05 kind::i8 (sa_ndft_i8.cu): complex128 8 int8 MMA terms x 4 MACs
    = 64 int ops per complex ⊙ (complex64: 4 terms, 32 ops), against the dense int8
    tensor rate (2 x the measured bf16 burst figure: B200 int8 runs at twice bf16;
    MEASURED_PEAKS has no int8 line).  Achieved is over the whole step (the digit
    prep kernel included)."""
    peaks, src = measured_peaks()
    peak = 2.0 * peaks.get("bf16_tflops", 1590.0)
    tr = ncu_traffic("k_ndft_i8<2" if dtype == "c128" else "k_ndft_i8<1")
    terms, per = (8, 64) if dtype == "c128" else (4, 32)
    return {"bound": "tensor", "achieved": round(achieved_tops, 1), "peak": round(peak, 1), "unit": "TOP/s",
            "frac": round(achieved_tops / peak, 4), "traffic": tr["bytes_per_launch"] if tr else None,
            "traffic_unit": "bytes/launch", "traffic_source": tr["source"] if tr else None,
            "kernel": "k_ndft_i8 + k_i8_prep" if dtype == "c128" else "k_ndft_i8 (x digit prep inside the kernel)",
            "algorithmic_bytes": 2 * 65536 * 1024 * (16 if dtype == "c128" else 8),
            "peak_source": f"2 x {src} bf16_tflops (int8 dense = 2 x bf16 on B200; int8 not measured)",
            "nominal_peak": 4500.0, "frac_nominal": round(achieved_tops / 4500.0, 4),
            "algorithmic": f"{per} int8 tensor ops per complex ⊙: {terms} digit x sign MMA terms x re/im x re/im MACs"}


def ncu_traffic(kernel_prefix):
    """DRAM bytes (read + write) per launch of a kernel, from the committed ncu
    --set full summary (profiles/*_kernels.json, tools/ncu_summary.py), or None.
    The newest round's file wins (files sort by round)."""
    import glob
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_kernels.json"))):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        for name, k in d.items():
            if name.startswith(kernel_prefix) and "dram_read_bytes" in k:
                best = {"bytes_per_launch": k["dram_read_bytes"] + k.get("dram_write_bytes", 0),
                        "source": os.path.relpath(f, ROOT),
                        "ncu": {key: round(k[key], 1) for key in ("issue_active_pct", "fma_pipe_pct",
                                                                   "alu_pipe_pct", "fp64_pipe_pct", "tensor_pipe_pct", "lts_pct",
                                                                   "dram_pct") if key in k}}
    return best


NDFT_KERNELS = {"c64": "k_ndft_fast_f32x2", "c128": "k_ndft_fast<double"}


def roof_alu(dtype, achieved_tflops, what="ndft"):
    peak = fma_peak_tflops(dtype)
    kern = NDFT_KERNELS[dtype] if what == "ndft" else what
    tr = ncu_traffic(kern)
    return {"bound": "fp32_alu" if dtype == "c64" else "fp64_alu", "achieved": round(achieved_tflops, 3),
            "peak": round(peak, 3), "unit": "TFLOP/s", "frac": round(achieved_tflops / peak, 4),
            "traffic": tr["bytes_per_launch"] if tr else None, "traffic_unit": "bytes/launch",
            "traffic_source": tr["source"] if tr else None,
            "kernel": kern,
            "peak_source": "measured live: sa_fma_peak, max(FFMA, FFMA2) for fp32 / DFMA for fp64 "
                           "(MEASURED_PEAKS.json has no CUDA-core figure)",
            "algorithmic": "8 FMA (16 flop) per complex ⊙ (sign-split identity)"}


def roof_hbm(bytes_per_step, ms, kernel=None):
    peaks, src = measured_peaks()
    ach = bytes_per_step / (ms * 1e-3) / 1e9
    tr = ncu_traffic(kernel) if kernel else None
    r = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
         "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": tr["bytes_per_launch"] if tr else None,
         "traffic_unit": "bytes/launch", "algorithmic_bytes": bytes_per_step, "kernel": kernel,
         "peak_source": src}
    if tr and tr.get("ncu"):  # issue / pipe utilisation of the same kernel (profiles/): the
        r["ncu_utilisation_pct"] = tr["ncu"]  # evidence SURVEY §8(d) asks for next to the HBM fraction
    return r


# --------------------------------------------------------------------------- CPU baselines
def cpu_ndft(x, P, rows=None):
    import oracle
    rows = rows or min(x.shape[0], 4096, max(256, 40 * P))  # ~10-30 s of CPU work at ~30 ms/vector/core
    sample = np.ascontiguousarray(x[:rows])
    t = time.perf_counter()
    oracle.ndft(sample, dtype="f32" if sample.dtype == np.complex64 else "f64", nthreads=P)
    dt = time.perf_counter() - t
    n = x.shape[1]
    return {"value": rows * n * n / dt, "unit": "⊙/s", "cores": P, "kind": "port",
            "sample": f"first {rows} of the vectors (N={n}), oracle/signadd_oracle.c or_ndft "
                      f"(sequential, op-for-op restatement of transforms.py:223-251), {P} threads, "
                      f"{dt:.2f}s wall"}


def cpu_nlfft(x, variant, P):
    import oracle
    n = x.shape[1]
    rows = min(x.shape[0], 8 * P)
    sample = np.ascontiguousarray(x[:rows])
    dts = "f32" if sample.dtype == np.complex64 else "f64"
    t = time.perf_counter()
    oracle.nfft(sample, variant, dtype=dts, nthreads=P)
    dt = time.perf_counter() - t
    per = n * (n.bit_length()) if variant == "dit" else (n // 2) * (n.bit_length() - 2) + 2 * n
    return {"value": rows * per / dt, "unit": "⊙/s", "cores": P, "kind": "port",
            "sample": f"first {rows} C3 vectors (N={n}), oracle/signadd_oracle.c or_nfft {variant.upper()} "
                      f"({'op-for-op restatement of transforms.py:254-298' if variant == 'dit' else 'the DIF convention, DESIGN §3.3 (no reference)'}), "
                      f"{P} threads, {dt:.2f}s wall"}


def cpu_map(surv, ref, L, M, P):
    import oracle
    rows = min(L, 4 * P)
    dts = "f32" if surv.dtype == np.complex64 else "f64"
    t = time.perf_counter()
    oracle.ambiguity_map(surv, ref, 0, rows, M, dtype=dts, nthreads=P)
    dt = time.perf_counter() - t
    ns = surv.size
    ops = rows * ns + rows * M * (M.bit_length())
    return {"value": rows * M / dt, "unit": "cells/s", "ops_per_s": ops / dt, "cores": P, "kind": "port",
            "sample": f"delay rows 0..{rows - 1} of {L} (Ns={ns}, M={M}), oracle/signadd_oracle.c "
                      f"or_ambiguity_map (lag_product_mf + block sums + nfft, ambiguity.py:146-187 composition), "
                      f"{P} threads, {dt:.2f}s wall"}


def numpy_ref_rows(kind, x, P, per_task, tasks_per_worker, all_rows=False):
    """The unmodified numpy reference on Pool(P) (tools/refcpu.py)."""
    from tools import refcpu
    ntask = P * tasks_per_worker
    rows = x.shape[0] if all_rows else min(x.shape[0], ntask * per_task)
    per_task = -(-rows // ntask)
    xs = x[:rows]
    tasks = lambda P_: [(kind, i, min(rows, i + per_task)) for i in range(0, rows, per_task)]  # noqa: E731
    try:
        r = refcpu.measure(kind, {"x": xs}, tasks, P)
    except Exception as ex:  # a baseline must not take the bench line down
        return {"unavailable": repr(ex)}
    r["sample"] = f"{rows} vectors, {per_task} per task, {len(tasks(P))} tasks on {P} workers"
    return r


def numpy_ref_map(surv, ref, L, M, P, rows_per_worker=4):
    from tools import refcpu
    lags = list(range(min(L, P * rows_per_worker)))
    tasks = lambda P_: [("map", lags[i:i + rows_per_worker], M) for i in range(0, len(lags), rows_per_worker)]  # noqa: E731
    try:
        r = refcpu.measure("map", {"surv": surv, "ref": ref}, tasks, P)
    except Exception as ex:
        return {"unavailable": repr(ex)}
    r["sample"] = (f"delay rows 0..{len(lags) - 1}: lag_product_mf(n={surv.size}) -> {surv.size // M}-sample block "
                   f"sums -> nfft({M}), {rows_per_worker} rows per worker")
    return r


def wl_nlfft(args, ws, rank, variant="dit", batch=4096, n=1 << 16, dtype=None):
    """C3: NL-FFT 2^16 x 4096 (inputs synthesised on the GPU, same model as workloads.c3)."""
    import torch
    import paper_1402_0532_b200 as sa
    dtype = dtype or args.dtype
    cdt = complex_dtype(dtype)
    g = torch.Generator(device="cuda").manual_seed(14020534 + rank)
    re = torch.randn(batch, n, device="cuda", dtype=torch.float64, generator=g)
    im = torch.randn(batch, n, device="cuda", dtype=torch.float64, generator=g)
    xd = torch.complex(re, im) * math.sqrt(0.5)
    del re, im
    t = torch.arange(n, device="cuda", dtype=torch.float64)
    k = torch.randint(1, 5, (batch,), device="cuda", generator=g)
    for j in range(4):
        a = torch.rand(batch, 1, device="cuda", dtype=torch.float64, generator=g) * 0.9 + 0.1
        f = torch.rand(batch, 1, device="cuda", dtype=torch.float64, generator=g) * n
        ph = torch.rand(batch, 1, device="cuda", dtype=torch.float64, generator=g) * 2 * math.pi
        on = (k > j).to(torch.float64)[:, None]
        xd += on * a * torch.exp(1j * (2 * math.pi * f * t[None] / n + ph))
    xd = xd.to(cdt)
    xd = xd.contiguous()
    torch.cuda.empty_cache()
    yd = torch.empty_like(xd)
    ops = batch * n * (int(math.log2(n)) + 1) if variant == "dit" else batch * sa.nfft_dif_complex_ops(n)
    step = lambda: sa.nfft_batch(xd, out=yd, variant=variant)  # noqa: E731
    bytes_step = 2 * xd.numel() * xd.element_size()
    res = {"ops": ops, "step": step, "launches_per_step": 1, "bytes": bytes_step,
           "config": {"workload": f"C3 NL-FFT {variant.upper()} (BASELINE.json configs[2])", "n": n,
                      "batch": batch, "dtype": str(cdt).replace("torch.", ""),
                      "inputs": "CN(0,1) + 1-4 off-grid tones, A~U[0.1,1] (SURVEY §8d model), torch RNG on the GPU",
                      "l2_policy": f"inputs ({bytes_step >> 20} MiB in + out) larger than L2; no flush"},
           "dtype": "f32" if dtype == "c64" else "f64"}
    kname = ("k_nlfft64k_dit" if variant == "dit" else "k_nlfft64k_dif") + (
        "<float" if dtype == "c64" else "<double")
    res["roofline"] = lambda ms: roof_hbm(bytes_step, ms, kname)
    sample = xd[: 64].cpu().numpy()  # host copy of the first rows for the CPU baselines
    res["cpu"] = lambda P: cpu_nlfft(sample, variant, P)
    if variant == "dit":
        res["cpu_numpy"] = lambda P: numpy_ref_rows("nfft", sample, P, per_task=1, tasks_per_worker=4)
    else:
        res["cpu_numpy"] = lambda P: {"unavailable": "the reference has no DIF NL-FFT (SPEC.md:14)"}
    if variant == "dit" and dtype == "c64" and not args.no_e2e:
        hin = torch.empty(xd.shape, dtype=xd.dtype, pin_memory=True)
        hin.copy_(xd)
        hout = torch.empty_like(hin).pin_memory()
        res["e2e_step"] = lambda: sa.nfft_batch(hin, out=hout, variant=variant)
        res["h2d"] = res["d2h"] = hin.numel() * hin.element_size()
        res["e2e_api"] = "paper_1402_0532_b200.nfft_batch(pinned host tensor, out=pinned host tensor)"
        res["e2e_launches"] = len(_pipeline_plan(batch, n * xd.element_size()))
    return res


def wl_detect(args, k=8):
    """§8(f)-1: peak search on a C5-shaped map (4096 x 2048, device-resident),
    sa_map_peaks through the C ABI with preallocated buffers (no host sync)."""
    import ctypes
    import torch
    from paper_1402_0532_b200 import _native
    rows, cols = 4096, 2048
    cdt = complex_dtype(args.dtype)
    g = torch.Generator(device="cuda").manual_seed(14020539)
    maps = [torch.randn(rows, cols, dtype=cdt, device="cuda", generator=g) for _ in range(4)]
    v = maps[0]
    need = ctypes.c_int64()
    _native.check(_native.lib().sa_peaks_workspace_bytes(rows, cols, k, ctypes.byref(need)))
    ws = torch.empty(need.value, dtype=torch.uint8, device="cuda")
    idx = torch.empty(k, dtype=torch.int64, device="cuda")
    mag = torch.empty(k, dtype=torch.float64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    d = _native.SA_C64 if args.dtype == "c64" else _native.SA_C128

    it = [0]

    def step():  # cycles through 4 maps (>= 256 MiB) so every read comes from HBM, not L2
        m = maps[it[0] % 4]
        it[0] += 1
        _native.check(_native.lib().sa_map_peaks(d, _native.ptr(m), rows, cols, k, _native.ptr(idx), _native.ptr(mag),
                                                 _native.ptr(cnt), _native.ptr(ws), need.value, _native.stream_ptr()))
    mb = v.numel() * v.element_size()
    return {"step": step, "ops": rows * cols, "map_bytes": mb, "launches_per_step": 2,
            "config": {"workload": "§8(f)-1 detection: top-k strict local maxima of |map|", "rows": rows,
                       "cols": cols, "k": k, "dtype": "complex64" if args.dtype == "c64" else "complex128",
                       "l2_policy": "4 maps cycled (> L2)"}}


def wl_writer(args):
    """§8(f)-4: the reference CLI's surface CSV (cli.py:184-191) for a C5-shaped
    map on the GPU: D2H + magnitude_db (numpy, the reference's arithmetic) + the
    native repr-exact formatter (writers.surface_csv_bytes).  Host-side work; the
    reference's Python csv/repr writer is timed on a bounded row sample."""
    import torch
    from paper_1402_0532_b200.writers import magnitude_db, surface_csv_bytes
    rows, cols = 4096, 2048
    g = torch.Generator(device="cuda").manual_seed(14020540)
    m = torch.randn(rows, cols, dtype=complex_dtype(args.dtype), device="cuda", generator=g)
    nbytes = [0]

    def step():
        nbytes[0] = len(surface_csv_bytes(magnitude_db(m), "map.manifest.json"))

    def cpu(P):
        import sys as _s
        from tools import refcpu
        if not refcpu.available():
            return {"unavailable": "baseline/_ref not installed"}
        if refcpu.REF not in _s.path:
            _s.path.insert(0, refcpu.REF)
        import signadd.cli as rcli
        db = magnitude_db(m[:128])
        t = time.perf_counter()
        rcli._write_csv(os.devnull, ["l", "p", "magnitude_db"],
                        ((l, p, float(db[l, p])) for l in range(128) for p in range(cols)), "map.manifest.json")
        dt = time.perf_counter() - t
        return {"value": 128 * cols / dt, "unit": "cells/s", "cores": 1, "kind": "reference (unmodified cli._write_csv)",
                "sample": f"128 of {rows} rows through the reference's csv/repr writer, {dt:.2f}s"}
    return {"step": step, "ops": rows * cols, "map_bytes": None, "host": True, "cpu": cpu,
            "config": {"workload": "§8(f)-4 surface CSV writer (cli.py:74-116, 184-191)", "rows": rows,
                       "cols": cols, "dtype": "complex64 map -> f64 dB -> repr() text",
                       "threads": len(os.sched_getaffinity(0))}}


def lag_is_i8():
    from paper_1402_0532_b200 import _native
    return _native.lib().sa_lag_kernel(-1) == 0


def lag_kernel(dtype):
    """The lag-integration kernel sa_ambiguity_integrate runs for T = 2048: the
    tcgen05 kind::i8 Hankel GEMM for complex64 (sa_lag_i8.cu; sa_lag_tc.cu's bf16
    kernel with SA_LAG_KIND=bf16), FP64 tiles otherwise."""
    if dtype != "c64":
        return "k_lag_integrate_fast<double>"
    return "k_lag_i8" if lag_is_i8() else "k_lag_tc"


def roof_lag(dtype, ns, lags, lms):
    """Lag stage roofline.  complex64: 32 tensor ops per lag ⊙ on tcgen05 -- int8
    (sa_lag_i8.cu: 8 sign x digit terms x 2 digits x re/im pairs = 16 int8 MACs)
    against the int8 rate (2 x the measured bf16 burst figure), or bf16 (sa_lag_tc.cu:
    8 sign-split terms x 2 pieces) against the bf16 figure.  lms is the whole lag
    stage (the reference digit prep included).  complex128 against the live DFMA
    peak (16 flop per ⊙)."""
    if dtype == "c64":
        peaks, src = measured_peaks()
        i8 = lag_is_i8()
        peak = peaks.get("bf16_tflops", 1590.0) * (2.0 if i8 else 1.0)
        ach = 32 * ns * lags / (lms * 1e-3) / 1e12
        tr = ncu_traffic(lag_kernel(dtype))
        return {"bound": "tensor", "achieved": round(ach, 1), "peak": round(peak, 1),
                "unit": "TOP/s" if i8 else "TFLOP/s",
                "frac": round(ach / peak, 4), "traffic": tr["bytes_per_launch"] if tr else None,
                "traffic_unit": "bytes/launch", "traffic_source": tr["source"] if tr else None,
                "kernel": lag_kernel(dtype) + (" (+ k_lag_cprep)" if i8 else ""), "kernel_ms": lms,
                "peak_source": (f"2 x {src} bf16_tflops (int8 dense = 2 x bf16 on B200; int8 not measured)" if i8
                                else f"{src} bf16_tflops (burst)"),
                "nominal_peak": 4500.0 if i8 else 2250.0, "frac_nominal": round(ach / (4500.0 if i8 else 2250.0), 4),
                "algorithmic": ("32 int8 tensor ops per lag ⊙ (sign x 2-digit terms: 16 MACs); K = T + 32 per block "
                                "(c-Hankel: no zero region)") if i8 else
                               ("32 bf16 tensor flop per lag ⊙ (8 sign-split terms x 2 pieces); the Hankel "
                                "K range (T + 1024 per T samples) is overhead, not counted"),
                **({"ncu_utilisation_pct": tr["ncu"]} if tr and tr.get("ncu") else {})}
    peak = fma_peak_tflops(dtype)
    ach = 16 * ns * lags / (lms * 1e-3) / 1e12
    return {"bound": "fp64_alu", "achieved": round(ach, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
            "frac": round(ach / peak, 4), "traffic": None, "kernel": lag_kernel(dtype), "kernel_ms": lms,
            "peak_source": "measured live sa_fma_peak"}


def wl_map(args, ws, rank, c5=False, e2e=False):
    """C4 (1 GPU) / C5 (sharded) ⊙ range-Doppler map."""
    import torch
    import paper_1402_0532_b200 as sa
    from paper_1402_0532_b200.workloads import c4_scene, c5_scene
    sc = c5_scene() if c5 else c4_scene()
    L, M = (4096, 2048) if c5 else (1024, 512)
    cdt = complex_dtype(args.dtype)
    surv = torch.from_numpy(sc.surv).to(cdt).cuda()
    ref = torch.from_numpy(sc.ref).to(cdt).cuda()
    ns = surv.numel()
    rows = L // ws
    l0 = rank * rows
    out = torch.empty((rows, M), dtype=cdt, device="cuda")
    ws_buf = torch.empty((rows + 30) * M * out.element_size(), dtype=torch.uint8, device="cuda")  # blocked z pads to whole tiles

    pm, zx, transport = None, None, "p2p"
    if ws > 1:  # rank 0's map, IPC-shared once: every rank's kernels store their rows into it
        from paper_1402_0532_b200.sharded import PeerMap, PeerMapUnavailable, ZExchange, blocks_shardable
        transport = args.map_transport
        if transport == "p2p":
            try:
                pm = PeerMap(L, M, cdt)
            except PeerMapUnavailable:  # (all ranks agree) NCCL gather instead
                transport = "gather"
        if pm is not None and blocks_shardable(surv, M, "fast", "mf", "nfft", L, ws):
            try:  # the z-row blocks of every rank, IPC-shared once (block-sharded lag stage)
                zx = ZExchange(L, M, cdt)
            except PeerMapUnavailable:
                zx = None
    full = torch.empty((L, M), dtype=cdt, device="cuda") if (ws > 1 and rank == 0 and pm is None) else None

    def step():
        if ws > 1:  # block-sharded lag stage + z rows to their owners, or delay-bin shards; rows into rank 0's map
            from paper_1402_0532_b200.sharded import ambiguity_map_sharded
            ambiguity_map_sharded(surv, ref, L, M, peer_map=pm, transport=transport, out_full=full,
                                  out_local=out, workspace=ws_buf, z_exchange=zx)
        else:
            sa.ambiguity_map(surv, ref, rows, M, l0=l0, out=out, workspace=ws_buf)

    z = torch.empty((rows + 30, M), dtype=cdt, device="cuda")
    from paper_1402_0532_b200 import _native
    zrows = torch.tensor([z.data_ptr()], dtype=torch.int64, device="cuda")

    def lag_only():
        # the lag stage exactly as the map runs it: complex64 writes the blocked z the
        # Doppler kernel reads (sa_ambiguity_integrate_blocks, one destination);
        # otherwise the row-major stage (sa_ambiguity_integrate)
        if args.dtype == "c64" and l0 == 0 and rows % 16 == 0 and \
                _native.lib().sa_ambiguity_integrate_blocks(
                    _native.SA_C64, _native.ptr(surv), _native.ptr(ref), ns, ns, 0, rows, M, 0, M, 1,
                    _native.ptr(zrows), 1, _native.stream_ptr()) == 0:
            return
        _native.check(_native.lib().sa_ambiguity_integrate(
            _native.SA_C64 if args.dtype == "c64" else _native.SA_C128, _native.ptr(surv), _native.ptr(ref),
            ns, ns, l0, rows, M, 1, _native.SA_NDFT_FAST, _native.ptr(z), _native.stream_ptr()))

    ops = sa.map_complex_ops(L, ns, M)

    def result():  # the map as delivered on rank 0 (None elsewhere)
        step()
        torch.cuda.synchronize()
        if ws > 1:
            return pm.full if pm is not None else full
        return out

    res = {"ops": ops, "cells": L * M, "step": step, "lag_only": lag_only, "launches_per_step": 4 if args.dtype == "c64" else 2,
           "result": result, "surv": surv, "ref": ref,
           "config": {"workload": ("C5" if c5 else "C4") + " ⊙ range-Doppler map (BASELINE.json configs["
                      + ("4" if c5 else "3") + "])", "ns": ns, "delay_bins": L, "doppler_bins": M,
                      "block_T": ns // M, "doppler": "NL-FFT DIT", "dtype": str(cdt).replace("torch.", ""),
                      "targets": len(sc.delays),
                      "parallelism": (f"Doppler-block shards x{ws} for the lag stage, z rows stored by the lag "
                                      "kernel into their owners' blocks over NVLink (fused all-to-all), delay-bin "
                                      "shards for the Doppler NL-FFT, rows stored into rank 0's IPC-shared map, "
                                      "two completion all-reduces") if zx is not None else (
                          f"delay-bin shards x{ws}" + (
                              (", rows stored by the transform kernels into rank 0's IPC-shared map over NVLink, "
                               "one completion all-reduce" if transport == "p2p" else ", NCCL gather to rank 0")
                              if ws > 1 else ""))},
           "dtype": (("int8 digits x sign, exact int32 accumulate, f64->f32 epilogue (lag)" if lag_is_i8() else
                      "bf16x2-split x sign, f32 accumulate (lag)") + "; f32 (NL-FFT)") if args.dtype == "c64"
           else "f64"}
    if ws == 1:
        def graph_step():
            mg = sa.MapGraph(ns, ns, L, M, dtype=cdt).load(surv, ref)
            mg.capture()
            return mg.replay
        res["graph_step"] = graph_step
    if e2e and not args.no_e2e:
        hs = torch.from_numpy(sc.surv).to(cdt).pin_memory()
        hr = torch.from_numpy(sc.ref).to(cdt).pin_memory()
        hout = torch.empty((L, M), dtype=cdt).pin_memory()
        res["e2e_step"] = lambda: sa.ambiguity_map(hs, hr, L, M, out=hout)
        res["h2d"] = 2 * hs.numel() * hs.element_size()
        res["d2h"] = hout.numel() * hout.element_size()
        res["e2e_api"] = ("paper_1402_0532_b200.ambiguity_map(pinned host surv, pinned host ref, L, M, "
                          "out=pinned host map)")
        res["e2e_launches"] = 4 if args.dtype == "c64" else 2
    sv = sc.surv.astype(np.complex64 if args.dtype == "c64" else np.complex128)
    rv = sc.ref.astype(sv.dtype)
    res["cpu"] = lambda P: cpu_map(sv, rv, L, M, P)
    res["cpu_numpy"] = lambda P: numpy_ref_map(sc.surv, sc.ref, L, M, P)
    return res


def wl_map_stream(args, ws, rank):
    """C5 map, streaming: each step submits one CPI to a sharded.MapStream (the
    lag stage of map i+1 overlaps the delivery of map i into rank 0's memory);
    timed over K steps including the flush of the last map."""
    import torch
    from paper_1402_0532_b200.sharded import MapStream, blocks_shardable
    from paper_1402_0532_b200.workloads import c5_scene
    sc = c5_scene()
    L, M = 4096, 2048
    cdt = complex_dtype(args.dtype)
    surv = torch.from_numpy(sc.surv).to(cdt).cuda()
    ref = torch.from_numpy(sc.ref).to(cdt).cuda()
    if not blocks_shardable(surv, M, "fast", "mf", "nfft", L, ws):
        return {"skipped": "not block-shardable"}
    ms_ = MapStream(L, M, cdt, depth=2)
    ems, _ = timed(lambda: ms_.submit(surv, ref), max(3, args.steps // 2), 3, ws, flush=ms_.flush)
    out = {"ms_per_step": ems, "cells_per_s": L * M / (ems * 1e-3), "n_gpus": ws, "scaling": "strong",
           "config": {"workload": "C5 ⊙ range-Doppler map, streaming CPIs (BASELINE.json configs[4])",
                      "delay_bins": L, "doppler_bins": M, "maps_in_flight": 2,
                      "parallelism": f"Doppler-block shards x{ws} (lag) + delay-bin shards (Doppler), map i "
                                     "delivered into rank 0 on a side stream while map i+1's lag stage runs"}}
    if args.check:
        full = ms_.submit(surv, ref)
        ms_.flush()
        torch.cuda.synchronize()
        if rank == 0:
            import paper_1402_0532_b200 as _sa
            out["map_check"] = {"bit_identical": bool(torch.equal(full, _sa.ambiguity_map(surv, ref, L, M)))}
    ms_.close()
    return out


def summarise(name, e):
    """One compact record per workload for the line's trailing ``summary`` key."""
    if "error" in e:
        return {"error": e["error"][:120]}
    if "ms_per_step" not in e:
        return {k: v for k, v in e.items() if k in ("skipped", "unavailable")}
    r = {"ms": round(e["ms_per_step"], 4)}
    for k in ("ops_per_s", "cells_per_s"):
        if k in e:
            r[k] = float(f"{e[k]:.4g}")
    rf = e.get("roofline")
    if rf:
        r["roofline"] = f"{rf['frac']:.3f} of {rf['bound']} ({rf['kernel']})"
    cb = e.get("cpu_baseline")
    if cb and "value" in cb:
        r["cpu_port"] = float(f"{cb['value']:.4g}")
        rn = cb.get("reference_numpy") or {}
        if "value" in rn:
            r["cpu_numpy"] = float(f"{rn.get('cells_per_s', rn['value']):.4g}")
            r["cpu_numpy_1core"] = float(f"{rn.get('one_core_cells_per_s', rn['one_core_value']):.4g}")
    if "e2e" in e:
        r["e2e_ms"] = round(e["e2e"]["ms_per_step"], 3)
    if "ms_per_step" in e.get("cuda_graph", {}):
        r["graph_ms"] = round(e["cuda_graph"]["ms_per_step"], 4)
    return r


# --------------------------------------------------------------------------- main
def run_extra(name, make, args, ws, rank):
    """One N=1 workload line: device-resident timing, roofline, CPU baselines
    (oracle port + unmodified numpy reference), e2e through the public API."""
    import torch
    r = make()
    steps = max(3, args.steps // 2)
    if r.get("host"):  # host-side work: wall clock, one warm-up
        r["step"]()
        t = time.perf_counter()
        for _ in range(2):
            r["step"]()
        hms = (time.perf_counter() - t) / 2 * 1e3
        e = {"ms_per_step": hms, "config": r["config"], "cells_per_s": r["ops"] / (hms * 1e-3),
             "timing": "host wall clock, 2 steps after 1 warm-up"}
        if not args.no_cpu and "cpu" in r:
            e["cpu_baseline"] = r["cpu"](len(os.sched_getaffinity(0)))
        del r
        return e
    ems, _ = timed(r["step"], steps, 3, 1)
    e = {"ms_per_step": ems, "config": r["config"], "dtype": r.get("dtype")}
    if "map_bytes" in r:  # detection: one read of the map
        e["cells_per_s"] = r["ops"] / (ems * 1e-3)
        e["roofline"] = roof_hbm(r["map_bytes"], ems, "k_peaks_tile")
    elif "cells" in r:
        e["cells_per_s"] = r["cells"] / (ems * 1e-3)
        e["ops_per_s"] = r["ops"] / (ems * 1e-3)
        lms, _ = timed(r["lag_only"], steps, 3, 1)
        e["roofline"] = roof_lag(args.dtype, r["config"]["ns"], r["config"]["delay_bins"], lms)
        e["roofline"]["share_of_step"] = round(lms / ems, 4)
        e["roofline"]["hbm_gbs_of_step"] = round((2 * r["config"]["ns"] * 8 + r["cells"] * 8) / (ems * 1e-3) / 1e9, 1)
    else:
        e["ops_per_s"] = r["ops"] / (ems * 1e-3)
        e["roofline"] = r["roofline"](ems)
    if "graph_step" in r:  # the same map call replayed from a CUDA graph (MapGraph)
        try:
            gms, _ = timed(r["graph_step"](), steps, 3, 1)
            e["cuda_graph"] = {"ms_per_step": gms, "cells_per_s": r["cells"] / (gms * 1e-3),
                               "api": "paper_1402_0532_b200.MapGraph(...).replay()"}
        except Exception as ex:  # capture is an extra: never fail the line
            e["cuda_graph"] = {"unavailable": repr(ex)[:200]}
    if "e2e_step" in r:
        xms, _ = timed(r["e2e_step"], max(2, steps // 2), 1, 1)
        unit = "cells/s" if "cells" in r else "⊙/s"
        e["e2e"] = {"value": (r["cells"] if "cells" in r else r["ops"]) / (xms * 1e-3), "unit": unit,
                    "ms_per_step": xms, "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"],
                    "api": r["e2e_api"]}
    if not args.no_cpu and "cpu" in r:
        P = len(os.sched_getaffinity(0))
        cb = r["cpu"](P)
        if "cpu_numpy" in r and not args.no_numpy_ref:
            cb["reference_numpy"] = r["cpu_numpy"](P)
        e["cpu_baseline"] = cb
    del r
    torch.cuda.empty_cache()
    return e


def run_ours(args):
    import torch
    ws, rank, local = dist_init(args.dist_backend, args.share_gpu)
    import paper_1402_0532_b200 as sa
    sa.require_native()
    w = args.workload
    if w == "ndft":
        res = wl_ndft(args, ws, rank)
    elif w == "nlfft":
        res = wl_nlfft(args, ws, rank)
    elif w in ("map", "map5"):
        res = wl_map(args, ws, rank, c5=(w == "map5"), e2e=(ws == 1))
    else:
        raise SystemExit(f"unknown workload {w}")
    sampler = ClockSampler(local) if rank == 0 else None
    ms, clocks = timed(res["step"], args.steps, args.warmup, ws, sampler)
    if w in ("map", "map5"):
        value = res["cells"] / (ms * 1e-3)
        unit = "cells/s"
    else:
        value = res["ops"] * ws / (ms * 1e-3)
        unit = "⊙/s"
    line = {"metric": METRIC, "value": value, "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if w in ("ndft", "nlfft") else "strong", "vs_baseline": None,
            "dtype": res.get("dtype", "f32" if args.dtype == "c64" else "f64"),
            "data": "synthetic (seeded, SURVEY §8d model)",
            "config": res["config"], "clocks": clocks,
            "gpu_launches": res["launches_per_step"] * args.steps}
    if w in ("map", "map5"):
        line["ops_per_s"] = res["ops"] / (ms * 1e-3)
    if rank == 0 and "roofline" in res:
        line["roofline"] = res["roofline"](ms)
    if args.check and w in ("map", "map5"):  # the delivered map vs a single-call map on this rank's GPU
        full = res["result"]()
        if rank == 0:
            import paper_1402_0532_b200 as _sa
            one = _sa.ambiguity_map(res["surv"], res["ref"], res["config"]["delay_bins"], res["config"]["doppler_bins"])
            line["map_check"] = {"bit_identical": bool(torch.equal(full, one)), "rows": int(full.shape[0])}
    if w == "map5" and ws > 1 and args.check:  # the streaming variant, checked too
        extras_stream = wl_map_stream(args, ws, rank)
        if rank == 0:
            line.setdefault("workloads", {})["C5_map_stream"] = extras_stream
    if w in ("map", "map5") and rank == 0:
        lms, _ = timed(res["lag_only"], args.steps, 3, 1)
        line["roofline"] = roof_lag(args.dtype, res["config"]["ns"], res["config"]["delay_bins"] // ws, lms)
        line["roofline"]["share_of_step"] = round(lms / ms, 4) if ws == 1 else None
    # e2e through the public API with host buffers
    if "e2e_step" in res:
        ems, _ = timed(res["e2e_step"], max(2, args.steps // 2), 1, ws)
        line["e2e"] = {"value": (res["cells"] if "cells" in res else res["ops"] * ws) / (ems * 1e-3), "unit": unit,
                       "ms_per_step": ems, "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"],
                       "api": res.get("e2e_api")}
        if w == "ndft":
            line["e2e"]["pipeline"] = ("H2D / transform / D2H overlapped over row chunks (32 MiB steady, "
                                       "16 MiB first and last)")
        line["gpu_launches"] += max(2, args.steps // 2) * res.get("e2e_launches", 1)
    # CPU baseline: rank 0, N=1 only
    if rank == 0 and ws == 1 and "cpu" in res and not args.no_cpu:
        P = len(os.sched_getaffinity(0))
        line["cpu_baseline"] = res["cpu"](P)
        if "cpu_numpy" in res and not args.no_numpy_ref:
            line["cpu_baseline"]["reference_numpy"] = res["cpu_numpy"](P)
    del res
    torch.cuda.empty_cache()
    # extras (N=1)
    extras = {}
    if rank == 0 and ws == 1 and not args.no_extras and w == "ndft":
        specs = [("C1_ndft_c128", lambda: wl_ndft64(args))]
        if args.ndft_mode == "tc8" and args.dtype == "c64":
            specs.append(("C2_ndft_bf16", lambda: {**wl_ndft(args, ws, rank, mode="tc", e2e=False), "cpu_skip": 1}))
        if args.ndft_mode in ("tc", "tc8") and args.dtype == "c64":
            specs.append(("C2_ndft_ffma2", lambda: {**wl_ndft(args, ws, rank, mode="fast", e2e=False), "cpu_skip": 1}))
        specs += [("C2_ndft_c128", lambda: wl_ndft(args, ws, rank, mode="tc", dtype="c128")),
                  ("C2_ndft_c128_dfma", lambda: {**wl_ndft(args, ws, rank, mode="fast", dtype="c128", e2e=False),
                                                 "cpu_skip": 1}),
                  ("C3_nlfft_dit", lambda: wl_nlfft(args, ws, rank, "dit", dtype="c64")),
                  ("C3_nlfft_dif", lambda: wl_nlfft(args, ws, rank, "dif", dtype="c64")),
                  ("C3_nlfft_dit_c128", lambda: wl_nlfft(args, ws, rank, "dit", dtype="c128")),
                  ("C3_nlfft_dif_c128", lambda: wl_nlfft(args, ws, rank, "dif", dtype="c128")),
                  ("C4_map", lambda: wl_map(args, ws, rank, e2e=True)),
                  ("C5_map_1gpu", lambda: wl_map(args, ws, rank, c5=True, e2e=True)),
                  ("C5_detect", lambda: wl_detect(args)),
                  ("C5_surface_csv", lambda: wl_writer(args))]
        for name, fn in specs:
            if args.only and name not in args.only.split(","):
                continue
            try:
                def make(fn=fn):
                    r = fn()
                    if r.pop("cpu_skip", None):  # same sample as the headline's baseline
                        r.pop("cpu", None)
                        r.pop("cpu_numpy", None)
                    return r
                extras[name] = run_extra(name, make, args, ws, rank)
                log(f"[bench] {name}: {extras[name]['ms_per_step']:.4f} ms")
            except Exception as ex:  # keep the headline line even if an extra fails
                extras[name] = {"error": repr(ex)}
                torch.cuda.empty_cache()
    # C5 map at every N (the north star asks map throughput at 1/2/4/8 GPUs):
    # all ranks take part -- Doppler-block shards for the lag stage, rows stored
    # into rank 0's map over peer memory -- timed as the max over ranks (strong scaling)
    if not args.no_extras and w == "ndft":
        try:
            r = wl_map(args, ws, rank, c5=True)
            ems, _ = timed(r["step"], max(3, args.steps // 2), 3, ws)
            e = {"ms_per_step": ems, "config": r["config"], "cells_per_s": r["cells"] / (ems * 1e-3),
                 "n_gpus": ws, "scaling": "strong"}
            del r
            torch.cuda.empty_cache()
        except Exception as ex:
            e = {"error": repr(ex)}
        extras["C5_map"] = e
        if ws > 1:  # CPIs back to back, two maps in flight (sharded.MapStream)
            try:
                e2 = wl_map_stream(args, ws, rank)
                extras["C5_map_stream"] = e2
            except Exception as ex:
                extras["C5_map_stream"] = {"error": repr(ex)}
    if rank == 0:
        if extras:
            line.setdefault("workloads", {}).update(extras)
        # compact per-workload record LAST, so a truncated stdout tail still shows it
        line["summary"] = {"headline": summarise("headline", {**line, "ops_per_s": line["value"]}),
                           **{k: summarise(k, v) for k, v in extras.items()}}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    """Reference CPU algorithm (oracle C port, all host threads) on the same workload."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    P = len(os.sched_getaffinity(0))
    w = args.workload
    if w == "ndft":
        from paper_1402_0532_b200.workloads import c2_ndft
        n, rows = 1024, max(64, 4 * P)
        x = c2_ndft(n, 65536, rows=slice(0, rows)).astype(np.complex64 if args.dtype == "c64" else np.complex128)
        dts = "f32" if args.dtype == "c64" else "f64"
        fn = lambda: oracle.ndft(x, dtype=dts, nthreads=P)  # noqa: E731
        ops = rows * n * n
        unit = "⊙/s"
        cfg = {"workload": "C2 batched NDFT (BASELINE.json configs[1])", "n": n, "batch": 65536,
               "dtype": "complex64" if args.dtype == "c64" else "complex128", "sample_rows_per_step": rows,
               "same_config": "rate vs rate: each step is the first rows of the same seeded C2 batch"}
        sample = f"first {rows} vectors of the C2 batch (N={n}) per step, oracle C port (sequential, op for op)"
    elif w == "nlfft":
        n, rows = 1 << 16, max(8, P)
        g = np.random.default_rng(1)
        x = (g.standard_normal((rows, n)) + 1j * g.standard_normal((rows, n))).astype(
            np.complex64 if args.dtype == "c64" else np.complex128)
        dts = "f32" if args.dtype == "c64" else "f64"
        fn = lambda: oracle.nfft(x, "dit", dtype=dts, nthreads=P)  # noqa: E731
        ops = rows * n * 17
        unit = "⊙/s"
        cfg = {"workload": "C3 NL-FFT DIT", "n": n, "batch": 4096, "sample_rows_per_step": rows}
        sample = f"{rows} vectors of 2^16 per step"
    else:
        from paper_1402_0532_b200.workloads import c4_scene, c5_scene
        sc = c5_scene() if w == "map5" else c4_scene()
        L, M = (4096, 2048) if w == "map5" else (1024, 512)
        rows = max(4, P)
        dts = "f32" if args.dtype == "c64" else "f64"
        s = sc.surv.astype(np.complex64 if dts == "f32" else np.complex128)
        r = sc.ref.astype(s.dtype)
        fn = lambda: oracle.ambiguity_map(s, r, 0, rows, M, dtype=dts, nthreads=P)  # noqa: E731
        ops = rows * M
        unit = "cells/s"
        cfg = {"workload": ("C5" if w == "map5" else "C4") + " ⊙ range-Doppler map", "delay_bins": L,
               "doppler_bins": M, "sample_rows_per_step": rows}
        sample = f"{rows} delay rows per step"
    for _ in range(args.warmup):
        fn()
    t = time.perf_counter()
    for _ in range(args.steps):
        fn()
    dt = (time.perf_counter() - t) / args.steps
    v = ops / dt
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": unit, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dts, "data": "synthetic (seeded)",
            "config": cfg,
            "cpu_baseline": {"value": v, "unit": unit, "cores": P, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="ndft", choices=["ndft", "nlfft", "map", "map5"])
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--ndft-mode", default="tc8", choices=["tc8", "tc", "fast"],
                    help="C2 NDFT kernel (complex64): tc8 = tcgen05 kind::i8 exact-digit GEMM, tc = tcgen05 "
                         "bf16x2-split GEMM, fast = FFMA2 CUDA-core kernel")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-numpy-ref", action="store_true",
                    help="skip the unmodified-numpy-reference Pool(P) figures (tools/refcpu.py)")
    ap.add_argument("--only", default="", help="comma-separated extra workloads to run (default: all)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo only for the shared-GPU test mode)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="test mode: all ranks on cuda:0 (NCCL refuses duplicate GPUs; use --dist-backend gloo)")
    ap.add_argument("--check", action="store_true", help="map workloads: compare the delivered map with a single call")
    ap.add_argument("--map-transport", default="p2p", choices=["p2p", "gather"],
                    help="N>1 map delivery: p2p = rows stored into rank 0's map over peer memory; "
                         "gather = delay-bin shards + NCCL gather (the north star's stated split)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: contract requires >= 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
