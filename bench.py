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
def dist_init():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(fn, steps, warmup, ws, sampler=None):
    """W untimed steps, then K steps between barrier+sync; CUDA events on the
    launching stream; returns (ms_per_step max over ranks, clocks)."""
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


def wl_ndft(args, ws, rank, mode=None, e2e=True):
    """C2: batched NDFT N=1024 x 65536.  mode "tc" (complex64 default): the
    fast-mode sum as a sign-split bf16 GEMM on tcgen05 (sa_ndft_tc.cu); "fast":
    the FFMA2 CUDA-core kernel (sa_ndft.cu)."""
    import torch
    import paper_1402_0532_b200 as sa
    from paper_1402_0532_b200.workloads import c2_ndft
    n, batch = 1024, 65536
    cdt = complex_dtype(args.dtype)
    mode = mode or (args.ndft_mode if args.dtype == "c64" else "fast")
    t0 = time.time()
    xh = torch.from_numpy(c2_ndft(n, batch)).to(cdt)
    log(f"[rank {rank}] C2 input generated in {time.time() - t0:.1f}s")
    xd = xh.cuda()
    yd = torch.empty_like(xd)
    ops = batch * n * n
    step = lambda: sa.ndft_batch(xd, out=yd, mode=mode)  # noqa: E731
    desc = ("tc (fast-mode sum as a sign-split bf16 GEMM on tcgen05 tensor cores, fp32 accumulation)"
            if mode == "tc" else "fast (sign-split regrouped accumulation, FFMA2)")
    res = {"ops": ops, "step": step, "launches_per_step": 1,
           "config": {"workload": "C2 batched NDFT (BASELINE.json configs[1])", "n": n,
                      "batch": batch, "mode": desc,
                      "dtype": "complex64" if args.dtype == "c64" else "complex128",
                      "l2_policy": "inputs (512 MiB c64) larger than L2; no flush",
                      "parallelism": f"dp{ws} (independent vectors, weak scaling)"}}
    if e2e and not args.no_e2e:
        hin = xh.pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        res["e2e_step"] = lambda: sa.ndft_batch(hin, out=hout, mode=mode)
        res["e2e_rows"], res["e2e_row_bytes"] = hin.shape[0], hin.shape[1] * hin.element_size()
        res["h2d"] = hin.numel() * hin.element_size()
        res["d2h"] = hout.numel() * hout.element_size()
        res["e2e_api"] = f"paper_1402_0532_b200.ndft_batch(pinned host tensor, out=pinned host tensor, mode={mode!r})"
    if mode == "tc":
        res["roofline"] = lambda ms: roof_tensor(ops * 32 / (ms * 1e-3) / 1e12)
    else:
        res["roofline"] = lambda ms: roof_alu(args.dtype, ops * 16 / (ms * 1e-3) / 1e12, args)
    res["cpu"] = lambda P: cpu_ndft(xh.numpy(), P)
    res["dtype"] = "f32" if args.dtype == "c64" else "f64"
    return res


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


def ncu_traffic(kernel_prefix):
    """DRAM bytes (read + write) per launch of a kernel, from the committed ncu
    --set full summary (profiles/*_kernels.json, tools/ncu_summary.py), or None."""
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


def roof_alu(dtype, achieved_tflops, args):
    peak = fma_peak_tflops(dtype)
    kern = "k_ndft_fast_f32x2" if dtype == "c64" else "k_ndft_fast<double"
    tr = ncu_traffic(kern)
    return {"bound": "fp32_alu" if dtype == "c64" else "fp64_alu", "achieved": round(achieved_tflops, 3),
            "peak": round(peak, 3), "unit": "TFLOP/s", "frac": round(achieved_tflops / peak, 4),
            "traffic": tr["bytes_per_launch"] if tr else None, "traffic_unit": "bytes/launch",
            "traffic_source": tr["source"] if tr else None,
            "algorithmic_bytes": 2 * 65536 * 1024 * (8 if dtype == "c64" else 16),
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


def cpu_ndft(x, P):
    import oracle
    rows = min(x.shape[0], 4096, max(256, 40 * P))  # ~10-30 s of CPU work at ~30 ms/vector/core
    sample = np.ascontiguousarray(x[:rows])
    t = time.perf_counter()
    oracle.ndft(sample, dtype="f32" if sample.dtype == np.complex64 else "f64", nthreads=P)
    dt = time.perf_counter() - t
    n = x.shape[1]
    return {"value": rows * n * n / dt, "unit": "⊙/s", "cores": P, "kind": "port",
            "sample": f"first {rows} of the C2 vectors (N={n}), oracle/signadd_oracle.c or_ndft "
                      f"(sequential, op-for-op restatement of transforms.py:223-251), {P} threads, "
                      f"{dt:.2f}s wall"}


def wl_nlfft(args, ws, rank, variant="dit", batch=4096, n=1 << 16):
    """C3: NL-FFT 2^16 x 4096 (inputs synthesised on the GPU, same model as workloads.c3)."""
    import torch
    import paper_1402_0532_b200 as sa
    cdt = complex_dtype(args.dtype)
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
    yd = torch.empty_like(xd)
    ops = batch * n * (int(math.log2(n)) + 1) if variant == "dit" else batch * sa.nfft_dif_complex_ops(n)
    step = lambda: sa.nfft_batch(xd, out=yd, variant=variant)  # noqa: E731
    bytes_step = 2 * xd.numel() * xd.element_size()
    res = {"ops": ops, "step": step, "launches_per_step": 2, "bytes": bytes_step,
           "config": {"workload": f"C3 NL-FFT {variant.upper()} (BASELINE.json configs[2])", "n": n,
                      "batch": batch, "dtype": str(cdt).replace("torch.", "")}}
    kname = ("k_nlfft64k_dit" if variant == "dit" else "k_nlfft64k_dif") + (
        "<float" if args.dtype == "c64" else "<double")
    res["roofline"] = lambda ms: roof_hbm(bytes_step, ms, kname)
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
    return {"step": step, "ops": rows * cols, "map_bytes": mb,
            "config": {"workload": "§8(f)-1 detection: top-k strict local maxima of |map|", "rows": rows,
                       "cols": cols, "k": k, "dtype": "complex64" if args.dtype == "c64" else "complex128",
                       "l2_policy": "4 maps cycled (> L2)"}}


def lag_kernel(dtype):
    """The lag-integration kernel sa_ambiguity_integrate runs for T = 2048: the
    tcgen05 Hankel GEMM for complex64 (sa_lag_tc.cu), FP64 tiles otherwise."""
    return "k_lag_tc" if dtype == "c64" else "k_lag_integrate_fast<double>"


def roof_lag(dtype, ns, lags, lms):
    """Lag stage roofline: complex64 on tcgen05 against the measured bf16 peak
    (32 tensor flop per ⊙: 8 sign-split terms x 2 bf16 pieces, as the NDFT);
    complex128 against the live DFMA peak (16 flop per ⊙)."""
    if dtype == "c64":
        peaks, src = measured_peaks()
        peak = peaks.get("bf16_tflops", 1590.0)
        ach = 32 * ns * lags / (lms * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(ach / peak, 4), "traffic": None, "kernel": lag_kernel(dtype), "kernel_ms": lms,
                "peak_source": f"{src} bf16_tflops (burst)", "nominal_peak": 2250.0,
                "frac_nominal": round(ach / 2250.0, 4),
                "algorithmic": "32 bf16 tensor flop per lag ⊙ (8 sign-split terms x 2 pieces); the Hankel "
                               "K range (T + 1024 per T samples) is overhead, not counted"}
    peak = fma_peak_tflops(dtype)
    ach = 16 * ns * lags / (lms * 1e-3) / 1e12
    return {"bound": "fp64_alu", "achieved": round(ach, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
            "frac": round(ach / peak, 4), "traffic": None, "kernel": lag_kernel(dtype), "kernel_ms": lms,
            "peak_source": "measured live sa_fma_peak"}


def wl_map(args, ws, rank, c5=False):
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
    ws_buf = torch.empty(rows * M * out.element_size(), dtype=torch.uint8, device="cuda")

    pm, zx, transport = None, None, "p2p"
    if ws > 1:  # rank 0's map, IPC-shared once: every rank's kernels store their rows into it
        from paper_1402_0532_b200.sharded import PeerMap, PeerMapUnavailable, ZExchange, blocks_shardable
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

    z = torch.empty((rows, M), dtype=cdt, device="cuda")
    from paper_1402_0532_b200 import _native

    def lag_only():
        _native.check(_native.lib().sa_ambiguity_integrate(
            _native.SA_C64 if args.dtype == "c64" else _native.SA_C128, _native.ptr(surv), _native.ptr(ref),
            ns, ns, l0, rows, M, 1, _native.SA_NDFT_FAST, _native.ptr(z), _native.stream_ptr()))

    ops = sa.map_complex_ops(L, ns, M)
    res = {"ops": ops, "cells": L * M, "step": step, "lag_only": lag_only, "launches_per_step": 2,
           "config": {"workload": ("C5" if c5 else "C4") + " ⊙ range-Doppler map (BASELINE.json configs["
                      + ("4" if c5 else "3") + "])", "ns": ns, "delay_bins": L, "doppler_bins": M,
                      "block_T": ns // M, "doppler": "NL-FFT DIT", "dtype": str(cdt).replace("torch.", ""),
                      "parallelism": (f"Doppler-block shards x{ws} for the lag stage, z rows stored by the lag "
                                      "kernel into their owners' blocks over NVLink (fused all-to-all), delay-bin "
                                      "shards for the Doppler NL-FFT, rows stored into rank 0's IPC-shared map, "
                                      "two completion all-reduces") if zx is not None else (
                          f"delay-bin shards x{ws}" + (
                              (", rows stored by the transform kernels into rank 0's IPC-shared map over NVLink, "
                               "one barrier" if transport == "p2p" else ", NCCL gather to rank 0") if ws > 1 else ""))}}
    return res


# --------------------------------------------------------------------------- main
def run_ours(args):
    import torch
    ws, rank, local = dist_init()
    import paper_1402_0532_b200 as sa
    sa.require_native()
    w = args.workload
    if w == "ndft":
        res = wl_ndft(args, ws, rank)
    elif w == "nlfft":
        res = wl_nlfft(args, ws, rank)
    elif w in ("map", "map5"):
        res = wl_map(args, ws, rank, c5=(w == "map5"))
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
            "dtype": res.get("dtype", "f32" if args.dtype == "c64" else "f64"), "data": "synthetic (seeded, SURVEY §8d model)",
            "config": res["config"], "clocks": clocks,
            "gpu_launches": res["launches_per_step"] * args.steps}
    if w in ("map", "map5"):
        line["ops_per_s"] = res["ops"] / (ms * 1e-3)
    if rank == 0 and "roofline" in res:
        line["roofline"] = res["roofline"](ms)
    if w in ("map", "map5") and rank == 0:
        lms, _ = timed(res["lag_only"], args.steps, 1, 1)
        line["roofline"] = roof_lag(args.dtype, res["config"]["ns"], res["config"]["delay_bins"] // ws, lms)
        line["roofline"]["share_of_step"] = round(lms / ms, 4) if ws == 1 else None
    # e2e through the public API with host buffers
    if "e2e_step" in res:
        ems, _ = timed(res["e2e_step"], max(2, args.steps // 2), 1, ws)
        line["e2e"] = {"value": res["ops"] * ws / (ems * 1e-3), "unit": unit, "ms_per_step": ems,
                       "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"],
                       "api": res.get("e2e_api"),
                       "pipeline": "H2D / transform / D2H overlapped over row chunks (32 MiB steady, "
                                   "16 MiB first and last)"}
        from paper_1402_0532_b200.transforms import pipeline_plan
        line["gpu_launches"] += max(2, args.steps // 2) * len(pipeline_plan(res["e2e_rows"], res["e2e_row_bytes"], 128))
    # CPU baseline: rank 0, N=1 only
    if rank == 0 and ws == 1 and "cpu" in res and not args.no_cpu:
        P = len(os.sched_getaffinity(0))
        line["cpu_baseline"] = res["cpu"](P)
    # extras (N=1)
    if rank == 0 and ws == 1 and not args.no_extras and w == "ndft":
        extras = {}
        other = "fast" if (args.ndft_mode == "tc" and args.dtype == "c64") else None
        for name, fn in ((("C2_ndft_ffma2", lambda: wl_ndft(args, ws, rank, mode="fast", e2e=False)),) if other else ()) + (
                         ("C3_nlfft_dit", lambda: wl_nlfft(args, ws, rank, "dit")),
                         ("C3_nlfft_dif", lambda: wl_nlfft(args, ws, rank, "dif")),
                         ("C4_map", lambda: wl_map(args, ws, rank)),
                         ("C5_detect", lambda: wl_detect(args))):
            try:
                r = fn()
                ems, _ = timed(r["step"], max(3, args.steps // 2), 2, 1)
                e = {"ms_per_step": ems, "config": r["config"], "ops_per_s": r["ops"] / (ems * 1e-3)}
                if "map_bytes" in r:  # detection: one read of the map
                    e = {"ms_per_step": ems, "config": r["config"], "cells_per_s": r["ops"] / (ems * 1e-3),
                         "roofline": roof_hbm(r["map_bytes"], ems, "k_peaks_tile")}
                elif "cells" in r:
                    e["cells_per_s"] = r["cells"] / (ems * 1e-3)
                    lms, _ = timed(r["lag_only"], 5, 1, 1)
                    e["roofline"] = roof_lag(args.dtype, r["config"]["ns"], r["config"]["delay_bins"], lms)
                    e["roofline"]["hbm_gbs_of_step"] = round(
                        (2 * r["config"]["ns"] * 8 + r["cells"] * 8) / (ems * 1e-3) / 1e9, 1)
                else:
                    e["roofline"] = r["roofline"](ems)
                extras[name] = e
                del r
                torch.cuda.empty_cache()
            except Exception as ex:  # keep the headline line even if an extra fails
                extras[name] = {"error": repr(ex)}
        line["workloads"] = extras
    # C5 map at every N (the north star asks map throughput at 1/2/4/8 GPUs):
    # all ranks take part -- delay-bin shards, rows stored into rank 0's map
    # over peer memory -- timed as the max over ranks (strong scaling)
    if not args.no_extras and w == "ndft":
        try:
            r = wl_map(args, ws, rank, c5=True)
            ems, _ = timed(r["step"], max(3, args.steps // 2), 2, ws)
            e = {"ms_per_step": ems, "config": r["config"], "cells_per_s": r["cells"] / (ems * 1e-3),
                 "n_gpus": ws, "scaling": "strong"}
            del r
            torch.cuda.empty_cache()
        except Exception as ex:
            e = {"error": repr(ex)}
        if rank == 0:
            line.setdefault("workloads", {})["C5_map"] = e
    if rank == 0:
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
        g = np.random.default_rng(14020532 + 1)
        x = (g.standard_normal((rows, n)) + 1j * g.standard_normal((rows, n))) / np.sqrt(2)
        x = x.astype(np.complex64 if args.dtype == "c64" else np.complex128)
        dts = "f32" if args.dtype == "c64" else "f64"
        fn = lambda: oracle.ndft(x, dtype=dts, nthreads=P)  # noqa: E731
        ops = rows * n * n
        unit = "⊙/s"
        cfg = {"workload": "C2 batched NDFT (BASELINE.json configs[1])", "n": n, "batch": 65536,
               "sample_rows_per_step": rows}
        sample = f"{rows} CN(0,1) vectors of N={n} per step (bounded sample of C2)"
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
    ap.add_argument("--ndft-mode", default="tc", choices=["tc", "fast"],
                    help="C2 NDFT kernel: tc = tcgen05 sign-split GEMM (complex64), fast = FFMA2 CUDA-core kernel")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: contract requires >= 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
