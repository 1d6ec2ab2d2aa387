"""Multi-GPU ⊙ range-Doppler map: delay-bin sharding, rows written into the root.

One process per GPU (torch.distributed).  Rows are independent
(ambiguity.py:27-28; test_ambiguity.py:208-217), so rank r computes the
contiguous delay rows [r*L/G, (r+1)*L/G) with no exchange, and the map's only
data movement is getting the row blocks to the root -- a rank's block lands at
offset r*rows, which is exactly the row-major map.

Block-sharded lag stage (complex64 fast mode, T % 128 == 0: the tensor-core lag
kernel).  That kernel amortises each surveillance read over all lags of a block,
so splitting delay rows would leave every rank re-reading its blocks for a
fraction of the lags.  Instead rank r integrates Doppler blocks
[shard_rows(M, G, r)] for ALL delay rows and its kernel stores each z row
straight into the z buffer of the rank that owns that delay row (CUDA IPC,
NVLink/NVSwitch peer stores: the all-to-all is fused into the compute).  After
one stream-ordered completion all-reduce every rank runs the Doppler transform
of its own delay rows into the root's map (``ZExchange``, ``ambiguity_map_sharded``).

Two transports for the map rows:
  * "p2p" (default): compute and collective fused.  The root's map is shared
    once by CUDA IPC (``PeerMap``); every rank's Doppler-transform kernel
    stores its rows straight into it over NVLink/NVSwitch, so there is no
    separate gather -- a 1-element, stream-ordered NCCL all-reduce after the
    kernels is the only exchange (gloo groups: a host barrier).
  * "gather": the rows land locally and ``dist.gather`` (NCCL) moves them.

The host logic (partition, gather layout) is backend-agnostic and covered with
gloo on CPU (tests/test_sharding_gloo.py); on B200s the backend is NCCL over
NVLink/NVSwitch.
"""

from __future__ import annotations

import ctypes


def shard_rows(l_bins: int, world: int, rank: int) -> tuple[int, int]:
    """(first row, row count) of rank's contiguous delay-bin shard.

    Uneven L is allowed: the first L % G ranks get one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(l_bins, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def _wire(t):
    """NCCL has no complex types: collectives move the interleaved (re, im) view."""
    import torch
    return torch.view_as_real(t) if t is not None and t.is_complex() else t


def gather_rows(local, full, l_bins: int, group=None, dst: int = 0):
    """Gather every rank's row block into ``full`` (L x M) on ``dst``.

    Uses ``dist.gather`` when all shards have equal size (one collective),
    else point-to-point sends/recvs of the uneven blocks."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_rows(l_bins, world, r)[1] for r in range(world)]
    if len(set(sizes)) == 1:
        if rank == dst:
            parts = [_wire(full[shard_rows(l_bins, world, r)[0]:][: sizes[r]]) for r in range(world)]
            dist.gather(_wire(local), parts, dst=dst, group=group)
        else:
            dist.gather(_wire(local), None, dst=dst, group=group)
        return full if rank == dst else None
    if rank == dst:
        for r in range(world):
            f, c = shard_rows(l_bins, world, r)
            if r == dst:
                full[f:f + c].copy_(local)
            elif c:
                dist.recv(_wire(full[f:f + c]), src=r, group=group)
        return full
    if local.shape[0]:
        dist.send(_wire(local), dst=dst, group=group)
    return None


class PeerMapUnavailable(RuntimeError):
    """CUDA IPC mapping of the root's map is not possible on this system."""


class PeerMap:
    """The root's (L x M) map, writable by every rank's kernels.

    The root allocates it and exports its CUDA IPC handle (torch's storage
    export: handle + offset); every other rank opens the handle in its OWN
    device's context with lazy peer access (``sa_ipc_open``), so kernels on that
    device store rows straight into the root's memory over NVLink/NVSwitch.
    Collective to construct and to ``close``."""

    def __init__(self, l_bins: int, m: int, dtype, group=None, dst: int = 0):
        import torch
        import torch.distributed as dist
        from . import _native
        self.l_bins, self.m, self.dst, self.group = l_bins, m, dst, group
        self.rank = dist.get_rank(group)
        self.full = None
        self._mapped = None
        payload = [None]
        world = dist.get_world_size(group)
        if self.rank == dst:
            self.full = torch.empty((l_bins, m), dtype=dtype, device="cuda")
        if self.rank == dst and world > 1:
            try:
                payload = [self._export()]
            except Exception:  # every rank still reaches the broadcast below
                payload = [None]
        ok = True
        if world > 1:
            dist.broadcast_object_list(payload, src=dst, group=group)
            ok = payload[0] is not None
        self.row_bytes = m * torch.empty((), dtype=dtype).element_size()
        if self.rank == dst:
            self.base = self.full.data_ptr()
        elif ok:
            handle, offset = payload[0]
            hbuf = ctypes.create_string_buffer(handle, len(handle))
            p = ctypes.c_void_p()
            ok = _native.lib().sa_ipc_open(hbuf, ctypes.byref(p)) == 0
            if ok:
                self._mapped = p
                self.base = p.value + offset
        if world > 1:  # all ranks agree, so a failure cannot strand a peer in a collective
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                                device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            if int(flag.item()) == 0:
                if self._mapped is not None:
                    _native.lib().sa_ipc_close(self._mapped)
                    self._mapped = None
                raise PeerMapUnavailable("CUDA IPC mapping of the root's map failed on some rank")

    def _export(self):
        """(64-byte IPC handle, byte offset of the map in its allocation)."""
        info = self.full.untyped_storage()._share_cuda_()
        handle, storage_offset = bytes(info[1]), int(info[3])
        # torch's caching allocator exports [version byte,] a type byte ('c' =
        # cudaMalloc segment) and the 64-byte cudaIpcMemHandle_t; expandable
        # segments use another format
        if len(handle) >= 65 and handle[-65:-64] == b"c":
            handle = handle[-64:]
        if len(handle) != 64:
            raise RuntimeError("PeerMap needs a cudaMalloc-backed map (set "
                               "PYTORCH_CUDA_ALLOC_CONF=expandable_segments:False)")
        return (handle, storage_offset + self.full.storage_offset() * self.full.element_size())

    def done_flag(self):
        """A 1-element device tensor for the completion all-reduce."""
        import torch
        if getattr(self, "_flag", None) is None:
            self._flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        return self._flag

    def rows_ptr(self, first: int) -> int:
        """Device address (valid on this rank's GPU) of the root's row ``first``."""
        return self.base + first * self.row_bytes

    def close(self, barrier: bool = True) -> None:
        """Unmap the root's map on this rank (after this rank's kernels finished;
        with ``barrier``, after every rank's).  The root keeps ``full``."""
        import torch
        import torch.distributed as dist
        from . import _native
        torch.cuda.current_stream().synchronize()  # this rank's stores into the mapping are done
        if barrier:
            dist.barrier(group=self.group)  # nobody still writes
        if self._mapped is not None:
            _native.check(_native.lib().sa_ipc_close(self._mapped))
            self._mapped = None


def _ipc_export(t):
    """(64-byte cudaIpcMemHandle_t, byte offset of ``t`` in its allocation)."""
    info = t.untyped_storage()._share_cuda_()
    handle, storage_offset = bytes(info[1]), int(info[3])
    if len(handle) >= 65 and handle[-65:-64] == b"c":
        handle = handle[-64:]
    if len(handle) != 64:
        raise RuntimeError("IPC export needs a cudaMalloc-backed tensor (set "
                           "PYTORCH_CUDA_ALLOC_CONF=expandable_segments:False)")
    return handle, storage_offset + t.storage_offset() * t.element_size()


class ZExchange:
    """Every rank's block of lag-integrated rows z (its delay rows x M), mapped
    into every other rank by CUDA IPC: the block-sharded lag kernel stores z rows
    straight into their owner's block.  ``table`` is the device array of the G
    row-block bases as seen from this rank's GPU.  Collective to construct/close."""

    def __init__(self, l_bins: int, m: int, dtype, group=None):
        import torch
        import torch.distributed as dist
        from . import _native
        self.group = group
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        self.first, self.count = shard_rows(l_bins, world, rank)
        self.z = torch.empty((max(1, self.count), m), dtype=dtype, device="cuda")
        self._mapped = []
        mine = None
        try:
            mine = _ipc_export(self.z)
        except Exception:
            mine = None
        allp = [None] * world
        dist.all_gather_object(allp, mine, group=group)
        ok = all(a is not None for a in allp)
        bases = []
        if ok:
            for r, (handle, offset) in enumerate(allp):
                if r == rank:
                    bases.append(self.z.data_ptr())
                    continue
                hbuf = ctypes.create_string_buffer(handle, len(handle))
                p = ctypes.c_void_p()
                if _native.lib().sa_ipc_open(hbuf, ctypes.byref(p)) != 0:
                    ok = False
                    break
                self._mapped.append(p)
                bases.append(p.value + offset)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                            device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()) == 0:
            self.close(barrier=False)
            raise PeerMapUnavailable("CUDA IPC mapping of the z row blocks failed on some rank")
        self.table = torch.tensor(bases, dtype=torch.int64, device="cuda")

    def close(self, barrier: bool = True) -> None:
        import torch
        import torch.distributed as dist
        from . import _native
        torch.cuda.current_stream().synchronize()  # this rank's peer stores are done
        if barrier:
            dist.barrier(group=self.group)
        for p in self._mapped:
            _native.lib().sa_ipc_close(p)
        self._mapped = []


def _done(flag, group):
    """Stream-ordered completion point across ranks (NCCL: the all-reduce waits
    for this rank's kernels; gloo: host sync + barrier)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(flag, group=group)
    else:
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=group)


def blocks_shardable(surv, m: int, mode: str, lag: str, doppler: str, l_bins: int | None = None,
                     world: int = 1) -> bool:
    """Whether the block-sharded map applies: the tensor-core lag path
    (sa_lag_tc_supported: complex64 fast ⊙ lags, T % 128 == 0, T <= 4096), the
    NL-FFT Doppler transform on the blocked z layout (sa_doppler_nlfft_blocked:
    M = 64 .. 2048), and whole 16-lag tiles per rank (sa_ambiguity_integrate_blocks:
    L % (16 G) == 0).  Shapes only, so every rank agrees."""
    import torch
    tb = surv.numel() // m if m else 0
    return (surv.dtype == torch.complex64 and mode == "fast" and lag == "mf" and doppler == "nfft"
            and 128 <= tb <= 4096 and tb % 128 == 0 and 64 <= m <= 2048 and (m & (m - 1)) == 0
            and (l_bins is None or (l_bins >= world and l_bins % (16 * world) == 0)))


def map_blocks_sharded(surv, ref, l_bins: int, m: int, zx: ZExchange, pm: PeerMap, *, gain: float = 1.0,
                       conjugate_ref: bool = True, doppler: str = "nfft", group=None) -> None:
    """Block-sharded map (see module doc): lag stage over this rank's Doppler
    blocks for all delay rows, z rows delivered to their owners, then the Doppler
    transform of this rank's delay rows into the root's map (``blocks_shardable``
    must hold)."""
    import torch.distributed as dist
    from . import _native
    from ._device import sa_dtype_of
    from .twiddle import device_twiddles
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    q0, qc = shard_rows(m, world, rank)
    d = sa_dtype_of(surv)
    ns = surv.numel()
    rc = _native.lib().sa_ambiguity_integrate_blocks(
        d, _native.ptr(surv), _native.ptr(ref), ns, ref.numel(), 0, l_bins, m, q0, qc, int(conjugate_ref),
        _native.ptr(zx.table), world, _native.stream_ptr())
    _native.check(rc)
    _done(pm.done_flag(), group)  # every rank's z rows are in their owners' blocks
    if zx.count:  # Doppler NL-FFT of this rank's delay rows (blocked z) into the root's map
        tw = device_twiddles(m, d, surv.device.index)
        _native.check(_native.lib().sa_doppler_nlfft_blocked(d, _native.ptr(zx.z), ctypes.c_void_p(
            pm.rows_ptr(zx.first)), zx.count, m, ctypes.c_void_p(tw), float(gain), _native.stream_ptr()))
    _done(pm.done_flag(), group)  # every rank's rows are in the root's map


class MapStream:
    """Streaming block-sharded maps: CPIs submitted back to back, ``depth`` map /
    z buffer sets in flight.  Map i's lag stage (with its fused z-tile exchange)
    runs on the caller's stream; its delivery -- the completion all-reduce, the
    Doppler NL-FFT of this rank's rows into the root's map, the final
    all-reduce -- runs on a delivery stream, so map i+1's lag stage overlaps
    the root's ingress of map i (the 56 MB ingress at 8 GPUs costs
    as much as the compute).  Stream-ordered throughout: set k is reused only
    after the Doppler of map i - depth has read its z tiles.  ``flush()`` makes
    the caller's stream wait for every submitted map.  Collective: every rank
    submits the same sequence."""

    def __init__(self, l_bins: int, m: int, dtype, depth: int = 2, group=None, dst: int = 0):
        import torch
        self.l_bins, self.m, self.group, self.dst, self.depth = l_bins, m, group, dst, depth
        self.pms = [PeerMap(l_bins, m, dtype, group=group, dst=dst) for _ in range(depth)]
        try:
            self.zxs = [ZExchange(l_bins, m, dtype, group=group) for _ in range(depth)]
        except PeerMapUnavailable:
            for pm in self.pms:
                pm.close(barrier=False)
            raise
        self.delivery = torch.cuda.Stream()
        self.z_free = [None] * depth  # event: the Doppler of the previous map in set k has read its z
        self.i = 0

    def submit(self, surv, ref, *, gain: float = 1.0, conjugate_ref: bool = True):
        """Enqueue one map; returns the root's (L x M) map of this submission
        (valid once the caller's stream has passed a later ``flush()``), None
        on other ranks."""
        import torch
        import torch.distributed as dist
        from . import _native
        from ._device import sa_dtype_of
        from .twiddle import device_twiddles
        k = self.i % self.depth
        self.i += 1
        pm, zx = self.pms[k], self.zxs[k]
        world = dist.get_world_size(self.group)
        rank = dist.get_rank(self.group)
        cur = torch.cuda.current_stream()
        if self.z_free[k] is not None:
            cur.wait_event(self.z_free[k])
        q0, qc = shard_rows(self.m, world, rank)
        d = sa_dtype_of(surv)
        ns = surv.numel()
        _native.check(_native.lib().sa_ambiguity_integrate_blocks(
            d, _native.ptr(surv), _native.ptr(ref), ns, ref.numel(), 0, self.l_bins, self.m, q0, qc,
            int(conjugate_ref), _native.ptr(zx.table), world, _native.stream_ptr()))
        lag_done = torch.cuda.Event()
        lag_done.record(cur)
        with torch.cuda.stream(self.delivery):
            self.delivery.wait_event(lag_done)
            _done(pm.done_flag(), self.group)  # every rank's z tiles are in their owners' blocks
            if zx.count:
                tw = device_twiddles(self.m, d, surv.device.index)
                _native.check(_native.lib().sa_doppler_nlfft_blocked(
                    d, _native.ptr(zx.z), ctypes.c_void_p(pm.rows_ptr(zx.first)), zx.count, self.m,
                    ctypes.c_void_p(tw), float(gain), _native.stream_ptr()))
            ev = torch.cuda.Event()
            ev.record(self.delivery)
            self.z_free[k] = ev
            _done(pm.done_flag(), self.group)  # every rank's rows are in the root's map
        return pm.full if rank == self.dst else None

    def flush(self) -> None:
        import torch
        torch.cuda.current_stream().wait_stream(self.delivery)

    def close(self) -> None:
        import torch
        torch.cuda.current_stream().wait_stream(self.delivery)
        for zx in self.zxs:
            zx.close()
        for pm in self.pms:
            pm.close()


def _map_p2p(surv, ref, l_bins, m, pm, z_exchange, *, gain, conjugate_ref, doppler, mode, lag, group, dst,
             workspace):
    import torch
    import torch.distributed as dist
    from .ambiguity import ambiguity_map
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    first, count = shard_rows(l_bins, world, rank)
    if world > 1 and blocks_shardable(surv, m, mode, lag, doppler, l_bins, world):
        if surv.data_ptr() % 16:  # the tensor-core lag kernel reads 16-byte sample pairs
            surv = surv.clone()
        zx = z_exchange
        try:
            if zx is None:
                zx = ZExchange(l_bins, m, surv.dtype, group=group)
        except PeerMapUnavailable:  # (all ranks agree) delay-row shards instead
            zx = None
        if zx is not None:
            try:
                map_blocks_sharded(surv, ref, l_bins, m, zx, pm, gain=gain, conjugate_ref=conjugate_ref,
                                   doppler=doppler, group=group)
            except BaseException:
                if z_exchange is None:  # built here: released on the error path too (no collective)
                    zx.close(barrier=False)
                raise
            if z_exchange is None:
                zx.close()
            return pm.full if rank == dst else None
    if count:
        ambiguity_map(surv, ref, count, m, l0=first, gain=gain, conjugate_ref=conjugate_ref,
                      doppler=doppler, mode=mode, lag=lag, out_ptr=pm.rows_ptr(first), workspace=workspace)
    if dist.get_backend(group) == "nccl":
        # stream-ordered: NCCL's stream waits for this rank's transform kernel,
        # the caller's stream waits for the all-reduce -- once it completes on
        # the root, every rank's row stores into its map are done (no host sync)
        dist.all_reduce(pm.done_flag(), group=group)
    else:
        torch.cuda.current_stream().synchronize()  # this rank's rows are in the root's memory
        dist.barrier(group=group)                  # ... and so are everyone's
    return pm.full if rank == dst else None


def ambiguity_map_sharded(surv, ref, l_bins: int, m: int, *, gain: float = 1.0,
                          conjugate_ref: bool = True, doppler: str = "nfft", mode: str = "fast",
                          lag: str = "mf", group=None, dst: int = 0, transport: str = "p2p",
                          peer_map: PeerMap | None = None, out_full=None, out_local=None, workspace=None,
                          z_exchange: ZExchange | None = None):
    """Compute this rank's delay rows on its GPU and deliver them to ``dst``.

    surv/ref: full CUDA tensors on every rank (broadcast beforehand if needed).
    transport "p2p": rows are stored by the transform kernel straight into the
    root's map (``peer_map``, built here if not given), then one barrier;
    "gather": local rows + ``dist.gather``.  Returns the (L x M) map on
    ``dst``, None elsewhere."""
    import torch
    import torch.distributed as dist
    from .ambiguity import ambiguity_map
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    first, count = shard_rows(l_bins, world, rank)
    own_pm = False
    if transport == "p2p" and peer_map is None:
        try:
            peer_map = PeerMap(l_bins, m, surv.dtype, group=group, dst=dst)
            own_pm = True
        except PeerMapUnavailable:
            transport = "gather"
    if transport == "p2p":
        from .ambiguity import _dev
        surv, ref = _dev(surv, surv.dtype), _dev(ref, surv.dtype)  # as ambiguity_map: flat, contiguous, one dtype
        try:
            out = _map_p2p(surv, ref, l_bins, m, peer_map, z_exchange, gain=gain, conjugate_ref=conjugate_ref,
                           doppler=doppler, mode=mode, lag=lag, group=group, dst=dst, workspace=workspace)
        except BaseException:
            if own_pm:  # a mapping opened here is released on the error path too (no collective)
                peer_map.close(barrier=False)
            raise
        if own_pm:  # ... and after the final completion point otherwise
            peer_map.close()
        return out
    if transport != "gather":
        raise ValueError(f"unknown transport {transport!r}")
    if out_local is None:
        out_local = torch.empty((count, m), dtype=surv.dtype, device=surv.device)
    if count:
        ambiguity_map(surv, ref, count, m, l0=first, gain=gain, conjugate_ref=conjugate_ref,
                      doppler=doppler, mode=mode, lag=lag, out=out_local, workspace=workspace)
    if rank == dst and out_full is None:
        out_full = torch.empty((l_bins, m), dtype=surv.dtype, device=surv.device)
    return gather_rows(out_local, out_full, l_bins, group=group, dst=dst)


def broadcast_inputs(surv, ref, src: int = 0, group=None):
    """ncclBroadcast of the two input streams from ``src``."""
    import torch.distributed as dist
    dist.broadcast(_wire(surv), src=src, group=group)
    dist.broadcast(_wire(ref), src=src, group=group)
    return surv, ref


def ambiguity_map_multi_device(survs, refs, l_bins: int, m: int, devices, *, l0: int = 0, gain: float = 1.0,
                               conjugate_ref: bool = True, doppler: str = "nfft", mode: str = "fast",
                               lag: str = "mf"):
    """Single-process multi-GPU map through ``sa_ambiguity_map_multi`` (no NCCL,
    no torch.distributed): ``survs[g]`` / ``refs[g]`` are the inputs resident on
    ``devices[g]``; shard g's transform kernel stores its delay rows straight into
    the returned (l_bins x m) map on ``devices[0]`` (peer access).  Each shard runs
    on its own stream; the caller's current stream on ``devices[0]`` waits for all
    of them, so the result is stream-ordered like any other call."""
    import torch
    from . import _native
    from ._device import sa_dtype_of
    from .twiddle import device_twiddles
    G = len(devices)
    if not (len(survs) == len(refs) == G >= 1):
        raise ValueError("one surveillance / reference tensor per device")
    d = sa_dtype_of(survs[0])
    out = torch.empty((l_bins, m), dtype=survs[0].dtype, device=f"cuda:{devices[0]}")
    dop = {"nfft": _native.SA_DOPPLER_NLFFT, "ndft": _native.SA_DOPPLER_NDFT,
           "fft": _native.SA_DOPPLER_FFT_EXACT}[doppler]
    md = {"fast": _native.SA_NDFT_FAST, "exact": _native.SA_NDFT_EXACT}[mode]
    lk = {"mf": _native.SA_LAG_MF, "exact": _native.SA_LAG_EXACT}[lag]
    streams, ws, tws, ws_bytes = [], [], [], []
    for g, dev in enumerate(devices):
        with torch.cuda.device(dev):
            first, count = shard_rows(l_bins, G, g)
            need = ctypes.c_int64()
            _native.check(_native.lib().sa_ambiguity_workspace_bytes(d, max(1, count), m, ctypes.byref(need)))
            ws.append(torch.empty(max(1, need.value), dtype=torch.uint8, device=f"cuda:{dev}"))
            ws_bytes.append(ws[-1].numel())
            tws.append(device_twiddles(m, d, dev))
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream(dev))  # inputs / out are ordered on the current streams
            if dev != devices[0]:
                s.wait_stream(torch.cuda.current_stream(devices[0]))
            streams.append(s)
    P = ctypes.c_void_p
    arr = lambda xs: (P * G)(*xs)  # noqa: E731
    _native.check(_native.lib().sa_ambiguity_map_multi(
        G, (ctypes.c_int * G)(*devices), d, lk, arr([t.data_ptr() for t in survs]),
        arr([t.data_ptr() for t in refs]), survs[0].numel(), refs[0].numel(), l0, l_bins, m, float(gain),
        int(conjugate_ref), dop, md, arr(tws), P(out.data_ptr()), arr([w.data_ptr() for w in ws]),
        (ctypes.c_int64 * G)(*ws_bytes), arr([s.cuda_stream for s in streams])))
    root = torch.cuda.current_stream(devices[0])
    for s, w in zip(streams, ws):
        root.wait_stream(s)
        w.record_stream(s)
    return out
