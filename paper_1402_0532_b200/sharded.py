"""Multi-GPU ⊙ range-Doppler map: delay-bin sharding, rows written into the root.

One process per GPU (torch.distributed).  Rows are independent
(ambiguity.py:27-28; test_ambiguity.py:208-217), so rank r computes the
contiguous delay rows [r*L/G, (r+1)*L/G) with no exchange, and the map's only
data movement is getting the row blocks to the root -- a rank's block lands at
offset r*rows, which is exactly the row-major map.

Two transports:
  * "p2p" (default): compute and collective fused.  The root's map is shared
    once by CUDA IPC (``PeerMap``); every rank's Doppler-transform kernel
    stores its rows straight into it over NVLink/NVSwitch, so there is no
    separate gather -- a host barrier after the kernels is the only exchange.
  * "gather": the rows land locally and ``dist.gather`` (NCCL) moves them.

The host logic (partition, gather layout) is backend-agnostic and covered with
gloo on CPU (tests/test_sharding_gloo.py); on B200s the backend is NCCL over
NVLink/NVSwitch.
"""

from __future__ import annotations


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


class PeerMap:
    """The root's (L x M) map, visible to every rank: the root allocates it and
    shares it once through CUDA IPC (torch's own tensor reduction); the other
    ranks open it and enable peer access from their device, so their kernels
    can store rows into it directly.  Collective to construct."""

    def __init__(self, l_bins: int, m: int, dtype, group=None, dst: int = 0):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        from . import _native
        self.l_bins, self.m, self.dst = l_bins, m, dst
        self.rank = dist.get_rank(group)
        self.full = None
        payload = [None]
        if self.rank == dst:
            self.full = torch.empty((l_bins, m), dtype=dtype, device="cuda")
            payload = [reduce_tensor(self.full)]
        dist.broadcast_object_list(payload, src=dst, group=group)
        if self.rank == dst:
            self.view = self.full
        else:
            fn, args = payload[0]
            self.view = fn(*args)  # IPC mapping of the root's map
            _native.check(_native.lib().sa_enable_peer_access(self.view.device.index))

    def rows(self, first: int, count: int):
        """The root's rows [first, first + count) as seen from this rank."""
        return self.view[first:first + count]


def ambiguity_map_sharded(surv, ref, l_bins: int, m: int, *, gain: float = 1.0,
                          conjugate_ref: bool = True, doppler: str = "nfft", mode: str = "fast",
                          lag: str = "mf", group=None, dst: int = 0, transport: str = "p2p",
                          peer_map: PeerMap | None = None, out_full=None, out_local=None, workspace=None):
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
    if transport == "p2p":
        pm = peer_map if peer_map is not None else PeerMap(l_bins, m, surv.dtype, group=group, dst=dst)
        if count:
            ambiguity_map(surv, ref, count, m, l0=first, gain=gain, conjugate_ref=conjugate_ref,
                          doppler=doppler, mode=mode, lag=lag, out=pm.rows(first, count), workspace=workspace)
        torch.cuda.current_stream().synchronize()  # this rank's rows are in the root's memory
        dist.barrier(group=group)                  # ... and so are everyone's
        return pm.full if rank == dst else None
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
