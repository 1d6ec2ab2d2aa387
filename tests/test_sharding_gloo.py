"""Multi-process (world_size 2, gloo, CPU) coverage of the delay-bin sharding
host logic used for the multi-GPU map (paper_1402_0532_b200/sharded.py).

The per-row compute is replaced by a deterministic row function (rows are
independent, ambiguity.py:27-28), so the test checks partition + gather layout
without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1402_0532_b200.sharded import gather_rows, shard_rows


def test_shard_rows_partition():
    for L in (1, 7, 64, 1024, 4096, 4097):
        for G in (1, 2, 3, 4, 8):
            spans = [shard_rows(L, G, r) for r in range(G)]
            cover = []
            for f, c in spans:
                cover.extend(range(f, f + c))
            assert cover == list(range(L))
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        shard_rows(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _row_value(l, m):
    return torch.arange(m, dtype=torch.float64) * 1000.0 + l


def _worker(rank, world, port, L, M, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f, c = shard_rows(L, world, rank)
        local = torch.stack([_row_value(l, M) for l in range(f, f + c)]) if c else torch.empty(0, M, dtype=torch.float64)
        full = torch.full((L, M), -1.0, dtype=torch.float64) if rank == 0 else None
        out = gather_rows(local, full, L)
        if rank == 0:
            ok = all(torch.equal(out[l], _row_value(l, M)) for l in range(L))
            q.put(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L", [8, 9])
def test_gather_rows_world2(L):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, L, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


def _owner_line(k, base):
    """Restatement of LagDst::line (sa_lag_tc.cu): owner rank of the 16-lag tile k
    of the blocked z layout and the tile's index inside the owner's block
    (16-aligned shards: base = L / G rows each, base % 16 == 0)."""
    o = (16 * k) // base
    return o, k - o * (base // 16)


def test_block_sharded_tile_owners_match_shard_rows():
    """The block-sharded lag kernel stores the 16-lag tile k into the block of
    the rank that shard_rows gives those delay rows (the rank that runs their
    Doppler transform), at the owner-local tile index."""
    for L in (16, 64, 1024, 4096):
        for G in (1, 2, 4, 8):
            if L % (16 * G):
                continue
            base = L // G
            for r in range(G):
                f, c = shard_rows(L, G, r)
                for lag in range(f, f + c):
                    k, j = divmod(lag, 16)
                    o, kl = _owner_line(k, base)
                    assert o == r and 16 * kl + j == lag - f


def _blocks_worker(rank, world, port, L, M, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank integrates Doppler blocks shard_rows(M) for every delay row ...
        q0, qc = shard_rows(M, world, rank)
        zpart = torch.tensor([[1000.0 * l + qq for qq in range(q0, q0 + qc)] for l in range(L)])
        # ... and each 16-lag tile reaches its owner in the blocked layout
        # zb[(k * M + q) * 16 + j] (CPU stand-in for the kernel's peer sector stores)
        parts = [None] * world
        dist.all_gather_object(parts, (q0, zpart))
        f, c = shard_rows(L, world, rank)
        zb = torch.zeros(c * M)
        for (p0, zp) in parts:
            for k in range(L // 16):
                o, kl = _owner_line(k, L // world)
                if o != rank:
                    continue
                for j in range(16):
                    for qq in range(zp.shape[1]):
                        zb[(kl * M + p0 + qq) * 16 + j] = zp[16 * k + j, qq]
        # the owner's Doppler stage reads row (16 kl + j) element q from the same place
        mine = torch.tensor([[float(zb[((r // 16) * M + qq) * 16 + r % 16]) for qq in range(M)] for r in range(c)])
        want = torch.tensor([[1000.0 * l + qq for qq in range(M)] for l in range(f, f + c)])
        q.put(bool(torch.equal(mine, want)))
    finally:
        dist.destroy_process_group()


def test_block_sharded_exchange_world2():
    """World 2 (gloo): block partition of the lag stage + owner tiles give every
    rank exactly its delay rows over all Doppler blocks (uneven M)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_blocks_worker, args=(r, 2, port, 64, 9, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(res)
