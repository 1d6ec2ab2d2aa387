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
