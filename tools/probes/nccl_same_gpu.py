"""Probe: can two NCCL ranks share one GPU (the 1-GPU box)?  Prints the outcome."""
import os, sys
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("nccl", rank=rank, world_size=2, device_id=torch.device("cuda", 0))
        t = torch.ones(4, device="cuda") * (rank + 1)
        dist.all_reduce(t)
        torch.cuda.synchronize()
        q.put((rank, "ok", float(t[0])))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e)[:400]))


if __name__ == "__main__":
    import socket
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, port, q)) for r in range(2)]
    for p in ps: p.start()
    res = []
    for _ in ps:
        try:
            res.append(q.get(timeout=90))
        except Exception as e:  # noqa: BLE001
            res.append(("?", "timeout", repr(e)))
    for p in ps:
        p.join(10)
        if p.is_alive(): p.kill()
    for r in sorted(res, key=str): print(r)
