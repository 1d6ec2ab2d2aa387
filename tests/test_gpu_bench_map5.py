"""The multi-GPU map path of bench.py (--workload map5, C5: 4096 x 2048 from
2^22 samples) with two ranks.  One GPU per box and NCCL refuses two ranks on
one device (profiles/round2_nccl_same_gpu.txt), so both ranks share cuda:0 with
a gloo process group for the handshake and barriers; everything else is the
production path: the block-sharded tensor-core lag stage storing 16-lag z
tiles into the owner rank's CUDA-IPC-mapped block, each rank's Doppler NL-FFT
storing its rows into rank 0's IPC-mapped map.  The delivered map must equal a
single-call map bit for bit (bench.py --check)."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_bench_map5_two_ranks_shared_gpu(sa):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--workload", "map5", "--dist-backend", "gloo", "--share-gpu", "--check", "--steps", "2",
           "--warmup", "3", "--no-cpu", "--no-e2e", "--no-extras"]
    env = dict(os.environ, PYTORCH_CUDA_ALLOC_CONF="expandable_segments:False")
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-4000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert "Doppler-block shards x2" in line["config"]["parallelism"]
    assert line["map_check"]["bit_identical"] is True, line["map_check"]
    st = line["workloads"]["C5_map_stream"]  # two CPIs in flight (sharded.MapStream)
    assert st["map_check"]["bit_identical"] is True and st["config"]["maps_in_flight"] == 2
