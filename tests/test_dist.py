"""Multi-process (N > 1) host logic of bench.py on CPU with the gloo backend,
world size 2: weak-scaling workload partition and the max-over-ranks / sum
aggregation, plus the torchrun launch of the reference arm."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    b, k, alpha = bench.workload(rank, 1)
    sig = float(b.ce_col.astype(np.int64).sum() % 1000003)
    vals = bench.aggregate([10.0 * (rank + 1), 3.0 + rank, sig, b.n], ["sum", "max", "max", "sum"], world, "cpu")
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, sig, b.n, b.n_layouts))
    if rank == 0:
        out.put((vals, gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_partition_and_aggregation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, q), nprocs=2, join=True, start_method="spawn")
    vals, gathered = q.get(timeout=60)
    (r0, sig0, n0, l0), (r1, sig1, n1, l1) = sorted(gathered)
    assert l0 == l1 == 10 and n0 == n1  # same shape of work per rank (weak scaling)
    assert sig0 != sig1  # but different seeded layouts
    assert vals[0] == 30.0 and vals[1] == 4.0 and vals[3] == n0 + n1


@pytest.mark.slow
def test_reference_arm_under_torchrun():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "0", "--replicas", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "components/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
