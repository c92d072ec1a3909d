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


def _worker_compact(rank, world, port, out):
    """bench.exchange_compact on CPU tensors: each rank owns a different part
    of one colouring (different list lengths); the gathered lists, applied to
    an all -1 array the way mpld_shard_import does, give the whole colouring."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    import bench
    n = 1000
    rng = np.random.default_rng(5)
    full = rng.integers(0, 4, n).astype(np.int32)
    owner = rng.choice(world + 1, n, p=[0.5, 0.2, 0.3])  # owner == world: a hidden vertex nobody searched
    mine = np.nonzero(owner == rank)[0]
    pairs = np.full(2 * n, 12345, dtype=np.int32)  # capacity 2n, garbage past the list (the export buffer)
    pairs[0:2 * mine.size:2] = mine
    pairs[1:2 * mine.size:2] = full[mine]
    got = bench.exchange_compact(torch.from_numpy(pairs), torch.tensor([mine.size], dtype=torch.int64), world)
    colors = np.full(n, -1, dtype=np.int32)
    g = got.numpy().reshape(-1, 2)
    for v, c in g:  # mpld_shard_import's rule
        if 0 <= v < n:
            colors[v] = c
    want = np.where(owner < world, full, -1)
    out.put((rank, bool(np.array_equal(colors, want)), int(g.shape[0]), int((g[:, 0] < 0).sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_compact_colour_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker_compact, args=(2, port, q), nprocs=2, join=True, start_method="spawn")
    res = sorted(q.get(timeout=60) for _ in range(2))
    assert all(ok for _, ok, _, _ in res)
    assert res[0][2] == res[1][2] and res[0][3] > 0  # equal gathered lengths; the shorter list was padded


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
