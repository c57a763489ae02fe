"""World-size-2 CPU tests (gloo) of the multi-GPU host logic:
row tiles of each problem are split into contiguous work-balanced shards by
msot_shard_tiles (the product library's host code, no GPU needed), each rank
reduces its rows, and an all-gather assembles the full potential vector.  The
assembled result must be bitwise identical to the single-process one — the
property the NCCL path relies on (every row reduced in a fixed order)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_02010_b200 import solver

TILE = 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tiles(n):
    return np.append(np.arange(0, n, TILE), n)


def _worker(rank, world, port, n, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        O.set_threads(1)
        rng = np.random.default_rng(11)
        x, y = rng.random((n, 3)), rng.random((m, 3))
        logw = np.log(np.full(m, 1.0 / m))
        h = 0.01 * rng.standard_normal(m)
        ts = _tiles(n)
        # uneven per-tile work (as after truncation): rows x kept columns
        kept = rng.integers(1, m + 1, len(ts) - 1).astype(np.float64)
        work = np.diff(ts) * kept
        b = solver.shard_tiles(work, world)
        r0, r1 = ts[b[rank]], ts[b[rank + 1]]
        part = O.softmin(x[r0:r1], y, logw, h, 1e-2) if r1 > r0 else np.zeros(0)
        gathered = [None] * world
        dist.all_gather_object(gathered, (int(r0), part))
        out = np.zeros(n)
        for s0, p in gathered:
            out[s0:s0 + len(p)] = p
        if rank == 0:
            full = O.softmin(x, y, logw, h, 1e-2)
            q.put((np.array_equal(out, full), [float(work[b[r]:b[r + 1]].sum())
                                               for r in range(world)], float(work.max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1000, 2049])
def test_sharded_softmin_gather_bitwise(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, 700, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    same, parts, wmax = q.get(timeout=10)
    assert same
    assert abs(parts[0] - parts[1]) <= wmax


def test_shard_bounds_cover_and_balance():
    rng = np.random.default_rng(3)
    for world in (1, 2, 4, 8):
        for nt in (1, 7, 300):
            w = rng.random(nt) * 1000 + 1
            b = solver.shard_tiles(w, world)
            assert b[0] == 0 and b[-1] == nt and np.all(np.diff(b) >= 0)
            if nt >= world:
                parts = np.array([w[b[r]:b[r + 1]].sum() for r in range(world)])
                assert parts.max() - parts.min() <= 2 * w.max() + 1e-9
