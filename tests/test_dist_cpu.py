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


def _sym_worker(rank, world, port, n, m, q):
    """Evaluate-once protocol of one scale: each rank owns a
    contiguous run of 256-row tiles of x; per tile it evaluates the cross
    block (rows x, all y) once -> row sums of its x rows and column partials
    for every y; the self block x-x over its diagonal + upper columns -> row
    sums, and column partials for the upper columns.  Column partials are
    all-reduced (NCCL in the product, gloo here), then every rank finalises
    its own rows (row part + column part) and all of a_xy.  Compared with the
    single-process dense sums."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        x, y = rng.random((n, 3)), rng.random((m, 3))
        a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
        f, g = 0.01 * rng.standard_normal(n), 0.01 * rng.standard_normal(m)
        eps = 0.05
        ts = _tiles(n)
        bnd = solver.shard_tiles(np.diff(ts).astype(np.float64) * m, world)
        row_cross = np.zeros(n)       # b_yx row sums (own rows)
        col_cross = np.zeros(m)       # a_xy column partials (all columns)
        row_self = np.zeros(n)        # a_xx row part (own rows)
        col_self = np.zeros(n)        # a_xx column part (all columns)
        for t in range(bnd[rank], bnd[rank + 1]):
            r0, r1 = ts[t], ts[t + 1]
            k = np.exp((f[r0:r1, None] + g[None, :]
                        - 0.5 * ((x[r0:r1, None] - y[None]) ** 2).sum(-1)) / eps)
            row_cross[r0:r1] = (k * b[None, :]).sum(1)
            col_cross += (k * a[r0:r1, None]).sum(0)
            ks = np.exp((f[r0:r1, None] + f[None, r0:] - 0.5 * ((x[r0:r1, None] - x[None, r0:]) ** 2).sum(-1)) / eps)
            row_self[r0:r1] = (ks * a[None, r0:]).sum(1)           # diagonal block + upper
            col_self[r1:] += (ks[:, r1 - r0:] * a[r0:r1, None]).sum(0)  # upper columns only
        ct = torch.from_numpy(np.concatenate([col_cross, col_self]))
        dist.all_reduce(ct, op=dist.ReduceOp.SUM)
        col_cross, col_self = ct.numpy()[:m], ct.numpy()[m:]
        r0, r1 = ts[bnd[rank]], ts[bnd[rank + 1]]
        mine = (int(r0), row_cross[r0:r1].copy(), (row_self + col_self)[r0:r1].copy())
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        byx, axx = np.zeros(n), np.zeros(n)
        for s0, rc, rs in gathered:
            byx[s0:s0 + len(rc)] = rc
            axx[s0:s0 + len(rs)] = rs
        if rank == 0:
            k = np.exp((f[:, None] + g[None, :] - 0.5 * ((x[:, None] - y[None]) ** 2).sum(-1)) / eps)
            ks = np.exp((f[:, None] + f[None, :] - 0.5 * ((x[:, None] - x[None]) ** 2).sum(-1)) / eps)
            ok = (np.allclose(byx, (k * b[None]).sum(1), rtol=1e-12)
                  and np.allclose(col_cross, (k * a[:, None]).sum(0), rtol=1e-12)
                  and np.allclose(axx, (ks * a[None]).sum(1), rtol=1e-12))
            q.put(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [700, 1300])
def test_evaluate_once_protocol_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sym_worker, args=(r, 2, port, n, 600, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10)
