"""Multi-rank solves on one GPU through the host-collective test seam
(msot_create_dist_host): two processes, each a rank with its own context on
cuda:0, exchanging column sums (all-reduce) and row shards (broadcast) over
gloo instead of NCCL.  The sharded result must match the single-rank solve:
bitwise for row-wise pair sets (dense solves, pair_eval 0: every row reduced
by one rank in an item order that does not depend on the rank count); for
the evaluate-once path the per-rank float64 column partials are all-reduced
and rounded once, which is bitwise in every case measured and bounded here
at 1e-5 eps."""
import math
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _mixture(n, seed):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.2, 0.8, (6, 3))
    return cen[rng.integers(0, 6, n)] + rng.normal(0, 0.05, (n, 3))


CASES = {
    "dense": dict(blur=0.05),
    "multiscale": dict(blur=0.01, multiscale=True, retruncate=1, cluster_scale=0.04),
    "unbalanced": dict(blur=0.02, reach=0.3, multiscale=True, retruncate=1, cluster_scale=0.04),
    # row-wise pair sets (pair_eval 0): every row reduced by its own rank in a
    # fixed item order -> bitwise identical for any number of GPUs
    "multiscale_rowwise": dict(blur=0.01, multiscale=True, retruncate=1, cluster_scale=0.04,
                               pair_eval=0),
}
BITWISE = ("dense", "multiscale_rowwise", "bench_rowwise")


def _inputs(case):
    if case.startswith("bench"):  # bench.py's generator and parameters at 30k
        import bench
        w = dict(bench.WORKLOAD, n=30000, m=30000)
        return bench.make_inputs(w)
    if case.startswith("hd"):
        from paper_2107_02010_b200 import workloads as W
        fa, _ = W.fibres(700, 3)
        fb, _ = W.fibres(600, 4)
        x, a = W.encode_fibers(fa)
        y, b = W.encode_fibers(fb)
        return x, a, y, b
    x, y = _mixture(4000, 1), _mixture(3500, 2)
    return x, np.full(4000, 1 / 4000), y, np.full(3500, 1 / 3500)


def _params(case):
    from paper_2107_02010_b200.abi import make_params
    if case.startswith("bench"):
        import bench
        prm = bench.params(dict(bench.WORKLOAD, n=30000, m=30000))
        if case == "bench_rowwise":
            prm.pair_eval = 0
        return prm
    if case == "hd":
        return make_params(blur=0.05, reach=0.3)
    if case == "hd_ms":
        return make_params(blur=0.03, reach=0.3, multiscale=True, retruncate=1,
                           switch_factor=1.0, clusters=10)
    return make_params(**CASES[case])


def _worker(rank, world, port, case, q, env=None):
    import sys
    import traceback
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(env or {})
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import datetime
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                timeout=datetime.timedelta(seconds=120))
        from paper_2107_02010_b200.solver import Context

        def ar(a):
            dist.all_reduce(torch.from_numpy(a))

        def bc(a, root):
            dist.broadcast(torch.from_numpy(a), src=root)

        ctx = Context(0, rank, world, host_collectives=(ar, bc))
        x, a, y, b = _inputs(case)
        loss, pots, st = ctx.sinkhorn(_params(case), x, a, y, b)
        ctx.close()
        q.put((rank, "ok", (loss, [pots.a_xx, pots.b_yy, pots.a_xy, pots.b_yx], st["world"])))
        dist.destroy_process_group()
    except BaseException:
        q.put((rank, "error", traceback.format_exc()))


def run_two_ranks(case, timeout=300, world=2, env=None):
    """Rank results {rank: (loss, potentials, world)}; raises with the worker
    traceback on failure and never leaves a worker behind."""
    import queue
    import torch.multiprocessing as mp
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, world, port, case, q, env), daemon=True)
             for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        while len(out) < world:
            rank, status, payload = q.get(timeout=timeout)
            if status != "ok":
                raise AssertionError(f"rank {rank} failed:\n{payload}")
            out[rank] = payload
    except queue.Empty:
        raise AssertionError(f"two-rank {case} solve timed out after {timeout}s")
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    return out


def _check_ranks(case, l1, p1, out, world):
    ref = [p1.a_xx, p1.b_yy, p1.a_xy, p1.b_yx]
    eps = _params(case).blur ** 2
    for rank in range(world):
        lw, pw, w = out[rank]
        assert w == world
        for u, v in zip(pw, ref):
            if case in BITWISE:
                np.testing.assert_array_equal(u, v)
            else:
                # evaluate-once: the per-rank float64 column partials are
                # added in another association and rounded once to float32,
                # so a column total can differ by one float32 ulp only where
                # the float64 sums straddle a rounding point (bitwise in
                # every case measured, tools/rank_diff.py)
                assert np.abs(u - v).max() <= 1e-5 * eps
        if case in BITWISE:
            assert lw == l1
        else:
            assert abs(lw - l1) <= 1e-9 * abs(l1) + 1e-15


@pytest.mark.parametrize("case", ["dense", "multiscale", "unbalanced", "hd", "hd_ms",
                                  "multiscale_rowwise"])
def test_two_ranks_match_one(ctx, case):
    x, a, y, b = _inputs(case)
    l1, p1, _ = ctx.sinkhorn(_params(case), x, a, y, b)
    _check_ranks(case, l1, p1, run_two_ranks(case), 2)


@pytest.mark.parametrize("case", ["multiscale", "hd_ms", "multiscale_rowwise"])
def test_three_ranks_match_one(ctx, case):
    """Uneven shards: three ranks (row tiles, mask rows and broadcast blocks
    split 3 ways)."""
    x, a, y, b = _inputs(case)
    l1, p1, _ = ctx.sinkhorn(_params(case), x, a, y, b)
    _check_ranks(case, l1, p1, run_two_ranks(case, world=3), 3)


def test_four_ranks_bench_parameters_rowwise_bitwise(ctx):
    """bench.py's parameters at 30k with row-wise pair sets on four ranks and
    forced small colpart batches: bitwise the one-rank solve (item cuts do
    not depend on the rank count)."""
    x, a, y, b = _inputs("bench_rowwise")
    l1, p1, _ = ctx.sinkhorn(_params("bench_rowwise"), x, a, y, b)
    out = run_two_ranks("bench_rowwise", world=4, env={"MSOT_COLPART_BUDGET": "200000"})
    _check_ranks("bench_rowwise", l1, p1, out, 4)


def test_four_ranks_bench_parameters_batched(ctx):
    """bench.py's C3 parameters (theta 12.5, switch r_max, automatic voxel edge
    and super level) at 30k on four ranks, with the column partials forced
    into many small batches per update (MSOT_COLPART_BUDGET): shard cuts,
    batch boundaries and the two exchange steps together, against the
    one-rank solve with the automatic budget."""
    x, a, y, b = _inputs("bench")
    l1, p1, s1 = ctx.sinkhorn(_params("bench"), x, a, y, b)
    assert s1["t_super"] > 0 or s1["t_switch"] > 0
    out = run_two_ranks("bench", world=4, env={"MSOT_COLPART_BUDGET": "200000"})
    _check_ranks("bench", l1, p1, out, 4)


@pytest.mark.parametrize("case", ["dense", "multiscale", "unbalanced", "hd_ms"])
def test_nccl_one_rank_communicator(ctx, case):
    """The product's NCCL path on one GPU: a context made by msot_create_dist
    with world = 1 holds a one-rank communicator, and the solver issues its
    real ncclAllReduce (column sums) and grouped ncclBroadcast (row shards,
    mask row blocks) calls on the solver stream.  With one rank they move no
    data, so the result must equal the communicator-less solve bitwise."""
    from paper_2107_02010_b200.solver import Context
    x, a, y, b = _inputs(case)
    l1, p1, _ = ctx.sinkhorn(_params(case), x, a, y, b)
    c1 = Context(0, 0, 1, Context.nccl_unique_id())
    try:
        assert c1.world_info() == (0, 1, 1)  # ncclCommCount
        l2, p2, st = c1.sinkhorn(_params(case), x, a, y, b)
    finally:
        c1.close()
    assert st["world"] == 1
    for u, v in zip([p2.a_xx, p2.b_yy, p2.a_xy, p2.b_yx], [p1.a_xx, p1.b_yy, p1.a_xy, p1.b_yx]):
        np.testing.assert_array_equal(u, v)
    assert l2 == l1


def test_nccl_one_rank_batched_bench_parameters(ctx):
    """The one-rank communicator under bench.py's parameters with the column
    partials in many small batches: the NCCL calls sit between batched
    updates on two streams; the result equals the communicator-less solve."""
    from paper_2107_02010_b200.solver import Context
    x, a, y, b = _inputs("bench")
    c0 = Context(0)
    c1 = Context(0, 0, 1, Context.nccl_unique_id())
    try:
        for c in (c0, c1):
            c.set_colpart_budget(200000)
        l0, p0, s0 = c0.sinkhorn(_params("bench"), x, a, y, b)
        l1, p1, s1 = c1.sinkhorn(_params("bench"), x, a, y, b)
    finally:
        c0.close()
        c1.close()
    assert s1["colpart_batches"] > 2
    for u, v in zip([p1.a_xx, p1.b_yy, p1.a_xy, p1.b_yx], [p0.a_xx, p0.b_yy, p0.a_xy, p0.b_yx]):
        np.testing.assert_array_equal(u, v)
    assert l1 == l0


if __name__ == "__main__":
    import sys
    for case in sys.argv[1:]:
        res = run_two_ranks(case)
        print(case, {r: v[0] for r, v in res.items()}, flush=True)
