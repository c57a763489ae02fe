"""The shared policies (policy.h) against an independent numpy restatement
(tests/independent.py), for the oracle (CPU) and the GPU: clustering
bit-exact, the automatic voxel edge, the switch and super-level indices of a
solve at bench.py's parameters, and the truncation mask up to pairs within
rounding of the threshold."""
import math

import numpy as np
import pytest

import bench
import independent as I
from paper_2107_02010_b200.abi import make_params


def _cloud(n, seed, d):
    rng = np.random.default_rng(seed)
    x = bench.mixture(n, seed, d) if d == 3 else rng.normal(0.5, 0.15, (n, d))
    # atoms exactly on voxel faces and duplicates
    x[: n // 20] = np.round(x[: n // 20] * 32) / 32
    x[n // 20: n // 10] = x[0]
    return x


def _check_clusters(got, ref):
    assert got["k"] == ref["k"]
    np.testing.assert_array_equal(got["perm"], ref["perm"])
    np.testing.assert_array_equal(got["labels"], ref["labels"])
    np.testing.assert_array_equal(got["offsets"], ref["offsets"])
    np.testing.assert_allclose(got["cweights"], ref["cweights"], rtol=1e-12)
    np.testing.assert_allclose(got["centroids"], ref["centroids"], rtol=0, atol=1e-6)
    # radii are float32, rounded up from the float64 distance
    r, r64 = np.asarray(got["radii"], np.float64), ref["radii"]
    assert np.all(r >= r64 * (1 - 1e-6) - 1e-7) and np.all(r <= r64 * (1 + 1e-5) + 1e-6)


def test_schedule_spec_examples():
    np.testing.assert_allclose(I.schedule(8.0, 1.0, 0.5), [8, 4, 2, 1])
    rng = np.random.default_rng(0)
    for _ in range(100):
        d, blur, q = rng.uniform(0.5, 4), rng.uniform(1e-3, 0.4), rng.uniform(0.3, 0.95)
        want = math.ceil(math.log(d / blur) / math.log(1 / q))
        assert len(I.schedule(d, blur, q)) in (want, want + 1)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_grid_cluster_oracle_vs_independent(oracle, d):
    x = _cloud(20000, 40 + d, d)
    w = np.random.default_rng(d).random(len(x)) + 0.5
    lo = x.min(0)
    _check_clusters(oracle.grid_cluster(x, w, lo, 0.03), I.grid_cluster(x, w, lo, 0.03))


def _policy_case(n):
    w = dict(bench.WORKLOAD, n=n, m=n)
    x, a, y, b = bench.make_inputs(w)
    return x, a, y, b, bench.params(w)


def _check_policies(st, x, y, prm):
    cell, lo, hi = I.auto_cell(x, y)
    assert st["cluster_scale"] == pytest.approx(cell, rel=1e-12)
    cx, cy = I.grid_cluster(x, np.ones(len(x)), lo, cell), I.grid_cluster(y, np.ones(len(y)), lo, cell)
    assert (st["kx"], st["ky"]) == (cx["k"], cy["k"])
    sig = I.schedule(math.dist(lo, hi), prm.blur, prm.scaling)
    assert st["n_scales"] == len(sig)
    rmax = max(cx["radii"].max(), cy["radii"].max())
    assert st["t_switch"] == I.switch_index(sig, rmax, prm.switch_factor)
    assert st["t_super"] == I.super_switch(sig, st["t_switch"], cell, x.shape[1],
                                           max(cx["k"], cy["k"]), prm.super_level)


def test_solver_policies_oracle_vs_independent(oracle):
    """Voxel edge, cluster counts, schedule, switch and super level of an
    oracle solve at bench.py's parameters (20k atoms: super level off)."""
    x, a, y, b, prm = _policy_case(20000)
    _, _, st = oracle.sinkhorn(prm, x, a, y, b, potentials=False)
    _check_policies(st, x, y, prm)


def _mask_case(seed, self_):
    rng = np.random.default_rng(seed)
    kx = 400
    ky = kx if self_ else 350
    f32 = lambda v: np.asarray(v, np.float32)
    cx = f32(rng.random((kx, 3)))
    cy = cx if self_ else f32(rng.random((ky, 3)))
    rx = f32(rng.random(kx) * 0.05)
    ry = rx if self_ else f32(rng.random(ky) * 0.05)
    fx = f32(rng.random(kx) * 0.01)
    gy = fx if self_ else f32(rng.random(ky) * 0.01)
    gx = f32(np.concatenate([rng.normal(0, 0.2, (kx, 3)), fx[:, None] + 0.001], 1))
    hy = gx if self_ else f32(np.concatenate([rng.normal(0, 0.2, (ky, 3)), gy[:, None] + 0.001], 1))
    # member boxes inside the radius ball's bounding cube, lo <= 0 <= hi
    bx = f32(np.concatenate([-rng.random((kx, 3)) * rx[:, None], rng.random((kx, 3)) * rx[:, None]], 1))
    by = bx if self_ else f32(np.concatenate([-rng.random((ky, 3)) * ry[:, None],
                                              rng.random((ky, 3)) * ry[:, None]], 1))
    return cx, rx, fx, cy, ry, gy, gx, hy, bx, by


def _check_mask(got, args, eps, theta, self_, slopes, boxes=False):
    cx, rx, fx, cy, ry, gy, gx, hy, bx, by = args
    sl = I.slack(cx, rx, fx, cy, ry, gy, gx if slopes else None, hy if slopes else None,
                 bx if boxes else None, by if boxes else None)
    want = I.mask(sl, eps, theta, self_)
    diff = got.astype(bool) != want
    # disagreements only where the slack is within rounding of the threshold
    near = np.abs(sl + theta * eps) <= 1e-9 * (1.0 + np.abs(sl))
    assert not (diff & ~near).any(), np.argwhere(diff & ~near)[:5]
    assert 0 < want.mean() < 1


RULES = [(False, False), (True, False), (True, True)]  # (slopes, boxes)


@pytest.mark.parametrize("self_", [False, True])
@pytest.mark.parametrize("slopes,boxes", RULES)
def test_mask_oracle_vs_independent(oracle, self_, slopes, boxes):
    args = _mask_case(7, self_)
    cx, rx, fx, cy, ry, gy, gx, hy, bx, by = args
    for eps, theta in ((1e-3, 20.0), (1e-4, 5.0)):
        got = oracle.truncation_mask(cx, rx, fx, cy, ry, gy, eps, theta, self_=self_,
                                     gx=gx if slopes else None, hy=hy if slopes else None,
                                     bx=bx if boxes else None, by=by if boxes else None)
        _check_mask(got, args, eps, theta, self_, slopes, boxes)


def test_box_bound_tightens(oracle):
    """The box bound only removes pairs (min of three bounds) and does remove
    some on this data."""
    args = _mask_case(9, False)
    cx, rx, fx, cy, ry, gy, gx, hy, bx, by = args
    a = oracle.truncation_mask(cx, rx, fx, cy, ry, gy, 1e-3, 20.0, gx=gx, hy=hy)
    b = oracle.truncation_mask(cx, rx, fx, cy, ry, gy, 1e-3, 20.0, gx=gx, hy=hy, bx=bx, by=by)
    assert not (b.astype(bool) & ~a.astype(bool)).any()
    assert b.sum() < a.sum()


# ------------------------------------------------------------------ GPU ---
@pytest.mark.gpu
@pytest.mark.parametrize("d", [1, 2, 3])
def test_grid_cluster_gpu_vs_independent(ctx, d):
    x = _cloud(50000, 50 + d, d)
    w = np.random.default_rng(d).random(len(x)) + 0.5
    lo = x.min(0)
    _check_clusters(ctx.grid_cluster(x, w, lo, 0.02), I.grid_cluster(x, w, lo, 0.02))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [20000, 1000000])
def test_solver_policies_gpu_vs_independent(ctx, n):
    """The same decisions on the GPU, up to C3 itself (1M: super level on)."""
    x, a, y, b, prm = _policy_case(n)
    _, _, st = ctx.sinkhorn(prm, x, a, y, b, potentials=False)
    _check_policies(st, x, y, prm)
    if n >= 1000000:
        assert st["t_super"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("self_", [False, True])
@pytest.mark.parametrize("slopes,boxes", RULES)
def test_mask_gpu_vs_independent(ctx, oracle, self_, slopes, boxes):
    """GPU masks against the restatement, and bit-exact against the oracle."""
    args = _mask_case(8, self_)
    cx, rx, fx, cy, ry, gy, gx, hy, bx, by = args
    for eps, theta in ((1e-3, 20.0), (1e-4, 5.0)):
        kw = dict(self_=self_, gx=gx if slopes else None, hy=hy if slopes else None,
                  bx=bx if boxes else None, by=by if boxes else None)
        got = ctx.kernel_truncation(cx, rx, fx, cy, ry, gy, eps, theta, **kw)
        _check_mask(got, args, eps, theta, self_, slopes, boxes)
        np.testing.assert_array_equal(got, oracle.truncation_mask(cx, rx, fx, cy, ry, gy, eps,
                                                                  theta, **kw))
