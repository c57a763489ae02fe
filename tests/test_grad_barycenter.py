"""grad_positions and the barycenter (BASELINE configs 5):
the oracle against finite differences / closed forms (CPU), the GPU against
the oracle on the same inputs (gpu)."""
import math

import numpy as np
import pytest

from paper_2107_02010_b200.abi import make_params


def test_oracle_grad_finite_differences(oracle):
    """Acceptance 3: central differences, h = 1e-4 d.  The
    envelope theorem needs converged potentials; with one averaged update
    per scale that takes q close to 1 (q=0.95 leaves ~10% error, q=0.9995
    1.5e-3), so the test runs the literal algorithm at q = 0.99995."""
    rng = np.random.default_rng(0)
    n, m = 8, 10
    x, y = rng.random((n, 2)), rng.random((m, 2))
    a = rng.random(n) + 0.5
    a /= a.sum()
    b = np.full(m, 1 / m)
    prm = make_params(blur=0.1, scaling=0.99995, max_full_iters=100000)
    nthreads = oracle.threads()
    oracle.set_threads(1)  # 5e4 tiny scales: the pool dispatch would dominate
    try:
        _, g = oracle.sinkhorn_grad(prm, x, a, y, b)
        fd = _fd(oracle, prm, x, a, y, b)
    finally:
        oracle.set_threads(nthreads)
    assert np.abs(fd - g).max() <= 1e-3 * np.abs(fd).max()


def _fd(oracle, prm, x, a, y, b):
    n = len(x)
    h = 1e-4 * math.sqrt(2)
    fd = np.zeros_like(x)
    for i in range(n):
        for k in range(2):
            xp, xm = x.copy(), x.copy()
            xp[i, k] += h
            xm[i, k] -= h
            fd[i, k] = (oracle.sinkhorn(prm, xp, a, y, b, False)[0] -
                        oracle.sinkhorn(prm, xm, a, y, b, False)[0]) / (2 * h)
    return fd


def test_oracle_grad_translation(oracle):
    """beta = alpha + t -> gradient ~ -alpha_i t (5%)."""
    rng = np.random.default_rng(1)
    x = rng.random((50, 2))
    t = np.array([0.3, 0.1])
    a = np.full(50, 1 / 50)
    _, g = oracle.sinkhorn_grad(make_params(blur=0.01), x, a, x + t, a)
    assert np.abs(g + a[:, None] * t).max() <= 0.05 * a[0] * np.linalg.norm(t)
    _, g0 = oracle.sinkhorn_grad(make_params(blur=0.01), x, a, x, a)
    assert np.abs(g0).max() <= 1e-6 * a[0]


def test_oracle_barycenter_midpoint(oracle):
    """targets delta_{-1}, delta_{+1}, init delta_{0.3} -> 0."""
    x, traj = oracle.barycenter(make_params(blur=0.01), np.array([[0.3]]), np.ones(1),
                                [(np.array([[-1.0]]), np.ones(1)),
                                 (np.array([[1.0]]), np.ones(1))], iters=20)
    assert abs(x[0, 0]) <= 0.01
    assert np.all(np.diff(traj) <= 0)


def blobs(seed, n, shift):
    rng = np.random.default_rng(seed)
    return rng.normal(0.5, 0.08, (n, 3)) + shift


@pytest.mark.gpu
@pytest.mark.parametrize("multiscale", [False, True])
def test_grad_matches_oracle(ctx, oracle, multiscale):
    n, m = 1500, 1300
    x, y = blobs(2, n, 0.0), blobs(3, m, 0.05)
    a = np.random.default_rng(4).random(n) + 0.5
    a /= a.sum()
    b = np.full(m, 1 / m)
    prm = make_params(blur=0.02, multiscale=multiscale, retruncate=1, cluster_scale=0.05)
    lg, gg, st = ctx.sinkhorn_grad(prm, x, a, y, b)
    lo, go = oracle.sinkhorn_grad(prm, x, a, y, b)
    assert abs(lg - lo) <= 1e-4 * abs(lo)
    scale = np.abs(go).max()
    assert np.abs(gg - go).max() <= 1e-3 * scale, np.abs(gg - go).max() / scale


@pytest.mark.gpu
def test_grad_translation_gpu(ctx):
    rng = np.random.default_rng(5)
    x = rng.random((4000, 3))
    t = np.array([0.2, -0.1, 0.05])
    a = np.full(4000, 1 / 4000)
    _, g, _ = ctx.sinkhorn_grad(make_params(blur=0.01, multiscale=True, retruncate=1), x, a,
                                x + t, a)
    assert np.abs(g + a[:, None] * t).max() <= 0.05 * a[0] * np.linalg.norm(t)


@pytest.mark.gpu
def test_barycenter_matches_oracle(ctx, oracle):
    """Config-5 shape at oracle size: 3 targets, positions after 3 steps."""
    rng = np.random.default_rng(6)
    targets = []
    for k in range(3):
        yk = blobs(10 + k, 400, 0.1 * np.array([k, -k, 0.5 * k]))
        targets.append((yk, np.full(400, 1 / 400)))
    x0 = blobs(20, 300, 0.05)
    a = np.full(300, 1 / 300)
    prm = make_params(blur=0.02)
    xg, tg, _ = ctx.barycenter(prm, x0, a, targets, iters=3)
    xo, to = oracle.barycenter(prm, x0, a, targets, iters=3)
    assert len(tg) == len(to)
    np.testing.assert_allclose(tg, to, rtol=1e-4)
    assert np.abs(xg - xo).max() <= 1e-4
    assert np.all(np.diff(tg) <= 0)


@pytest.mark.gpu
def test_barycenter_midpoint_gpu(ctx):
    x, traj, _ = ctx.barycenter(make_params(blur=0.01), np.array([[0.3]]), np.ones(1),
                                [(np.array([[-1.0]]), np.ones(1)),
                                 (np.array([[1.0]]), np.ones(1))], iters=20)
    assert abs(x[0, 0]) <= 0.01


@pytest.mark.gpu
def test_barycenter_multiscale_matches_oracle(ctx, oracle):
    """Config-5 path at oracle size: multiscale solves with
    the shared x-x self term — target 0 records a_xx and the self-plan
    payload, targets 1..K-1 skip the x-x problem (Plan::skip_p0 in the masks,
    the coarse and the fine tiles) — against oracle_barycenter, which shares
    the self term the same way."""
    targets = []
    for k in range(3):
        yk = blobs(30 + k, 2500, 0.1 * np.array([k, -k, 0.5 * k]))
        targets.append((yk, np.full(2500, 1 / 2500)))
    x0 = blobs(40, 3000, 0.05)
    a = np.full(3000, 1 / 3000)
    prm = make_params(blur=0.01, multiscale=True, retruncate=1, cluster_scale=0.04,
                      switch_factor=1.0)
    # the solves really ran the multiscale path with a fine phase
    _, _, s1 = ctx.sinkhorn(prm, x0, a, *targets[1], potentials=False)
    assert 0 < s1["t_switch"] < s1["n_scales"] and s1["pairs_fine"] > 0
    # every descent step from identical positions agrees to 1e-4 (x0 and the
    # GPU's own second iterate)
    x2, _, _ = ctx.barycenter(prm, x0, a, targets, iters=2)
    for xs in (x0, x2):
        xg, tg, _ = ctx.barycenter(prm, xs, a, targets, iters=1)
        xo, to = oracle.barycenter(prm, xs, a, targets, iters=1)
        np.testing.assert_allclose(tg, to, rtol=1e-4)
        assert np.abs(xg - xo).max() <= 1e-4
    # three chained steps: the loss trajectory stays within 1e-4.  Positions
    # drift further apart: the float32/float64 difference of one step (~3e-5)
    # moves atoms across voxel faces in one run and not the other, so later
    # solves use different clusters and tiles (measured 1.4e-3 max after 3
    # steps, tools/diag_bary.py); bounded here by blur / 4.
    xg, tg, _ = ctx.barycenter(prm, x0, a, targets, iters=3)
    xo, to = oracle.barycenter(prm, x0, a, targets, iters=3)
    assert len(tg) == len(to) == 4
    np.testing.assert_allclose(tg, to, rtol=1e-4)
    assert np.abs(xg - xo).max() <= 0.25 * 0.01
    assert np.all(np.diff(tg) <= 0)
