"""exact_ot (module exact_oracle): the
host network simplex of csrc/exact_ot.cpp against independent ground truths —
brute-force permutation enumeration, the closed-form 1D
monotone matching, and scipy's HiGHS LP — plus the contract's invariants and
errors.  GPU tests: acceptance criteria 1 (Sinkhorn divergence at blur 1e-3 d
against the exact value) and 9 (barycenter of translated copies, matched per
atom by exact_ot)."""
import itertools
import math

import numpy as np
import pytest

from paper_2107_02010_b200.abi import DataError, make_params
from paper_2107_02010_b200.solver import exact_ot


def _cost(x, y):
    return 0.5 * ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)


def test_dirac_pair():
    v, plan = exact_ot(np.array([[0.0, 1.0]]), [1.0], np.array([[2.0, 1.0]]), [1.0])
    assert v == 2.0 and plan.tolist() == [[1.0]]


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_brute_force_permutations(n):
    rng = np.random.default_rng(n)
    for _ in range(10):
        x, y = rng.random((n, 2)), rng.random((n, 2))
        w = np.full(n, 1.0 / n)
        v, plan = exact_ot(x, w, y, w)
        C = _cost(x, y)
        best = min(sum(C[i, s[i]] for i in range(n)) / n for s in itertools.permutations(range(n)))
        assert abs(v - best) <= 1e-14
        np.testing.assert_allclose(plan.sum(1), w, atol=1e-12)
        np.testing.assert_allclose(plan.sum(0), w, atol=1e-12)


def test_one_dimensional_monotone():
    rng = np.random.default_rng(3)
    x, y = rng.normal(size=40), rng.normal(size=40) + 0.5
    w = np.full(40, 1 / 40)
    v, plan = exact_ot(x, w, y, w)
    ref = np.sum((np.sort(x) - np.sort(y)) ** 2) / (2 * 40)
    assert abs(v - ref) <= 1e-13
    # monotone: the i-th smallest x goes to the i-th smallest y
    ox, oy = np.argsort(x), np.argsort(y)
    np.testing.assert_allclose(plan[ox, oy], w, atol=1e-12)


@pytest.mark.parametrize("shape", [(32, 32), (50, 70), (128, 100), (200, 256)])
def test_matches_highs(shape):
    from scipy.optimize import linprog
    n, m = shape
    rng = np.random.default_rng(n + m)
    x, y = rng.random((n, 3)), rng.random((m, 3))
    a, b = rng.random(n), rng.random(m)
    a /= a.sum()
    b *= a.sum() / b.sum()
    v, plan = exact_ot(x, a, y, b)
    C = _cost(x, y)
    A = np.zeros((n + m, n * m))
    for i in range(n):
        A[i, i * m:(i + 1) * m] = 1
    for j in range(m):
        A[n + j, j::m] = 1
    r = linprog(C.ravel(), A_eq=A, b_eq=np.r_[a, b], method="highs")
    assert r.status == 0
    assert abs(v - r.fun) <= 1e-12 * max(1.0, r.fun) + 1e-14
    assert plan.min() >= 0
    np.testing.assert_allclose(plan.sum(1), a, atol=1e-9)
    np.testing.assert_allclose(plan.sum(0), b, atol=1e-9)
    assert abs((plan * C).sum() - v) <= 1e-14
    # an optimal vertex: at most n + m - 1 nonzeros
    assert np.count_nonzero(plan) <= n + m - 1


def test_invariants():
    rng = np.random.default_rng(11)
    x, y = rng.random((30, 2)), rng.random((25, 2))
    a = np.full(30, 1 / 30)
    b = np.full(25, 1 / 25)
    v, _ = exact_ot(x, a, y, b, plan=False)
    v3, _ = exact_ot(3 * x, a, 3 * y, b, plan=False)
    assert abs(v3 - 9 * v) <= 1e-12 * v3  # scale covariance, p = 2
    v0, plan = exact_ot(x, a, x, a)
    assert v0 == 0.0
    np.testing.assert_allclose(np.diag(plan), a, atol=1e-15)  # identity-supported
    # p = 1 against HiGHS-free check: 1D p=1 value = integral |F - G|
    xs, ys = rng.random(20), rng.random(20)
    w = np.full(20, 0.05)
    v1, _ = exact_ot(xs, w, ys, w, p=1.0)
    assert abs(v1 - np.abs(np.sort(xs) - np.sort(ys)).sum() * 0.05) <= 1e-13


def test_zero_weights_and_degenerate_ties():
    x = np.array([[0.0], [1.0], [2.0], [3.0]])
    a = np.array([0.5, 0.0, 0.5, 0.0])
    y = np.array([[0.0], [2.0]])
    v, plan = exact_ot(x, a, y, [0.5, 0.5])
    assert v == 0.0
    # every point equidistant: any permutation is optimal
    x = np.zeros((8, 2))
    v, plan = exact_ot(x, np.full(8, 1 / 8), x + 1.0, np.full(8, 1 / 8))
    assert abs(v - 1.0) <= 1e-14


def test_errors():
    with pytest.raises(DataError):
        exact_ot([[0.0]], [1.0], [[1.0]], [0.5])  # unbalanced
    with pytest.raises(DataError):
        exact_ot(np.zeros((1001, 1)), np.full(1001, 1 / 1001), np.zeros((1000, 1)),
                 np.full(1000, 1e-3))  # N*M > 1e6
    with pytest.raises(DataError):
        exact_ot([[0.0]], [-1.0], [[1.0]], [-1.0])
    with pytest.raises(DataError):
        exact_ot([[0.0]], [1.0], [[1.0]], [1.0], p=3.0)


@pytest.mark.gpu
def test_acceptance_oracle_agreement(ctx):
    """SPEC.md:587 (criterion 1): 20 random balanced pairs, N = M = 32, D = 2,
    p = 2, reach = inf, blur = 1e-3 d -> |S - exact| <= 1e-2 exact.

    The schedule-driven algorithm (one update per scale)
    meets it only with a slow enough schedule: the FP64 oracle's worst error
    over these fixtures is 8.2% at q = 0.9, 4.7% at 0.95, 1.1% at 0.99 and
    0.49% at q = 0.995 (1379 scales), the value used here."""
    rng = np.random.default_rng(587)
    for _ in range(20):
        x, y = rng.random((32, 2)), rng.random((32, 2))
        a, b = rng.random(32) + 0.1, rng.random(32) + 0.1
        a /= a.sum()
        b /= b.sum()
        d = math.dist(np.minimum(x.min(0), y.min(0)), np.maximum(x.max(0), y.max(0)))
        s, _, _ = ctx.sinkhorn(make_params(blur=1e-3 * d, scaling=0.995), x, a, y, b,
                               potentials=False)
        v, _ = exact_ot(x, a, y, b, plan=False)
        assert abs(s - v) <= 1e-2 * v


@pytest.mark.gpu
def test_acceptance_barycenter_of_translates(ctx):
    """SPEC.md:595 (criterion 9): K = 4 translated copies of a 200-atom cloud ->
    the barycenter lies within blur of the mean-translated cloud, per atom
    after the optimal matching computed by exact_ot."""
    rng = np.random.default_rng(595)
    base = rng.random((200, 2)) * 0.5 + 0.25
    shifts = rng.normal(0, 0.1, (4, 2))
    w = np.full(200, 1 / 200)
    blur = 0.01
    targets = [(base + s, w) for s in shifts]
    want = base + shifts.mean(0)
    # initialised at the first target, or at a slightly jittered copy of the
    # cloud (a 0.02 jitter lets gradient descent trap one atom in a local
    # minimum 0.04 away — the FP64 oracle stops at the same point)
    for x0 in (targets[0][0], base + rng.normal(0, 0.005, base.shape)):
        x, traj, _ = ctx.barycenter(make_params(blur=blur), x0, w, targets, iters=60, tol=1e-9)
        _, plan = exact_ot(x, w, want, w)
        match = plan.argmax(1)
        err = np.linalg.norm(x - want[match], axis=1)
        assert err.max() <= blur, (err.max(), len(traj))
