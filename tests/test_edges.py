"""Edge cases of the GPU path against the FP64 oracle (SURVEY.md §4 / §8c:
empty-ish and ragged inputs, tile and block boundaries, low dimensions in the
multiscale path, degenerate geometry, invalid input).  Same contract as
tests/test_gpu_parity.py: potentials within 1e-3 eps, loss within 1e-4."""
import math

import numpy as np
import pytest

from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import DataError, make_params

pytestmark = pytest.mark.gpu

POT_TOL, LOSS_TOL = 1e-3, 1e-4


def mixture(n, seed, d=3, k=6, sigma=0.05):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.2, 0.8, (k, d))
    return cen[rng.integers(0, k, n)] + rng.normal(0, sigma, (n, d))


def check(ctx, oracle, prm, x, a, y, b, eps):
    lg, pg, sg = ctx.sinkhorn(prm, x, a, y, b)
    lo, po, so = oracle.sinkhorn(prm, x, a, y, b)
    for name, g in zip(("a_xx", "b_yy", "a_xy", "b_yx"), (pg.a_xx, pg.b_yy, pg.a_xy, pg.b_yx)):
        # plus 16 float32 ulps of the potential: potentials of clouds far
        # apart (|t|^2 / 2 ~ 4e3) are stored to ~2e-4 and averaged over ~70 scales
        err = np.abs(g - po[name]) - 16 * np.spacing(np.abs(po[name]).astype(np.float32))
        assert err.max() <= POT_TOL * eps, f"{name}: {err.max() / eps:.3e} eps"
    assert abs(lg - lo) <= LOSS_TOL * abs(lo) + 1e-12, (lg, lo)
    return sg, so


@pytest.mark.parametrize("d", [1, 2])
def test_multiscale_low_dim(ctx, oracle, d):
    """The voxel multiscale path (super level, masks, evaluate-once) in 1D / 2D."""
    n, m = 5000, 4300
    x, y = mixture(n, 21, d), mixture(m, 22, d)
    a, b = np.full(n, 1 / n), np.full(m, 1 / m)
    prm = make_params(blur=0.01, multiscale=True, retruncate=1,
                      cluster_scale=0.02 if d == 1 else 0.03, super_level=1)
    sg, so = check(ctx, oracle, prm, x, a, y, b, 1e-4)
    assert (sg["kx"], sg["t_switch"], sg["t_super"]) == (so["kx"], so["t_switch"], so["t_super"])
    assert sg["pairs_fine"] < sg["pairs_fine_dense"]


@pytest.mark.parametrize("n,m", [(1, 1), (1, 700), (255, 257), (256, 256), (257, 513)])
@pytest.mark.parametrize("multiscale", [False, True])
def test_ragged_sizes(ctx, oracle, n, m, multiscale):
    """Tile (256 rows), column-stage (128) and warp boundaries, single atoms."""
    x, y = mixture(n, n + 1), mixture(m, m + 2)
    rng = np.random.default_rng(n * m)
    a = rng.random(n) + 0.1
    b = rng.random(m) + 0.1
    a /= a.sum()
    b /= b.sum()
    prm = make_params(blur=0.02, multiscale=multiscale, retruncate=1, cluster_scale=0.05)
    check(ctx, oracle, prm, x, a, y, b, 4e-4)


def test_unbalanced_masses_and_reach(ctx, oracle):
    """Total masses 1 and 2.5 with a finite reach (mass term and damping)."""
    x, y = mixture(900, 31), mixture(1100, 32)
    a = np.full(900, 1 / 900)
    b = np.full(1100, 2.5 / 1100)
    check(ctx, oracle, make_params(blur=0.03, reach=0.2), x, a, y, b, 9e-4)


def test_coincident_atoms(ctx, oracle):
    """Many atoms at the same position (zero-radius clusters, ties in the sort)."""
    rng = np.random.default_rng(41)
    base = rng.random((20, 3))
    x = base[rng.integers(0, 20, 3000)]
    y = base[rng.integers(0, 20, 2500)] + 0.01
    a, b = np.full(3000, 1 / 3000), np.full(2500, 1 / 2500)
    for ms in (False, True):
        check(ctx, oracle, make_params(blur=0.02, multiscale=ms, retruncate=1, cluster_scale=0.05),
              x, a, y, b, 4e-4)


@pytest.mark.parametrize("n,m", [(1, 1), (130, 127), (300, 513)])
def test_high_dim_ragged(ctx, oracle, n, m):
    """The tcgen05 path off its 128-row / 128-column blocks (D = 60 fibres)."""
    fa, _ = W.fibres(n, 51)
    fb, _ = W.fibres(m, 52)
    x, a = W.encode_fibers(fa)
    y, b = W.encode_fibers(fb)
    check(ctx, oracle, make_params(blur=0.05, reach=0.3), x, a, y, b, 0.05 ** 2)


def test_non_finite_inputs(ctx):
    x = np.zeros((4, 3))
    w = np.full(4, 0.25)
    bad = x.copy()
    bad[2, 1] = np.nan
    with pytest.raises(DataError):
        ctx.sinkhorn(make_params(), bad, w, x, w)
    bad[2, 1] = np.inf
    with pytest.raises(DataError):
        ctx.sinkhorn(make_params(), x, w, bad, w)
    with pytest.raises(DataError):
        ctx.sinkhorn(make_params(), x, np.array([0.25, np.nan, 0.25, 0.25]), x, w)


def test_far_apart_clouds(ctx, oracle):
    """Clouds 50 units apart: large potentials, the fixed-reference window."""
    x, y = mixture(800, 61), mixture(700, 62) + 50.0
    a, b = np.full(800, 1 / 800), np.full(700, 1 / 700)
    sg, so = check(ctx, oracle, make_params(blur=0.05), x, a, y, b, 0.05 ** 2)


@pytest.mark.parametrize("multiscale", [False, True])
def test_deterministic(ctx, multiscale):
    """Fixed-order reductions everywhere (no float atomics): a repeated solve
    is bitwise identical."""
    x, y = mixture(6000, 71), mixture(5000, 72)
    a, b = np.full(6000, 1 / 6000), np.full(5000, 1 / 5000)
    prm = make_params(blur=0.01, multiscale=multiscale, retruncate=1, cluster_scale=0.04,
                      super_level=1)
    l1, p1, _ = ctx.sinkhorn(prm, x, a, y, b)
    l2, p2, _ = ctx.sinkhorn(prm, x, a, y, b)
    assert l1 == l2
    for u, v in zip((p1.a_xx, p1.b_yy, p1.a_xy, p1.b_yx), (p2.a_xx, p2.b_yy, p2.a_xy, p2.b_yx)):
        np.testing.assert_array_equal(u, v)



@pytest.mark.parametrize("multiscale", [False, True])
def test_numeric_error_names_scale(ctx, multiscale):
    """SPEC.md:178 / common.hpp:15-19: a non-finite potential raises
    NumericError naming the scale where it first appeared.  blur = 1e-30 puts
    eps = sigma^2 below float32's range ~400 scales into the schedule; the
    device flags the first non-finite store (atomicMin over the scale index)."""
    from paper_2107_02010_b200.abi import NumericError
    x, y = mixture(500, 81), mixture(400, 82)
    a, b = np.full(500, 1 / 500), np.full(400, 1 / 400)
    prm = make_params(blur=1e-30, multiscale=multiscale, cluster_scale=0.1 if multiscale else 0.0)
    with pytest.raises(NumericError, match=r"non-finite potential at scale (\d+) of (\d+)") as ei:
        ctx.sinkhorn(prm, x, a, y, b)
    import re
    t, n = map(int, re.search(r"scale (\d+) of (\d+)", str(ei.value)).groups())
    assert 0 < t <= n
    # the context stays usable after the error
    l, _, _ = ctx.sinkhorn(make_params(blur=0.05), x, a, y, b, potentials=False)
    assert np.isfinite(l)
