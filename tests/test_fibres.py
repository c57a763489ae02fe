"""Config-4 path (D = 60 fibre features, unbalanced): the tcgen05 split-f16
softmin (softmin_hd.cu) against the FP64 oracle, on encoded, flip-augmented
synthetic fibres."""
import math

import numpy as np
import pytest

from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import make_params


def fibre_measures(n, m, seed):
    fa, _ = W.fibres(n, seed)
    fb, _ = W.fibres(m, seed + 1)
    x, a = W.encode_fibers(fa)
    y, b = W.encode_fibers(fb)
    return x, a, y, b


def test_encode_and_flip():
    line = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    x, w = W.encode_fibers([line], P=3)
    np.testing.assert_allclose(x[0].reshape(3, 3)[:, 0], np.array([0, 0.5, 1]) / math.sqrt(3))
    xf, wf = W.flip_augment(x, w, P=3)
    np.testing.assert_allclose(xf[1].reshape(3, 3)[:, 0], np.array([1, 0.5, 0]) / math.sqrt(3))
    assert wf.sum() == 1.0 and len(xf) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("reach", [math.inf, 0.3])
def test_hd_sinkhorn_matches_oracle(ctx, oracle, reach):
    x, a, y, b = fibre_measures(700, 600, 7)
    x, a = W.flip_augment(x, a)
    y, b = W.flip_augment(y, b)
    prm = make_params(blur=0.03, reach=reach)
    lg, pg, sg = ctx.sinkhorn(prm, x, a, y, b)
    lo, po, so = oracle.sinkhorn(prm, x, a, y, b)
    assert sg["n_scales"] == so["n_scales"]
    eps = 0.03 ** 2
    for name in ("a_xx", "b_yy", "a_xy", "b_yx"):
        err = np.abs(getattr(pg, name) - po[name]).max()
        assert err <= 1e-3 * eps, f"{name}: {err / eps:.3e} eps"
    assert abs(lg - lo) <= 1e-4 * abs(lo), (lg, lo)


@pytest.mark.gpu
def test_hd_softmin_kernel_dims(ctx, oracle):
    """Odd dimensions and sizes that are not multiples of the 128/256 tiles."""
    rng = np.random.default_rng(3)
    for d, n, m in ((4, 300, 257), (17, 513, 129), (64, 260, 1000)):
        x = rng.random((n, d)) * 0.3
        y = rng.random((m, d)) * 0.3
        prm = make_params(blur=0.05)
        lg, pg, _ = ctx.sinkhorn(prm, x, np.full(n, 1 / n), y, np.full(m, 1 / m))
        lo, po, _ = oracle.sinkhorn(prm, x, np.full(n, 1 / n), y, np.full(m, 1 / m))
        for name in ("a_xx", "b_yy", "a_xy", "b_yx"):
            assert np.abs(getattr(pg, name) - po[name]).max() <= 1e-3 * 0.05 ** 2, (d, name)
        assert abs(lg - lo) <= 1e-4 * abs(lo)


@pytest.mark.gpu
@pytest.mark.parametrize("reach", [math.inf, 0.3])
def test_hd_multiscale_matches_oracle(ctx, oracle, reach):
    """K-means multiscale at D = 60: padded cluster
    layout, centroid/radius masks, evaluate-once block-sparse tcgen05 phase,
    against the oracle's restatement on the same inputs."""
    x, a, y, b = fibre_measures(900, 800, 21)
    x, a = W.flip_augment(x, a)
    y, b = W.flip_augment(y, b)
    # ~120 atoms per cluster keeps the 128-atom padding small for the oracle
    prm = make_params(blur=0.03, reach=reach, multiscale=True, retruncate=1, switch_factor=1.0,
                      clusters=15)
    lg, pg, sg = ctx.sinkhorn(prm, x, a, y, b)
    lo, po, so = oracle.sinkhorn(prm, x, a, y, b)
    assert (sg["kx"], sg["ky"], sg["t_switch"]) == (so["kx"], so["ky"], so["t_switch"])
    assert 0 < sg["t_switch"] < sg["n_scales"]
    eps = 0.03 ** 2
    for name in ("a_xx", "b_yy", "a_xy", "b_yx"):
        err = np.abs(getattr(pg, name) - po[name]).max()
        assert err <= 1e-3 * eps, f"{name}: {err / eps:.3e} eps"
    assert abs(lg - lo) <= 1e-4 * abs(lo), (lg, lo)
    # and close to the dense solve
    ld, _, _ = ctx.sinkhorn(make_params(blur=0.03, reach=reach), x, a, y, b, potentials=False)
    assert abs(lg - ld) <= 1e-3 * abs(ld), (lg, ld)


@pytest.mark.gpu
@pytest.mark.parametrize("reach", [math.inf, 0.3])
def test_hd_multiscale_extrapolation_matches_oracle(ctx, oracle, reach):
    """transfer_rule 1 on the K-means path (D = 60): the extrapolation softmin
    runs on the tcgen05 kernel against the centroid measure, padding slots
    included, against the oracle."""
    x, a, y, b = fibre_measures(900, 800, 23)
    x, a = W.flip_augment(x, a)
    y, b = W.flip_augment(y, b)
    prm = make_params(blur=0.03, reach=reach, multiscale=True, retruncate=1, switch_factor=1.0,
                      clusters=15, transfer_rule=1)
    lg, pg, sg = ctx.sinkhorn(prm, x, a, y, b)
    lo, po, so = oracle.sinkhorn(prm, x, a, y, b)
    assert (sg["kx"], sg["ky"], sg["t_switch"]) == (so["kx"], so["ky"], so["t_switch"])
    assert 0 < sg["t_switch"] < sg["n_scales"]
    eps = 0.03 ** 2
    for name in ("a_xx", "b_yy", "a_xy", "b_yx"):
        err = np.abs(getattr(pg, name) - po[name]).max()
        assert err <= 1e-3 * eps, f"{name}: {err / eps:.3e} eps"
    assert abs(lg - lo) <= 1e-4 * abs(lo), (lg, lo)


@pytest.mark.gpu
def test_hd_colpart_batches(ctx):
    """Batched column partials on the tcgen05 path (dense pair sets, hd_colsum,
    two streams).  Batched high-D updates size their work items per batch, so
    the row sums associate differently than one batch: equal to rounding, and
    bitwise reproducible for a given budget."""
    x, a, y, b = fibre_measures(1500, 1300, 25)
    prm = make_params(blur=0.03, reach=0.3)
    ctx.set_colpart_budget(1 << 30)
    try:
        l1, p1, s1 = ctx.sinkhorn(prm, x, a, y, b)
        ctx.set_colpart_budget(3000)
        l2, p2, s2 = ctx.sinkhorn(prm, x, a, y, b)
        l3, p3, _ = ctx.sinkhorn(prm, x, a, y, b)
    finally:
        ctx.set_colpart_budget(0)
    assert s1["colpart_batches"] == 1 and s2["colpart_batches"] > 2
    assert l2 == l3 and abs(l1 - l2) <= 1e-6 * abs(l1)
    eps = 0.03 ** 2
    for k in ("a_xx", "b_yy", "a_xy", "b_yx"):
        np.testing.assert_array_equal(getattr(p2, k), getattr(p3, k))
        assert np.abs(getattr(p1, k) - getattr(p2, k)).max() <= 1e-5 * eps
