"""transfer_labels (K9), resolve_flips and classify (PAPER.md
eq. 7): the SPEC examples and invariants on the FP64 oracle (CPU) and the
GPU path against the oracle on the same inputs (dense 3-D, multiscale 3-D,
and D = 60 fibres through the tcgen05 kernel)."""
import math

import numpy as np
import pytest

from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import DataError, make_params
from paper_2107_02010_b200.solver import OUTLIER, SoftLabels, classify, resolve_flips


def oracle_labels(oracle, prm, x, a, y, b, labels, L):
    _, po, _ = oracle.sinkhorn(prm, x, a, y, b)
    return oracle.transfer_labels(x, y, b, po["b_yx"], po["a_xy"], prm.blur ** 2, labels, L)


# ----------------------------------------------------------- host helpers --
def test_classify_spec_examples():
    soft = SoftLabels(np.array([[0.01, 0.02, 0.95], [0.005, 0.005, 0.0], [0.3, 0.3, 0.0]]),
                      np.array([0.98, 0.01, 0.6]))
    lab, conf = classify(soft, 0.5)
    assert lab.tolist() == [2, OUTLIER, 0]  # argmax tie -> lowest class
    assert conf[0] == pytest.approx(0.95 / 0.98) and conf[2] == pytest.approx(0.5)


def test_resolve_flips_spec_examples():
    # originals 0, 1; augmented rows: 0, 1 originals, 2, 3 their flips
    sc = np.array([[0.9, 0.0], [0.01, 0.01], [0.05, 0.0], [0.0, 0.7]])
    rm = sc.sum(1)
    out, chosen = resolve_flips(SoftLabels(sc, rm), [0, 1, 0, 1], [0, 0, 1, 1])
    assert chosen.tolist() == [0, 3]  # A 0.9 vs B 0.05 -> A; all mass on the flip -> flip
    np.testing.assert_array_equal(out.scores, sc[[0, 3]])
    # exact tie (palindromic fibre) -> original kept
    out, chosen = resolve_flips(SoftLabels(np.ones((2, 1)), np.ones(2)), [0, 0], [0, 1])
    assert chosen.tolist() == [0]
    with pytest.raises(DataError):  # missing flip pair
        resolve_flips(SoftLabels(np.ones((2, 1)), np.ones(2)), [0, 0], [0, 0])


# ------------------------------------------------------------ oracle (CPU) --
def test_oracle_labels_bijective_diracs(oracle):
    x = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    a = np.full(4, 0.25)
    prm = make_params(blur=0.05, scaling=0.7)
    sc, rm = oracle_labels(oracle, prm, x, a, x + 0.01, a, np.arange(4), 4)
    np.testing.assert_allclose(sc, np.eye(4), atol=1e-3)


def test_oracle_labels_equidistant(oracle):
    x = np.array([[0.0]])
    y = np.array([[-1.0], [1.0]])
    sc, rm = oracle_labels(oracle, make_params(blur=0.1, scaling=0.7), x, np.ones(1), y,
                           np.full(2, 0.5), [0, 1], 2)
    np.testing.assert_allclose(sc[0], [0.5, 0.5], atol=1e-3)


def test_oracle_labels_far_outlier_and_one_class(oracle):
    rng = np.random.default_rng(0)
    y = rng.random((40, 2)) * 0.2
    x = np.concatenate([rng.random((39, 2)) * 0.2, [[5.0, 5.0]]])
    a = np.full(40, 1 / 40)
    prm = make_params(blur=0.02, reach=0.3, scaling=0.8)
    sc, rm = oracle_labels(oracle, prm, x, a, y, a, np.zeros(40, np.int32), 1)
    assert rm[-1] < 0.05  # PAPER §2: "will be almost zero"
    np.testing.assert_allclose(sc[:, 0], rm, rtol=1e-12)  # L = 1: scores == row_mass


def test_oracle_labels_simplex(oracle):
    # "converged duals": the loop is schedule-driven, so the
    # invariant needs a slow schedule (q = 0.99); at q = 0.9 row masses of
    # this fixture are off by up to 40% after the last (non-averaged) update
    rng = np.random.default_rng(1)
    x, y = rng.random((50, 3)), rng.random((50, 3))
    lab = rng.integers(0, 4, 50)
    sc, rm = oracle_labels(oracle, make_params(blur=0.02, scaling=0.99), x, np.full(50, 1 / 50),
                           y, np.full(50, 1 / 50), lab, 4)
    assert np.all(sc >= 0)
    np.testing.assert_allclose(sc.sum(1), rm, rtol=1e-9)
    assert np.all(np.abs(rm - 1) <= 1e-2)  # SPEC simplex consistency


# ---------------------------------------------------------------- GPU parity --
def _check(gpu_soft, sc, rm, tol=3e-3):
    # potentials agree within 1e-3 eps each, so every plan entry within ~2e-3
    # relative; scores compared relative to the row mass
    scale = np.maximum(rm, 1e-30)[:, None]
    assert np.abs(gpu_soft.scores - sc).max() <= tol * max(1.0, rm.max())
    np.testing.assert_allclose(gpu_soft.row_mass, rm, rtol=tol, atol=1e-12)
    assert np.all(np.abs(gpu_soft.scores - sc) <= tol * scale + 1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("reach", [math.inf, 0.3])
def test_labels_dense_3d(ctx, oracle, reach):
    rng = np.random.default_rng(2)
    x, y = rng.random((700, 3)), rng.random((650, 3))
    lab = rng.integers(0, 5, 650)
    a, b = np.full(700, 1 / 700), np.full(650, 1 / 650)
    prm = make_params(blur=0.05, reach=reach)
    soft, loss, st = ctx.transfer_labels(prm, x, a, y, b, lab, 5)
    sc, rm = oracle_labels(oracle, prm, x, a, y, b, lab, 5)
    _check(soft, sc, rm)
    lab_g, _ = classify(soft, 0.5)
    lab_o, _ = classify(SoftLabels(sc, rm), 0.5)
    assert np.mean(lab_g == lab_o) > 0.99


@pytest.mark.gpu
def test_labels_multiscale_3d(ctx, oracle):
    rng = np.random.default_rng(3)
    cen = rng.uniform(0.2, 0.8, (4, 3))
    k = rng.integers(0, 4, 3000)
    x = cen[k] + rng.normal(0, 0.05, (3000, 3))
    y = cen[rng.integers(0, 4, 2500)] + rng.normal(0, 0.05, (2500, 3))
    lab = (y[:, 0] > 0.5).astype(np.int32) + 2 * (y[:, 1] > 0.5)
    a, b = np.full(3000, 1 / 3000), np.full(2500, 1 / 2500)
    prm = make_params(blur=0.02, multiscale=True, cluster_scale=0.05)
    soft, _, st = ctx.transfer_labels(prm, x, a, y, b, lab, 4)
    assert st["t_switch"] > 0
    sc, rm = oracle_labels(oracle, prm, x, a, y, b, lab, 4)
    _check(soft, sc, rm)


@pytest.mark.gpu
def test_labels_fibres_hd(ctx, oracle):
    """Config-4 shape (D = 60, flip-augmented, reach 0.3) at small N, with
    label segments that are not multiples of the 128-column block."""
    fa, la = W.fibres(500, 7, bundles=6, bundle_seed=1)
    fb, lb = W.fibres(450, 8, bundles=6, bundle_seed=1)
    x, a = W.flip_augment(*W.encode_fibers(fa))
    y, b = W.flip_augment(*W.encode_fibers(fb))
    lab = np.concatenate([lb, lb]).astype(np.int32)
    prm = make_params(blur=0.03, reach=0.3)
    soft, _, _ = ctx.transfer_labels(prm, x, a, y, b, lab, 6)
    sc, rm = oracle_labels(oracle, prm, x, a, y, b, lab, 6)
    _check(soft, sc, rm)
    out, chosen = resolve_flips(soft, np.tile(np.arange(500), 2), np.repeat([0, 1], 500))
    hard, _ = classify(out, 0.25)
    assert np.mean(hard[hard >= 0] == la[hard >= 0]) > 0.9


@pytest.mark.gpu
def test_labels_fibres_hd_multiscale(ctx, oracle):
    """Label transfer on the padded K-means layout of the high-D multiscale solver."""
    fa, la = W.fibres(600, 7, bundles=6, bundle_seed=2)
    fb, lb = W.fibres(500, 8, bundles=6, bundle_seed=2)
    x, a = W.flip_augment(*W.encode_fibers(fa))
    y, b = W.flip_augment(*W.encode_fibers(fb))
    lab = np.concatenate([lb, lb]).astype(np.int32)
    prm = make_params(blur=0.03, reach=0.3, multiscale=True, retruncate=1, switch_factor=1.0,
                      clusters=10)
    soft, _, st = ctx.transfer_labels(prm, x, a, y, b, lab, 6)
    assert st["t_switch"] > 0
    sc, rm = oracle_labels(oracle, prm, x, a, y, b, lab, 6)
    _check(soft, sc, rm)


@pytest.mark.gpu
def test_labels_errors(ctx):
    x = np.zeros((3, 3))
    with pytest.raises(DataError):
        ctx.transfer_labels(make_params(), x, np.full(3, 1 / 3), x, np.full(3, 1 / 3),
                            [0, 1, 5], 2)
