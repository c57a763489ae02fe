"""K-means coarsening: the FP64
oracle against SPEC's examples, and the GPU kernels bit-exact against the
oracle (labels, permutation, offsets, centroids, weights, radii)."""
import numpy as np
import pytest

from paper_2107_02010_b200 import workloads as W


def test_oracle_kmeans_spec_examples(oracle):
    rng = np.random.default_rng(0)
    x = rng.random((40, 5))
    w = rng.random(40) + 0.5
    r = oracle.kmeans(x, w, 40)  # K = N: every atom its own cluster
    assert np.all(np.diff(r["offsets"]) == 1)
    np.testing.assert_allclose(r["centroids"][r["labels"]], x, rtol=1e-15)  # (w x) / w
    assert np.all(r["radii"] <= 1e-15)
    r = oracle.kmeans(x, w, 1)  # K = 1: the weighted mean, the total mass
    np.testing.assert_allclose(r["centroids"][0], (w[:, None] * x).sum(0) / w.sum(), rtol=1e-12)
    assert r["cweights"][0] == pytest.approx(w.sum(), rel=1e-12)
    a = rng.normal(0, 0.01, (50, 3))
    b = rng.normal(5, 0.01, (50, 3))
    x2 = np.concatenate([a, b])
    r = oracle.kmeans(x2, np.ones(100), 2)
    means = sorted([a.mean(0).tolist(), b.mean(0).tolist()])
    got = sorted(r["centroids"].tolist())
    np.testing.assert_allclose(got, means, atol=1e-6)
    assert np.all(np.diff(r["labels"][r["perm"]]) >= 0)  # clusters contiguous


@pytest.mark.gpu
@pytest.mark.parametrize("d,n,k", [(3, 3000, 55), (17, 2000, 45), (60, 4000, 63)])
def test_kmeans_bit_exact(ctx, oracle, d, n, k):
    rng = np.random.default_rng(d)
    if d == 60:
        fa, _ = W.fibres(n // 2, 3, bundles=12)
        x, w = W.flip_augment(*W.encode_fibers(fa))
    else:
        cen = rng.random((7, d))
        x = cen[rng.integers(0, 7, n)] + rng.normal(0, 0.05, (n, d))
        w = rng.random(n) + 0.5
    g = ctx.kmeans(x, w, k, seed=11)
    o = oracle.kmeans(x, w, k, seed=11)
    assert g["iters"] == o["iters"]
    for key in ("labels", "perm", "offsets", "centroids", "cweights", "radii"):
        np.testing.assert_array_equal(g[key], o[key], err_msg=key)
