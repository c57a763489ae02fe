"""Independent restatement of the multiscale policies (test infrastructure).

The GPU solver and the FP64 oracle share the integer policies of
paper_2107_02010_b200/csrc/policy.h (schedule, Morton cube ids, automatic voxel
edge, switch and super-level indices), so a GPU-vs-oracle comparison of those
rules alone would be tautological.  This module
re-derives them in numpy from their specifications — SPEC.md and DESIGN.md,
not the C sources — as a third implementation both are checked against
(tests/test_independent.py).  Nothing here is shared with, or imported by,
the product or the oracle.

  schedule       SPEC.md:153-162 (n = floor(log(d/blur)/log(1/q)) + 1, sigma_t
                 = d q^t, last = blur; d=8, blur=1, q=1/2 -> [8,4,2,1])
  voxel grid     north star: cube id floor((x - lo)/cell) per axis (clamped to
                 10 bits), Morton-interleaved; clusters = runs of a stable sort
                 by cube id (labels, permutation, weights,
                 centroids, radii)
  voxel edge     DESIGN.md §8c: ~28 atoms per cell of the joint bounding box,
                 then twice rescaled by (occupied / target)^(1/d)
  switch         SPEC.md:306: first sigma_t < factor * r_max
  super level    DESIGN.md §8c: 2x voxel edge, switch at sigma < 2 x (half
                 diagonal of a super voxel), only with >= 16384 clusters and
                 >= 4 scales taken off the cluster level
  mask           DESIGN.md §3 K3: keep (I, J) iff min(B_a, B_b) >= -theta eps,
                 plus the best pair of every row (and column) with none
"""
import math

import numpy as np

BITS = 10
ATOMS_PER_CELL = 28.0


def schedule(diameter, blur, q):
    """(sigma_t) of SPEC.md:153-162."""
    if not diameter > blur:
        return np.array([blur])
    r = math.log(diameter / blur) / math.log(1.0 / q)
    k = math.floor(r)
    if r - k > 1.0 - 1e-9:  # an integer ratio up to rounding (d=8, blur=1, q=1/2)
        k += 1
    n = int(k) + 1
    s = diameter * q ** np.arange(n, dtype=np.float64)
    s[-1] = blur
    return s


def cube_coords(x, lo, cell):
    q = np.floor((x - lo) / cell)
    return np.clip(q, 0, (1 << BITS) - 1).astype(np.int64)


def morton(q):
    """Interleave the per-axis voxel coordinates bit by bit (axis 0 lowest)."""
    n, d = q.shape
    key = np.zeros(n, np.int64)
    for b in range(BITS):
        for k in range(d):
            key |= ((q[:, k] >> b) & 1) << (b * d + k)
    return key


def grid_cluster(x, w, lo, cell):
    """Clusters of the voxel grid: dict(perm, labels (sorted order), offsets,
    k, cweights, centroids, radii) in float64."""
    x = np.asarray(x, np.float64)
    if x.ndim == 1:
        x = x[:, None]
    key = morton(cube_coords(x, lo, cell))
    perm = np.argsort(key, kind="stable")
    ks = key[perm]
    start = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    offsets = np.r_[start, len(ks)]
    k = len(start)
    labels = np.repeat(np.arange(k), np.diff(offsets))
    xs, ws = x[perm], np.asarray(w, np.float64)[perm]
    cw = np.add.reduceat(ws, start)
    cen = np.add.reduceat(xs * ws[:, None], start) / cw[:, None]
    dist = np.sqrt(((xs - cen[labels]) ** 2).sum(1))
    rad = np.maximum.reduceat(dist, start)
    return dict(perm=perm.astype(np.int32), labels=labels.astype(np.int32),
                offsets=offsets.astype(np.int32), k=k, cweights=cw, centroids=cen, radii=rad)


def occupied(x, lo, cell):
    return len(np.unique(morton(cube_coords(np.asarray(x, np.float64), lo, cell))))


def auto_cell(x, y):
    """The automatic voxel edge and the joint bounding box (lo, hi)."""
    lo = np.minimum(x.min(0), y.min(0))
    hi = np.maximum(x.max(0), y.max(0))
    d = x.shape[1]
    n = max(len(x), len(y))
    target = max(n / ATOMS_PER_CELL, 1.0)
    ext = hi - lo
    emax = ext.max()
    if emax <= 0:
        return 1.0, lo, hi
    live = ext > 1e-6 * emax
    s = (np.prod(ext[live]) / target) ** (1.0 / max(int(live.sum()), 1))
    smin = emax / ((1 << BITS) - 2)
    s = max(s, smin)
    for _ in range(2):  # two occupancy refinements
        k = max(occupied(x, lo, s), occupied(y, lo, s), 1)
        s = s * (k / target) ** (1.0 / d)
        s = min(max(s, smin), 2.0 * emax)
    return s, lo, hi


def switch_index(sigma, r_max, factor):
    for t, s in enumerate(sigma):
        if s < factor * r_max:
            return t
    return len(sigma)


def super_switch(sigma, tsw, cell, d, kmax, mode=-1):
    if mode == 0 or (mode < 0 and kmax < 16384):
        return 0
    r = 0.5 * math.sqrt(d) * cell * 2.0
    t2 = switch_index(sigma[:tsw], r, 2.0)
    return t2 if tsw - t2 >= 4 else 0


def box_quad(u, v, l1, h1, l2, h2):
    """max over a in [l1, h1], b in [l2, h2] of u a + v b - (a - b)^2 / 2,
    by brute force on a fine grid plus the exact edge candidates."""
    g = lambda aa, bb: u * aa + v * bb - 0.5 * (aa - bb) ** 2
    best = np.full(np.broadcast(u, v, l1, l2).shape, -np.inf)
    for aa in (l1, h1):
        best = np.maximum(best, g(aa, np.clip(aa + v, l2, h2)))
    for bb in (l2, h2):
        best = np.maximum(best, g(np.clip(bb + u, l1, h1), bb))
    return best


def slack(cx, rx, fx, cy, ry, gy, gx=None, hy=None, bx=None, by=None):
    """min(B_a, B_b[, B_c]) for every cluster pair (float64); bx / by: member
    boxes (K, 6) {lo[3], hi[3]} (DESIGN.md §3 K3, the box bound)."""
    cx, cy = np.asarray(cx, np.float64), np.asarray(cy, np.float64)
    rx, ry = np.asarray(rx, np.float64), np.asarray(ry, np.float64)
    fx, gy = np.asarray(fx, np.float64), np.asarray(gy, np.float64)
    D = cx[:, None, :] - cy[None, :, :]
    dist = np.sqrt((D ** 2).sum(-1))
    gap = np.maximum(0.0, dist - (rx[:, None] + ry[None, :]))
    ba = fx[:, None] + gy[None, :] - 0.5 * gap ** 2
    if gx is None:
        return ba
    gx, hy = np.asarray(gx, np.float64), np.asarray(hy, np.float64)
    S, Fp = gx[:, :3], gx[:, 3]
    T, Gp = hy[:, :3], hy[:, 3]
    U, V = S[:, None, :] - D, T[None, :, :] + D
    bb = (Fp[:, None] + Gp[None, :]
          + rx[:, None] * np.sqrt((U ** 2).sum(-1))
          + ry[None, :] * np.sqrt((V ** 2).sum(-1))
          - 0.5 * dist ** 2)
    out = np.minimum(ba, bb)
    if bx is None:
        return out
    bx, by = np.asarray(bx, np.float64), np.asarray(by, np.float64)
    q = sum(box_quad(U[..., k], V[..., k], bx[:, None, k], bx[:, None, 3 + k],
                     by[None, :, k], by[None, :, 3 + k]) for k in range(cx.shape[1]))
    return np.minimum(out, Fp[:, None] + Gp[None, :] + q - 0.5 * dist ** 2)


def mask(sl, eps, theta, self_=False):
    """Kept cluster pairs plus best pairs (ties -> lowest index)."""
    m = sl >= -theta * eps
    for i in np.flatnonzero(~m.any(1)):
        j = int(np.argmax(sl[i]))
        m[i, j] = True
        if self_:  # a self mask stays symmetric
            m[j, i] = True
    if not self_:
        for j in np.flatnonzero(~m.any(0)):
            m[int(np.argmax(sl[:, j])), j] = True
    return m
