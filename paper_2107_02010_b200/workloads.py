"""Synthetic inputs of the BASELINE configs, seeded.

C1  uniform 3D clouds                      uniform(n, seed)
C2/C3 3D Gaussian mixtures                 mixture(n, seed)
C4  tractogram fibres (D = 60 features)    fibres(n, seed) -> polylines, bundle labels
C5  track-density maps on a 128^3 grid     density_maps(k, seed0) -> list of (ijk, value)

Plus the measure constructors the barycenter needs on the host:
density_to_measure and upsample.
"""
import numpy as np


def uniform(n, seed, d=3):
    return np.random.default_rng(seed).random((n, d))


def mixture(n, seed, d=3, k=8, sigma=0.05):
    """k Gaussian components, sigma 0.05, centres ~ U[0.2, 0.8]^d."""
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.2, 0.8, (k, d))
    return cen[rng.integers(0, k, n)] + rng.normal(0, sigma, (n, d))


# ------------------------------------------------------------------ C5 -----
def _tube_curve(rng, s):
    """A common smooth curve through the unit cube, randomly perturbed."""
    a = rng.normal(0, 0.03, (3, 3))
    ph = rng.uniform(0, 2 * np.pi, (3, 3))
    base = np.stack([0.2 + 0.6 * s, 0.5 + 0.15 * np.sin(2 * np.pi * s),
                     0.5 + 0.1 * np.cos(3 * np.pi * s)], 1)
    pert = sum(a[:, q][None, :] * np.sin((q + 1) * np.pi * s[:, None] + ph[:, q][None, :])
               for q in range(3))
    return base + pert


def density_map(seed, grid=128, radius_vox=3.0, samples=400, cutoff=1e-2):
    """Gaussian-profile tube (radius ~3 voxels) along a perturbed curve.
    Returns (ijk int array (K,3), values (K,)) for the nonzero voxels."""
    rng = np.random.default_rng(seed)
    s = np.linspace(0, 1, samples)
    c = _tube_curve(rng, s) * grid  # voxel units
    vol = np.zeros((grid, grid, grid), np.float32)
    r = int(np.ceil(3 * radius_vox))
    off = np.arange(-r, r + 1)
    dz, dy, dx = np.meshgrid(off, off, off, indexing="ij")
    for p in c:
        ctr = np.floor(p).astype(int)
        ii, jj, kk = ctr[0] + dz, ctr[1] + dy, ctr[2] + dx
        ok = (ii >= 0) & (ii < grid) & (jj >= 0) & (jj < grid) & (kk >= 0) & (kk < grid)
        d2 = (ii + 0.5 - p[0]) ** 2 + (jj + 0.5 - p[1]) ** 2 + (kk + 0.5 - p[2]) ** 2
        vol[ii[ok], jj[ok], kk[ok]] += np.exp(-d2[ok] / (2 * radius_vox ** 2)).astype(np.float32)
    vol[vol < cutoff * vol.max()] = 0.0
    ijk = np.argwhere(vol > 0)
    return ijk, vol[ijk[:, 0], ijk[:, 1], ijk[:, 2]].astype(np.float64)


def density_maps(k=10, seed0=9, grid=128, **kw):
    return [density_map(seed0 + q, grid, **kw) for q in range(k)]


def density_to_measure(ijk, values, voxel=1.0 / 128, origin=(0.0, 0.0, 0.0)):
    """One atom per nonzero voxel at its centre, weights normalised to 1
    (compensated summation via math.fsum)."""
    import math
    keep = values > 0
    pts = (np.asarray(ijk)[keep] + 0.5) * voxel + np.asarray(origin)
    w = np.asarray(values, np.float64)[keep]
    return pts, w / math.fsum(w)


def average_density(maps, grid=128):
    """Arithmetic average of the maps' normalised densities."""
    import math
    vol = np.zeros((grid, grid, grid))
    for ijk, v in maps:
        vol[ijk[:, 0], ijk[:, 1], ijk[:, 2]] += v / math.fsum(v)
    vol /= len(maps)
    ijk = np.argwhere(vol > 0)
    return ijk, vol[ijk[:, 0], ijk[:, 1], ijk[:, 2]]


def upsample(pts, w, factor, jitter, seed):
    """Each atom -> `factor` copies with weight w/factor and uniform jitter in
    [-jitter, jitter]^D; deterministic under `seed`."""
    rng = np.random.default_rng(seed)
    p = np.repeat(pts, factor, axis=0)
    if jitter > 0:
        p = p + rng.uniform(-jitter, jitter, p.shape)
    return p, np.repeat(w / factor, factor)


# ------------------------------------------------------------------ C4 -----
def fibres(n, seed, bundles=50, points=24, bundle_seed=None):
    """Smooth random cubic curves in [0,1]^3 grouped into `bundles` bundles:
    returns (list of (points, 3) polylines, bundle label per fibre).  The
    bundle geometry comes from `bundle_seed` (default: `seed`), so an atlas
    and a subject drawn with one bundle_seed share their bundles."""
    rng = np.random.default_rng(seed)
    ctrl = np.random.default_rng(seed if bundle_seed is None else bundle_seed).uniform(
        0.15, 0.85, (bundles, 4, 3))
    lab = rng.integers(0, bundles, n)
    t = np.linspace(0, 1, points)[:, None]
    bern = np.concatenate([(1 - t) ** 3, 3 * t * (1 - t) ** 2, 3 * t ** 2 * (1 - t), t ** 3], 1)
    out = []
    for i in range(n):
        cp = ctrl[lab[i]] + rng.normal(0, 0.02, (4, 3))
        out.append(bern @ cp)
    return out, lab


def encode_fibers(polylines, P=20):
    """Arc-length resampling to P points, flattened to 3P coordinates scaled
    by 1/sqrt(P), uniform weights 1/N."""
    out = np.empty((len(polylines), 3 * P))
    for i, line in enumerate(polylines):
        line = np.asarray(line, np.float64)
        seg = np.sqrt(((line[1:] - line[:-1]) ** 2).sum(1))
        arc = np.concatenate([[0.0], np.cumsum(seg)])
        if not arc[-1] > 0:
            raise ValueError(f"fiber {i} is degenerate")
        t = np.linspace(0.0, arc[-1], P)
        out[i] = np.stack([np.interp(t, arc, line[:, k]) for k in range(3)], 1).reshape(-1)
    return out / np.sqrt(P), np.full(len(polylines), 1.0 / len(polylines))


def flip_augment(x, w, P=20):
    """Append every fibre's point-order reversal, halving all weights
    (SPEC.md:76-84); atoms [0, N) originals, [N, 2N) flips."""
    flipped = x.reshape(len(x), P, 3)[:, ::-1, :].reshape(len(x), 3 * P)
    return np.concatenate([x, flipped]), np.concatenate([w, w]) / 2.0
