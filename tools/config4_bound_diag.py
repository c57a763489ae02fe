"""High-D truncation bounds on config 4: fraction of atom pairs kept by the
centroid/radius bound B_a alone, by min(B_a, B_b) with per-cluster slopes
(diagonal and ridge least squares), against the true fraction
f_i + g_j - C_ij >= -theta eps, at the final potentials of a dense solve.
    python tools/config4_bound_diag.py [n_fibres] [K]"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 0
fa, _ = W.fibres(n, 7, bundles=50, bundle_seed=1)
fb, _ = W.fibres(n, 8, bundles=50, bundle_seed=1)
x, a = W.flip_augment(*W.encode_fibers(fa))
y, b = W.flip_augment(*W.encode_fibers(fb))
N = len(x)
K = K or int(math.ceil(math.sqrt(N)))
ctx = Context(0)
prm = make_params(blur=0.03, reach=0.3)
loss, P, st = ctx.sinkhorn(prm, x, a, y, b)
eps, theta = 0.03 ** 2, 12.5
dev = torch.device("cuda")
X, Y = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
f = torch.from_numpy(P.b_yx).to(dev)  # cross potentials: rows x
g = torch.from_numpy(P.a_xy).to(dev)
out = dict(N=N, K=K)
# true kept fraction on a row sample
rows = torch.randperm(N, generator=torch.Generator().manual_seed(0))[:2000].to(dev)
C = 0.5 * torch.cdist(X[rows], Y) ** 2
out["true"] = float(((f[rows, None] + g[None, :] - C) >= -theta * eps).double().mean())
del C


def clusters(pts, w):
    km = ctx.kmeans(pts, w, K)
    lab = np.empty(len(pts), np.int64)
    perm, off = km["perm"], km["offsets"]
    for I in range(K):
        lab[perm[off[I]:off[I + 1]]] = I
    return torch.from_numpy(lab).to(dev), torch.from_numpy(km["centroids"]).to(dev)


def stats(P_, pot, lab, cen, mode):
    D = P_.shape[1]
    u = P_ - cen[lab]
    r = torch.zeros(K, device=dev, dtype=torch.float64).scatter_reduce(0, lab, u.norm(dim=1), "amax")
    F = torch.full((K,), -math.inf, device=dev, dtype=torch.float64).scatter_reduce(0, lab, pot, "amax")
    if mode == "none":
        return r, F, None, None
    cnt = torch.zeros(K, device=dev, dtype=torch.float64).index_add_(0, lab, torch.ones_like(pot))
    fm = torch.zeros(K, device=dev, dtype=torch.float64).index_add_(0, lab, pot) / cnt
    fc = pot - fm[lab]
    if mode == "diag":
        num = torch.zeros(K, D, device=dev, dtype=torch.float64).index_add_(0, lab, u * fc[:, None])
        den = torch.zeros(K, D, device=dev, dtype=torch.float64).index_add_(0, lab, u * u)
        S = num / (den + 1e-12)
    else:  # ridge least squares per cluster
        S = torch.zeros(K, D, device=dev, dtype=torch.float64)
        for I in range(K):
            m = lab == I
            U, v = u[m], fc[m]
            A = U.T @ U + 1e-6 * torch.eye(D, device=dev, dtype=torch.float64) * (U * U).sum()
            S[I] = torch.linalg.solve(A, U.T @ v)
    Fp = torch.full((K,), -math.inf, device=dev, dtype=torch.float64).scatter_reduce(
        0, lab, pot - (u * S[lab]).sum(1), "amax")
    return r, F, S, Fp


lx, cx = clusters(x, a)
ly, cy = clusters(y, b)
nx = torch.bincount(lx, minlength=K).double()
ny = torch.bincount(ly, minlength=K).double()
Dm = cx[:, None, :] - cy[None, :, :]
dn = Dm.norm(dim=2)
for mode in ("none", "diag", "ridge"):
    rx, Fx, Sx, Fpx = stats(X, f, lx, cx, mode)
    ry, Gy, Ty, Gpy = stats(Y, g, ly, cy, mode)
    Ba = Fx[:, None] + Gy[None, :] - 0.5 * torch.clamp(dn - rx[:, None] - ry[None, :], min=0) ** 2
    B = Ba
    if Sx is not None:
        ma = (Sx[:, None, :] - Dm).norm(dim=2)
        mb = (Ty[None, :, :] + Dm).norm(dim=2)
        Bb = Fpx[:, None] + Gpy[None, :] + rx[:, None] * ma + ry[None, :] * mb - 0.5 * dn ** 2
        B = torch.minimum(Ba, Bb)
    keep = (B >= -theta * eps).double()
    out[mode] = float((keep * nx[:, None] * ny[None, :]).sum() / (N * len(y)))
out["radius_mean"] = float(stats(X, f, lx, cx, "none")[0].mean())
print(json.dumps(out))
