"""Config 4 (D = 60 fibres): would the member-box bound of the voxel path
(mask.cu B_c) tighten the K-means truncation?  At the final potentials of a
multiscale solve, per K-means cluster: max potential, least-squares slope,
F' and the 60-D member box; the pair-weighted kept fraction of the cluster
pairs under
  ball   B_a (today's high-D mask)
  slope  min(B_a, B_b)
  box    min(B_a, B_b, B_c)
  exact  pairs with f + g - C >= -theta eps (sampled rows)
python tools/c4_bound_probe.py [n_fibres]"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
fa, _ = W.fibres(nf, 7, bundles=50, bundle_seed=1)
fb, _ = W.fibres(nf, 8, bundles=50, bundle_seed=1)
x, a = W.flip_augment(*W.encode_fibers(fa))
y, b = W.flip_augment(*W.encode_fibers(fb))
prm = make_params(blur=0.03, reach=0.3, multiscale=True, retruncate=1, switch_factor=2.0, theta=12.5)
ctx = Context(0)
_, P, st = ctx.sinkhorn(prm, x, a, y, b)
eps, theta = 0.03 ** 2, 12.5
K = math.ceil(math.sqrt(len(x)))
dev = torch.device("cuda")
T = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev, torch.float64)


def stats(pts, f, k):
    km = ctx.kmeans(pts, np.full(len(pts), 1.0), k)
    L = torch.from_numpy(km["labels"].astype(np.int64)).to(dev)
    Pt, F = T(pts), T(f)
    n, d = Pt.shape
    cnt = torch.zeros(k, device=dev, dtype=torch.float64).index_add_(0, L, torch.ones(n, device=dev, dtype=torch.float64))
    cen = torch.zeros(k, d, device=dev, dtype=torch.float64).index_add_(0, L, Pt) / cnt[:, None]
    u = Pt - cen[L]
    rad = torch.zeros(k, device=dev, dtype=torch.float64).scatter_reduce_(0, L, u.norm(dim=1), "amax")
    lo = torch.zeros(k, d, device=dev, dtype=torch.float64).scatter_reduce_(0, L[:, None].expand(-1, d), u, "amin")
    hi = torch.zeros(k, d, device=dev, dtype=torch.float64).scatter_reduce_(0, L[:, None].expand(-1, d), u, "amax")
    fmax = torch.full((k,), -1e300, device=dev, dtype=torch.float64).scatter_reduce_(0, L, F, "amax")
    fbar = torch.zeros(k, device=dev, dtype=torch.float64).index_add_(0, L, F) / cnt
    Muu = torch.zeros(k, d, d, device=dev, dtype=torch.float64).index_add_(0, L, u[:, :, None] * u[:, None, :])
    Muf = torch.zeros(k, d, device=dev, dtype=torch.float64).index_add_(0, L, u * (F - fbar[L])[:, None])
    S = torch.linalg.solve(Muu + 1e-9 * torch.eye(d, device=dev, dtype=torch.float64), Muf[:, :, None])[:, :, 0]
    Fp = torch.full((k,), -1e300, device=dev, dtype=torch.float64).scatter_reduce_(0, L, F - (u * S[L]).sum(1), "amax")
    return dict(cnt=cnt, cen=cen, rad=rad, lo=lo, hi=hi, fmax=fmax, S=S, Fp=Fp)


X, Y = stats(x, P.b_yx, K), stats(y, P.a_xy, K)


def box_quad(u, v, l1, h1, l2, h2):
    g = lambda A, B: u * A + v * B - 0.5 * (A - B) ** 2
    return torch.maximum(torch.maximum(g(l1, torch.clamp(l1 + v, l2, h2)), g(h1, torch.clamp(h1 + v, l2, h2))),
                         torch.maximum(g(torch.clamp(l2 + u, l1, h1), l2), g(torch.clamp(h2 + u, l1, h1), h2)))


thr = -theta * eps
w = X["cnt"][:, None] * Y["cnt"][None, :]
tot = float(w.sum())
res = {}
keep = {"ball": [], "slope": [], "box": []}
for i0 in range(0, K, 64):
    I = slice(i0, min(K, i0 + 64))
    D = X["cen"][I][:, None, :] - Y["cen"][None, :, :]
    dist = D.norm(dim=2)
    ba = X["fmax"][I][:, None] + Y["fmax"][None, :] - 0.5 * torch.clamp(dist - X["rad"][I][:, None] - Y["rad"][None, :], min=0) ** 2
    U = X["S"][I][:, None, :] - D
    V = Y["S"][None, :, :] + D
    base = X["Fp"][I][:, None] + Y["Fp"][None, :] - 0.5 * dist ** 2
    bb = base + X["rad"][I][:, None] * U.norm(dim=2) + Y["rad"][None, :] * V.norm(dim=2)
    q = box_quad(U, V, X["lo"][I][:, None, :], X["hi"][I][:, None, :], Y["lo"][None, :, :], Y["hi"][None, :, :]).sum(-1)
    bc = base + q
    wi = w[I]
    keep["ball"].append(float((wi * (ba >= thr)).sum()))
    keep["slope"].append(float((wi * (torch.minimum(ba, bb) >= thr)).sum()))
    keep["box"].append(float((wi * (torch.minimum(torch.minimum(ba, bb), bc) >= thr)).sum()))
for k, v in keep.items():
    res[k] = sum(v) / tot
rows = np.random.default_rng(0).choice(len(x), 1000, replace=False)
Xr, f = T(x[rows]), T(P.b_yx[rows])
Yt, g = T(y), T(P.a_xy)
kept = 0
for r0 in range(0, 1000, 100):
    C = 0.5 * torch.cdist(Xr[r0:r0 + 100], Yt) ** 2
    kept += int(((f[r0:r0 + 100, None] + g[None, :] - C) >= thr).sum())
res["exact"] = kept / (1000 * len(y))
print(json.dumps(dict(K=K, fine_kept_solver=st["pairs_fine"] / st["pairs_fine_dense"], **res)))
