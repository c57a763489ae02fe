"""Rigorous two-level (voxel -> octant) column refinement of the C3 fine
phase, at tile granularity: for sampled 256-row tiles of the cross problem at
one fine update, the columns evaluated today (the union of the tile's kept
column clusters) against the columns kept by min(B_a, B_b, B_c) >= -theta eps
(mask.cu's three bounds) evaluated between the TILE's rows (centroid, radius,
max potential, fitted slope, F', member box) and each OCTANT of every kept
column cluster, and against the exact per-pair need (octant_probe.py).
python tools/octant_bound_probe.py [t_offset_from_switch]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from oracle import oracle as O
from paper_2107_02010_b200.solver import Context

w = dict(bench.WORKLOAD)
x, a, y, b = bench.make_inputs(w)
n, m = len(x), len(y)
prm = bench.params(w)
ctx = Context(0)
_, _, st = ctx.sinkhorn(prm, x, a, y, b, potentials=False)
tsw, ns = st["t_switch"], st["n_scales"]
off = int(sys.argv[1]) if len(sys.argv) > 1 else 0
t = min(tsw + off, ns)
_, eps_s, _ = O.schedule(st["diameter"], prm)
eps = eps_s[min(t, ns - 1)]
thr = -prm.theta * eps
before, _ = ctx.debug_capture(t, n, m)
ctx.sinkhorn(prm, x, a, y, b, potentials=False)
ctx.debug_capture(-1, 0, 0)
mask, rl, cl = ctx.debug_mask(2, n, m)
cell = st["cluster_scale"]
lo = np.minimum(x.min(0), y.min(0))
q = np.floor((y - lo) / (cell / 2)).astype(np.int64) & 1
octant = q[:, 0] | (q[:, 1] << 1) | (q[:, 2] << 2)
dev = torch.device("cuda")
T64 = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev, torch.float64)
order = np.argsort(rl, kind="stable")
g_all = T64(before["a_xy"])
f_all = before["b_yx"]
Y = T64(y)
# octant groups of the column clusters: id = 8 J + o
gid = torch.from_numpy(cl.astype(np.int64) * 8 + octant).to(dev)
K8 = mask.shape[1] * 8


def group_stats(P, F, L, k):
    cnt = torch.zeros(k, device=dev, dtype=torch.float64).index_add_(0, L, torch.ones_like(F))
    cen = torch.zeros(k, 3, device=dev, dtype=torch.float64).index_add_(0, L, P) / cnt.clamp(min=1)[:, None]
    u = P - cen[L]
    rad = torch.zeros(k, device=dev, dtype=torch.float64).scatter_reduce_(0, L, u.norm(dim=1), "amax")
    lo_ = torch.zeros(k, 3, device=dev, dtype=torch.float64)
    hi_ = torch.zeros(k, 3, device=dev, dtype=torch.float64)
    for d in range(3):
        lo_[:, d] = torch.zeros(k, device=dev, dtype=torch.float64).scatter_reduce_(0, L, u[:, d], "amin")
        hi_[:, d] = torch.zeros(k, device=dev, dtype=torch.float64).scatter_reduce_(0, L, u[:, d], "amax")
    fmax = torch.full((k,), -1e300, device=dev, dtype=torch.float64).scatter_reduce_(0, L, F, "amax")
    fbar = torch.zeros(k, device=dev, dtype=torch.float64).index_add_(0, L, F) / cnt.clamp(min=1)
    Muu = torch.zeros(k, 3, 3, device=dev, dtype=torch.float64).index_add_(0, L, u[:, :, None] * u[:, None, :])
    Muf = torch.zeros(k, 3, device=dev, dtype=torch.float64).index_add_(0, L, u * (F - fbar[L])[:, None])
    S = torch.linalg.solve(Muu + 1e-12 * torch.eye(3, device=dev, dtype=torch.float64), Muf[:, :, None])[:, :, 0]
    Fp = torch.full((k,), -1e300, device=dev, dtype=torch.float64).scatter_reduce_(0, L, F - (u * S[L]).sum(1), "amax")
    return dict(cnt=cnt, cen=cen, rad=rad, lo=lo_, hi=hi_, fmax=fmax, S=S, Fp=Fp)


Gs = group_stats(Y, g_all, gid, K8)


def q_axis(u, v, l1, h1, l2, h2):
    g = lambda aa, bb: u * aa + v * bb - 0.5 * (aa - bb) ** 2
    return torch.maximum(torch.maximum(g(l1, torch.clamp(l1 + v, l2, h2)), g(h1, torch.clamp(h1 + v, l2, h2))),
                         torch.maximum(g(torch.clamp(l2 + u, l1, h1), l2), g(torch.clamp(h2 + u, l1, h1), h2)))


rng = np.random.default_rng(0)
T = (n + 255) // 256
tot = dict(now=0.0, octant_bound=0.0, cluster_bound_tile=0.0, exact_octant=0.0, exact_pairs=0.0)
col_of_cluster = None
for tile in rng.choice(T - 1, 200, replace=False):
    rows = order[tile * 256:(tile + 1) * 256]
    kept = np.flatnonzero(mask[np.unique(rl[rows])].any(0))
    if len(kept) == 0:
        continue
    P = T64(x[rows])
    F = T64(f_all[rows])
    R = group_stats(P, F, torch.zeros(len(rows), dtype=torch.int64, device=dev), 1)
    groups = torch.from_numpy((kept[:, None] * 8 + np.arange(8)[None, :]).ravel()).to(dev)
    groups = groups[Gs["cnt"][groups] > 0]
    D = R["cen"][0][None, :] - Gs["cen"][groups]
    dist = D.norm(dim=1)
    ba = R["fmax"][0] + Gs["fmax"][groups] - 0.5 * torch.clamp(dist - R["rad"][0] - Gs["rad"][groups], min=0) ** 2
    U = R["S"][0][None, :] - D
    V = Gs["S"][groups] + D
    base = R["Fp"][0] + Gs["Fp"][groups] - 0.5 * dist ** 2
    bb = base + R["rad"][0] * U.norm(dim=1) + Gs["rad"][groups] * V.norm(dim=1)
    qs = sum(q_axis(U[:, k], V[:, k], R["lo"][0][k], R["hi"][0][k], Gs["lo"][groups][:, k], Gs["hi"][groups][:, k])
             for k in range(3))
    bc = base + qs
    keep = torch.minimum(torch.minimum(ba, bb), bc) >= thr
    sizes = Gs["cnt"][groups]
    nr = len(rows)
    tot["now"] += nr * float(sizes.sum())
    tot["octant_bound"] += nr * float(sizes[keep].sum())
    # same bound at cluster granularity (tile rows vs whole column cluster)
    cl_keep = keep.view(-1) if False else None
    # exact need per octant
    cols = torch.nonzero(torch.isin(gid, groups)).squeeze(1)
    C = 0.5 * torch.cdist(P, Y[cols]) ** 2
    need = (F[:, None] + g_all[cols][None, :] - C) >= thr
    tot["exact_pairs"] += float(need.sum())
    need_g = torch.zeros(K8, dtype=torch.bool, device=dev)
    need_g[gid[cols][need.any(0)]] = True
    tot["exact_octant"] += nr * float(Gs["cnt"][groups][need_g[groups]].sum())
print(json.dumps(dict(t=int(t), eps=float(eps), octant_bound=tot["octant_bound"] / tot["now"],
                      exact_octant=tot["exact_octant"] / tot["now"], ball=tot["exact_pairs"] / tot["now"])))
