"""Would a tighter cluster-pair bound shrink the C3 fine-phase pair sets?
For one fine update of the cross problem, recompute per cluster (from the
captured input potentials) the mask inputs — centroid, radius, max potential,
least-squares slope S and F' = max(f - <S, u>) — plus the axis-aligned box of
the members' offsets, and compare on sampled 256-row tiles the evaluated
(tile-union) pairs of
  now   min(B_a, B_b)          B_b = F' + G' + r_I|S - D| + r_J|T + D| - |D|^2/2
  box   min(B_a, B_c)          B_c = F' + G' - |D|^2/2 + sum_k max_{a_k, b_k in the
                               boxes} [(S - D)_k a_k + (T + D)_k b_k - (a_k - b_k)^2/2]
  exact the clusters holding a pair with f + g - C >= -theta eps
(B_c keeps the -|a - b|^2/2 term B_b drops; per axis a concave quadratic on a
rectangle, maximised over its four edges).  python tools/box_bound_probe.py [t_offset]"""
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
t = min(tsw + (int(sys.argv[1]) if len(sys.argv) > 1 else 0), ns)
_, eps_s, _ = O.schedule(st["diameter"], prm)
eps = eps_s[min(t, ns - 1)]
thr = -prm.theta * eps
before, _ = ctx.debug_capture(t, n, m)
ctx.sinkhorn(prm, x, a, y, b, potentials=False)
ctx.debug_capture(-1, 0, 0)
mask, rl, cl = ctx.debug_mask(2, n, m)
dev = torch.device("cuda")
T64 = lambda v: torch.from_numpy(np.ascontiguousarray(v)).to(dev, torch.float64)


def stats(pts, f, lab, k):
    P, F, L = T64(pts), T64(f), torch.from_numpy(lab.astype(np.int64)).to(dev)
    cnt = torch.zeros(k, device=dev, dtype=torch.float64).index_add_(0, L, torch.ones_like(F))
    cen = torch.zeros(k, 3, device=dev, dtype=torch.float64).index_add_(0, L, P) / cnt[:, None]
    u = P - cen[L]
    rad = torch.zeros(k, device=dev, dtype=torch.float64).scatter_reduce_(0, L, u.norm(dim=1), "amax")
    lo = torch.zeros(k, 3, device=dev, dtype=torch.float64)
    hi = torch.zeros(k, 3, device=dev, dtype=torch.float64)
    for d in range(3):
        lo[:, d] = torch.zeros(k, device=dev, dtype=torch.float64).scatter_reduce_(0, L, u[:, d], "amin")
        hi[:, d] = torch.zeros(k, device=dev, dtype=torch.float64).scatter_reduce_(0, L, u[:, d], "amax")
    fmax = torch.full((k,), -1e300, device=dev, dtype=torch.float64).scatter_reduce_(0, L, F, "amax")
    Muu = torch.zeros(k, 3, 3, device=dev, dtype=torch.float64).index_add_(0, L, u[:, :, None] * u[:, None, :])
    fbar = torch.zeros(k, device=dev, dtype=torch.float64).index_add_(0, L, F) / cnt
    Muf = torch.zeros(k, 3, device=dev, dtype=torch.float64).index_add_(0, L, u * (F - fbar[L])[:, None])
    S = torch.linalg.solve(Muu + 1e-12 * torch.eye(3, device=dev, dtype=torch.float64), Muf[:, :, None])[:, :, 0]
    Fp = torch.full((k,), -1e300, device=dev, dtype=torch.float64).scatter_reduce_(
        0, L, F - (u * S[L]).sum(1), "amax")
    return dict(cen=cen, rad=rad, lo=lo, hi=hi, fmax=fmax, S=S, Fp=Fp)


kx, ky = mask.shape
X = stats(x, before["b_yx"], rl, kx)
Y = stats(y, before["a_xy"], cl, ky)


def q_axis(u, v, l1, h1, l2, h2):
    g = lambda aa, bb: u * aa + v * bb - 0.5 * (aa - bb) ** 2
    c1 = g(l1, torch.clamp(l1 + v, l2, h2))
    c2 = g(h1, torch.clamp(h1 + v, l2, h2))
    c3 = g(torch.clamp(l2 + u, l1, h1), l2)
    c4 = g(torch.clamp(h2 + u, l1, h1), h2)
    return torch.maximum(torch.maximum(c1, c2), torch.maximum(c3, c4))


def bounds(I):
    I = torch.as_tensor(I, device=dev)
    D = X["cen"][I][:, None, :] - Y["cen"][None, :, :]
    dist = D.norm(dim=2)
    rI, rJ = X["rad"][I][:, None], Y["rad"][None, :]
    ba = X["fmax"][I][:, None] + Y["fmax"][None, :] - 0.5 * torch.clamp(dist - rI - rJ, min=0) ** 2
    u = X["S"][I][:, None, :] - D
    v = Y["S"][None, :, :] + D
    base = X["Fp"][I][:, None] + Y["Fp"][None, :] - 0.5 * dist ** 2
    bb = base + rI * u.norm(dim=2) + rJ * v.norm(dim=2)
    qs = sum(q_axis(u[..., k], v[..., k], X["lo"][I][:, None, k], X["hi"][I][:, None, k],
                    Y["lo"][None, :, k], Y["hi"][None, :, k]) for k in range(3))
    bc = base + qs
    return torch.minimum(ba, bb) >= thr, torch.minimum(ba, bc) >= thr


order = np.argsort(rl, kind="stable")
csize = torch.from_numpy(np.bincount(cl, minlength=ky).astype(np.float64)).to(dev)
rng = np.random.default_rng(0)
T = (n + 255) // 256
tot = {"mask": 0.0, "now": 0.0, "box": 0.0}
for tile in rng.choice(T, 300, replace=False):
    rows = order[tile * 256:(tile + 1) * 256]
    I = np.unique(rl[rows])
    now, box = bounds(I)
    nr = len(rows)
    tot["mask"] += nr * float(csize[torch.from_numpy(mask[I].any(0)).to(dev)].sum())
    tot["now"] += nr * float(csize[now.any(0)].sum())
    tot["box"] += nr * float(csize[box.any(0)].sum())
print(json.dumps(dict(t=int(t), eps=float(eps), mask_captured=1.0,
                      bound_now=tot["now"] / tot["mask"], bound_box=tot["box"] / tot["mask"])))
