"""Upper bound of a two-level (voxel -> octant) column refinement of the C3
fine-phase pair sets: for sampled 256-row tiles of the cross
problem at one fine update, the columns the kernel evaluates today (the tile's
union of kept column clusters) against the columns an EXACT per-pair test
would need at cluster and at octant (sub-voxel) granularity, plus octants
trimmed to one contiguous run per cluster.  Exact = f_i + g_j - C_ij >=
-theta eps at that update's input potentials, so any rigorous bound keeps at
least this much.  python tools/octant_probe.py [t_offset_from_switch]"""
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
before, _ = ctx.debug_capture(t, n, m)
ctx.sinkhorn(prm, x, a, y, b, potentials=False)
ctx.debug_capture(-1, 0, 0)
mask, rl, cl = ctx.debug_mask(2, n, m)
cell = st["cluster_scale"]
lo = np.minimum(x.min(0), y.min(0))
# octant of every column atom: the next bit of its cube coordinates
q = np.floor((y - lo) / (cell / 2)).astype(np.int64) & 1
octant = q[:, 0] | (q[:, 1] << 1) | (q[:, 2] << 2)
# Morton order of octants inside a voxel (x lowest): octant id is already that order
order = np.argsort(rl, kind="stable")  # cluster-sorted rows
kc = mask.shape[1]
col_of_cluster = [[] for _ in range(kc)]
for j, J in enumerate(cl):
    col_of_cluster[J].append(j)
col_of_cluster = [np.array(v, np.int64) for v in col_of_cluster]
dev = torch.device("cuda")
Y = torch.from_numpy(y).to(dev)
g = torch.from_numpy(before["a_xy"]).to(dev)
f_all = before["b_yx"]
rng = np.random.default_rng(0)
T = (n + 255) // 256
tot = dict(now=0.0, cluster=0.0, octant=0.0, octant_run=0.0, ball=0.0)
for tile in rng.choice(T, 300, replace=False):
    rows = order[tile * 256:(tile + 1) * 256]
    kept = np.flatnonzero(mask[np.unique(rl[rows])].any(0))
    cols = np.concatenate([col_of_cluster[J] for J in kept]) if len(kept) else np.zeros(0, np.int64)
    if len(cols) == 0:
        continue
    X = torch.from_numpy(x[rows]).to(dev)
    f = torch.from_numpy(f_all[rows]).to(dev)
    cj = torch.from_numpy(cols).to(dev)
    C = 0.5 * torch.cdist(X, Y[cj]) ** 2
    inball = ((f[:, None] + g[cj][None, :] - C) >= -prm.theta * eps).any(0).cpu().numpy()
    nr = len(rows)
    tot["now"] += nr * len(cols)
    tot["ball"] += float(((f[:, None] + g[cj][None, :] - C) >= -prm.theta * eps).sum())
    # per cluster / octant need
    pos = 0
    for J in kept:
        cj_ = col_of_cluster[J]
        need = inball[pos:pos + len(cj_)]
        oc = octant[cj_]
        pos += len(cj_)
        if need.any():
            tot["cluster"] += nr * len(cj_)
            needed_oct = np.unique(oc[need])
            tot["octant"] += nr * np.isin(oc, needed_oct).sum()
            lo_o, hi_o = needed_oct.min(), needed_oct.max()
            tot["octant_run"] += nr * ((oc >= lo_o) & (oc <= hi_o)).sum()
print(json.dumps(dict(t=int(t), eps=float(eps), **{k: v / tot["now"] for k, v in tot.items()})))
