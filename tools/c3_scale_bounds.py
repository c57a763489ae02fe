"""C3 truncation tightness per fine scale (cross problem x-y), at bench.py's
parameters: for every fine update t (t_switch .. final assignment) the
fraction of atom pairs
  ball    f_i + g_j - C_ij >= -theta eps_t   at that update's input potentials
          (2000 sampled rows against all columns)
  mask    inside kept cluster pairs (the captured cluster mask)
  tiles   inside the column ranges of the 256-row tile (the union of its row
          clusters' kept columns: what the kernel evaluates)
so the evaluated / needed ratio splits into the ball-size part (the eps
schedule), the cluster granularity and the tile union.
python tools/c3_scale_bounds.py [n]  -> JSON lines"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from oracle import oracle as O
from paper_2107_02010_b200.solver import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
w = dict(bench.WORKLOAD, n=n, m=n)
x, a, y, b = bench.make_inputs(w)
prm = bench.params(w)
ctx = Context(0)
_, _, st = ctx.sinkhorn(prm, x, a, y, b, potentials=False)
ns, tsw = st["n_scales"], st["t_switch"]
sig, eps_s, _ = O.schedule(st["diameter"], prm)
dev = torch.device("cuda")
Y = torch.from_numpy(y).to(dev)
rows = np.sort(np.random.default_rng(0).choice(n, 2000, replace=False))
X = torch.from_numpy(x[rows]).to(dev)
for t in range(tsw, ns + 1):
    before, _ = ctx.debug_capture(t, n, n)
    try:
        ctx.sinkhorn(prm, x, a, y, b, potentials=False)
    finally:
        ctx.debug_capture(-1, 0, 0)
    eps = eps_s[min(t, ns - 1)]
    f = torch.from_numpy(before["b_yx"][rows]).to(dev)
    g = torch.from_numpy(before["a_xy"]).to(dev)
    kept = 0
    for k in range(0, len(rows), 250):
        C = 0.5 * torch.cdist(X[k:k + 250], Y) ** 2
        kept += int(((f[k:k + 250, None] + g[None, :] - C) >= -prm.theta * eps).sum())
    ball = kept / (len(rows) * n)
    mask, rl, cl = ctx.debug_mask(2, n, n)
    kr, kc = mask.shape
    rsz = np.bincount(rl, minlength=kr).astype(np.float64)
    csz = np.bincount(cl, minlength=kc).astype(np.float64)
    mfrac = float(rsz @ mask.astype(np.float64) @ csz) / (float(n) * n)
    # uniform 256-row tiles of the cluster-sorted rows (policy.h msot_row_tiles)
    lab_sorted = np.sort(rl)
    tile_pairs = 0.0
    for s in range(0, n, 256):
        cs = np.unique(lab_sorted[s:s + 256])
        union = mask[cs].any(axis=0)
        tile_pairs += min(256, n - s) * float(csz[union].sum())
    tfrac = tile_pairs / (float(n) * n)
    print(json.dumps(dict(t=int(t), sigma=float(sig[min(t, ns - 1)]), final=t == ns, ball=ball,
                          mask=mfrac, tiles=tfrac, mask_over_ball=mfrac / ball,
                          tiles_over_mask=tfrac / mfrac)), flush=True)
