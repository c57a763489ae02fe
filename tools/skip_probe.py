"""In-kernel skip headroom of K4s on the C3 fine phase: for sampled 256-row
tiles of the cross problem at one fine update, the fraction of the kernel's
(warp rows x column pair) units that hold at least one pair with
f_i + g_j - C_ij >= -theta eps (at that update's input potentials), for the
current strided row layout (thread t: rows t + 64 q, each warp spans the
tile) and for a contiguous one (warp w: rows 128 w .. 128 w + 127).
python tools/skip_probe.py [t_offset_from_switch]"""
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
order = np.argsort(rl, kind="stable")
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
strided = [np.arange(256).reshape(4, 64)[:, w0 * 32:(w0 + 1) * 32].ravel() for w0 in range(2)]
contig = [np.arange(128) + 128 * w0 for w0 in range(2)]
tot = dict(units=0, strided=0, contig=0, contig64=0, pairs=0, ball=0)
for tile in rng.choice(T, 300, replace=False):
    rows = order[tile * 256:(tile + 1) * 256]
    if len(rows) < 256:
        continue
    kept = np.flatnonzero(mask[np.unique(rl[rows])].any(0))
    cols = np.concatenate([col_of_cluster[J] for J in kept]) if len(kept) else np.zeros(0, np.int64)
    if len(cols) == 0:
        continue
    cols = np.sort(cols)
    if len(cols) % 2:
        cols = cols[:-1]
    X = torch.from_numpy(x[rows]).to(dev)
    f = torch.from_numpy(f_all[rows]).to(dev)
    cj = torch.from_numpy(cols).to(dev)
    C = 0.5 * torch.cdist(X, Y[cj]) ** 2
    need = (f[:, None] + g[cj][None, :] - C) >= -prm.theta * eps  # 256 x nc
    pairs = need.view(256, -1, 2).any(2)  # per column pair
    tot["units"] += 2 * pairs.shape[1]
    tot["pairs"] += 256 * len(cols)
    tot["ball"] += int(need.sum())
    for lay, key in ((strided, "strided"), (contig, "contig")):
        for rr in lay:
            tot[key] += int(pairs[torch.as_tensor(rr, device=dev)].any(0).sum())
    for w0 in range(4):
        tot["contig64"] += int(pairs[64 * w0:64 * (w0 + 1)].any(0).sum()) / 2
print(json.dumps(dict(t=int(t), eps=float(eps), ball=tot["ball"] / tot["pairs"],
                      strided=tot["strided"] / tot["units"], contig=tot["contig"] / tot["units"],
                      contig64=tot["contig64"] / tot["units"])))
