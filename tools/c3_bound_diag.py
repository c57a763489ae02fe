"""C3: fraction of the (x_i, y_j) pairs with f_i + g_j - C_ij >= -theta eps at the
final cross potentials (row sample), against the fine phase's evaluated fraction."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2107_02010_b200.solver import Context

w = dict(bench.WORKLOAD)
x, a, y, b = bench.make_inputs(w)
ctx = Context(0)
loss, P, st = ctx.sinkhorn(bench.params(w), x, a, y, b)
eps, theta = w["blur"] ** 2, w["theta"]
dev = torch.device("cuda")
Y = torch.from_numpy(y).to(dev)
g = torch.from_numpy(P.a_xy).to(dev)
rows = torch.randperm(len(x), generator=torch.Generator().manual_seed(0))[:2000]
X = torch.from_numpy(x[rows.numpy()]).to(dev)
f = torch.from_numpy(P.b_yx[rows.numpy()]).to(dev)
kept = 0
for k in range(0, len(rows), 250):
    C = 0.5 * torch.cdist(X[k:k + 250], Y) ** 2
    kept += int(((f[k:k + 250, None] + g[None, :] - C) >= -theta * eps).sum())
true = kept / (len(rows) * len(y))
print(json.dumps(dict(true_kept_final=true, fine_evaluated_avg=st["pairs_fine"] / st["pairs_fine_dense"],
                      ratio=st["pairs_fine"] / st["pairs_fine_dense"] / true, loss=loss)))
