"""How tight is the high-D truncation?  Fraction of (x_i, y_j) pairs with
f_i + g_j - C_ij >= -theta eps at the final potentials, on a row sample."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
fa, _ = W.fibres(n, 7, bundles=50, bundle_seed=1)
fb, _ = W.fibres(n, 8, bundles=50, bundle_seed=1)
x, a = W.flip_augment(*W.encode_fibers(fa))
y, b = W.flip_augment(*W.encode_fibers(fb))
ctx = Context(0)
prm = make_params(blur=0.03, reach=0.3)
loss, P, st = ctx.sinkhorn(prm, x, a, y, b)
eps = 0.03 ** 2
rng = np.random.default_rng(0)
rows = rng.choice(len(x), 300, replace=False)
out = {}
for theta in (20.0, 12.5):
    kept = 0
    for i in rows:
        c = 0.5 * ((y - x[i]) ** 2).sum(1)
        kept += np.count_nonzero(P.b_yx[i] + P.a_xy - c >= -theta * eps)
    out[theta] = kept / (len(rows) * len(y))
# distances between fibres: nearest-neighbour and within-bundle scales
d2 = ((y[:2000, None, :] - y[None, :2000, :]) ** 2).sum(-1)
print(json.dumps(dict(kept_fraction_true=out, loss=loss, eps=eps,
                      dist_quantiles=np.quantile(np.sqrt(d2[np.triu_indices(2000, 1)]),
                                                 [0.01, 0.05, 0.1, 0.5]).tolist())))
