import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context
def mixture(n, seed, d=3, k=8, sigma=0.05):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.2, 0.8, (k, d))
    return cen[rng.integers(0, k, n)] + rng.normal(0, sigma, (n, d))
ctx = Context(0)
rng = np.random.default_rng(7)
n = 10000
xb = np.concatenate([rng.normal(0, 0.03, (n // 2, 3)), rng.normal(1, 0.03, (n // 2, 3))])
yb = np.concatenate([rng.normal(0.02, 0.03, (n // 2, 3)), rng.normal(1.02, 0.03, (n // 2, 3))])
for name, x, y in [("mix20k", mixture(20000, 5), mixture(20000, 6)), ("blobs10k", xb, yb)]:
    a = np.full(len(x), 1 / len(x))
    ld, _, _ = ctx.sinkhorn(make_params(blur=0.01), x, a, y, a, potentials=False)
    for sf in (2.0, 1.0):
        for th in (20.0, 5.0):
            for rt in (0, 1):
                lm, _, st = ctx.sinkhorn(make_params(blur=0.01, multiscale=True, retruncate=rt, theta=th, switch_factor=sf), x, a, y, a, potentials=False)
                print(name, sf, th, rt, st['kx'], st['t_switch'], st['n_scales'], round(st['pairs_fine'] / st['pairs_fine_dense'], 4), f"{(lm - ld) / ld:.2e}", flush=True)
