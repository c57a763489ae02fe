import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

def mixture(n, seed, d=3, k=8, sigma=0.05):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.2, 0.8, (k, d))
    return cen[rng.integers(0, k, n)] + rng.normal(0, sigma, (n, d))


def uniform(n, seed, d=3):
    return np.random.default_rng(seed).random((n, d))
ctx = Context(0)
rng = np.random.default_rng(590)
for k in range(20):
    d = 2 + k % 2
    n, m = int(rng.integers(200, 2001)), int(rng.integers(200, 2001))
    kind = k % 3
    if kind == 0:
        x, y = mixture(n, 100 + k, d), mixture(m, 200 + k, d)
    elif kind == 1:
        x, y = uniform(n, 100 + k, d), uniform(m, 200 + k, d) * 0.8 + 0.1
    else:
        x = mixture(n, 100 + k, d, k=3, sigma=0.08)
        y = x[rng.integers(0, n, m)] + 0.05 + rng.normal(0, 0.02, (m, d))
    a, b = rng.random(n) + 0.5, rng.random(m) + 0.5
    a, b = a / a.sum(), b / b.sum()
    blur = float(rng.choice([0.01, 0.02, 0.05]))
    ld, _, _ = ctx.sinkhorn(make_params(blur=blur), x, a, y, b, potentials=False)
    out = []
    for kw in (dict(), dict(transfer_rule=1), dict(switch_factor=3.0), dict(transfer_rule=1, switch_factor=3.0)):
        lm, _, st = ctx.sinkhorn(make_params(blur=blur, multiscale=True, retruncate=1, **kw), x, a, y, b, potentials=False)
        out.append((round(abs(lm-ld)/abs(ld)*1e4, 2), st["t_switch"], st["n_scales"], st["kx"], st["ky"], round(st["cluster_scale"], 4)))
    print(k, n, m, d, blur, kind, out, flush=True)
