"""One S_eps solve (for ncu captures): python tools/one_solve.py N [ms] [cell] [theta]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

def mixture(n, seed, d=3, k=8, sigma=0.05):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.2, 0.8, (k, d))
    return cen[rng.integers(0, k, n)] + rng.normal(0, sigma, (n, d))

n = int(sys.argv[1]); ms = len(sys.argv) > 2 and sys.argv[2] == "ms"
cell = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
theta = float(sys.argv[4]) if len(sys.argv) > 4 else 20.0
blur = 0.01 if ms else 0.5
x, y = mixture(n, 5), mixture(n, 6)
a = np.full(n, 1 / n)
ctx = Context(0)
loss, _, st = ctx.sinkhorn(make_params(blur=blur, multiscale=ms, retruncate=1, cluster_scale=cell, theta=theta), x, a, y, a, potentials=False)
print(loss, st)
