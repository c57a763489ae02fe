import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context
from oracle import oracle as O
def blobs(seed, n, shift):
    rng = np.random.default_rng(seed)
    return rng.normal(0.5, 0.08, (n, 3)) + shift
targets = []
for k in range(3):
    yk = blobs(30 + k, 2500, 0.1 * np.array([k, -k, 0.5 * k]))
    targets.append((yk, np.full(2500, 1 / 2500)))
x0 = blobs(40, 3000, 0.05)
a = np.full(3000, 1 / 3000)
prm = make_params(blur=0.01, multiscale=True, retruncate=1, cluster_scale=0.04, switch_factor=1.0)
ctx = Context(0)
for k in range(3):
    lg, gg, sg = ctx.sinkhorn_grad(prm, x0, a, *targets[k])
    lo, go = O.sinkhorn_grad(prm, x0, a, *targets[k])
    fg, fo = gg / a[:, None], go / a[:, None]
    e = np.abs(fg - fo).max(1)
    i = int(e.argmax())
    print(k, "loss", lg, lo, "field err max", e.max(), "at", i, "field", fo[i], "median err", np.median(e), "n>1e-4", (e > 1e-4).sum())
    d = np.linalg.norm(targets[k][0] - x0[i], axis=1)
    print("   atom", x0[i], "nearest target dist", d.min(), "|field|", np.linalg.norm(fo[i]))
for it in (1, 2, 3):
    xg, tg, _ = ctx.barycenter(prm, x0, a, targets, iters=it)
    xo, to = O.barycenter(prm, x0, a, targets, iters=it)
    e = np.abs(xg - xo).max(1)
    print("iters", it, "traj", tg, to, "pos err", e.max(), "at", int(e.argmax()), "n>1e-4", (e > 1e-4).sum())
