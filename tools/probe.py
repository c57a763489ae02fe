"""Quick GPU probe: multiscale solves (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

def mixture(n, seed, d=3, k=8, sigma=0.05):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.2, 0.8, (k, d))
    return cen[rng.integers(0, k, n)] + rng.normal(0, sigma, (n, d))

ctx = Context(0)
ctx.set_profiling(True)
cfgs = []
for sf in (2.0, 1.0):
    for th in (20.0, 5.0):
        cfgs.append((1000000, dict(blur=0.01, multiscale=True, retruncate=1, theta=th, switch_factor=sf)))
cfgs.append((1000000, dict(blur=0.01, multiscale=True, retruncate=1, theta=20.0, switch_factor=1.0, cluster_scale=0.03)))
for n, kw in cfgs:
    x, y = mixture(n, 5), mixture(n, 6)
    a = np.full(n, 1 / n)
    t = time.time()
    loss, _, st = ctx.sinkhorn(make_params(**kw), x, a, y, a, potentials=False)
    wall = time.time() - t
    print(f"n={n} {kw} loss={loss:.8g} wall={wall:.3f}s total_ms={st['total_ms']:.1f} "
          f"softmin_ms={st['softmin_ms']:.1f} pairs={st['pairs_evaluated']:.3e} "
          f"rate={st['pairs_evaluated']/st['softmin_ms']*1e3:.3e} launches={st['gpu_launches']} "
          f"kx={st['kx']} cell={st['cluster_scale']:.4f} tsw={st['t_switch']}/{st['n_scales']} fine={st['pairs_fine']/max(st['pairs_fine_dense'],1):.4f} fb={st['fallback_rows']} phases={ {k: round(v, 1) for k, v in st['phase_ms'].items()} }", flush=True)
