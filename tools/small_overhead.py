"""Fixed cost of the multiscale path at small N: SPEC.md:590's 10k two-blob
fixture, dense vs multiscale device time, per-phase split, launches and
host waits.  python tools/small_overhead.py [n]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
rng = np.random.default_rng(7)
x = np.concatenate([rng.normal(0, 0.03, (n // 2, 3)), rng.normal(1, 0.03, (n // 2, 3))])
y = np.concatenate([rng.normal(0.02, 0.03, (n // 2, 3)), rng.normal(1.02, 0.03, (n // 2, 3))])
a = np.full(n, 1 / n)
ctx = Context(0)
for name, prm in (("dense", make_params(blur=0.01)),
                  ("ms", make_params(blur=0.01, multiscale=True, retruncate=1))):
    for _ in range(3):
        _, _, st = ctx.sinkhorn(prm, x, a, y, a, potentials=False)
    ctx.set_profiling(True)
    _, _, sp = ctx.sinkhorn(prm, x, a, y, a, potentials=False)
    ctx.set_profiling(False)
    print(json.dumps(dict(mode=name, n=n, device_ms=st["total_ms"], launches=st["gpu_launches"],
                          host_syncs=st["host_syncs"], n_scales=st["n_scales"],
                          t_switch=st["t_switch"], t_super=st["t_super"], kx=st["kx"],
                          softmin_ms_prof=sp["softmin_ms"], phases_prof=sp["phase_ms"],
                          total_prof=sp["total_ms"])), flush=True)
