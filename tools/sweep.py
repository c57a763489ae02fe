"""Parameter sweep of the C3 solve: python tools/sweep.py key=v1,v2,... [key2=...]
(times one solve per setting after a warm-up; prints phase times)."""
import itertools, json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

grid = {}
shape = "mixture"
for a in sys.argv[1:]:
    k, v = a.split("=")
    if k == "shape":
        shape = v
        continue
    grid[k] = [float(x) for x in v.split(",")]
w = dict(bench.WORKLOAD)
x, a, y, b = bench.make_inputs(w)
if shape == "uniform":  # SURVEY.md §8d C3 second shape
    import numpy as np
    x = np.random.default_rng(5).random((w["n"], 3))
    y = np.random.default_rng(6).random((w["m"], 3))
ctx = Context(0)
ctx.set_profiling(True)
base = dict(blur=w["blur"], reach=math.inf, scaling=w["scaling"], multiscale=True,
            retruncate=w["retruncate"], theta=w["theta"], switch_factor=w["switch_factor"])
for combo in itertools.product(*grid.values()):
    kw = dict(base)
    for k, v in zip(grid.keys(), combo):
        kw[k] = int(v) if k in ("retruncate", "pair_eval", "mask_rule", "transfer_rule") else v
    prm = make_params(**kw)
    ctx.sinkhorn(prm, x, a, y, b, potentials=False)
    loss, _, st = ctx.sinkhorn(prm, x, a, y, b, potentials=False)
    print(json.dumps(dict(zip(grid.keys(), combo), total_ms=round(st["total_ms"], 1),
                          softmin_ms=round(st["softmin_ms"], 1),
                          phases={k: round(v, 1) for k, v in st["phase_ms"].items()},
                          pairs=st["pairs_evaluated"], kx=st["kx"], t_switch=st["t_switch"],
                          loss=loss)), flush=True)
