"""Config 2: N=M=100k 3D Gaussian mixtures (seeds 3/4), multiscale voxel grid with
kernel truncation, blur 0.01, one B200.  python tools/config2.py"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
x, y = bench.mixture(n, 3), bench.mixture(n, 4)
a = np.full(n, 1.0 / n)
ctx = Context(0)
ctx.set_profiling(True)
prm = make_params(blur=0.01, multiscale=True, retruncate=1, switch_factor=1.0)
for rep in range(3):
    t = time.perf_counter()
    loss, _, st = ctx.sinkhorn(prm, x, a, y, a, potentials=False)
    wall = time.perf_counter() - t
ld, _, sd = ctx.sinkhorn(make_params(blur=0.01), x, a, y, a, potentials=False)
print(json.dumps(dict(n=n, device_ms=st["total_ms"], wall_s=wall, softmin_ms=st["softmin_ms"],
                      phases=st["phase_ms"], loss=loss, dense_loss=ld, rel_vs_dense=loss / ld - 1,
                      dense_ms=sd["total_ms"], kx=st["kx"], t_switch=st["t_switch"],
                      pairs=st["pairs_evaluated"])))
