"""Phase times of one config-5 solve + gradient (barycenter atoms vs one target)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

maps = W.density_maps(10)
targets = [W.density_to_measure(*m) for m in maps]
p, w = W.density_to_measure(*W.average_density(maps))
x0, a = W.upsample(p, w, 6, 0.5 / 128, 0)
ctx = Context(0)
ctx.set_profiling(True)
for kw in (dict(), dict(theta=12.5), dict(switch_factor=2.0)):
    prm = make_params(blur=1 / 128, multiscale=True, retruncate=1, switch_factor=kw.get("switch_factor", 1.0),
                      theta=kw.get("theta", 20.0))
    y, b = targets[0]
    for rep in range(2):
        l, g, st = ctx.sinkhorn_grad(prm, x0, a, y, b)
    print(json.dumps(dict(kw=kw, n=len(x0), m=len(y), loss=l, total_ms=st["total_ms"],
                          softmin_ms=st["softmin_ms"], phases=st["phase_ms"], kx=st["kx"],
                          ky=st["ky"], t_switch=st["t_switch"], n_scales=st["n_scales"],
                          pairs=st["pairs_evaluated"], launches=st["gpu_launches"])))
