"""Config 5: Wasserstein barycenter of 10 synthetic 128^3 track-density maps
(blur = voxel, reach = inf, init = average density upsampled x6)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
maps = W.density_maps(10)
targets = [W.density_to_measure(*m) for m in maps]
p, w = W.density_to_measure(*W.average_density(maps))
x0, a = W.upsample(p, w, 6, 0.5 / 128, 0)
prm = make_params(blur=1 / 128, multiscale=True, retruncate=1, switch_factor=1.0)
ctx = Context(0)
t = time.perf_counter()
x, traj, st = ctx.barycenter(prm, x0, a, targets, iters=iters, step=1.0, tol=0.0)
dt = time.perf_counter() - t
out = dict(atoms=len(x0), target_atoms=[len(b) for _, b in targets], iters=len(traj) - 1,
           seconds=dt, seconds_per_iter=dt / max(1, len(traj) - 1), loss=list(traj),
           device_ms=st["total_ms"], pairs=st["pairs_evaluated"], solves=st["softmin_launches"])
print(json.dumps(out))
