"""Config 5 barycenter (3 descent steps after a warm-up) with per-phase
device times (profiling mode: launches serialised): where an iteration goes.
python tools/config5_profile.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

maps = W.density_maps(10)
targets = [W.density_to_measure(*m) for m in maps]
p, w = W.density_to_measure(*W.average_density(maps))
x0, a = W.upsample(p, w, 6, 0.5 / 128, 0)
prm = make_params(blur=1 / 128, multiscale=True, retruncate=1, switch_factor=1.0)
ctx = Context(0)
ctx.barycenter(prm, x0, a, targets, iters=1, step=1.0, tol=0.0)
for prof in (False, True):
    ctx.set_profiling(prof)
    x, traj, st = ctx.barycenter(prm, x0, a, targets, iters=3, step=1.0, tol=0.0)
    print(json.dumps(dict(profiling=prof, device_ms=st["total_ms"], softmin_ms=st.get("softmin_ms"),
                          phases=st.get("phase_ms"), pairs=st["pairs_evaluated"],
                          launches=st["gpu_launches"], host_syncs=st.get("host_syncs"))), flush=True)
