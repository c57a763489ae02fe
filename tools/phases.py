"""Per-phase device time of one C3-style solve: python tools/phases.py [N]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_02010_b200.solver import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
w = dict(bench.WORKLOAD, n=n, m=n)
x, a, y, b = bench.make_inputs(w)
ctx = Context(0)
ctx.set_profiling(True)
prm = bench.params(w)
for rep in range(2):
    loss, _, st = ctx.sinkhorn(prm, x, a, y, b, potentials=False)
names = ["setup", "coarse", "extrapolate", "masks", "fine", "loss"]
print(json.dumps(dict(n=n, loss=loss, total_ms=st["total_ms"], softmin_ms=st["softmin_ms"],
                      phases=st["phase_ms"],
                      pairs=st["pairs_evaluated"], terms=st["pairs_terms"],
                      mask_terms=st["pairs_mask_terms"], fine=st["pairs_fine"], kept=st["pairs_fine"] / st["pairs_fine_dense"],
                      kx=st["kx"], t_switch=st["t_switch"], n_scales=st["n_scales"])))
