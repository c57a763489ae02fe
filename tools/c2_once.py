"""One C2 solve (100k vs 100k mixtures, seeds 3/4, bench parameters) after two
warm-ups, for launch lists: python tools/c2_once.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_02010_b200.solver import Context
w = dict(bench.WORKLOAD, n=100000, m=100000)
x, y = bench.mixture(100000, 3), bench.mixture(100000, 4)
a = np.full(100000, 1e-5)
ctx = Context(0)
for _ in range(3):
    loss, _, st = ctx.sinkhorn(bench.params(w), x, a, y, a, potentials=False)
print(loss, st["total_ms"], st["gpu_launches"], st["host_syncs"], flush=True)
