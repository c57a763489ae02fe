"""One C2 solve (100k vs 100k mixtures, seeds 3/4, bench.py's parameters)
after two warm-ups, for launch lists: python tools/c2_once.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_02010_b200.solver import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
x, y = bench.mixture(n, 3), bench.mixture(n, 4)
a = np.full(n, 1.0 / n)
w = dict(bench.WORKLOAD, n=n, m=n)
ctx = Context(0)
for _ in range(3):
    loss, _, st = ctx.sinkhorn(bench.params(w), x, a, y, a, potentials=False)
print(loss, st["total_ms"], st["gpu_launches"], st["host_syncs"], flush=True)
