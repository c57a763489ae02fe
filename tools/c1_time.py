"""C1 (10k vs 10k uniform 3D, blur 0.05, dense eps-scaling): device ms of the
solve (min of 5 after a warm-up).  python tools/c1_time.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

x = np.random.default_rng(1).random((10000, 3))
y = np.random.default_rng(2).random((10000, 3))
w = np.full(10000, 1e-4)
ctx = Context(0)
ts = []
for _ in range(6):
    loss, _, st = ctx.sinkhorn(make_params(blur=0.05), x, w, y, w, potentials=False)
    ts.append(st["total_ms"])
print("C1 ms", min(ts[1:]), "S", loss)
