"""Softmin throughput vs the MUFU/FMA exp2 split (MSOT_POLY16 set by the caller)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context
ctx = Context(0)
ctx.set_profiling(True)
x, y = bench.mixture(300000, 5), bench.mixture(300000, 6)
a = np.full(300000, 1 / 300000)
l, _, st = ctx.sinkhorn(make_params(blur=0.5), x, a, y, a, potentials=False)
l, _, st = ctx.sinkhorn(make_params(blur=0.5), x, a, y, a, potentials=False)
print("poly16", os.environ.get("MSOT_POLY16"), "dense rate", st["pairs_evaluated"] / st["softmin_ms"] * 1e3, "loss", repr(l), flush=True)
w = dict(bench.WORKLOAD)
X, A, Y, B = bench.make_inputs(w)
ls = []
for _ in range(2):
    l, _, st = ctx.sinkhorn(bench.params(w), X, A, Y, B, potentials=False)
print("poly16", os.environ.get("MSOT_POLY16"), "C3 total_ms", st["total_ms"], "softmin_ms", st["softmin_ms"], "rate", st["pairs_evaluated"] / st["softmin_ms"] * 1e3, "loss", repr(l), "fb", st["fallback_rows"], flush=True)
