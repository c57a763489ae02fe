"""Dense (no truncation, no coarsening) S_eps of the C3 workload on the GPU:
the reference value the multiscale bench config is compared against."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context
w = dict(bench.WORKLOAD)
x, a, y, b = bench.make_inputs(w)
ctx = Context(0)
ld, _, sd = ctx.sinkhorn(make_params(blur=w["blur"], scaling=w["scaling"]), x, a, y, b, potentials=False)
lm, _, sm = ctx.sinkhorn(bench.params(w), x, a, y, b, potentials=False)
out = dict(dense_S_eps=ld, dense_ms=sd["total_ms"], multiscale_S_eps=lm, multiscale_ms=sm["total_ms"],
           rel_diff=(lm - ld) / ld, pairs_dense=sd["pairs_evaluated"], pairs_multiscale=sm["pairs_evaluated"])
print(json.dumps(out))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/c3_dense_vs_multiscale.json", "w"), indent=1)
