"""One C3 solve at bench.py's parameters after a warm-up (for ncu captures):
python tools/c3_once.py [n] [colpart_budget]   (budget 0 = automatic)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2107_02010_b200.solver import Context
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 0
w = dict(bench.WORKLOAD, n=n, m=n)
x, a, y, b = bench.make_inputs(w)
ctx = Context(0)
ctx.set_colpart_budget(budget)
loss, _, st = ctx.sinkhorn(bench.params(w), x, a, y, b, potentials=False)
print(loss, st["total_ms"], st["gpu_launches"], st["colpart_batches"], flush=True)
