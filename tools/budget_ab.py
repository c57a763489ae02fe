"""C3 device time with the automatic colpart budget (bounded, batched on two
streams) against one batch per update: python tools/budget_ab.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2107_02010_b200.solver import Context
w = dict(bench.WORKLOAD)
x, a, y, b = bench.make_inputs(w)
ctx = Context(0)
for budget in [0, 1 << 40, 0, 1 << 40]:
    ctx.set_colpart_budget(budget)
    ts = []
    for _ in range(4):
        loss, _, st = ctx.sinkhorn(bench.params(w), x, a, y, b, potentials=False)
        ts.append(st["total_ms"])
    print(json.dumps(dict(budget=budget, ms=sorted(ts)[:3], batches=st["colpart_batches"], launches=st["gpu_launches"])), flush=True)
