"""Cost of the bounded column-partial batches: C2 (100k) and C3 (1M) at bench
parameters, phases and launches, for several MSOT_COLPART_BUDGET values:
python tools/batch_cost.py n budget [budget ...]   (0 = automatic)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2107_02010_b200.solver import Context
n = int(sys.argv[1])
w = dict(bench.WORKLOAD, n=n, m=n)
x, a, y, b = bench.make_inputs(w)
for bud in sys.argv[2:]:
    os.environ["MSOT_COLPART_BUDGET"] = bud
    ctx = Context(0)
    ctx.set_profiling(True)
    for _ in range(3):
        loss, _, st = ctx.sinkhorn(bench.params(w), x, a, y, b, potentials=False)
    ctx.set_profiling(False)
    for _ in range(3):
        loss, _, s2 = ctx.sinkhorn(bench.params(w), x, a, y, b, potentials=False)
    print(json.dumps(dict(n=n, budget=bud, total_ms=s2["total_ms"], prof_total_ms=st["total_ms"],
                          softmin_ms=st["softmin_ms"], launches=s2["gpu_launches"], host_syncs=s2["host_syncs"],
                          softmin_launches=st["softmin_launches"], batches=st["colpart_batches"],
                          device_mb=st["device_bytes"] / 1e6,
                          phases={k: round(v, 2) for k, v in st["phase_ms"].items()}, loss=loss)),
          flush=True)
    ctx.close()
