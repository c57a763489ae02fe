"""Coarse -> fine transfer rule on C3 / C2 at bench parameters: inheritance
(transfer_rule 0) vs the GeomLoss extrapolation softmin
(transfer_rule 1): device time and distance of S_eps from the dense solve.
python tools/transfer_compare.py [n ...]  -> JSON lines"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dense_c3 = json.load(open(os.path.join(ROOT, "profiles", "r1_c3_dense_vs_multiscale.json")))["dense_S_eps"]
ctx = Context(0)
for n in [int(v) for v in sys.argv[1:]] or [1000000, 100000]:
    w = dict(bench.WORKLOAD, n=n, m=n)
    x, a, y, b = bench.make_inputs(w)
    if n == 1000000:
        dense = dense_c3
    else:
        dense, _, _ = ctx.sinkhorn(make_params(blur=0.01), x, a, y, b, potentials=False)
    for rule in [int(r) for r in os.environ.get("RULES", "0,1").split(",")]:
        prm = bench.params(w)
        prm.transfer_rule = rule
        for _ in range(3):
            loss, _, st = ctx.sinkhorn(prm, x, a, y, b, potentials=False)
        print(json.dumps(dict(n=n, transfer_rule=rule, device_ms=st["total_ms"], S_eps=loss,
                              dense_S_eps=dense, rel_vs_dense=loss / dense - 1,
                              pairs=st["pairs_evaluated"], t_switch=st["t_switch"])), flush=True)
