"""C3 (and C2) at bench parameters with the round-1 mask (mask_rule 2: min of
the radius and slope bounds) and with the member-box bound (mask_rule 0):
device time, evaluated pairs, S_eps and its distance from the dense solve.
python tools/mask_rule_ab.py [n ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2107_02010_b200.solver import Context

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dense_c3 = json.load(open(os.path.join(ROOT, "profiles", "r1_c3_dense_vs_multiscale.json")))["dense_S_eps"]
ctx = Context(0)
for n in [int(v) for v in sys.argv[1:]] or [1000000, 100000]:
    w = dict(bench.WORKLOAD, n=n, m=n)
    x, a, y, b = bench.make_inputs(w)
    for rule in (2, 0):
        prm = bench.params(w)
        prm.mask_rule = rule
        ts = []
        for _ in range(4):
            loss, _, st = ctx.sinkhorn(prm, x, a, y, b, potentials=False)
            ts.append(st["total_ms"])
        print(json.dumps(dict(n=n, mask_rule=rule, device_ms=min(ts[1:]), S_eps=loss,
                              rel_vs_dense=(loss / dense_c3 - 1) if n == 1000000 else None,
                              pairs=st["pairs_evaluated"], fine_kept=st["pairs_fine"] / st["pairs_fine_dense"],
                              fallback_rows=st["fallback_rows"])), flush=True)
