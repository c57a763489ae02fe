"""Multi-rank (host-collective seam, one GPU) vs one-rank solve: largest
potential difference in units of eps and the loss difference, per case.
python tools/rank_diff.py [world]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import test_dist_gpu as T
from paper_2107_02010_b200.solver import Context

if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ctx = Context(0)
    for case in ["multiscale", "unbalanced", "hd_ms", "bench"]:
        x, a, y, b = T._inputs(case)
        l1, p1, _ = ctx.sinkhorn(T._params(case), x, a, y, b)
        out = T.run_two_ranks(case, world=world)
        eps = T._params(case).blur ** 2
        ref = [p1.a_xx, p1.b_yy, p1.a_xy, p1.b_yx]
        d = max(float(np.abs(u - v).max()) for r in range(world) for u, v in zip(out[r][1], ref))
        ne = sum(int((u != v).sum()) for u, v in zip(out[0][1], ref))
        print(json.dumps(dict(case=case, world=world, max_diff_eps=d / eps, n_differ=ne,
                              loss_rel=abs(out[0][0] - l1) / abs(l1))), flush=True)
