"""C3 at bench.py's parameters with the voxel edge overridden: device time,
pairs and distance of S_eps from the dense solve.
python tools/cell_sweep.py edge1 edge2 ...   (0 = automatic)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2107_02010_b200.solver import Context

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dense = json.load(open(os.path.join(ROOT, "profiles", "r1_c3_dense_vs_multiscale.json")))["dense_S_eps"]
w = dict(bench.WORKLOAD)
x, a, y, b = bench.make_inputs(w)
ctx = Context(0)
for edge in [float(v) for v in sys.argv[1:]] or [0.0]:
    prm = bench.params(w)
    if edge > 0:
        prm.cluster_scale = edge
    ts = []
    for _ in range(4):
        loss, _, st = ctx.sinkhorn(prm, x, a, y, b, potentials=False)
        ts.append(st["total_ms"])
    print(json.dumps(dict(edge=edge or st["cluster_scale"], device_ms=min(ts[1:]), S_eps=loss,
                          rel_vs_dense=loss / dense - 1, pairs=st["pairs_evaluated"], kx=st["kx"],
                          t_switch=st["t_switch"])), flush=True)
