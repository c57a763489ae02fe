"""Device memory held by a context after one solve (C2 100k, C3 1M):
python tools/memory.py [n ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2107_02010_b200.solver import Context

for n in [int(v) for v in sys.argv[1:]] or [100000, 1000000]:
    w = dict(bench.WORKLOAD, n=n, m=n)
    if n <= 100000:
        w.update(blur=0.01)
    x, a, y, b = bench.make_inputs(w)
    torch.cuda.init()
    free0 = torch.cuda.mem_get_info(0)[0]
    ctx = Context(0)
    loss, _, st = ctx.sinkhorn(bench.params(w), x, a, y, b, potentials=False)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info(0)[0]
    print(json.dumps(dict(n=n, device_bytes=free0 - free1, per_atom=(free0 - free1) / (2 * n),
                          pairs=st["pairs_evaluated"], loss=loss)), flush=True)
    ctx.close()
