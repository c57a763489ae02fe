"""Device buffer table after one bench-parameter solve (MSOT_DEBUG_BUFS):
python tools/membufs.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MSOT_DEBUG_BUFS"] = "1"
import bench
from paper_2107_02010_b200.solver import Context
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
w = dict(bench.WORKLOAD, n=n, m=n)
x, a, y, b = bench.make_inputs(w)
ctx = Context(0)
loss, _, st = ctx.sinkhorn(bench.params(w), x, a, y, b, potentials=False)
print(n, "device_bytes", st["device_bytes"], "batches", st["colpart_batches"], "total_ms", st["total_ms"], flush=True)
ctx.close()
