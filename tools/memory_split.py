"""Device memory at C2 (1e5 vs 1e5) split into the library's module/context
share (after creating a context, before any solve) and the solver's buffers
(stats.device_bytes and the cudaMemGetInfo delta of the solve).
python tools/memory_split.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2107_02010_b200.solver import Context

w = dict(bench.WORKLOAD, n=100000, m=100000, blur=0.01)
x, a, y, b = bench.make_inputs(w)
torch.cuda.init()
free0 = torch.cuda.mem_get_info(0)[0]
ctx = Context(0)
torch.cuda.synchronize()
free1 = torch.cuda.mem_get_info(0)[0]
loss, _, st = ctx.sinkhorn(bench.params(w), x, a, y, b, potentials=False)
torch.cuda.synchronize()
free2 = torch.cuda.mem_get_info(0)[0]
print(json.dumps(dict(context_and_modules=free0 - free1, solve_delta=free1 - free2,
                      total=free0 - free2, solver_device_bytes=st["device_bytes"])))
