"""Times msot_kmeans on the config-4 fibre features: python tools/kmeans_time.py [n_fibres] [K]"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.solver import Context
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
fa, _ = W.fibres(n, 7, bundles=50, bundle_seed=1)
x, a = W.flip_augment(*W.encode_fibers(fa))
K = int(sys.argv[2]) if len(sys.argv) > 2 else int(math.ceil(math.sqrt(len(x))))
ctx = Context(0)
for rep in range(2):
    t = time.perf_counter()
    km = ctx.kmeans(x, a, K)
    print(f"K-means N={len(x)} D={x.shape[1]} K={K}: {1e3 * (time.perf_counter() - t):.1f} ms wall, "
          f"{km['iters']} Lloyd iterations", flush=True)
