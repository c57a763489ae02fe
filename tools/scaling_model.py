"""Strong-scaling model of the C3 solve, from a measured one-GPU
per-kernel launch list (profiles/r2_launches_c3.txt, second table: one batch
per update, whose total equals the timed step) and the NVLink references of
the B200 profiling guide (8-rank all-reduce bus bandwidth 725 GB/s, peer copy
770 GB/s per direction), with the per-solve exchange volumes of the sharded
solver (solver.cu: coll_allreduce64 / coll_bcast_rows):

    T(N) = replicated + sharded x (1 + imbalance) / N + comm(N) + host waits

python tools/scaling_model.py [launch_summary.txt] > profiles/r2_scaling_model.json"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r2_launches_c3.txt")

# kernels whose work is split across ranks by row tiles (each rank runs the
# work items / rows of its own tiles); everything else runs on every rank
SHARDED = ("softmin_sym_kernel", "sym_colsum_kernel", "mask_rows_kernel", "hd_colsum_kernel",
           "softmin_finalize", "softmin_rowsum")

blocks = open(path).read().split("\n\n")
table = blocks[-1] if len(blocks) > 1 else blocks[0]  # one batch per update
kern = {}
for line in table.splitlines():
    m = re.match(r"\s*([\d.]+)\s+[\d.]+%\s+(\d+)\s+(.+)$", line)
    if m:
        kern[m.group(3).strip()] = (float(m.group(1)), int(m.group(2)))
sharded = sum(t for k, (t, _) in kern.items() if k.startswith(SHARDED))
replicated = sum(t for k, (t, _) in kern.items() if not k.startswith(SHARDED))

# exchange volumes per C3 solve (N = M = 1e6, 33930 / 32285 clusters, 44
# coarse-level scales incl. the super level, 6 fine updates, 5 mask rebuilds)
n = m = 1_000_000
kx, ky = 33930, 32285
fine_updates, coarse_scales, rebuilds = 6, 44, 5
words = lambda k: (k + 31) // 32
mask_bytes = 4 * (kx * words(kx) + ky * words(ky) + kx * words(ky))
AR_BUS, P2P, LAT = 725e9, 770e9, 25e-6  # bytes/s, bytes/s, s per collective call


def comm_ms(N):
    if N == 1:
        return 0.0
    f = (N - 1) / N
    ar = lambda b: LAT + b * 2 * f / AR_BUS          # ring all-reduce
    bc = lambda b: LAT + b * f / P2P                 # grouped row-shard broadcast
    t = fine_updates * (ar(8 * (n + 2 * m)) + bc(4 * (2 * n + m)))  # float64 column totals
    t += coarse_scales * (ar(8 * (kx + 2 * ky)) + bc(4 * (2 * kx + ky)))
    t += rebuilds * bc(mask_bytes)
    return 1e3 * t


host_waits_ms = 12 * 0.03  # 12 host waits per solve, ~30 us of device idle each
imbalance = 0.03           # tile shards balanced on evaluated pairs per tile
out = {"source": os.path.relpath(path, ROOT), "replicated_ms": replicated,
       "sharded_ms": sharded, "mask_bytes_per_rebuild": mask_bytes, "predicted": {}}
t1 = replicated + sharded + host_waits_ms
for N in (1, 2, 4, 8):
    t = replicated + sharded * (1 + (imbalance if N > 1 else 0)) / N + comm_ms(N) + host_waits_ms
    out["predicted"][N] = {"ms": round(t, 1), "comm_ms": round(comm_ms(N), 2),
                           "speedup": round(t1 / t, 2), "efficiency": round(t1 / t / N, 3)}
print(json.dumps(out, indent=1))
