"""Config 4: 200k vs 200k synthetic fibres (D = 60, P = 20), flip-augmented
to 400k vs 400k, reach = 0.3, blur = 0.03, dense
eps-scaling with the tcgen05 softmin, then label transfer (K9) of the atlas
bundle labels, resolve_flips and classify.
    python tools/config4.py [n_fibres] [bundles] [dense|ms] [clusters]
(ms: K-means multiscale + block-sparse fine phase; dense: all pairs)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2107_02010_b200 import workloads as W
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context, classify, resolve_flips

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 50
mode = sys.argv[3] if len(sys.argv) > 3 else "ms"
kcl = int(sys.argv[4]) if len(sys.argv) > 4 else 0
sf = float(sys.argv[5]) if len(sys.argv) > 5 else 2.0
tr = int(sys.argv[6]) if len(sys.argv) > 6 else 0
th = float(sys.argv[7]) if len(sys.argv) > 7 else 12.5
t = time.perf_counter()
fa, la = W.fibres(n, 7, bundles=L, bundle_seed=1)   # subject
fb, lb = W.fibres(n, 8, bundles=L, bundle_seed=1)   # atlas (shares the bundles)
x, a = W.flip_augment(*W.encode_fibers(fa))
y, b = W.flip_augment(*W.encode_fibers(fb))
lab = np.concatenate([lb, lb]).astype(np.int32)
prep = time.perf_counter() - t
ctx = Context(0)
ctx.set_profiling(True)
prm = make_params(blur=0.03, reach=0.3, multiscale=(mode == "ms"), retruncate=1,
                  switch_factor=sf, clusters=kcl, transfer_rule=tr, theta=th)
for rep in range(2):
    t = time.perf_counter()
    soft, loss, st = ctx.transfer_labels(prm, x, a, y, b, lab, L)
    wall = time.perf_counter() - t
ctx.set_profiling(False)
_, _, st_np = ctx.transfer_labels(prm, x, a, y, b, lab, L)  # unprofiled: batches overlapped
out, chosen = resolve_flips(soft, np.tile(np.arange(n), 2), np.repeat([0, 1], n))
hard, conf = classify(out, 0.5)
inl = hard >= 0
print(json.dumps(dict(mode=mode, switch_factor=sf, transfer_rule=tr, theta=th, kx=st["kx"],
                      t_switch=st["t_switch"],
                      fine_kept=st["pairs_fine"] / max(st["pairs_fine_dense"], 1.0),
                      atoms=[len(x), len(y)], D=x.shape[1], classes=L, prep_s=prep, wall_s=wall,
                      device_ms=st["total_ms"], device_ms_unprofiled=st_np["total_ms"],
                      batches=st["colpart_batches"], device_mb=st["device_bytes"] / 1e6,
                      softmin_ms=st["softmin_ms"],
                      phases=st["phase_ms"], loss=loss, n_scales=st["n_scales"],
                      pairs=st["pairs_evaluated"],
                      pairs_per_s=st["pairs_evaluated"] / (st["softmin_ms"] * 1e-3),
                      fallback_rows=st["fallback_rows"], inlier_fraction=float(inl.mean()),
                      label_accuracy=float((hard[inl] == la[inl]).mean()) if inl.any() else None,
                      mean_row_mass=float(out.row_mass.mean()))))
