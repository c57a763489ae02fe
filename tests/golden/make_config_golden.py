"""Generates tests/golden/config_golden.json — FP64 oracle results at the
BASELINE.json configurations, so the GPU parity tests can check the product
at full size without rerunning the oracle (C2 takes ~6 min on 8 threads).

  C1  BASELINE.json configs[0]: N=M=10k uniform 3D (seeds 1/2), blur 0.05,
      dense single-scale eps-scaling.
  C2  BASELINE.json configs[1]: N=M=100k 3D Gaussian mixtures (seeds 3/4),
      multiscale with bench.py's exact params(): theta 12.5, switch_factor 1,
      retruncate every scale, automatic voxel edge (policy.h: 28 atoms per
      occupied voxel + 2 occupancy refinements), automatic super level
      (SPEC.md:290-303).

Stored per config: the loss, the four potentials (canonical gauge, caller
order) on 2048 fixed sampled rows, the schedule length and — multiscale —
the integer decisions kx / ky / t_switch / t_super / k_super and the
voxel edge, plus input checksums so a generator drift is caught.  The
oracle is the checker here (tests/ only); the product never reads this file.

Run:  python tests/golden/make_config_golden.py [c1] [c2]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config_golden.json")
N_SAMPLE = 2048


def c1_inputs():
    x = np.random.default_rng(1).random((10000, 3))
    y = np.random.default_rng(2).random((10000, 3))
    w = np.full(10000, 1e-4)
    return x, w, y, w


def c2_inputs(n=100000):
    import bench
    x, y = bench.mixture(n, 3), bench.mixture(n, 4)
    w = np.full(n, 1.0 / n)
    return x, w, y, w


def c1_params():
    from paper_2107_02010_b200.abi import make_params
    return make_params(blur=0.05)


def c2_params(n=100000):
    import bench
    w = dict(bench.WORKLOAD)
    w["n"] = w["m"] = n
    return bench.params(w)


def sample_rows(n, seed):
    return np.sort(np.random.default_rng(seed).choice(n, N_SAMPLE, replace=False))


def checksum(a):
    return [float(np.sum(a)), float(np.sum(a * a))]


def run(name, inputs, prm, seed):
    from oracle import oracle as O
    x, a, y, b = inputs
    t = time.perf_counter()
    loss, pots, st = O.sinkhorn(prm, x, a, y, b)
    dt = time.perf_counter() - t
    ix, iy = sample_rows(len(x), seed), sample_rows(len(y), seed + 1)
    rec = {
        "loss": loss, "oracle_seconds": dt, "oracle_threads": O.threads(),
        "rows_x": ix.tolist(), "rows_y": iy.tolist(),
        "a_xx": pots["a_xx"][ix].tolist(), "b_yx": pots["b_yx"][ix].tolist(),
        "b_yy": pots["b_yy"][iy].tolist(), "a_xy": pots["a_xy"][iy].tolist(),
        "n_scales": st["n_scales"], "t_switch": st["t_switch"], "kx": st["kx"],
        "ky": st["ky"], "t_super": st["t_super"], "k_super_x": st["k_super_x"],
        "k_super_y": st["k_super_y"], "cluster_scale": st["cluster_scale"],
        "diameter": st["diameter"], "pairs_evaluated": st["pairs_evaluated"],
        "checksum_x": checksum(x), "checksum_y": checksum(y),
    }
    print(f"{name}: loss {loss:.12g} in {dt:.1f} s, kx {st['kx']} t_switch {st['t_switch']}",
          flush=True)
    return rec


def main(which):
    g = json.load(open(OUT)) if os.path.exists(OUT) else {}
    if "c1" in which:
        g["c1"] = {"cite": "BASELINE.json configs[0]; SPEC.md:174-182",
                   **run("c1", c1_inputs(), c1_params(), 11)}
    if "c2" in which:
        g["c2"] = {"cite": "BASELINE.json configs[1]; SPEC.md:290-303; bench.py params()",
                   **run("c2", c2_inputs(), c2_params(), 21)}
    with open(OUT, "w") as f:
        json.dump(g, f)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2"])
