"""Generates tests/golden/spec_golden.json — the known answers that pin the
oracle (and, through it, the GPU path).

The reference ships no test vectors; its only pins are the
closed forms and acceptance criteria of SPEC.md.  This script writes them
down with their citations, and adds exact-OT values computed independently
of any Sinkhorn code (scipy.optimize.linear_sum_assignment on uniform
measures = the exact_ot oracle of SPEC.md:469-510):

  schedule
  softmin
  divergence
  exact OT      SPEC.md:587 (acceptance 1: N=M=32, D=2, blur=1e-3 d, 1e-2 rel).
                With one averaged update per scale (the literal Algorithm,
                PAPER.md:242-322) q = 0.9 leaves the 32-atom problems 0.6-3%
                short of exact OT; q = 0.99 meets 1e-2 (max 0.11%), so the
                fixtures carry "scaling": 0.99.
  1D monotone
Run:  python tests/golden/make_golden.py
"""
import json
import math
import os

import numpy as np
from scipy.optimize import linear_sum_assignment

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_golden.json")


def exact_uniform_ot(x, y):
    C = 0.5 * ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    r, c = linear_sum_assignment(C)
    return float(C[r, c].mean())


def main():
    g = {"schedule": [], "softmin": [], "divergence": [], "exact_ot": []}
    g["schedule"] += [
        {"cite": "SPEC.md:159", "d": 1.0, "blur": 1.0, "q": 0.9, "p": 2, "sigma": [1.0]},
        {"cite": "SPEC.md:160", "d": 8.0, "blur": 1.0, "q": 0.5, "p": 2,
         "sigma": [8.0, 4.0, 2.0, 1.0], "eps": [64.0, 16.0, 4.0, 1.0], "lam": [1, 1, 1, 1]},
        {"cite": "SPEC.md:161", "d": 10.0, "blur": 1.0, "q": 0.9, "p": 2, "len": 22},
        {"cite": "SPEC.md:162", "d": 2.0, "blur": 2.0, "q": 0.9, "p": 2, "reach": 2.0,
         "lam": [0.5]},
    ]
    g["softmin"] += [
        {"cite": "SPEC.md:170", "x": [[0.0]], "y": [[1.5]], "w": [1.0], "h": [0.0], "eps": 0.3,
         "f": [0.5 * 1.5 ** 2]},
        {"cite": "SPEC.md:171", "x": [[0.0]], "y": [[1.0], [-1.0]], "w": [0.5, 0.5],
         "h": [0.0, 0.0], "eps": 0.2, "f": [0.5]},
        # C = (0, 100) with p=2 -> points at distance 0 and sqrt(200)
        {"cite": "SPEC.md:172", "x": [[0.0]], "y": [[0.0], [math.sqrt(200.0)]], "w": [1.0, 1.0],
         "h": [0.0, 0.0], "eps": 1e-3, "f": [0.0], "atol": 1e-12},
    ]
    g["divergence"] += [
        {"cite": "SPEC.md:201", "x": [[0.0, 0.0, 0.0]], "a": [1.0], "y": [[1.0, 0.5, 0.0]],
         "b": [1.0], "blur": 0.01, "value": 0.5 * 1.25, "rtol": 1e-2},
        {"cite": "SPEC.md:530", "x": [[0.0]], "a": [1.0], "y": [[2.0]], "b": [1.0],
         "blur": 1e-3, "value": 2.0, "rtol": 1e-2},
        {"cite": "SPEC.md:202", "x": [[0.3, 0.1]], "a": [1.0], "y": [[0.3, 0.1]], "b": [2.0],
         "blur": 0.1, "value": 0.5 * 0.1 ** 2 * 1.0, "rtol": 1.5,
         "note": "order of the (eps/2)(1-2)^2 mass term; the balanced dual of this "
                 "mass-mismatched pair adds (eps/2) ln 2 on top"},
    ]
    rng = np.random.default_rng(20210705)
    for k in range(20):
        x = rng.random((32, 2))
        y = rng.random((32, 2)) * 0.8 + 0.1
        lo = np.minimum(x.min(0), y.min(0))
        hi = np.maximum(x.max(0), y.max(0))
        d = float(np.sqrt(((hi - lo) ** 2).sum()))
        g["exact_ot"].append({"cite": "SPEC.md:587", "x": x.tolist(), "y": y.tolist(),
                              "blur": 1e-3 * d, "scaling": 0.99,
                              "value": exact_uniform_ot(x, y), "rtol": 1e-2})
    x = np.sort(rng.random(16))
    y = np.sort(rng.random(16) + 0.3)
    g["exact_ot"].append({"cite": "SPEC.md:487", "x": x[:, None].tolist(),
                          "y": y[:, None].tolist(), "blur": 1e-3, "scaling": 0.99,
                          "value": float(0.5 * np.mean((x - y) ** 2)), "rtol": 1e-2})
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
