"""compute-sanitizer on the product kernels: one small
multiscale 3-D solve (clustering, masks, evaluate-once fine phase, loss)
and one small high-D solve (tcgen05 / TMA / mbarrier kernels) under memcheck,
the 3-D solve under racecheck (shared-memory hazards) and synccheck, and the
truncation-mask ABI (upper-half self masks + mask_mirror) under memcheck and
racecheck.
The solve runs in a child process through the C ABI (no torch)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
from paper_2107_02010_b200.abi import make_params
from paper_2107_02010_b200.solver import Context
kind = sys.argv[1]
rng = np.random.default_rng(0)
ctx = Context(0)
if kind == "3d":
    cen = rng.uniform(0.2, 0.8, (4, 3))
    x = cen[rng.integers(0, 4, 3000)] + rng.normal(0, 0.05, (3000, 3))
    y = cen[rng.integers(0, 4, 2600)] + rng.normal(0, 0.05, (2600, 3)) + 0.01
    a, b = np.full(3000, 1 / 3000), np.full(2600, 1 / 2600)
    prm = make_params(blur=0.02, multiscale=True, retruncate=1, cluster_scale=0.06, super_level=1)
elif kind == "mask":
    # truncation masks through the ABI: self (upper half + mask_mirror) and
    # cross, with slopes and member boxes
    k = 1100
    c = rng.random((k, 3)).astype(np.float32)
    r = (rng.random(k) * 0.05).astype(np.float32)
    f = (rng.random(k) * 0.01).astype(np.float32)
    g = np.concatenate([rng.normal(0, 0.2, (k, 3)), f[:, None] + 0.001], 1).astype(np.float32)
    box = np.concatenate([-rng.random((k, 3)) * r[:, None], rng.random((k, 3)) * r[:, None]],
                         1).astype(np.float32)
    m1 = ctx.kernel_truncation(c, r, f, c, r, f, 1e-3, 10.0, self_=True, gx=g, hy=g, bx=box, by=box)
    m2 = ctx.kernel_truncation(c, r, f, c[::-1].copy(), r, f, 1e-3, 10.0, gx=g, hy=g, bx=box, by=box)
    assert (m1 == m1.T).all() and 0 < m1.mean() < 1 and 0 < m2.mean() < 1
    print("ok", m1.mean(), m2.mean())
    ctx.close()
    sys.exit(0)
else:
    x, y = rng.random((700, 60)) * 0.2, rng.random((600, 60)) * 0.2
    a, b = np.full(700, 1 / 700), np.full(600, 1 / 600)
    prm = make_params(blur=0.05, multiscale=True, retruncate=1, clusters=4, switch_factor=1.0)
loss, _, st = ctx.sinkhorn(prm, x, a, y, b)
assert np.isfinite(loss) and st["gpu_launches"] > 0
print("ok", loss, st["gpu_launches"])
ctx.close()
"""


@pytest.mark.parametrize("tool,kind", [("memcheck", "3d"), ("memcheck", "hd"),
                                       ("racecheck", "3d"), ("synccheck", "3d"),
                                       ("memcheck", "mask"), ("racecheck", "mask")])
def test_compute_sanitizer(tmp_path, tool, kind):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    script = tmp_path / "child.py"
    script.write_text(CHILD.format(root=ROOT))
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    r = subprocess.run(cmd + [sys.executable, str(script), kind], capture_output=True, text=True,
                       timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "ok" in r.stdout, out[-4000:]
    # memcheck/synccheck: "ERROR SUMMARY: 0 errors"; racecheck: "RACECHECK
    # SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    assert ("ERROR SUMMARY: 0 errors" in out or "(0 errors, 0 warnings)" in out), out[-4000:]
