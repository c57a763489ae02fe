"""bench.py keeps the driver's JSON contract (one line, the required keys and
their types) — run at a reduced size; the reference arm prints its own line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line_contract():
    d = _run("--steps", "3", "--warmup", "3", "--n", "100000", "--no-cpu", "--no-extras")
    for k, t in [("metric", str), ("value", float), ("unit", str), ("n_gpus", int),
                 ("steps", int), ("warmup", int), ("ms_per_step", float),
                 ("higher_is_better", bool), ("scaling", str), ("dtype", str), ("data", str),
                 ("config", dict), ("gpu_launches", int), ("e2e", dict), ("roofline", dict),
                 ("clocks", dict)]:
        assert isinstance(d[k], t), k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["higher_is_better"] is False and d["vs_baseline"] is None
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] <= 1.05
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "workload" in d["config"]


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-n", "5000")
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_self_spawn_ranks_gloo():
    """`bench.py --gpus N` without torchrun spawns N ranks itself (RANK /
    WORLD_SIZE / MASTER_ADDR=127.0.0.1 / MASTER_PORT), rendezvous over gloo,
    reduces the step time as the max over ranks and prints one line on rank 0
    (the driver's --gpus 8 must not run a single GPU)."""
    env_clean = {k: v for k, v in os.environ.items()
                 if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    for n in (2, 3):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                            "--dist-probe"], cwd=ROOT, capture_output=True, text=True,
                           timeout=300, env=env_clean)
        assert r.returncode == 0, r.stderr[-2000:]
        lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, r.stdout
        d = json.loads(lines[0])
        assert d["n_gpus"] == n and d["ranks_seen"] == n and d["ms_per_step"] == float(n)
