"""The `msot` command line: file
formats, exit codes (0 ok, 2 usage, 3 data, 4 numeric) and the commands'
SPEC examples."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2107_02010_b200 import _build, workloads as W

CLI = _build.CLI


@pytest.fixture(scope="module")
def cli():
    _build.build_lib()
    return _build.build_cli()


def run(cli, *args, timeout=300):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout, r.stderr


def write_points(path, pts, w=None):
    pts = np.atleast_2d(pts)
    w = np.ones(len(pts)) / len(pts) if w is None else w
    with open(path, "w") as f:
        f.write("# weight coords\n")
        for wi, p in zip(w, pts):
            f.write(" ".join(map(repr, [float(wi), *map(float, p)])) + "\n")


def write_fibers(path, lines):
    with open(path, "w") as f:
        for ln in lines:
            f.write(f"fiber {len(ln)}\n")
            for p in ln:
                f.write(f"{float(p[0])!r} {float(p[1])!r} {float(p[2])!r}\n")


def test_usage_and_data_errors(cli, tmp_path):
    assert run(cli)[0] == 2
    assert run(cli, "frobnicate")[0] == 2
    code, _, err = run(cli, "divergence", tmp_path / "missing.txt", tmp_path / "missing.txt")
    assert code == 3 and "missing.txt" in err  # the error names the path
    bad = tmp_path / "bad.txt"
    bad.write_text("0.5 0 0\n0.5 1 zz\n")
    code, _, err = run(cli, "divergence", bad, bad)
    assert code == 3 and ":2:" in err  # parse failure with the line number
    good = tmp_path / "a.txt"
    write_points(good, [[0.0], [1.0]])
    assert run(cli, "divergence", good, good, "--blur", "-1")[0] == 2
    assert run(cli, "bench", "--sizes", "0")[0] == 2


@pytest.mark.gpu
def test_divergence_and_verify(cli, tmp_path):
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    write_points(a, [[0.0]], [1.0])
    write_points(b, [[2.0]], [1.0])
    code, out, _ = run(cli, "divergence", a, b, "--blur", "1e-3", "--format", "json")
    assert code == 0
    rep = json.loads(out)
    assert abs(rep["value"] - 2.0) < 2e-2 and rep["atoms"] == [1, 1]
    rng = np.random.default_rng(0)
    c = tmp_path / "c.txt"
    write_points(c, rng.random((300, 3)))
    code, out, _ = run(cli, "divergence", c, c, "--format", "json")
    assert code == 0 and abs(json.loads(out)["value"]) < 1e-9  # identical files -> 0
    assert run(cli, "verify")[0] == 0


@pytest.mark.gpu
def test_plan_cluster_bench(cli, tmp_path):
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    write_points(a, [[0.0, 0.0], [1.0, 0.0]])
    write_points(b, [[0.0, 0.1], [1.0, 0.1]])
    code, out, _ = run(cli, "plan", a, b, "--blur", "0.01", "--tau", "1e-3")
    rows = [l.split() for l in out.splitlines()]
    assert code == 0 and sorted((int(i), int(j)) for i, j, _ in rows) == [(0, 0), (1, 1)]
    assert all(abs(float(m) - 0.5) < 1e-3 for _, _, m in rows)
    c = tmp_path / "c.txt"
    rng = np.random.default_rng(1)
    write_points(c, np.concatenate([rng.normal(0, 0.01, (40, 3)), rng.normal(5, 0.01, (40, 3))]))
    code, out, _ = run(cli, "cluster", c, "--clusters", "2")
    lab = np.array([int(l.split()[1]) for l in out.splitlines() if l and l[0].isdigit()])
    assert code == 0 and len(set(lab[:40])) == 1 and len(set(lab[40:])) == 1 and lab[0] != lab[40]
    code, out, _ = run(cli, "bench", "--sizes", "1000")
    reps = [json.loads(l) for l in out.splitlines()]
    assert code == 0 and reps[1]["pairs"] <= reps[0]["pairs"]  # multiscale <= dense


@pytest.mark.gpu
def test_transfer_identity_and_flips(cli, tmp_path):
    """atlas = subject -> every fibre keeps its label; reversed subject -> same
    labels through flip resolution."""
    fa, la = W.fibres(120, 3, bundles=3, bundle_seed=5)
    subj, atlas, labels = tmp_path / "s.fib", tmp_path / "a.fib", tmp_path / "a.lab"
    write_fibers(subj, fa)
    write_fibers(atlas, fa)
    labels.write_text("".join(f"{i} bundle{l}\n" for i, l in enumerate(la)))
    res = tmp_path / "labels.out"
    code, out, err = run(cli, "transfer", subj, atlas, labels, "--blur", "0.02", "--reach", "0.3",
                         "--out", res)
    assert code == 0, err
    got = [l.split()[1] for l in res.read_text().splitlines()]
    assert got == [f"bundle{l}" for l in la]
    assert "OUTLIER" not in out  # summary counts per class on stdout
    write_fibers(subj, [np.asarray(f)[::-1] for f in fa])
    code, out, _ = run(cli, "transfer", subj, atlas, labels, "--blur", "0.02", "--reach", "0.3",
                       "--out", res)
    assert code == 0
    assert [l.split()[1] for l in res.read_text().splitlines()] == [f"bundle{l}" for l in la]


@pytest.mark.gpu
def test_barycenter_two_maps(cli, tmp_path):
    paths = []
    for k, off in enumerate((4, 12)):
        p = tmp_path / f"d{k}.txt"
        p.write_text("density 20 20 20 1.0 0 0 0\n" + f"{off} 10 10 1.0\n")
        paths.append(p)
    out_p = tmp_path / "bary.txt"
    code, _, err = run(cli, "barycenter", *paths, "--upsample", "1", "--iters", "20",
                       "--out", out_p)
    assert code == 0, err
    lines = out_p.read_text().splitlines()
    loss = [float(v) for v in lines[0].split()[2:]]
    pts = np.array([[float(v) for v in l.split()[1:]] for l in lines[1:]])
    assert loss[-1] <= loss[0]
    assert np.abs(pts[:, 0].mean() - 8.5).max() < 0.5  # the midpoint of the voxel centres


def test_barycenter_mismatched_grids(cli, tmp_path):
    """maps on different grids are a data error (exit 3), checked
    before any device work (runs without a GPU)."""
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    a.write_text("density 20 20 20 1.0 0 0 0\n4 10 10 1.0\n")
    b.write_text("density 20 20 20 2.0 0 0 0\n12 10 10 1.0\n")  # voxel size differs
    code, _, err = run(cli, "barycenter", a, b, "--iters", "1")
    assert code == 3 and "grid" in err
    b.write_text("density 20 20 20 1.0 5 0 0\n12 10 10 1.0\n")  # origin differs
    assert run(cli, "barycenter", a, b, "--iters", "1")[0] == 3
