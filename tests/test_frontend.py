"""The msot:: C++ front-end (include/msot/*.hpp) compiled as a user would:
g++ against include/ and libmsot_b200.so.  CPU mode covers the measure
constructors and the schedule; GPU mode runs solves."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2107_02010_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "frontend_test.cpp")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "frontend_test")
    cmd = ["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), SRC, "-L" + PKG,
           "-lmsot_b200", "-Wl,-rpath," + PKG, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_frontend_cpu(exe):
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr + r.stdout


@pytest.mark.gpu
def test_frontend_gpu(exe):
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
