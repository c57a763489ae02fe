"""CPU tests of the drop-in boundary: the C-ABI library loads without a GPU,
exports every symbol include/msot_gpu.h declares, and its host-side logic
(schedule, shard split) agrees with the oracle.  No compute calls."""
import ctypes as C
import math
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2107_02010_b200 import solver
from paper_2107_02010_b200.abi import make_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "msot_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(msot_[a-z_0-9]+)\s*\(", src)))


def test_header_matches_binding():
    assert declared_symbols() == sorted(solver.EXPORTS)


def test_library_exports_every_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", solver.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    have = {l.split()[-1] for l in out.splitlines() if l.strip()}
    missing = [s for s in declared_symbols() if s not in have]
    assert not missing, missing


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", solver.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_loads_and_params_default():
    L = solver.lib()
    p = make_params()
    L.msot_params_default(p)
    assert p.scaling == 0.9 and p.theta == 20.0 and p.switch_factor == 2.0
    assert math.isinf(p.reach) and p.p == 2.0


def test_schedule_matches_oracle(oracle):
    rng = np.random.default_rng(0)
    for _ in range(50):
        blur = 10 ** rng.uniform(-3, 0)
        d = blur * 10 ** rng.uniform(-0.5, 3)
        q = rng.uniform(0.2, 0.97)
        reach = [math.inf, 10 ** rng.uniform(-2, 1)][rng.integers(2)]
        prm = make_params(blur=blur, scaling=q, reach=reach)
        a = solver.make_schedule(d, prm)
        b = oracle.schedule(d, prm)
        for u, v in zip(a, b):
            np.testing.assert_array_equal(u, v)


def test_shard_tiles_balanced():
    rng = np.random.default_rng(1)
    w = rng.random(1000) * 100
    for world in (1, 2, 3, 8):
        b = solver.shard_tiles(w, world)
        assert b[0] == 0 and b[-1] == 1000 and np.all(np.diff(b) >= 0)
        parts = [w[b[r]:b[r + 1]].sum() for r in range(world)]
        assert max(parts) - min(parts) <= 2 * w.max()


def test_no_oracle_in_product():
    """The product package must never import or link the oracle."""
    pkg = os.path.join(ROOT, "paper_2107_02010_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                if f == "_build.py":  # builds the checker next to the product
                    continue
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"(from|import)\s+oracle|liboracle|oracle_[a-z]", txt), f
    out = subprocess.run(["ldd", solver.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "msotref" not in out


def test_binding_rejects_short_arrays():
    """the ctypes binding validates every array length before the
    C ABI reads n / m entries behind the pointers (no GPU needed: the checks
    run before any library call)."""
    import numpy as np
    from paper_2107_02010_b200.abi import DataError, UsageError, make_params
    from paper_2107_02010_b200.solver import Context, grad_weights, DualPotentials

    ctx = Context.__new__(Context)  # no device: the checks fire first
    ctx._h = None
    x, y = np.zeros((5, 3)), np.zeros((4, 3))
    prm = make_params()
    with pytest.raises(DataError):
        ctx.sinkhorn(prm, x, np.ones(4), y, np.ones(4))
    with pytest.raises(DataError):
        ctx.sinkhorn(prm, x, np.ones(5), y, np.ones(3))
    with pytest.raises(DataError):
        ctx.sinkhorn_grad(prm, x, np.ones(5), y, np.ones(5))
    with pytest.raises(DataError):
        ctx.transfer_labels(prm, x, np.ones(5), y, np.ones(4), np.zeros(3, np.int32))
    with pytest.raises(DataError):
        ctx.barycenter(prm, x, np.ones(5), [(y, np.ones(4)), (y, np.ones(2))])
    with pytest.raises(DataError):
        ctx.plan_apply(x, np.ones(5), y, np.ones(4), np.zeros(5), np.zeros(4), 1.0, np.ones(3))
    with pytest.raises(DataError):
        ctx.softmin(x, y, np.zeros(3), np.zeros(4), 1.0)
    d = DualPotentials(np.zeros(5), np.zeros(4), np.zeros(4), np.zeros(5), 1.0)
    with pytest.raises(UsageError):  # reach must be > 0 or inf
        grad_weights(make_params(reach=0.0), np.ones(5), np.ones(4), d)
    with pytest.raises(UsageError):
        grad_weights(make_params(reach=-1.0), np.ones(5), np.ones(4), d)


def _span_fn(lib, name, nargs):
    f = getattr(lib, name)
    f.restype = C.c_double
    f.argtypes = [C.c_void_p, C.c_size_t] * nargs  # std::span<const double> by value
    return f


def test_numeric_bitwise_vs_reference():
    """include/msot/numeric.hpp (reference proj/include/msot/numeric.hpp:9-15),
    implemented in libmsot_b200.so, against the reference's own numeric.cpp
    compiled unmodified into oracle/_ref: bitwise equal on every length."""
    ref_path = os.path.join(ROOT, "oracle", "_ref", "libmsotref.so")
    if not os.path.exists(ref_path):
        pytest.skip("oracle/_ref not built")
    ours, ref = C.CDLL(solver.LIB_PATH), C.CDLL(ref_path)
    names = {"kahan": ("_ZN4msot9kahan_sumESt4spanIKdLm18446744073709551615EE", 1),
             "sum": ("_ZN4msot12pairwise_sumESt4spanIKdLm18446744073709551615EE", 1),
             "dot": ("_ZN4msot12pairwise_dotESt4spanIKdLm18446744073709551615EES2_", 2)}
    rng = np.random.default_rng(7)
    for n in [0, 1, 2, 31, 32, 33, 64, 65, 100, 1000, 4097, 123457]:
        a = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))
        b = rng.standard_normal(n)
        for key, (sym, k) in names.items():
            fo, fr = _span_fn(ours, sym, k), _span_fn(ref, sym, k)
            args = [a.ctypes.data, n] if k == 1 else [a.ctypes.data, n, b.ctypes.data, n - n // 3]
            vo, vr = fo(*args), fr(*args)
            assert vo == vr or (math.isnan(vo) and math.isnan(vr)), (key, n, vo, vr)
