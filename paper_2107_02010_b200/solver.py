"""Python binding of the C ABI (include/msot_gpu.h) over ctypes.

This is a thin harness for tests and the bench: every call goes through
`libmsot_b200.so` (CUDA, sm_100a).  There is no CPU fallback — if the
library or a GPU is missing the calls raise.

Names mirror the reference operations of SPEC.md: `softmin` (:164),
`symmetric_sinkhorn` / `multiscale_sinkhorn` (:174, :290), `divergence`
(:194), `make_schedule` (:153), plus the north-star kernels
`grid_cluster` and `kernel_truncation` (:280).
"""
import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from .abi import Params, Stats, make_params, raise_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmsot_b200.so")
_LIB = None

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_bp = C.POINTER(C.c_uint8)


_AR_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_float), C.c_int64, C.c_void_p)
_BC_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_float), C.c_int64, C.c_int, C.c_void_p)


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() — "
                               "the solver has no CPU fallback")
        # libmsot links libnccl.so.2: when torch is installed, load it first
        # so its bundled (newer) NCCL is the process's libnccl — loading the
        # system one first would leave torch's CUDA library unresolvable
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        L = C.CDLL(LIB_PATH)
        L.msot_last_error.restype = C.c_char_p
        L.msot_params_default.argtypes = [C.POINTER(Params)]
        L.msot_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        L.msot_nccl_unique_id.argtypes = [C.c_char_p]
        L.msot_create_dist.argtypes = [C.c_int, C.c_int, C.c_int, C.c_char_p,
                                       C.POINTER(C.c_void_p)]
        L.msot_create_dist_host.argtypes = [C.c_int, C.c_int, C.c_int, _AR_FN, _BC_FN, C.c_void_p,
                                            C.POINTER(C.c_void_p)]
        L.msot_world_info.argtypes = [C.c_void_p, _ip, _ip, _ip]
        L.msot_debug_mask.argtypes = [C.c_void_p, C.c_int, _ip, _ip, _bp, _ip, _ip]
        L.msot_debug_capture.argtypes = [C.c_void_p, C.c_int, C.POINTER(_dp), C.POINTER(_dp)]
        L.msot_destroy.argtypes = [C.c_void_p]
        L.msot_destroy.restype = None
        L.msot_set_profiling.argtypes = [C.c_void_p, C.c_int]
        L.msot_set_colpart_budget.argtypes = [C.c_void_p, C.c_int64]
        L.msot_schedule.argtypes = [C.c_double, C.POINTER(Params), _dp, _dp, _dp, C.c_int]
        L.msot_shard_tiles.argtypes = [_dp, C.c_int64, C.c_int, _lp]
        L.msot_softmin.argtypes = [C.c_void_p, _dp, C.c_int64, _dp, C.c_int64, C.c_int, _dp,
                                   _dp, C.c_double, C.c_double, _dp, _dp]
        L.msot_grid_cluster.argtypes = [C.c_void_p, _dp, _dp, C.c_int64, C.c_int, _dp,
                                        C.c_double, _ip, _ip, _ip, _ip, _dp, _dp, _fp]
        L.msot_truncation_mask.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, _fp,
                                           _fp, _fp, _fp, _fp, _fp, _fp, _fp, C.c_double,
                                           C.c_double, C.c_double, C.c_int, _bp]
        L.msot_truncation_mask_box.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, _fp,
                                               _fp, _fp, _fp, _fp, _fp, _fp, _fp, _fp, _fp,
                                               C.c_double, C.c_double, C.c_double, C.c_int, _bp]
        L.msot_sinkhorn.argtypes = [C.c_void_p, C.POINTER(Params), _dp, _dp, C.c_int64, _dp,
                                    _dp, C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp,
                                    C.POINTER(Stats)]
        L.msot_probe_ex2.argtypes = [C.c_void_p, _dp]
        L.msot_sinkhorn_grad.argtypes = [C.c_void_p, C.POINTER(Params), _dp, _dp, C.c_int64, _dp,
                                         _dp, C.c_int64, C.c_int, _dp, _dp, C.POINTER(Stats)]
        L.msot_barycenter.argtypes = [C.c_void_p, C.POINTER(Params), _dp, _dp, C.c_int64,
                                      C.c_int, C.POINTER(_dp), C.POINTER(_dp), _lp, C.c_int,
                                      C.c_int, C.c_double, C.c_double, _dp, _dp,
                                      C.POINTER(C.c_int), C.POINTER(Stats)]
        L.msot_sinkhorn_device.argtypes = [C.c_void_p, C.POINTER(Params), C.c_void_p,
                                           C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                           C.c_int64, C.c_int, _dp, C.POINTER(Stats)]
        L.msot_transfer_labels.argtypes = [C.c_void_p, C.POINTER(Params), _dp, _dp, C.c_int64,
                                           _dp, _dp, C.c_int64, C.c_int, _ip, C.c_int, _dp, _dp,
                                           _dp, C.POINTER(Stats)]
        L.msot_resolve_flips.argtypes = [_dp, _dp, C.c_int64, C.c_int, _ip, _ip, _dp, _dp,
                                         _ip]
        L.msot_classify.argtypes = [_dp, _dp, C.c_int64, C.c_int, C.c_double, _ip, _dp]
        L.msot_kmeans.argtypes = [C.c_void_p, _dp, _dp, C.c_int64, C.c_int, C.c_int, C.c_uint64,
                                  _ip, _ip, _ip, _dp, _dp, _fp, C.POINTER(C.c_int)]
        L.msot_plan_apply.argtypes = [C.c_void_p, _dp, _dp, C.c_int64, _dp, _dp, C.c_int64,
                                      C.c_int, _dp, _dp, C.c_double, _dp, _dp]
        L.msot_exact_ot.argtypes = [_dp, _dp, C.c_int64, _dp, _dp, C.c_int64, C.c_int,
                                    C.c_double, _dp, _dp]
        _LIB = L
    return _LIB


# Symbols include/msot_gpu.h declares (checked by the CPU test suite).
EXPORTS = ["msot_last_error", "msot_params_default", "msot_create", "msot_nccl_unique_id",
           "msot_create_dist", "msot_destroy", "msot_set_profiling", "msot_schedule",
           "msot_shard_tiles", "msot_softmin", "msot_grid_cluster", "msot_truncation_mask",
           "msot_sinkhorn", "msot_sinkhorn_device", "msot_probe_ex2", "msot_sinkhorn_grad",
           "msot_barycenter", "msot_transfer_labels", "msot_resolve_flips", "msot_classify",
           "msot_plan_apply", "msot_kmeans", "msot_create_dist_host", "msot_exact_ot",
           "msot_world_info", "msot_debug_capture", "msot_debug_mask",
           "msot_set_colpart_budget", "msot_truncation_mask_box"]


def _check(rc):
    if rc != 0:
        raise_status(rc, lib().msot_last_error().decode())


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _d(a):
    return a.ctypes.data_as(_dp)


def _measures(x, a, y, b):
    """Shape checks of a pair of measures before any ABI call: the C ABI reads
    n (m) weights behind the caller's pointers, so a short array must be a
    DataError here, not an out-of-bounds host read (msot::DiscreteMeasure
    enforces the same on the C++ side, measure.hpp:26-37)."""
    from .abi import DataError
    x, a, y, b = _c64(x), _c64(a), _c64(y), _c64(b)
    if x.ndim == 1:
        x = x[:, None]
    if y.ndim == 1:
        y = y[:, None]
    if x.ndim != 2 or y.ndim != 2:
        raise DataError("points must be (N, D) arrays")
    n, d = x.shape
    m = y.shape[0]
    if y.shape[1] != d:
        raise DataError("dimension mismatch")
    if a.ndim != 1 or a.size != n:
        raise DataError(f"weights of x: expected {n} entries, got {a.size}")
    if b.ndim != 1 or b.size != m:
        raise DataError(f"weights of y: expected {m} entries, got {b.size}")
    return x, a, y, b, n, m, d


def _reach_inf(prm):
    """reach = +inf is balanced OT; reach must otherwise be > 0."""
    from .abi import UsageError
    if not prm.reach > 0:
        raise UsageError("reach must be > 0 (or +inf for balanced OT)")
    return math.isinf(prm.reach)


def _vec(v, size, what):
    from .abi import DataError
    v = _c64(v)
    if v.ndim != 1 or v.size != size:
        raise DataError(f"{what}: expected {size} entries, got {v.size}")
    return v


def default_params(**kw):
    return make_params(**kw)


def make_schedule(diameter, prm):
    cap = 100000
    s, e, l = (np.zeros(cap) for _ in range(3))
    n = lib().msot_schedule(diameter, C.byref(prm), _d(s), _d(e), _d(l), cap)
    if n <= 0:
        from .abi import UsageError
        raise UsageError(lib().msot_last_error().decode() if n == 0 else "schedule too long")
    return s[:n].copy(), e[:n].copy(), l[:n].copy()


def shard_tiles(work, world):
    w = _c64(work)
    b = np.zeros(world + 1, np.int64)
    _check(lib().msot_shard_tiles(_d(w), w.size, world, b.ctypes.data_as(_lp)))
    return b


def exact_ot(x, a, y, b, p=2.0, plan=True):
    """exact_ot(a, b, spec) -> DensePlan: the exact
    transport value and (optionally) an optimal N x M plan, by the host network
    simplex of csrc/exact_ot.cpp.  Returns (value, plan or None)."""
    x, a, y, b = _c64(x), _c64(a), _c64(y), _c64(b)
    if x.ndim == 1:
        x = x[:, None]
    if y.ndim == 1:
        y = y[:, None]
    n, d = x.shape
    m = y.shape[0]
    if y.shape[1] != d or a.size != n or b.size != m:
        from .abi import DataError
        raise DataError("exact_ot: dimension mismatch")
    out = np.zeros((n, m)) if plan else None
    v = C.c_double()
    _check(lib().msot_exact_ot(_d(x), _d(a), n, _d(y), _d(b), m, d, float(p),
                               _d(out) if plan else None, C.byref(v)))
    return v.value, out


@dataclass
class DualPotentials:
    """The four dual vectors of SPEC.md:137-140 (caller's atom order)."""

    a_xx: np.ndarray
    b_yy: np.ndarray
    a_xy: np.ndarray
    b_yx: np.ndarray
    eps: float


@dataclass
class SoftLabels:
    """scores (N x L, >= 0) and row_mass (N)."""
    scores: np.ndarray
    row_mass: np.ndarray


OUTLIER = -1  # classify(): label of rows whose mass is below tau


def plan_entry(i, j, x, a, y, b, duals):
    """a_i b_j exp((f_i + g_j - C(x_i, y_j)) / eps), p = 2 (host)."""
    x, y = np.atleast_2d(_c64(x)), np.atleast_2d(_c64(y))
    if x.shape[0] == 1 and x.shape[1] != y.shape[1]:
        x, y = x.T, y.T
    c = 0.5 * float(((x[i] - y[j]) ** 2).sum())
    return float(a[i] * b[j] * math.exp((duals.b_yx[i] + duals.a_xy[j] - c) / duals.eps))


def grad_weights(prm, a, b, duals):
    """gradient of S with respect to the weights of alpha with
    the potentials frozen: (rho + eps/2)(exp(-a_xx/rho) - exp(-b_yx/rho)) for a
    finite reach, b_yx - a_xx + eps (sum a - sum b) for reach = inf (host)."""
    a, b = _c64(a), _c64(b)
    eps = duals.eps
    if _reach_inf(prm):
        return duals.b_yx - duals.a_xx + eps * (a.sum() - b.sum())
    rho = prm.reach ** prm.p
    return (rho + eps / 2) * (np.exp(-duals.a_xx / rho) - np.exp(-duals.b_yx / rho))


def resolve_flips(soft, flip_of, orientation):
    """soft labels of a flip-augmented subject -> one row per
    original fibre, keeping the orientation with the larger row mass (ties to
    the original orientation).  flip_of[i] = original fibre of augmented row
    i, orientation[i] = 0 (original) or 1 (flipped).  Returns (SoftLabels,
    chosen augmented row per original)."""
    sc = _c64(soft.scores)
    rm = _c64(soft.row_mass)
    n, L = sc.shape
    fo = np.ascontiguousarray(flip_of, dtype=np.int32)
    ori = np.ascontiguousarray(orientation, dtype=np.int32)
    n_orig = n // 2
    out_s = np.zeros((n_orig, L))
    out_m = np.zeros(n_orig)
    chosen = np.zeros(n_orig, np.int32)
    _check(lib().msot_resolve_flips(_d(sc), _d(rm), n, L, fo.ctypes.data_as(_ip),
                                    ori.ctypes.data_as(_ip), _d(out_s), _d(out_m),
                                    chosen.ctypes.data_as(_ip)))
    return SoftLabels(out_s, out_m), chosen


def classify(soft, tau=0.5):
    """hard labels (OUTLIER = -1 where row_mass < tau;
    argmax with ties to the lowest class) and confidence max/row_mass."""
    sc = _c64(soft.scores)
    rm = _c64(soft.row_mass)
    n, L = sc.shape
    lab = np.zeros(n, np.int32)
    conf = np.zeros(n)
    _check(lib().msot_classify(_d(sc), _d(rm), n, L, tau, lab.ctypes.data_as(_ip), _d(conf)))
    return lab, conf


class Context:
    """One GPU (one process per GPU; optional NCCL communicator)."""

    def __init__(self, device=0, rank=0, world=1, nccl_id=None, host_collectives=None):
        """host_collectives: (allreduce(np.ndarray), broadcast(np.ndarray, root))
        callables — the msot_create_dist_host test seam (several processes on
        one GPU) instead of NCCL."""
        self._h = C.c_void_p()
        if host_collectives is not None:
            ar, bc = host_collectives

            def _ar(ptr, count, user):
                try:
                    ar(np.ctypeslib.as_array(ptr, shape=(count,)))
                    return 0
                except Exception:
                    return 1

            def _bc(ptr, count, root, user):
                try:
                    bc(np.ctypeslib.as_array(ptr, shape=(count,)), root)
                    return 0
                except Exception:
                    return 1

            self._cbs = (_AR_FN(_ar), _BC_FN(_bc))  # keep alive
            _check(lib().msot_create_dist_host(device, rank, world, self._cbs[0], self._cbs[1],
                                               None, C.byref(self._h)))
        elif world > 1 or nccl_id is not None:
            # one process per GPU; world 1 with an id = a one-rank communicator
            # (the NCCL calls run, as no-ops on the data)
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("world > 1 needs the 128-byte NCCL id of rank 0")
            _check(lib().msot_create_dist(device, rank, world, bytes(nccl_id), C.byref(self._h)))
        else:
            _check(lib().msot_create(device, C.byref(self._h)))
        self.rank, self.world = rank, world

    @staticmethod
    def nccl_unique_id():
        buf = C.create_string_buffer(128)
        _check(lib().msot_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if self._h:
            lib().msot_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def world_info(self):
        """(rank, world, ranks in the NCCL communicator per ncclCommCount)."""
        r, w, n = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().msot_world_info(self._h, C.byref(r), C.byref(w), C.byref(n)))
        return r.value, w.value, n.value

    def debug_capture(self, scale, n, m):
        """Arms the parity seam for schedule index `scale`: returns (before,
        after) dicts of caller-order float64 arrays that the next solves fill;
        scale < 0 disarms."""
        if scale < 0:
            _check(lib().msot_debug_capture(self._h, -1, None, None))
            return None, None
        keys, sizes = ("a_xx", "b_yy", "a_xy", "b_yx"), (n, m, m, n)
        before = {k: np.full(s, np.nan) for k, s in zip(keys, sizes)}
        after = {k: np.full(s, np.nan) for k, s in zip(keys, sizes)}
        self._cap = ((_dp * 4)(*[_d(before[k]) for k in keys]),
                     (_dp * 4)(*[_d(after[k]) for k in keys]), before, after)
        _check(lib().msot_debug_capture(self._h, int(scale), self._cap[0], self._cap[1]))
        return before, after

    def debug_mask(self, which, n_rows, n_cols):
        """The captured cluster mask (0 = x-x, 1 = y-y, 2 = x-y) as a (Kr, Kc)
        uint8 array, plus the row / column atom -> cluster maps."""
        kr, kc = C.c_int32(), C.c_int32()
        _check(lib().msot_debug_mask(self._h, which, C.byref(kr), C.byref(kc), None, None, None))
        mask = np.zeros((kr.value, kc.value), np.uint8)
        rl, cl = np.zeros(n_rows, np.int32), np.zeros(n_cols, np.int32)
        _check(lib().msot_debug_mask(self._h, which, None, None, mask.ctypes.data_as(_bp),
                                     rl.ctypes.data_as(_ip), cl.ctypes.data_as(_ip)))
        return mask, rl, cl

    def set_colpart_budget(self, slots=0):
        """Column-partial slots of one evaluate-once batch pair (0 = automatic)."""
        _check(lib().msot_set_colpart_budget(self._h, int(slots)))

    def set_profiling(self, on=True):
        _check(lib().msot_set_profiling(self._h, int(bool(on))))

    def probe_ex2(self):
        """Measured MUFU.EX2 rate of this GPU (ex2/s): the softmin roofline."""
        r = C.c_double()
        _check(lib().msot_probe_ex2(self._h, C.byref(r)))
        return r.value

    # -- SPEC.md:164-172
    def softmin(self, x, y, logw, h, eps, lam=1.0, f_est=None):
        x, _, y, _, n, m, d = _measures(x, np.zeros(np.shape(x)[0]), y, np.zeros(np.shape(y)[0]))
        logw, h = _vec(logw, m, "logw"), _vec(h, m, "h")
        out = np.zeros(n)
        fe = None if f_est is None else _d(_vec(f_est, n, "f_est"))
        _check(lib().msot_softmin(self._h, _d(x), n, _d(y), y.shape[0], d, _d(logw), _d(h),
                                  eps, lam, fe, _d(out)))
        return out

    # -- voxel-grid clustering (K2)
    def grid_cluster(self, x, w, origin, cell):
        x, w, origin = _c64(x), _c64(w), _c64(origin)
        n, d = x.shape
        w = _vec(w, n, "weights")
        origin = _vec(origin, d, "origin")
        perm = np.zeros(n, np.int32)
        labels = np.zeros(n, np.int32)
        offsets = np.zeros(n + 1, np.int32)
        k = C.c_int32()
        cen = np.zeros((n, d))
        cw = np.zeros(n)
        rad = np.zeros(n, np.float32)
        _check(lib().msot_grid_cluster(self._h, _d(x), _d(w), n, d, _d(origin), cell,
                                       perm.ctypes.data_as(_ip), labels.ctypes.data_as(_ip),
                                       offsets.ctypes.data_as(_ip), C.byref(k), _d(cen),
                                       _d(cw), rad.ctypes.data_as(_fp)))
        K = k.value
        return dict(perm=perm, labels=labels, offsets=offsets[:K + 1].copy(), k=K,
                    centroids=cen[:K].copy(), cweights=cw[:K].copy(), radii=rad[:K].copy())

    # -- kmeans_coarsen
    def kmeans(self, x, w, k, seed=0):
        x, w = _c64(x), _c64(w)
        if x.ndim == 1:
            x = x[:, None]
        n, d = x.shape
        w = _vec(w, n, "weights")
        perm = np.zeros(n, np.int32)
        off = np.zeros(k + 1, np.int32)
        lab = np.zeros(n, np.int32)
        cen = np.zeros((k, d))
        cw = np.zeros(k)
        rad = np.zeros(k, np.float32)
        it = C.c_int()
        _check(lib().msot_kmeans(self._h, _d(x), _d(w), n, d, k, seed, perm.ctypes.data_as(_ip),
                                 off.ctypes.data_as(_ip), lab.ctypes.data_as(_ip), _d(cen), _d(cw),
                                 rad.ctypes.data_as(_fp), C.byref(it)))
        return dict(perm=perm, offsets=off, labels=lab, centroids=cen, cweights=cw, radii=rad,
                    iters=it.value)

    # -- kernel_truncation on explicit coarse inputs (K3)
    def kernel_truncation(self, cx, rx, fx, cy, ry, gy, eps, theta, self_=False, gx=None,
                          hy=None, bx=None, by=None):
        """gx / hy: optional (K, 4) {slope, F'} arrays for the slope bound;
        bx / by: optional (K, 6) member boxes {lo[3], hi[3]} for the box bound."""
        f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
        cx, rx, fx, cy, ry, gy = map(f32, (cx, rx, fx, cy, ry, gy))
        kx, d = cx.shape
        ky = cy.shape[0]
        out = np.zeros((kx, ky), np.uint8)
        fp = lambda a: None if a is None else a.ctypes.data_as(_fp)
        gx = None if gx is None else f32(gx)
        hy = None if hy is None else f32(hy)
        if bx is None and by is None:
            _check(lib().msot_truncation_mask(self._h, kx, ky, d, fp(cx), fp(rx), fp(fx), fp(gx),
                                              fp(cy), fp(ry), fp(gy), fp(hy), eps, theta, 2.0,
                                              int(self_), out.ctypes.data_as(_bp)))
        else:
            bx = None if bx is None else _vec(np.ravel(bx), kx * 6, "bx").astype(np.float32)
            by = None if by is None else _vec(np.ravel(by), ky * 6, "by").astype(np.float32)
            _check(lib().msot_truncation_mask_box(self._h, kx, ky, d, fp(cx), fp(rx), fp(fx),
                                                  fp(gx), fp(bx), fp(cy), fp(ry), fp(gy), fp(hy),
                                                  fp(by), eps, theta, 2.0, int(self_),
                                                  out.ctypes.data_as(_bp)))
        return out

    # -- symmetric_sinkhorn / multiscale_sinkhorn + divergence
    def sinkhorn(self, prm, x, a, y, b, potentials=True):
        x, a, y, b, n, m, d = _measures(x, a, y, b)
        loss = C.c_double()
        st = Stats()
        pots = None
        ptrs = [None] * 4
        if potentials:
            pots = [np.zeros(n), np.zeros(m), np.zeros(m), np.zeros(n)]
            ptrs = [_d(p) for p in pots]
        _check(lib().msot_sinkhorn(self._h, C.byref(prm), _d(x), _d(a), n, _d(y), _d(b), m, d,
                                   *ptrs, C.byref(loss), C.byref(st)))
        duals = None
        if potentials:
            s, e, _ = make_schedule(st.diameter, prm)
            duals = DualPotentials(*pots, eps=float(e[-1]))
        return loss.value, duals, st.as_dict()

    # -- grad_positions
    def sinkhorn_grad(self, prm, x, a, y, b):
        """Returns (loss, grad_x (N x D), stats)."""
        x, a, y, b, n, m, d = _measures(x, a, y, b)
        loss = C.c_double()
        st = Stats()
        g = np.zeros((n, d))
        _check(lib().msot_sinkhorn_grad(self._h, C.byref(prm), _d(x), _d(a), n, _d(y), _d(b),
                                        y.shape[0], d, C.byref(loss), _d(g), C.byref(st)))
        return loss.value, g, st.as_dict()

    # -- barycenter
    def barycenter(self, prm, x0, a, targets, iters=10, step=1.0, tol=1e-4):
        """targets: list of (points, weights).  Returns (x, loss trajectory, stats)."""
        if not targets:
            from .abi import DataError
            raise DataError("barycenter needs at least one target")
        ys, bs = [], []
        for t in targets:
            x0, a, yt, bt, n, _, d = _measures(x0, a, t[0], t[1])
            ys.append(yt)
            bs.append(bt)
        k = len(targets)
        yp = (_dp * k)(*[_d(v) for v in ys])
        bp = (_dp * k)(*[_d(v) for v in bs])
        ms = np.array([len(v) for v in bs], np.int64)
        x = np.zeros((n, d))
        traj = np.zeros(iters + 1)
        done = C.c_int()
        st = Stats()
        _check(lib().msot_barycenter(self._h, C.byref(prm), _d(x0), _d(a), n, k, yp, bp,
                                     ms.ctypes.data_as(_lp), d, iters, step, tol, _d(x),
                                     _d(traj), C.byref(done), C.byref(st)))
        return x, traj[:done.value + 1].copy(), st.as_dict()

    # -- transfer_labels (eq. 7)
    def transfer_labels(self, prm, x, a, y, b, labels, n_classes=None):
        """Solves S(alpha, beta) and transfers the atlas labels of y to x.
        Returns (SoftLabels(scores N x L, row_mass N), loss, stats)."""
        x, a, y, b, n, m, d = _measures(x, a, y, b)
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        if lab.ndim != 1 or lab.size != m:
            from .abi import DataError
            raise DataError(f"labels: expected {m} entries, got {lab.size}")
        L = int(lab.max()) + 1 if n_classes is None else int(n_classes)
        scores = np.zeros((n, L))
        mass = np.zeros(n)
        loss = C.c_double()
        st = Stats()
        _check(lib().msot_transfer_labels(self._h, C.byref(prm), _d(x), _d(a), n, _d(y), _d(b),
                                          y.shape[0], d, lab.ctypes.data_as(_ip), L,
                                          _d(scores), _d(mass), C.byref(loss), C.byref(st)))
        return SoftLabels(scores, mass), loss.value, st.as_dict()

    # -- plan_apply
    def plan_apply(self, x, a, y, b, f, g, eps, v):
        """(pi v)_i = sum_j a_i b_j exp((f_i + g_j - C_ij)/eps) v_j on the GPU."""
        x, a, y, b, n, m, d = _measures(x, a, y, b)
        f, g, v = _vec(f, n, "f"), _vec(g, m, "g"), _vec(v, m, "v")
        out = np.zeros(n)
        _check(lib().msot_plan_apply(self._h, _d(x), _d(a), n, _d(y), _d(b), y.shape[0], d,
                                     _d(f), _d(g), eps, _d(v), _d(out)))
        return out

    def ot_value(self, prm, x, a, y, b, duals):
        """the dual objective of Eq. (3) at (f, g) = (b_yx, a_xy);
        reach = inf uses the limit <a,f> + <b,g> + eps <a x b, 1 - exp((f+g-C)/eps)>,
        whose plan mass comes from plan_apply(1)."""
        eps = duals.eps
        f, g = duals.b_yx, duals.a_xy
        a, b = _c64(a), _c64(b)
        if _reach_inf(prm):
            mass = self.plan_apply(x, a, y, b, f, g, eps, np.ones(len(b))).sum()
            return float(a @ f + b @ g + eps * (a.sum() * b.sum() - mass))
        rho = prm.reach ** prm.p  # PAPER.md eq. 3
        mass = self.plan_apply(x, a, y, b, f, g, eps, np.ones(len(b))).sum()
        return float(rho * (a @ (1 - np.exp(-f / rho))) + rho * (b @ (1 - np.exp(-g / rho)))
                     + eps * (a.sum() * b.sum() - mass))

    def sinkhorn_device(self, prm, x_ptr, a_ptr, n, y_ptr, b_ptr, m, d):
        """Inputs already resident in HBM (float64 device pointers)."""
        loss = C.c_double()
        st = Stats()
        _check(lib().msot_sinkhorn_device(self._h, C.byref(prm), x_ptr, a_ptr, n, y_ptr, b_ptr,
                                          m, d, C.byref(loss), C.byref(st)))
        return loss.value, st.as_dict()

    def divergence(self, x, a, y, b, blur=0.05, reach=math.inf, scaling=0.9, multiscale=False,
                   **kw):
        prm = make_params(blur=blur, reach=reach, scaling=scaling, multiscale=multiscale, **kw)
        return self.sinkhorn(prm, x, a, y, b, potentials=False)[0]


def params_struct(**kw):
    return make_params(**kw)
