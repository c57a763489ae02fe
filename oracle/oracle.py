"""ctypes binding of oracle/liboracle.so — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker / the timed CPU baseline.  The
product path (paper_2107_02010_b200) never imports it.
"""
import ctypes as C
import os

import numpy as np

from paper_2107_02010_b200.abi import Params, Stats, raise_status

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_bp = C.POINTER(C.c_uint8)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/liboracle.so missing: run `make -C oracle`")
        L = C.CDLL(path)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_threads.restype = C.c_int
        L.oracle_schedule.restype = C.c_int
        L.oracle_schedule.argtypes = [C.c_double, C.POINTER(Params), _dp, _dp, _dp, C.c_int]
        L.oracle_softmin.restype = None
        L.oracle_softmin.argtypes = [_dp, C.c_int64, _dp, C.c_int64, C.c_int, _dp, _dp,
                                     C.c_double, C.c_double, C.c_double, _dp]
        L.oracle_grid_cluster.restype = C.c_int
        L.oracle_grid_cluster.argtypes = [_dp, _dp, C.c_int64, C.c_int, _dp, C.c_double, _ip,
                                          _ip, _ip, _ip, _dp, _dp, _fp]
        L.oracle_truncation_mask.restype = None
        L.oracle_truncation_mask.argtypes = [C.c_int64, C.c_int64, C.c_int, _fp, _fp, _fp,
                                             _fp, _fp, _fp, _fp, _fp, C.c_double, C.c_double,
                                             C.c_double, C.c_int, _bp]
        L.oracle_truncation_mask_box.restype = None
        L.oracle_truncation_mask_box.argtypes = [C.c_int64, C.c_int64, C.c_int, _fp, _fp, _fp, _fp,
                                                 _fp, _fp, _fp, _fp, _fp, _fp, C.c_double,
                                                 C.c_double, C.c_double, C.c_int, _bp]
        L.oracle_tile_ranges.restype = C.c_int64
        L.oracle_tile_ranges.argtypes = [_ip, _ip, C.c_int64, C.c_int64, _ip, C.c_int64, _bp,
                                         _lp, _lp, _lp, _ip, C.c_int64]
        L.oracle_sinkhorn.restype = C.c_int
        L.oracle_sinkhorn.argtypes = [C.POINTER(Params), _dp, _dp, C.c_int64, _dp, _dp,
                                      C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp,
                                      C.POINTER(Stats)]
        L.oracle_divergence_from_potentials.restype = C.c_double
        L.oracle_divergence_from_potentials.argtypes = [C.POINTER(Params), C.c_double, _dp,
                                                        C.c_int64, _dp, C.c_int64, _dp, _dp,
                                                        _dp, _dp]
        _LIB = L
    return _LIB


def _d(a):
    return a.ctypes.data_as(_dp)


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n):
    lib().oracle_set_threads(int(n))


def threads():
    return lib().oracle_threads()


def schedule(diameter, prm):
    cap = 100000
    s, e, l = (np.zeros(cap) for _ in range(3))
    n = lib().oracle_schedule(diameter, C.byref(prm), _d(s), _d(e), _d(l), cap)
    return s[:n].copy(), e[:n].copy(), l[:n].copy()


def softmin(x, y, logw, h, eps, lam=1.0, p=2.0):
    x, y, logw, h = _c64(x), _c64(y), _c64(logw), _c64(h)
    n, d = x.shape
    m = y.shape[0]
    out = np.zeros(n)
    lib().oracle_softmin(_d(x), n, _d(y), m, d, _d(logw), _d(h), eps, lam, p, _d(out))
    return out


def grid_cluster(x, w, origin, cell):
    x, w, origin = _c64(x), _c64(w), _c64(origin)
    n, d = x.shape
    perm = np.zeros(n, np.int32)
    labels = np.zeros(n, np.int32)
    offsets = np.zeros(n + 1, np.int32)
    k = C.c_int32(0)
    cen = np.zeros((n, d))
    cw = np.zeros(n)
    rad = np.zeros(n, np.float32)
    rc = lib().oracle_grid_cluster(_d(x), _d(w), n, d, _d(origin), cell,
                                   perm.ctypes.data_as(_ip), labels.ctypes.data_as(_ip),
                                   offsets.ctypes.data_as(_ip), C.byref(k), _d(cen), _d(cw),
                                   rad.ctypes.data_as(_fp))
    raise_status(rc, lib().oracle_last_error().decode())
    K = k.value
    return dict(perm=perm, labels=labels, offsets=offsets[:K + 1].copy(), k=K,
                centroids=cen[:K].copy(), cweights=cw[:K].copy(), radii=rad[:K].copy())


def kmeans(x, w, k, seed=0):
    L = lib()
    L.oracle_kmeans.restype = C.c_int
    L.oracle_kmeans.argtypes = [_dp, _dp, C.c_int64, C.c_int, C.c_int, C.c_uint64, _ip, _ip, _ip,
                                _dp, _dp, _fp, C.POINTER(C.c_int)]
    x, w = _c64(x), _c64(w)
    if x.ndim == 1:
        x = x[:, None]
    n, d = x.shape
    perm = np.zeros(n, np.int32)
    off = np.zeros(k + 1, np.int32)
    lab = np.zeros(n, np.int32)
    cen = np.zeros((k, d))
    cw = np.zeros(k)
    rad = np.zeros(k, np.float32)
    it = C.c_int()
    rc = L.oracle_kmeans(_d(x), _d(w), n, d, k, seed, perm.ctypes.data_as(_ip),
                         off.ctypes.data_as(_ip), lab.ctypes.data_as(_ip), _d(cen), _d(cw),
                         rad.ctypes.data_as(_fp), C.byref(it))
    raise_status(rc, L.oracle_last_error().decode())
    return dict(perm=perm, offsets=off, labels=lab, centroids=cen, cweights=cw, radii=rad,
                iters=it.value)


def truncation_mask(cx, rx, fx, cy, ry, gy, eps, theta, p=2.0, self_=False, gx=None, hy=None,
                    bx=None, by=None):
    """bx / by: member boxes (K x 6: lo[3], hi[3]) for the box bound."""
    f32 = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    cx, rx, fx, cy, ry, gy = map(f32, (cx, rx, fx, cy, ry, gy))
    kx, d = cx.shape
    ky = cy.shape[0]
    out = np.zeros((kx, ky), np.uint8)
    fp = lambda a: None if a is None else a.ctypes.data_as(_fp)
    gx = None if gx is None else f32(gx)
    hy = None if hy is None else f32(hy)
    if bx is None:
        lib().oracle_truncation_mask(kx, ky, d, fp(cx), fp(rx), fp(fx), fp(gx), fp(cy), fp(ry),
                                     fp(gy), fp(hy), eps, theta, p, int(self_),
                                     out.ctypes.data_as(_bp))
    else:
        bx, by = f32(bx), f32(by)
        lib().oracle_truncation_mask_box(kx, ky, d, fp(cx), fp(rx), fp(fx), fp(gx), fp(bx),
                                         fp(cy), fp(ry), fp(gy), fp(hy), fp(by), eps, theta, p,
                                         int(self_), out.ctypes.data_as(_bp))
    return out


def tile_ranges(row_labels, row_offsets, col_offsets, mask):
    """Returns (tile_start, tile_ptr, ranges) — cluster-aligned row tiles."""
    row_labels = np.ascontiguousarray(row_labels, np.int32)
    row_offsets = np.ascontiguousarray(row_offsets, np.int32)
    col_offsets = np.ascontiguousarray(col_offsets, np.int32)
    mask = np.ascontiguousarray(mask, np.uint8)
    n = row_labels.shape[0]
    kx, ky = mask.shape
    cap = kx + n // 256 + 2
    ts = np.zeros(cap, np.int64)
    ptr = np.zeros(cap, np.int64)
    nt = C.c_int64()
    args = (row_labels.ctypes.data_as(_ip), row_offsets.ctypes.data_as(_ip), n, kx,
            col_offsets.ctypes.data_as(_ip), ky, mask.ctypes.data_as(_bp), C.byref(nt),
            ts.ctypes.data_as(_lp), ptr.ctypes.data_as(_lp))
    cnt = lib().oracle_tile_ranges(*args, None, 0)
    rg = np.zeros((max(cnt, 1), 2), np.int32)
    lib().oracle_tile_ranges(*args, rg.ctypes.data_as(_ip), cnt)
    T = nt.value
    return ts[:T + 1].copy(), ptr[:T + 1].copy(), rg[:cnt]


def sinkhorn(prm, x, a, y, b, potentials=True):
    """Returns (loss, dict of potentials or None, stats dict)."""
    x, a, y, b = _c64(x), _c64(a), _c64(y), _c64(b)
    if x.ndim == 1:
        x = x[:, None]
    if y.ndim == 1:
        y = y[:, None]
    n, d = x.shape
    m = y.shape[0]
    loss = C.c_double(0)
    st = Stats()
    pots = None
    args = [None] * 4
    if potentials:
        pots = dict(a_xx=np.zeros(n), b_yy=np.zeros(m), a_xy=np.zeros(m), b_yx=np.zeros(n))
        args = [_d(pots[k]) for k in ("a_xx", "b_yy", "a_xy", "b_yx")]
    rc = lib().oracle_sinkhorn(C.byref(prm), _d(x), _d(a), n, _d(y), _d(b), m, d, *args,
                               C.byref(loss), C.byref(st))
    raise_status(rc, lib().oracle_last_error().decode())
    return loss.value, pots, st.as_dict()


def divergence_from_potentials(prm, eps, a, b, pots):
    a, b = _c64(a), _c64(b)
    P = {k: _c64(v) for k, v in pots.items()}
    return lib().oracle_divergence_from_potentials(C.byref(prm), eps, _d(a), a.size, _d(b),
                                                   b.size, _d(P["a_xx"]), _d(P["b_yy"]),
                                                   _d(P["a_xy"]), _d(P["b_yx"]))


def _setup_grad(L):
    L.oracle_sinkhorn_grad.restype = C.c_int
    L.oracle_sinkhorn_grad.argtypes = [C.POINTER(Params), _dp, _dp, C.c_int64, _dp, _dp,
                                       C.c_int64, C.c_int, _dp, _dp]
    L.oracle_barycenter.restype = C.c_int
    L.oracle_barycenter.argtypes = [C.POINTER(Params), _dp, _dp, C.c_int64, C.c_int,
                                    C.POINTER(_dp), C.POINTER(_dp), _lp, C.c_int, C.c_int,
                                    C.c_double, C.c_double, _dp, _dp, C.POINTER(C.c_int)]


def sinkhorn_grad(prm, x, a, y, b):
    L = lib()
    _setup_grad(L)
    x, a, y, b = _c64(x), _c64(a), _c64(y), _c64(b)
    if x.ndim == 1:
        x = x[:, None]
    if y.ndim == 1:
        y = y[:, None]
    n, d = x.shape
    loss = C.c_double()
    g = np.zeros((n, d))
    rc = L.oracle_sinkhorn_grad(C.byref(prm), _d(x), _d(a), n, _d(y), _d(b), y.shape[0], d,
                                C.byref(loss), _d(g))
    raise_status(rc, L.oracle_last_error().decode())
    return loss.value, g


def transfer_labels(x, y, b, f, g, eps, labels, n_classes):
    """Dense FP64 soft labels: returns (scores N x L, row_mass N)."""
    L = lib()
    L.oracle_transfer_labels.restype = C.c_int
    L.oracle_transfer_labels.argtypes = [_dp, C.c_int64, _dp, _dp, C.c_int64, C.c_int, _dp, _dp,
                                         C.c_double, _ip, C.c_int, _dp, _dp]
    x, y, b, f, g = _c64(x), _c64(y), _c64(b), _c64(f), _c64(g)
    if x.ndim == 1:
        x = x[:, None]
    if y.ndim == 1:
        y = y[:, None]
    n, d = x.shape
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    sc = np.zeros((n, n_classes))
    rm = np.zeros(n)
    rc = L.oracle_transfer_labels(_d(x), n, _d(y), _d(b), y.shape[0], d, _d(f), _d(g), eps,
                                  lab.ctypes.data_as(_ip), n_classes, _d(sc), _d(rm))
    raise_status(rc, L.oracle_last_error().decode())
    return sc, rm


def plan_apply(x, a, y, b, f, g, eps, v):
    L = lib()
    L.oracle_plan_apply.restype = None
    L.oracle_plan_apply.argtypes = [_dp, _dp, C.c_int64, _dp, _dp, C.c_int64, C.c_int, _dp, _dp,
                                    C.c_double, _dp, _dp]
    x, a, y, b, f, g, v = map(_c64, (x, a, y, b, f, g, v))
    if x.ndim == 1:
        x = x[:, None]
    if y.ndim == 1:
        y = y[:, None]
    out = np.zeros(len(a))
    L.oracle_plan_apply(_d(x), _d(a), len(a), _d(y), _d(b), len(b), x.shape[1], _d(f), _d(g),
                        eps, _d(v), _d(out))
    return out


def barycenter(prm, x0, a, targets, iters=10, step=1.0, tol=1e-4):
    L = lib()
    _setup_grad(L)
    x0, a = _c64(x0), _c64(a)
    n, d = x0.shape
    ys = [_c64(t[0]).reshape(-1, d) for t in targets]
    bs = [_c64(t[1]) for t in targets]
    k = len(targets)
    yp = (_dp * k)(*[_d(v) for v in ys])
    bp = (_dp * k)(*[_d(v) for v in bs])
    ms = np.array([len(v) for v in bs], np.int64)
    x = np.zeros((n, d))
    traj = np.zeros(iters + 1)
    done = C.c_int()
    rc = L.oracle_barycenter(C.byref(prm), _d(x0), _d(a), n, k, yp, bp, ms.ctypes.data_as(_lp),
                             d, iters, step, tol, _d(x), _d(traj), C.byref(done))
    raise_status(rc, L.oracle_last_error().decode())
    return x, traj[:done.value + 1].copy()
