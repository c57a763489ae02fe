"""ctypes mirror of include/msot_gpu.h (structs + status codes).

Shared by the product binding (`paper_2107_02010_b200.solver`) and the test
oracle binding (`oracle/oracle.py`); contains no compute.
"""
import ctypes as C
import math

OK, EUSAGE, EDATA, ENUMERIC, ECUDA = 0, 2, 3, 4, 5


class Params(C.Structure):
    """msot_params (SolverParams of SPEC.md:127-130 + multiscale knobs)."""

    _fields_ = [
        ("blur", C.c_double),
        ("reach", C.c_double),
        ("p", C.c_double),
        ("scaling", C.c_double),
        ("multiscale", C.c_int32),
        ("retruncate", C.c_int32),
        ("cluster_scale", C.c_double),
        ("theta", C.c_double),
        ("switch_factor", C.c_double),
        ("max_full_iters", C.c_int32),
        ("mask_rule", C.c_int32),
        ("transfer_rule", C.c_int32),
        ("pair_eval", C.c_int32),
        ("clusters", C.c_int32),
        ("seed", C.c_int32),
        ("super_level", C.c_int32),
    ]


def make_params(blur=0.05, reach=math.inf, p=2.0, scaling=0.9, multiscale=False,
                retruncate=0, cluster_scale=0.0, theta=20.0, switch_factor=2.0,
                max_full_iters=10000, mask_rule=0, transfer_rule=0, pair_eval=1, clusters=0,
                seed=0, super_level=-1):
    """Defaults follow SPEC.md:128 (q=0.9), :306 (switch 2 r_max), :308 (theta 20),
    :270-274 (coarse duals inherited by the fine atoms)."""
    return Params(blur, math.inf if reach is None else reach, p, scaling, int(bool(multiscale)),
                  int(retruncate), cluster_scale, theta, switch_factor, int(max_full_iters),
                  int(mask_rule), int(transfer_rule), int(pair_eval), int(clusters), int(seed),
                  int(super_level))


class Stats(C.Structure):
    _fields_ = [
        ("n_scales", C.c_int32),
        ("t_switch", C.c_int32),
        ("kx", C.c_int32),
        ("ky", C.c_int32),
        ("diameter", C.c_double),
        ("cluster_scale", C.c_double),
        ("pairs_dense", C.c_double),
        ("pairs_evaluated", C.c_double),
        ("pairs_fine", C.c_double),
        ("pairs_fine_dense", C.c_double),
        ("softmin_ms", C.c_double),
        ("softmin_launches", C.c_int64),
        ("total_ms", C.c_double),
        ("fallback_rows", C.c_int64),
        ("gpu_launches", C.c_int64),
        ("h2d_bytes", C.c_double),
        ("d2h_bytes", C.c_double),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("phase_ms", C.c_double * 8),
        ("pairs_terms", C.c_double),
        ("pairs_mask_terms", C.c_double),
        ("t_super", C.c_int32),
        ("k_super_x", C.c_int32),
        ("k_super_y", C.c_int32),
        ("colpart_batches", C.c_int32),
        ("device_bytes", C.c_double),
        ("host_syncs", C.c_int64),
    ]

    PHASES = ("setup", "coarse", "extrapolate", "masks", "updates", "loss", "labels")

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "phase_ms"}
        d["phase_ms"] = {p: self.phase_ms[i] for i, p in enumerate(self.PHASES)}
        return d


TILE_ROWS = 256  # MSOT_TILE_ROWS in csrc/policy.h


class DataError(ValueError):
    """msot::DataError (common.hpp:10-13): malformed/inconsistent input."""


class NumericError(ArithmeticError):
    """msot::NumericError (common.hpp:15-19): non-finite intermediates."""


class UsageError(ValueError):
    """Invalid parameters (CLI exit code 2)."""


class CudaError(RuntimeError):
    """CUDA/NCCL failure (status 5)."""


def raise_status(code, msg):
    if code == OK:
        return
    cls = {EUSAGE: UsageError, EDATA: DataError, ENUMERIC: NumericError}.get(code, CudaError)
    raise cls(msg)
