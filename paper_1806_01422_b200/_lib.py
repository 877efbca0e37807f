"""ctypes binding of ``libsemb200.so`` (the C ABI in ``include/sem1d.h``).

The library is built in-tree by ``make -C paper_1806_01422_b200/csrc`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is
missing, or no CUDA device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# SEM1D_LIB selects an alternative build of the same ABI (A/B kernel experiments)
LIB_PATH = os.environ.get("SEM1D_LIB") or os.path.join(_HERE, "libsemb200.so")

SEM1D_FLAG_STATE_NONFINITE = 1
SEM1D_FLAG_INPUT2_NONFINITE = 2
SEM1D_FLAG_STEP_NONFINITE = 4
MAX_TERMS = 5

c_int, c_int64, c_double, c_void_p = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)

SEM1D_CN_OK = 0
SEM1D_CN_GMRES_FAILED = 1
SEM1D_CN_NEWTON_STALLED = 2
SEM1D_CN_RESIDUAL_NONFINITE = 3
SEM1D_CN_INPUT_NONFINITE = 4


class CnParams(ctypes.Structure):
    """sem1d_cn_params (TsConfig's Newton / GMRES settings, timeloop.py:49-53)."""
    _fields_ = [("newton_tol", c_double), ("newton_max", c_int), ("gmres_tol", c_double),
                ("gmres_max", c_int), ("gmres_restart", c_int)]


class CnStats(ctypes.Structure):
    """sem1d_cn_stats (accumulating counters + status of the last call)."""
    _fields_ = [("newton_iters", c_int64), ("gmres_iters", c_int64), ("rhs_applies", c_int64),
                ("jac_applies", c_int64), ("jact_applies", c_int64), ("status", c_int),
                ("gmres_info", c_int), ("last_residual", c_double)]


# name -> (restype, argtypes); exactly the declarations of include/sem1d.h
SIGNATURES = {
    "sem1d_version": (c_int, []),
    "sem1d_set_kernel_path": (c_int, [c_int]),
    "sem1d_set_tile_variant": (c_int, [c_int]),
    "sem1d_last_error": (ctypes.c_char_p, []),
    "sem1d_max_degree": (c_int, []),
    "sem1d_plan_create": (c_int, [c_int64, c_int, c_int, c_double, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_int64, ctypes.POINTER(c_void_p)]),
    "sem1d_plan_destroy": (c_int, [c_void_p]),
    "sem1d_plan_ndof": (c_int64, [c_void_p]),
    "sem1d_plan_set_advection": (c_int, [c_void_p, c_int, c_double]),
    "sem1d_rhs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem1d_jac": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem1d_jact": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem1d_rk_stage": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                               c_double, c_void_p, c_int, c_void_p, c_void_p]),
    "sem1d_adj_stage": (c_int, [c_void_p, c_void_p, c_void_p, c_double, c_int, c_void_p, c_void_p,
                                c_double, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem1d_ens_forward": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                  c_void_p, c_void_p]),
    "sem1d_ens_adjoint": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                  c_void_p, c_void_p]),
    "sem1d_ens_adjoint_ex": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                                     c_void_p, c_void_p]),
    "sem1d_step_supported": (c_int, [c_void_p]),
    "sem1d_step_stages_supported": (c_int, [c_void_p]),
    "sem1d_rk_step_stages": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int, c_void_p,
                                     c_void_p]),
    "sem1d_adj_step_stages": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int,
                                      c_void_p, c_void_p]),
    "sem1d_rk_step": (c_int, [c_void_p, c_void_p, c_void_p, c_double, c_int, c_void_p, c_void_p]),
    "sem1d_rk_step_ex": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int, c_int, c_int, c_int,
                                 c_void_p, c_void_p]),
    "sem1d_adj_step_ex": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int, c_int, c_int,
                                  c_int, c_void_p, c_void_p]),
    "sem1d_step_tiling": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "sem1d_adj_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_int, c_void_p,
                               c_void_p]),
    "sem1d_terminal_work_size": (c_int64, [c_void_p]),
    "sem1d_terminal": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem1d_scatter": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem1d_gather": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem1d_cn_work_size": (c_int64, [c_void_p, c_int]),
    "sem1d_cn_step": (c_int, [c_void_p, c_void_p, c_void_p, c_double, ctypes.POINTER(CnParams),
                              c_void_p, c_void_p, ctypes.POINTER(CnStats), c_void_p]),
    "sem1d_cn_adjoint_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double,
                                      ctypes.POINTER(CnParams), c_void_p, c_void_p,
                                      ctypes.POINTER(CnStats), c_void_p]),
    "sem1d_gmres": (c_int, [c_void_p, c_int, c_void_p, c_double, c_void_p, c_void_p,
                            ctypes.POINTER(CnParams), c_void_p, c_void_p, ctypes.POINTER(CnStats),
                            c_void_p]),
    "sem1d_reduce_work_size": (c_int64, []),
    "sem1d_vec_dot": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem1d_rk_error_norm": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_double, c_double,
                                    c_double, c_int, c_void_p, c_void_p, c_void_p]),
    "sem1d_vec_rk_combine": (c_int, [c_int64, c_void_p, c_double, c_int, c_void_p, c_void_p, c_void_p,
                                     c_int, c_void_p, c_void_p]),
    "sem1d_vec_adj_combine": (c_int, [c_int64, c_void_p, c_double, c_int, c_void_p, c_void_p, c_void_p,
                                      c_void_p]),
    "sem1d_vec_accumulate": (c_int, [c_int64, c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "sem1d_vec_scale": (c_int, [c_int64, c_void_p, c_double, c_void_p, c_void_p]),
    "sem3d_max_degree": (c_int, []),
    "sem3d_plan_create": (c_int, [c_void_p, c_int, c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                                  c_void_p, ctypes.POINTER(c_void_p)]),
    "sem3d_plan_destroy": (c_int, [c_void_p]),
    "sem3d_plan_ndof": (c_int64, [c_void_p]),
    "sem3d_work_size": (c_int64, [c_void_p]),
    "sem3d_rhs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem3d_jac": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem3d_jact": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem3d_terminal": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "sem3d_cn_work_size": (c_int64, [c_void_p, c_int]),
    "sem3d_cn_step": (c_int, [c_void_p, c_void_p, c_void_p, c_double, ctypes.POINTER(CnParams),
                              c_void_p, c_void_p, ctypes.POINTER(CnStats), c_void_p]),
    "sem3d_cn_adjoint_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double,
                                      ctypes.POINTER(CnParams), c_void_p, c_void_p,
                                      ctypes.POINTER(CnStats), c_void_p]),
    "sem3d_gmres": (c_int, [c_void_p, c_int, c_void_p, c_double, c_void_p, c_void_p,
                            ctypes.POINTER(CnParams), c_void_p, c_void_p, ctypes.POINTER(CnStats),
                            c_void_p]),
}

_lock = threading.Lock()
_lib = None


class LibraryMissing(RuntimeError):
    """libsemb200.so is not built or cannot be loaded (no CPU fallback exists)."""


def load():
    """Load (once) and return the ctypes handle; raises LibraryMissing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not found: build it with `make -C {os.path.join(_HERE, 'csrc')} -j` "
                "or __graft_entry__.build(); there is no CPU fallback")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - environment specific
            raise LibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error():
    return load().sem1d_last_error().decode("utf-8", "replace")


def check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed ({rc}): {last_error()}")


def ptr_array(ptrs):
    """ctypes array of device pointers (None -> NULL)."""
    arr = (c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def dbl_array(vals):
    arr = (c_double * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = float(v)
    return arr
