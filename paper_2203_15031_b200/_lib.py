"""ctypes binding of libspmesl.so (include/spmesl.h).  Argument marshalling only.

The library must exist in-tree (built by ``paper_2203_15031_b200.build`` /
``__graft_entry__.build()``); there is no fallback of any kind: a missing library raises.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libspmesl.so")

OK = 0
WARN_NOT_CONVERGED = 1
ERR_ARG = -1
ERR_CONSTANT_COLUMN = -2
ERR_NONFINITE = -3
ERR_CUDA = -4
ERR_OOM = -6
ERR_UNSUPPORTED = -7


class Options(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_int32),
        ("max_inner", ctypes.c_int32),
        ("standardize", ctypes.c_int32),
        ("symmetrize", ctypes.c_int32),
        ("sigma_floor", ctypes.c_double),
        ("mode", ctypes.c_int32),
        ("tile_cols", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("tail_after", ctypes.c_int32),
        ("solver", ctypes.c_int32),
        ("eager", ctypes.c_int32),
        ("num_devices", ctypes.c_int32),
        ("exchange", ctypes.c_int32),
        ("device_ids", ctypes.POINTER(ctypes.c_int32)),
        ("reserved", ctypes.c_int32 * 2),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("coord_updates", ctypes.c_int64),
        ("total_sweeps", ctypes.c_int64),
        ("max_sweeps", ctypes.c_int32),
        ("max_outer", ctypes.c_int32),
        ("n_unconverged", ctypes.c_int32),
        ("tile_cols", ctypes.c_int32),
        ("num_ctas", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("bad_column", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("ms_standardize", ctypes.c_double),
        ("ms_cd", ctypes.c_double),
        ("ms_assemble", ctypes.c_double),
        ("ms_total", ctypes.c_double),
        ("ms_tail", ctypes.c_double),
        ("tail_columns", ctypes.c_int64),
        ("tail_gram_ondemand", ctypes.c_int64),
        ("tail_sweeps", ctypes.c_int64),
        ("solver", ctypes.c_int32),
        ("gram_fallback", ctypes.c_int32),
        ("ms_gram", ctypes.c_double),
        ("screen_candidates", ctypes.c_int64),
        ("ms_screen", ctypes.c_double),
        ("screen_fill_bytes", ctypes.c_int64),
        ("graph_replay", ctypes.c_int32),
        ("pad1", ctypes.c_int32),
        ("tail_changes", ctypes.c_int64),
        ("tail_passes", ctypes.c_int64),
        ("ms_comm", ctypes.c_double),
        ("num_devices", ctypes.c_int32),
        ("exchange", ctypes.c_int32),
    ]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = [
    "spmesl_default_options", "spmesl_fit", "spmesl_fit_ex", "spmesl_fit_device",
    "spmesl_fit_columns_device", "spmesl_assemble_device", "spmesl_gram_tile_count",
    "spmesl_gram_screen_device", "spmesl_fit_columns_gram_device", "spmesl_gram_supported",
    "spmesl_fit_path_device", "spmesl_screen_tile_count", "spmesl_fit_sparse_device",
    "spmesl_screen_accumulators_device", "spmesl_fit_sparse", "spmesl_lambda_univ",
    "spmesl_lambda_ub", "spmesl_lambda_pb", "spmesl_solve_k", "spmesl_last_error",
    "spmesl_release_workspace", "spmesl_version",
]

_lib = None


def load() -> ctypes.CDLL:
    """Load libspmesl.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m "
                           "paper_2203_15031_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    popt = ctypes.POINTER(Options)
    pst = ctypes.POINTER(Stats)
    L.spmesl_default_options.argtypes = [popt]
    L.spmesl_default_options.restype = None
    L.spmesl_fit.argtypes = [vp, i64, i64, dbl, dbl, i32, vp, vp, vp]
    L.spmesl_fit.restype = ctypes.c_int
    L.spmesl_fit_ex.argtypes = [vp, i64, i64, dbl, dbl, i32, popt, vp, vp, vp, vp, vp, pst]
    L.spmesl_fit_ex.restype = ctypes.c_int
    L.spmesl_fit_device.argtypes = [vp, i64, i64, dbl, dbl, i32, popt, vp, vp, vp, vp, vp, vp, pst]
    L.spmesl_fit_device.restype = ctypes.c_int
    L.spmesl_fit_columns_device.argtypes = [vp, i64, i64, i64, i64, dbl, dbl, i32, popt, vp, vp,
                                            vp, i64, ctypes.POINTER(i64), vp, vp, vp, vp, vp, vp,
                                            pst]
    L.spmesl_fit_columns_device.restype = ctypes.c_int
    L.spmesl_fit_path_device.argtypes = [vp, i64, i64, vp, i32, dbl, i32, popt, vp, vp, vp, vp, vp,
                                         vp, pst]
    L.spmesl_fit_path_device.restype = ctypes.c_int
    L.spmesl_gram_supported.argtypes = [i64, i64]
    L.spmesl_gram_supported.restype = ctypes.c_int
    L.spmesl_gram_tile_count.argtypes = [i64]
    L.spmesl_gram_tile_count.restype = i64
    L.spmesl_fit_sparse_device.argtypes = [vp, i64, i64, dbl, dbl, i32, popt, vp, vp, vp, i64,
                                           ctypes.POINTER(ctypes.c_int64), vp, vp, vp, vp, vp, pst]
    L.spmesl_fit_sparse_device.restype = ctypes.c_int
    L.spmesl_screen_tile_count.argtypes = [i64, popt]
    L.spmesl_screen_tile_count.restype = i64
    L.spmesl_gram_screen_device.argtypes = [vp, i64, i64, dbl, i64, i64, popt, vp, vp, pst]
    L.spmesl_gram_screen_device.restype = ctypes.c_int
    L.spmesl_fit_columns_gram_device.argtypes = [vp, i64, i64, i64, i64, dbl, dbl, i32, popt, vp,
                                                 vp, vp, vp, i64, ctypes.POINTER(i64), vp, vp, vp,
                                                 vp, vp, vp, pst]
    L.spmesl_fit_columns_gram_device.restype = ctypes.c_int
    L.spmesl_assemble_device.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, popt, vp, vp, vp]
    L.spmesl_assemble_device.restype = ctypes.c_int
    L.spmesl_screen_accumulators_device.argtypes = [vp, i64, i64, popt, vp, i64, vp, vp, vp]
    L.spmesl_screen_accumulators_device.restype = ctypes.c_int
    L.spmesl_fit_sparse.argtypes = [vp, i64, i64, dbl, dbl, i32, popt, vp, vp, vp, i64,
                                    ctypes.POINTER(i64), vp, vp, vp, vp, pst]
    L.spmesl_fit_sparse.restype = ctypes.c_int
    for f in ("spmesl_lambda_univ",):
        getattr(L, f).argtypes = [i64, i64]
        getattr(L, f).restype = dbl
    for f in ("spmesl_lambda_ub", "spmesl_lambda_pb"):
        getattr(L, f).argtypes = [i64, i64, dbl]
        getattr(L, f).restype = dbl
    L.spmesl_solve_k.argtypes = [i64]
    L.spmesl_solve_k.restype = dbl
    L.spmesl_last_error.argtypes = []
    L.spmesl_last_error.restype = ctypes.c_char_p
    L.spmesl_release_workspace.restype = ctypes.c_int
    L.spmesl_version.restype = ctypes.c_char_p
    _lib = L
    return L


def default_options(**kw) -> Options:
    o = Options()
    load().spmesl_default_options(ctypes.byref(o))
    for k, v in kw.items():
        if v is None:
            continue
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, v)
    return o


class SpmeslError(RuntimeError):
    def __init__(self, code: int, msg: str, bad_column: int = -1):
        super().__init__(f"spmesl error {code}: {msg}")
        self.code = code
        self.bad_column = bad_column


def check(rc: int, stats: Stats | None = None) -> int:
    if rc < 0:
        msg = load().spmesl_last_error().decode()
        raise SpmeslError(rc, msg, stats.bad_column if stats is not None else -1)
    return rc
