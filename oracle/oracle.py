"""SPMESL CPU oracle — TEST INFRASTRUCTURE ONLY.

Python side of the oracle: a ctypes wrapper around ``spmesl_oracle.c`` (Algorithm 2 of
arXiv 2203.15031 written out literally in fp64) plus the penalty-level helpers of §2.2
written with scipy's normal quantile as the library primitive.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module.  The product package
``paper_2203_15031_b200`` never imports it; the two share no code.

Citations are PAPER.md lines (``P:<line>``).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spmesl_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK = 0
WARN_NOT_CONVERGED = 1
ERR_ARG = -1
ERR_CONSTANT_COLUMN = -2
ERR_NONFINITE = -3


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, -O2, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        vp = ctypes.c_void_p
        L.oracle_soft_threshold.restype = ctypes.c_double
        L.oracle_soft_threshold.argtypes = [ctypes.c_double, ctypes.c_double]
        L.oracle_standardize.argtypes = [vp, i64, i64, vp, vp, vp, vp]
        L.oracle_scaled_lasso.argtypes = [vp, i64, i64, vp, ctypes.c_double, ctypes.c_double, i32,
                                          i32, ctypes.c_double, vp, vp, vp, vp, vp, vp, vp, vp]
        L.oracle_lasso_cd.argtypes = [vp, i64, i64, vp, ctypes.c_double, ctypes.c_double, i32, vp,
                                      vp]
        L.oracle_spmesl_columns.argtypes = [vp, i64, i64, vp, i64, ctypes.c_double,
                                            ctypes.c_double, i32, i32, ctypes.c_double, i32, vp,
                                            vp, vp, vp, vp, vp]
        L.oracle_assemble.argtypes = [vp, vp, vp, i64, vp]
        L.oracle_symmetrize.argtypes = [vp, i64]
        L.oracle_spmesl_fit.argtypes = [vp, i64, i64, ctypes.c_double, ctypes.c_double, i32, i32,
                                        ctypes.c_double, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp,
                                        vp]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_joint_columns.argtypes = [vp, i64, i64, vp, i64, ctypes.c_double, ctypes.c_double,
                                           i32, i32, ctypes.c_double, vp, vp, vp, vp, vp]
        L.oracle_spmesl_fit_joint.argtypes = [vp, i64, i64, ctypes.c_double, ctypes.c_double, i32,
                                              i32, ctypes.c_double, i32, vp, vp, vp, vp, vp, vp, vp]
        del dp
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _colmajor(X) -> np.ndarray:
    return np.asfortranarray(np.asarray(X, dtype=np.float64))


class OracleError(RuntimeError):
    def __init__(self, code, bad_col=None):
        super().__init__(f"oracle error {code} (column {bad_col})")
        self.code = code
        self.bad_col = bad_col


def soft_threshold(a: float, lam: float) -> float:
    """P:595 Soft_lambda(a) = sign(a)(|a| - lambda)_+."""
    return lib().oracle_soft_threshold(float(a), float(lam))


def standardize(X):
    """P:305-307. Returns (Xs, mu, s) with Xs column-major."""
    X = _colmajor(X)
    n, p = X.shape
    Xs = np.zeros((n, p), order="F")
    mu = np.zeros(p)
    s = np.zeros(p)
    bad = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_standardize(_p(X), n, p, _p(Xs), _p(mu), _p(s), _p(bad))
    if rc:
        raise OracleError(rc, int(bad[0]))
    return Xs, mu, s


@dataclass
class ScaledLassoResult:
    beta: np.ndarray
    sigma: float
    outer: int
    sweeps: int
    converged: bool
    inner_capped: bool
    sigma_trace: np.ndarray
    margin: np.ndarray
    resid: np.ndarray


def scaled_lasso(X, y, lambda0, delta=1e-4, max_outer=100, max_inner=10000, sigma_floor=1e-8):
    """Algorithm 1 on response y with design X (no standardization applied)."""
    X = _colmajor(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, q = X.shape
    beta = np.zeros(q)
    sig = np.zeros(1)
    outer = np.zeros(1, np.int32)
    sweeps = np.zeros(1, np.int32)
    flags = np.zeros(1, np.int32)
    trace = np.zeros(max_outer + 1)
    margin = np.zeros(q)
    resid = np.zeros(n)
    rc = lib().oracle_scaled_lasso(_p(X), n, q, _p(y), lambda0, delta, max_outer, max_inner,
                                   sigma_floor, _p(beta), _p(sig), _p(outer), _p(sweeps),
                                   _p(flags), _p(trace), _p(margin), _p(resid))
    if rc < 0:
        raise OracleError(rc)
    return ScaledLassoResult(beta, float(sig[0]), int(outer[0]), int(sweeps[0]),
                             bool(flags[0] & 1), bool(flags[0] & 2), trace[: outer[0] + 1],
                             margin, resid)


def lasso_cd(X, y, lam, delta=1e-12, max_inner=100000, beta0=None):
    """Inner lasso of Alg. 1 (Eq. lasso) at a fixed lambda, warm-started at beta0."""
    X = _colmajor(X)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n, q = X.shape
    beta = np.zeros(q) if beta0 is None else np.array(beta0, dtype=np.float64)
    sw = np.zeros(1, np.int32)
    rc = lib().oracle_lasso_cd(_p(X), n, q, _p(y), lam, delta, max_inner, _p(beta), _p(sw))
    if rc < 0:
        raise OracleError(rc)
    return beta, int(sw[0])


@dataclass
class ColumnsResult:
    B: np.ndarray        # p x ncols (column c = beta_{-cols[c]})
    sigma: np.ndarray    # standardized-scale sigma
    outer: np.ndarray
    sweeps: np.ndarray
    converged: np.ndarray
    margin: np.ndarray


def spmesl_columns(Xs, cols, lambda0, delta=1e-4, max_outer=100, max_inner=10000,
                   sigma_floor=1e-8, nthreads=0, want_margin=True):
    """Algorithm 2 first loop for a subset of columns of standardized Xs."""
    Xs = _colmajor(Xs)
    n, p = Xs.shape
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    m = len(cols)
    B = np.zeros((p, m), order="F")
    sig = np.zeros(m)
    outer = np.zeros(m, np.int32)
    sweeps = np.zeros(m, np.int32)
    conv = np.zeros(m, np.uint8)
    margin = np.zeros((p, m), order="F") if want_margin else None
    rc = lib().oracle_spmesl_columns(_p(Xs), n, p, _p(cols), m, lambda0, delta, max_outer,
                                     max_inner, sigma_floor, nthreads, _p(B), _p(sig), _p(outer),
                                     _p(sweeps), _p(conv), _p(margin))
    if rc < 0:
        raise OracleError(rc)
    return ColumnsResult(B, sig, outer, sweeps, conv.astype(bool), margin)


def assemble(B, sigma, s=None):
    """Alg. 2 P:698-708 + Prop. 1."""
    B = _colmajor(B)
    p = B.shape[0]
    T = np.zeros((p, p), order="F")
    sigma = np.ascontiguousarray(sigma, dtype=np.float64)
    s = None if s is None else np.ascontiguousarray(s, dtype=np.float64)
    lib().oracle_assemble(_p(B), _p(sigma), _p(s), p, _p(T))
    return T


def symmetrize(T):
    """Alg. 2 P:709-719 (Eq. symm)."""
    T = np.array(T, dtype=np.float64, order="F", copy=True)
    lib().oracle_symmetrize(_p(T), T.shape[0])
    return T


@dataclass
class FitResult:
    code: int
    Theta: np.ndarray
    sigma: np.ndarray
    outer: np.ndarray
    sweeps: np.ndarray
    converged: np.ndarray
    B: np.ndarray
    Theta1: np.ndarray
    margin: np.ndarray


def spmesl_fit(X, lambda0, delta=1e-4, max_outer=100, max_inner=10000, sigma_floor=1e-8,
               standardize=True, nthreads=0, want_margin=True):
    """The whole Algorithm 2 pipeline with Prop. 1 rescaling."""
    X = _colmajor(X)
    n, p = X.shape
    T = np.zeros((p, p), order="F")
    T1 = np.zeros((p, p), order="F")
    B = np.zeros((p, p), order="F")
    margin = np.zeros((p, p), order="F") if want_margin else None
    sig = np.zeros(p)
    outer = np.zeros(p, np.int32)
    sweeps = np.zeros(p, np.int32)
    conv = np.zeros(p, np.uint8)
    bad = np.zeros(1, np.int64)
    rc = lib().oracle_spmesl_fit(_p(X), n, p, lambda0, delta, max_outer, max_inner, sigma_floor,
                                 1 if standardize else 0, nthreads, _p(T), _p(sig), _p(outer),
                                 _p(sweeps), _p(conv), _p(B), _p(T1), _p(margin), _p(bad))
    if rc < 0:
        raise OracleError(rc, int(bad[0]))
    return FitResult(rc, T, sig, outer, sweeps, conv.astype(bool), B, T1, margin)


def joint_columns(Xs, cols, lambda0, delta=1e-4, max_outer=100, max_inner=10000,
                  sigma_floor=1e-8):
    """Algorithm 3 (joint stop) for a subset of columns of standardized Xs."""
    Xs = _colmajor(Xs)
    n, p = Xs.shape
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    m = len(cols)
    B = np.zeros((p, m), order="F")
    sig = np.zeros(m)
    outer = np.zeros(m, np.int32)
    sweeps = np.zeros(m, np.int32)
    conv = np.zeros(m, np.uint8)
    rc = lib().oracle_joint_columns(_p(Xs), n, p, _p(cols), m, lambda0, delta, max_outer,
                                    max_inner, sigma_floor, _p(B), _p(sig), _p(outer),
                                    _p(sweeps), _p(conv))
    if rc < 0:
        raise OracleError(rc)
    return ColumnsResult(B, sig, outer, sweeps, conv.astype(bool), None)


def spmesl_fit_joint(X, lambda0, delta=1e-4, max_outer=100, max_inner=10000, sigma_floor=1e-8,
                     standardize=True):
    """Algorithm 3 end to end with Prop. 1 rescaling and Eq. (symm)."""
    X = _colmajor(X)
    n, p = X.shape
    T = np.zeros((p, p), order="F")
    B = np.zeros((p, p), order="F")
    sig = np.zeros(p)
    outer = np.zeros(p, np.int32)
    sweeps = np.zeros(p, np.int32)
    conv = np.zeros(p, np.uint8)
    bad = np.zeros(1, np.int64)
    rc = lib().oracle_spmesl_fit_joint(_p(X), n, p, lambda0, delta, max_outer, max_inner,
                                       sigma_floor, 1 if standardize else 0, _p(T), _p(sig),
                                       _p(outer), _p(sweeps), _p(conv), _p(B), _p(bad))
    if rc < 0:
        raise OracleError(rc, int(bad[0]))
    return FitResult(rc, T, sig, outer, sweeps, conv.astype(bool), B, None, None)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ----------------------------------------------------------------------------------------
# Penalty levels, §2.2.  scipy's normal quantile is the library primitive.
# ----------------------------------------------------------------------------------------

def lambda_univ(n: int, p: int) -> float:
    """Universal level as used for SPMESL, sqrt(2 log(p-1)/n) (reading g13)."""
    return math.sqrt(2.0 * math.log(p - 1) / n)


def lambda_ub(n: int, p: int, A: float = 1.0) -> float:
    """Union-bound level A sqrt(4 log p / n)."""
    return A * math.sqrt(4.0 * math.log(p) / n)


def _L(n: float, t: float) -> float:
    """L_n(t) = n^{-1/2} Phi^{-1}(1 - t)."""
    from scipy.special import ndtri
    return float(ndtri(1.0 - t)) / math.sqrt(n)


def solve_k(p: int, tol: float = 1e-12, max_iter: int = 400) -> float:
    """Real solution of k = L_1^4(k/p) + 2 L_1^2(k/p) by bisection (reading
    g12: the text form, not the caption's sign)."""
    def f(k):
        L1 = _L(1.0, k / p)
        return k - L1 ** 4 - 2.0 * L1 ** 2
    lo, hi = 1e-9, p / 2.0
    flo, fhi = f(lo), f(hi)
    if flo * fhi > 0:
        raise ValueError("no bracket")
    for _ in range(max_iter):
        mid = 0.5 * (lo + hi)
        fm = f(mid)
        if (fm < 0) == (flo < 0):
            lo, flo = mid, fm
        else:
            hi = mid
        if hi - lo < tol * max(1.0, abs(mid)):
            break
    return 0.5 * (lo + hi)


def lambda_pb(n: int, p: int, A: float = math.sqrt(2.0)) -> float:
    """Probabilistic-bound level A L_n(k/p)."""
    return A * _L(n, solve_k(p) / p)
