"""B200-native SPMESL hot path (arXiv 2203.15031): Python binding of libspmesl.so.

Every step of the path runs in the CUDA kernels behind the C ABI (include/spmesl.h); this
module only marshals arguments (numpy host arrays or torch CUDA tensors) and names the
results.  There is no CPU fallback: without the built library every call raises.

Public API (same names as the C ABI):
    fit(X, lambda0, tol, max_iter, ...)          host arrays in/out   -> FitResult
    fit_device(X, lambda0, tol, max_iter, ...)   torch CUDA tensors   -> FitResult (tensors)
    fit_columns_device / assemble_device         multi-GPU building blocks (see distributed.py)
    lambda_univ / lambda_ub / lambda_pb / solve_k  penalty levels
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _lib
from ._lib import SpmeslError, Stats, default_options, load  # noqa: F401

__all__ = ["fit", "fit_device", "fit_columns_device", "assemble_device", "gram_tile_count",
           "gram_screen_device", "fit_columns_gram_device", "gram_supported", "fit_path_device",
           "lambda_univ",
           "lambda_ub", "lambda_pb", "solve_k", "FitResult", "SpmeslError", "load",
           "release_workspace", "version"]


@dataclass
class FitResult:
    code: int
    Theta: Any            # p x p (numpy Fortran array or torch tensor view, column-major)
    sigma: Any
    iters: Any
    sweeps: Any
    converged: Any
    stats: dict = field(default_factory=dict)


def _vp(a) -> ctypes.c_void_p:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


MODES = {"per_column": 0, "joint": 1}
SOLVERS = {"auto": 0, "residual": 1, "gram": 2, "gram16": 3}
EXCHANGES = {"auto": 0, "nccl": 1, "p2p": 2}


_OPTS_CACHE = {}


def _opts(**kw) -> _lib.Options:
    """Options for these keyword arguments (cached: the device path is called per fit)."""
    key = tuple(sorted((k, tuple(v) if isinstance(v, list) else v) for k, v in kw.items()))
    o = _OPTS_CACHE.get(key)
    if o is None:
        o = _OPTS_CACHE[key] = _make_opts(**kw)
    return o


def _make_opts(max_inner=10000, standardize=True, symmetrize=True, sigma_floor=1e-8, tile_cols=0,
               device=-1, tail_after=1, mode="per_column", solver="auto",
               eager=False, num_devices=0, device_ids=None, exchange="auto") -> _lib.Options:
    """mode: "per_column" (Algorithm 1 stop per column) or "joint" (Algorithm 3).
    solver: "auto", "residual" (CD on X~) or "gram" (covariance updates on X~^T X~ / n).
    num_devices / device_ids (host entry points): fit on several devices; exchange: "auto",
    "nccl" (collectives) or "p2p" (peer reads; device ids may repeat) — DESIGN.md §8."""
    o = default_options(max_inner=int(max_inner), standardize=int(bool(standardize)),
                        symmetrize=int(bool(symmetrize)), sigma_floor=float(sigma_floor),
                        tile_cols=int(tile_cols), device=int(device),
                        tail_after=int(tail_after),
                        mode=MODES[mode] if isinstance(mode, str) else int(mode),
                        solver=SOLVERS[solver] if isinstance(solver, str) else int(solver),
                        eager=int(bool(eager)), num_devices=int(num_devices),
                        exchange=EXCHANGES[exchange] if isinstance(exchange, str) else int(exchange))
    if device_ids is not None:
        ids = (ctypes.c_int32 * len(device_ids))(*[int(d) for d in device_ids])
        o._ids = ids   # (kept alive with the options)
        o.device_ids = ctypes.cast(ids, ctypes.POINTER(ctypes.c_int32))
    return o


def fit(X, lambda0: float, tol: float = 1e-4, max_iter: int = 100, *, out_theta=None,
        **options) -> FitResult:
    """spmesl_fit_ex on host memory.  X: n x p (any numpy layout; copied to column-major)."""
    X = np.asfortranarray(np.asarray(X, dtype=np.float64))
    n, p = X.shape
    Theta = out_theta if out_theta is not None else np.empty((p, p), order="F")
    sigma = np.empty(p)
    iters = np.empty(p, np.int32)
    sweeps = np.empty(p, np.int32)
    conv = np.empty(p, np.uint8)
    st = Stats()
    o = _opts(**options)
    rc = load().spmesl_fit_ex(_vp(X), n, p, float(lambda0), float(tol), int(max_iter),
                              ctypes.byref(o), _vp(Theta), _vp(sigma), _vp(iters), _vp(sweeps),
                              _vp(conv), ctypes.byref(st))
    _lib.check(rc, st)
    return FitResult(rc, Theta, sigma, iters, sweeps, conv.astype(bool), st.asdict())


def fit_sparse(X, lambda0: float, tol: float = 1e-4, max_iter: int = 100, *, cap=None,
               **options) -> dict:
    """spmesl_fit_sparse on host memory: Theta as CSC numpy arrays (col_ptr int64 [p+1], rows
    int32, vals float64; symmetric, so also CSR) without the dense p x p array, plus sigma /
    iters / sweeps / converged.  cap: entry capacity (default p + 16 p; retried once with the
    count needed)."""
    X = np.asfortranarray(np.asarray(X, dtype=np.float64))
    n, p = X.shape
    cap = int(cap) if cap is not None else p + 16 * p
    col_ptr = np.empty(p + 1, np.int64)
    sigma = np.empty(p)
    iters = np.empty(p, np.int32)
    sweeps = np.empty(p, np.int32)
    conv = np.empty(p, np.uint8)
    o = _opts(**options)
    for attempt in range(2):
        rows = np.empty(max(cap, 1), np.int32)
        vals = np.empty(max(cap, 1), np.float64)
        nnz = ctypes.c_int64(0)
        st = Stats()
        rc = load().spmesl_fit_sparse(_vp(X), n, p, float(lambda0), float(tol), int(max_iter),
                                      ctypes.byref(o), _vp(col_ptr), _vp(rows), _vp(vals), cap,
                                      ctypes.byref(nnz), _vp(sigma), _vp(iters), _vp(sweeps),
                                      _vp(conv), ctypes.byref(st))
        if rc == _lib.ERR_ARG and nnz.value > cap:
            cap = int(nnz.value)
            continue
        _lib.check(rc, st)
        break
    k = nnz.value
    return dict(code=rc, col_ptr=col_ptr, rows=rows[:k], vals=vals[:k], sigma=sigma, iters=iters,
                sweeps=sweeps, converged=conv.astype(bool), stats=st.asdict())


def as_colmajor(X):
    """torch (n, p) tensor -> same values with column-major (Fortran) strides."""
    if X.dim() != 2:
        raise ValueError("X must be 2-D")
    if X.stride(0) == 1 and X.stride(1) == X.shape[0]:
        return X
    return X.t().contiguous().t()


_OUT_KEYS = ("theta", "sigma", "iters", "sweeps", "conv")
_STATS_NAMES = tuple(k for k, _ in Stats._fields_)
_FAST = {}   # repeated device fits on the same buffers: the marshalled call, reused


def _fast_key(X, lambda0, tol, max_iter, s, out, options):
    try:
        key = (X.data_ptr(), X.shape, X.stride(), X.dtype, X.device, float(lambda0), float(tol),
               int(max_iter), s.cuda_stream, tuple(out[k].data_ptr() for k in _OUT_KEYS),
               tuple(out[k].dtype for k in _OUT_KEYS), out["theta"].shape,
               tuple(sorted(options.items())))
        hash(key)
        return key
    except (TypeError, KeyError, AttributeError):
        return None


def _result(rc, out, st):
    import torch
    # the buffer holds Theta column-major: element (j, k) at j + k p -> view as its transpose
    # (uint8 0/1 reinterpreted as bool: a view, no conversion kernel)
    return FitResult(rc, out["theta"].t(), out["sigma"], out["iters"], out["sweeps"],
                     out["conv"].view(torch.bool), {k: getattr(st, k) for k in _STATS_NAMES})


def fit_device(X, lambda0: float, tol: float = 1e-4, max_iter: int = 100, *, stream=None,
               out=None, **options) -> FitResult:
    """spmesl_fit_device on torch CUDA tensors.  X: (n, p) float64 on the current device.
    A repeat of an earlier call with the same tensors (`out` given), stream and options — a
    fit loop on reused buffers — reuses the marshalled ctypes arguments (one native call)."""
    import torch
    key = None
    if out is not None and getattr(X, "is_cuda", False):
        s = stream if stream is not None else torch.cuda.current_stream(X.device)
        key = _fast_key(X, lambda0, tol, max_iter, s, out, options)
        ent = _FAST.get(key) if key is not None else None
        if ent is not None:
            fn, args, st, dev = ent
            if torch.cuda.current_device() != dev:
                with torch.cuda.device(dev):
                    rc = fn(*args)
            else:
                rc = fn(*args)
            _lib.check(rc, st)
            return _result(rc, out, st)
    if not X.is_cuda or X.dtype != torch.float64:
        raise TypeError("X must be a float64 CUDA tensor")
    Xc = as_colmajor(X)
    n, p = Xc.shape
    dev = Xc.device
    if out is None:
        out = dict(
            theta=torch.empty((p, p), dtype=torch.float64, device=dev),
            sigma=torch.empty(p, dtype=torch.float64, device=dev),
            iters=torch.empty(p, dtype=torch.int32, device=dev),
            sweeps=torch.empty(p, dtype=torch.int32, device=dev),
            conv=torch.empty(p, dtype=torch.uint8, device=dev))
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    st = Stats()
    o = _opts(**options)
    fn = load().spmesl_fit_device
    args = (_vp(Xc), n, p, float(lambda0), float(tol), int(max_iter), ctypes.byref(o),
            _vp(out["theta"]), _vp(out["sigma"]), _vp(out["iters"]), _vp(out["sweeps"]),
            _vp(out["conv"]), ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
    with torch.cuda.device(dev):
        rc = fn(*args)
    _lib.check(rc, st)
    # (cached only when X was used as given: the arguments hold raw pointers, valid for as
    # long as tensors with these addresses, shapes and dtypes exist — which the key checks)
    if key is not None and Xc is X and len(_FAST) < 64:
        _FAST[key] = (fn, args, st, dev.index)
    return _result(rc, out, st)


def fit_sparse_device(X, lambda0: float, tol: float = 1e-4, max_iter: int = 100, *,
                      stream=None, cap=None, out=None, **options) -> dict:
    """spmesl_fit_sparse_device: Theta in CSC form (col_ptr int64 [p+1], rows int32, vals
    float64; symmetric, so also CSR) without the dense p x p array, plus sigma / iters / sweeps
    / converged.  cap: entry capacity (default p + 64 p; grown and retried once if short).
    out (optional): preallocated col_ptr / rows / vals / sigma / iters / sweeps / conv tensors
    (reused buffers let repeated fits replay their CUDA graph)."""
    import torch
    if not X.is_cuda or X.dtype != torch.float64:
        raise TypeError("X must be a float64 CUDA tensor")
    X = as_colmajor(X)
    n, p = X.shape
    dev = X.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    o = _opts(**options)
    if out is not None:
        cap = out["rows"].numel()
    cap = int(cap) if cap is not None else p + 64 * p
    out = out or {}
    col_ptr = out.get("col_ptr", None)
    col_ptr = col_ptr if col_ptr is not None else torch.empty(p + 1, dtype=torch.int64, device=dev)
    sigma = out["sigma"] if "sigma" in out else torch.empty(p, dtype=torch.float64, device=dev)
    iters = out["iters"] if "iters" in out else torch.empty(p, dtype=torch.int32, device=dev)
    sweeps = out["sweeps"] if "sweeps" in out else torch.empty(p, dtype=torch.int32, device=dev)
    conv = out["conv"] if "conv" in out else torch.empty(p, dtype=torch.uint8, device=dev)
    for attempt in range(2):
        if attempt == 0 and "rows" in out and "vals" in out:
            rows, vals = out["rows"], out["vals"]
        else:
            rows = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
            vals = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
        nnz = ctypes.c_int64(0)
        st = Stats()
        with torch.cuda.device(dev):
            rc = load().spmesl_fit_sparse_device(
                _vp(X), n, p, float(lambda0), float(tol), int(max_iter), ctypes.byref(o),
                _vp(col_ptr), _vp(rows), _vp(vals), cap, ctypes.byref(nnz), _vp(sigma),
                _vp(iters), _vp(sweeps), _vp(conv), ctypes.c_void_p(s.cuda_stream),
                ctypes.byref(st))
        if rc == _lib.ERR_ARG and nnz.value > cap:
            cap = int(nnz.value)
            continue
        _lib.check(rc, st)
        break
    k = nnz.value
    return dict(code=rc, col_ptr=col_ptr, rows=rows[:k], vals=vals[:k], sigma=sigma,
                iters=iters, sweeps=sweeps, converged=conv.view(torch.bool), stats=st.asdict())


def sparse_to_dense(col_ptr, rows, vals, p: int):
    """Dense p x p (column-major view) of a CSC matrix from fit_sparse_device (testing aid)."""
    import torch
    T = torch.zeros((p, p), dtype=torch.float64, device=vals.device)   # T[k, j] = Theta[j, k]
    cols = torch.repeat_interleave(torch.arange(p, device=vals.device),
                                   (col_ptr[1:] - col_ptr[:-1]))
    T[cols, rows.long()] = vals
    return T.t()


def gram_supported(n: int, p: int) -> bool:
    """spmesl_gram_supported: the Gram solver's sweep state fits on chip for (n, p)."""
    return bool(load().spmesl_gram_supported(int(n), int(p)))


def gram_tile_count(p: int, solver=None) -> int:
    """Tiles of the screening pass: spmesl_gram_tile_count (the 128 x 128 upper-triangle tiles
    of S = X~^T X~ / n, solver "gram") or, with `solver`, spmesl_screen_tile_count for that
    solver ("auto"/"gram16": the 128 x 256 tiles of the certified f16 screening)."""
    if solver is None:
        return int(load().spmesl_gram_tile_count(int(p)))
    o = _opts(solver=solver)
    return int(load().spmesl_screen_tile_count(int(p), ctypes.byref(o)))


def gram_screen_device(X, lambda0: float, tile_begin: int, tile_end: int, hit, *, stream=None,
                       **options) -> dict:
    """spmesl_gram_screen_device: OR the screening flags of tiles [tile_begin, tile_end) into
    `hit` (uint8 CUDA tensor [p], zero-filled by the caller).  solver "gram": exact hits of the
    FP64 Gram tiles; "auto"/"gram16" (default): candidates of the certified f16 screening
    (a superset of the hits; fit_columns_gram_device with the same solver decides them)."""
    import torch
    X = as_colmajor(X)
    n, p = X.shape
    if hit.dtype != torch.uint8 or hit.numel() != p or not hit.is_cuda:
        raise TypeError("hit must be a uint8 CUDA tensor of length p")
    s = stream if stream is not None else torch.cuda.current_stream(X.device)
    st = Stats()
    o = _opts(**options)
    with torch.cuda.device(X.device):
        rc = load().spmesl_gram_screen_device(_vp(X), n, p, float(lambda0), int(tile_begin),
                                              int(tile_end), ctypes.byref(o), _vp(hit),
                                              ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
    _lib.check(rc, st)
    return st.asdict()


def _columns_outputs(X, m, p, cap):
    import torch
    dev = X.device
    n = X.shape[0]
    if cap is None:
        cap = m * min(p, ((n + 31) // 32) * 32 + 64)
    return dict(counts=torch.empty(m, dtype=torch.int32, device=dev),
                rows=torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
                vals=torch.empty(max(cap, 1), dtype=torch.float64, device=dev),
                sigma_std=torch.empty(m, dtype=torch.float64, device=dev),
                scale=torch.empty(p, dtype=torch.float64, device=dev),
                iters=torch.empty(m, dtype=torch.int32, device=dev),
                sweeps=torch.empty(m, dtype=torch.int32, device=dev),
                conv=torch.empty(m, dtype=torch.uint8, device=dev)), cap


def screen_accumulators_device(X, *, stream=None, **options):
    """spmesl_screen_accumulators_device (TEST-ONLY): the raw f32 accumulators n R_hat of the
    certified f16 screening (tcgen05) for every pair its tiles cover, as a (p_pad, p_pad) float32
    tensor A with A[c, j] = acc_jc (NaN where no tile wrote), plus the candidate flags at
    lambda0 = 0, and the f16 operands as a (p_pad, n64) float16 tensor (variable, sample; the
    tile layout undone).  X: (n, p) float64 CUDA tensor."""
    import torch
    X = as_colmajor(X)
    n, p = X.shape
    ld = -(-p // 256) * 256
    n_pad = -(-n // 32) * 32
    nc = -(-n_pad // 64)
    acc = torch.full((ld, ld), float("nan"), dtype=torch.float32, device=X.device)
    cand = torch.zeros(p, dtype=torch.uint8, device=X.device)
    y16 = torch.empty((ld // 128, nc, 128, 8, 8), dtype=torch.float16, device=X.device)
    s = stream if stream is not None else torch.cuda.current_stream(X.device)
    o = _opts(**options)
    with torch.cuda.device(X.device):
        rc = load().spmesl_screen_accumulators_device(_vp(X), n, p, ctypes.byref(o), _vp(acc), ld,
                                                      _vp(cand), _vp(y16),
                                                      ctypes.c_void_p(s.cuda_stream))
    _lib.check(rc)
    # undo the 16-byte-group swizzle (group g of row r sits at g ^ (r & 7)), then the tiling
    r = torch.arange(128, device=X.device)
    g = torch.arange(8, device=X.device)
    src = (g[None, :] ^ (r[:, None] & 7))                       # [128, 8]
    y = torch.gather(y16, 3, src[None, None, :, :, None].expand(y16.shape))
    Y = y.permute(0, 2, 1, 3, 4).reshape(ld, nc * 64)
    return acc, cand, Y


def fit_columns_gram_device(X, col_begin: int, col_end: int, lambda0: float, hit,
                            tol: float = 1e-4, max_iter: int = 100, *, stream=None, cap=None,
                            **options):
    """spmesl_fit_columns_gram_device: Gram-solver CSC coefficients of columns
    [col_begin, col_end) given the global screening flags `hit` (uint8 CUDA tensor [p]) of
    gram_screen_device with the same solver."""
    import torch
    X = as_colmajor(X)
    n, p = X.shape
    m = col_end - col_begin
    b, cap = _columns_outputs(X, m, p, cap)
    nnz = ctypes.c_int64(0)
    s = stream if stream is not None else torch.cuda.current_stream(X.device)
    st = Stats()
    o = _opts(**options)
    with torch.cuda.device(X.device):
        rc = load().spmesl_fit_columns_gram_device(
            _vp(X), n, p, col_begin, col_end, float(lambda0), float(tol), int(max_iter),
            ctypes.byref(o), _vp(hit), _vp(b["counts"]), _vp(b["rows"]), _vp(b["vals"]), cap,
            ctypes.byref(nnz), _vp(b["sigma_std"]), _vp(b["scale"]), _vp(b["iters"]),
            _vp(b["sweeps"]), _vp(b["conv"]), ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
    _lib.check(rc, st)
    k = nnz.value
    return dict(code=rc, counts=b["counts"], rows=b["rows"][:k], vals=b["vals"][:k],
                sigma_std=b["sigma_std"], scale=b["scale"], iters=b["iters"],
                sweeps=b["sweeps"], converged=b["conv"].bool(), stats=st.asdict())


def fit_path_device(X, lambdas, tol: float = 1e-4, max_iter: int = 100, *, stream=None,
                    **options) -> list:
    """spmesl_fit_path_device: one fit per penalty level in `lambdas` (1..8 levels) sharing
    X~, S = X~^T X~ / n and the screening pass.  Returns a list of FitResult (device tensors)."""
    import torch
    if not X.is_cuda or X.dtype != torch.float64:
        raise TypeError("X must be a float64 CUDA tensor")
    X = as_colmajor(X)
    n, p = X.shape
    lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.float64).ravel())
    L = lam.size
    dev = X.device
    theta = torch.empty((L, p, p), dtype=torch.float64, device=dev)
    sigma = torch.empty((L, p), dtype=torch.float64, device=dev)
    iters = torch.empty((L, p), dtype=torch.int32, device=dev)
    sweeps = torch.empty((L, p), dtype=torch.int32, device=dev)
    conv = torch.empty((L, p), dtype=torch.uint8, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    st = Stats()
    o = _opts(**options)
    with torch.cuda.device(dev):
        rc = load().spmesl_fit_path_device(_vp(X), n, p, _vp(lam), L, float(tol), int(max_iter),
                                           ctypes.byref(o), _vp(theta), _vp(sigma), _vp(iters),
                                           _vp(sweeps), _vp(conv), ctypes.c_void_p(s.cuda_stream),
                                           ctypes.byref(st))
    _lib.check(rc, st)
    stats = st.asdict()
    return [FitResult(rc, theta[l].t(), sigma[l], iters[l], sweeps[l], conv[l].bool(), stats)
            for l in range(L)]


def fit_columns_device(X, col_begin: int, col_end: int, lambda0: float, tol: float = 1e-4,
                       max_iter: int = 100, *, stream=None, cap=None, **options):
    """spmesl_fit_columns_device: CSC coefficients of columns [col_begin, col_end)."""
    import torch
    X = as_colmajor(X)
    n, p = X.shape
    m = col_end - col_begin
    dev = X.device
    if cap is None:
        cap = m * min(p, ((n + 31) // 32) * 32 + 64)
    counts = torch.empty(m, dtype=torch.int32, device=dev)
    rows = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
    sigma_std = torch.empty(m, dtype=torch.float64, device=dev)
    scale = torch.empty(p, dtype=torch.float64, device=dev)
    iters = torch.empty(m, dtype=torch.int32, device=dev)
    sweeps = torch.empty(m, dtype=torch.int32, device=dev)
    conv = torch.empty(m, dtype=torch.uint8, device=dev)
    nnz = ctypes.c_int64(0)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    st = Stats()
    o = _opts(**options)
    with torch.cuda.device(dev):
        rc = load().spmesl_fit_columns_device(
            _vp(X), n, p, col_begin, col_end, float(lambda0), float(tol), int(max_iter),
            ctypes.byref(o), _vp(counts), _vp(rows), _vp(vals), cap, ctypes.byref(nnz),
            _vp(sigma_std), _vp(scale), _vp(iters), _vp(sweeps), _vp(conv),
            ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))
    _lib.check(rc, st)
    k = nnz.value
    return dict(code=rc, counts=counts, rows=rows[:k], vals=vals[:k], sigma_std=sigma_std,
                scale=scale, iters=iters, sweeps=sweeps, converged=conv.bool(),
                stats=st.asdict())


def assemble_device(p: int, col_begin: int, col_end: int, col_ptr, rows, vals, sigma_std, scale,
                    *, stream=None, out_theta=None, out_sigma=None, **options):
    """spmesl_assemble_device: columns [col_begin, col_end) of Theta from the global CSC."""
    import torch
    dev = col_ptr.device
    m = col_end - col_begin
    theta = out_theta if out_theta is not None else torch.empty((m, p), dtype=torch.float64,
                                                                device=dev)
    sig = out_sigma if out_sigma is not None else torch.empty(m, dtype=torch.float64, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    o = _opts(**options)
    with torch.cuda.device(dev):
        rc = load().spmesl_assemble_device(p, col_begin, col_end, _vp(col_ptr), _vp(rows),
                                           _vp(vals), _vp(sigma_std), _vp(scale),
                                           ctypes.byref(o), _vp(theta), _vp(sig),
                                           ctypes.c_void_p(s.cuda_stream))
    _lib.check(rc)
    return theta.t(), sig   # (p, m) column block, column-major


def lambda_univ(n: int, p: int) -> float:
    return load().spmesl_lambda_univ(n, p)


def lambda_ub(n: int, p: int, A: float = 1.0) -> float:
    return load().spmesl_lambda_ub(n, p, A)


def lambda_pb(n: int, p: int, A: float = 2 ** 0.5) -> float:
    return load().spmesl_lambda_pb(n, p, A)


def solve_k(p: int) -> float:
    return load().spmesl_solve_k(p)


def release_workspace() -> int:
    return load().spmesl_release_workspace()


def version() -> str:
    return load().spmesl_version().decode()
