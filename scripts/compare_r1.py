"""Development check: the current library against the round-1 library (scripts/_r1/, built from
commit e5ba4ad; not committed) on the same inputs, bit for bit.  Both are loaded into one
process with ctypes (separate workspaces)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2203_15031_b200 as S
from paper_2203_15031_b200 import _lib
from synth import generators as G

old = ctypes.CDLL(sys.argv[1] if len(sys.argv) > 1 else "scripts/_r1/libspmesl.so")
vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
old.spmesl_fit_device.argtypes = [vp, i64, i64, dbl, dbl, i32, ctypes.POINTER(_lib.Options), vp,
                                  vp, vp, vp, vp, vp, vp]
old.spmesl_default_options.argtypes = [ctypes.POINTER(_lib.Options)]


def run_old(Xd, lam, solver):
    n, p = Xd.shape
    o = _lib.Options()
    old.spmesl_default_options(ctypes.byref(o))
    o.solver = solver
    o.eager = 1
    th = torch.empty((p, p), dtype=torch.float64, device="cuda")
    sg = torch.empty(p, dtype=torch.float64, device="cuda")
    it = torch.empty(p, dtype=torch.int32, device="cuda")
    sw = torch.empty(p, dtype=torch.int32, device="cuda")
    cv = torch.empty(p, dtype=torch.uint8, device="cuda")
    rc = old.spmesl_fit_device(ctypes.c_void_p(Xd.data_ptr()), n, p, lam, 1e-4, 100,
                               ctypes.byref(o), ctypes.c_void_p(th.data_ptr()),
                               ctypes.c_void_p(sg.data_ptr()), ctypes.c_void_p(it.data_ptr()),
                               ctypes.c_void_p(sw.data_ptr()), ctypes.c_void_p(cv.data_ptr()),
                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), None)
    if rc < 0:
        return None
    return th, sg, it, sw


cases = [(4, dict(family="hub"), "ub"), (4, dict(family="band3"), "ub"), (4, dict(family="hub"), "ub"), (5, {}, "univ"),
         (5, {}, "ub"), (4, dict(p=777, n=203), "univ"), (2, {}, "univ"), (3, {}, "univ")]
for cfg, over, rule in cases:
    X, _, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = S.lambda_ub(n, p) if rule == "ub" else S.lambda_univ(n, p)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()   # n x p, column-major
    for solver in (3, 1):
        if solver == 1 and p > 6000:
            continue
        a = run_old(Xd, lam, solver)
        if a is None:
            print(cfg, over, rule, "solver", solver, "round-1 library declined", flush=True)
            continue
        b = S.fit_device(Xd, lam, eager=True, solver={3: "gram16", 1: "residual"}[solver])
        same = [torch.equal(a[0], b.Theta.t().contiguous().t() if False else b.Theta.t()),
                torch.equal(a[1], b.sigma), torch.equal(a[2], b.iters), torch.equal(a[3], b.sweeps)]
        dth = (a[0] - b.Theta.t()).abs().max().item()
        print(cfg, over, rule, "solver", solver, "identical (Theta, sigma, iters, sweeps):", same,
              "max |dTheta|", dth, flush=True)
