"""Development check: two builds (paths) bit for bit, eager fits: the exact-Gram-column path of the
certified screening (config 5 at lambda_ub: 65 candidates; lower penalties: several 96-column
vector groups) and the multi-sweep workloads (config 4 band(3) / hub, odd p)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_15031_b200 import _lib
from synth import generators as G

libs = [ctypes.CDLL(a) for a in sys.argv[1:3]]
vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
for L in libs:
    L.spmesl_fit_device.argtypes = [vp, i64, i64, dbl, dbl, i32, ctypes.POINTER(_lib.Options), vp,
                                    vp, vp, vp, vp, vp, ctypes.POINTER(_lib.Stats)]
    L.spmesl_default_options.argtypes = [ctypes.POINTER(_lib.Options)]
    L.spmesl_lambda_ub.restype = dbl
    L.spmesl_lambda_ub.argtypes = [i64, i64, dbl]


def run(L, Xd, lam):
    n, p = Xd.shape
    o = _lib.Options()
    L.spmesl_default_options(ctypes.byref(o))
    o.eager = 1
    st = _lib.Stats()
    th = torch.empty((p, p), dtype=torch.float64, device="cuda")
    sg = torch.empty(p, dtype=torch.float64, device="cuda")
    it = torch.empty(p, dtype=torch.int32, device="cuda")
    sw = torch.empty(p, dtype=torch.int32, device="cuda")
    cv = torch.empty(p, dtype=torch.uint8, device="cuda")
    rc = L.spmesl_fit_device(ctypes.c_void_p(Xd.data_ptr()), n, p, lam, 1e-4, 100, ctypes.byref(o),
                             ctypes.c_void_p(th.data_ptr()), ctypes.c_void_p(sg.data_ptr()),
                             ctypes.c_void_p(it.data_ptr()), ctypes.c_void_p(sw.data_ptr()),
                             ctypes.c_void_p(cv.data_ptr()),
                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(st))
    assert rc >= 0, rc
    return (th, sg, it, sw), st


bad = 0
CASES = ((5, {}, 1.0), (5, {}, 0.9), (5, {}, 0.8), (3, {}, 1.0), (3, {}, 0.85), (5, dict(p=3001), 0.8),
         (4, dict(family="band3"), 1.0), (4, dict(family="hub"), 1.0),
         (4, dict(family="hub", seed=3207), 1.0), (4, dict(family="band3"), 0.7),
         (4, dict(family="band3", p=3001), 1.0), (4, dict(family="hub", p=1999), 0.8))
for cfg, over, scale in CASES:
    X, _, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = libs[0].spmesl_lambda_ub(n, p, 1.0) * scale
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    a, sa = run(libs[0], Xd, lam)
    b, sb = run(libs[1], Xd, lam)
    same = [torch.equal(x, y) for x, y in zip(a, b)]
    bad += not all(same)
    print(f"config {cfg} {over} lambda_ub x {scale}: candidates {sa.screen_candidates}/{sb.screen_candidates}"
          f" fallback {sa.gram_fallback}/{sb.gram_fallback} identical {same}", flush=True)
print("ALL IDENTICAL" if bad == 0 else f"{bad} DIFFER")
