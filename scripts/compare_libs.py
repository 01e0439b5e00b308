"""Development check: two builds of the library (paths) on the same inputs, bit for bit."""
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
                                    vp, vp, vp, vp, vp, vp]
    L.spmesl_default_options.argtypes = [ctypes.POINTER(_lib.Options)]
    L.spmesl_lambda_ub.restype = dbl
    L.spmesl_lambda_ub.argtypes = [i64, i64, dbl]


def run(L, Xd, lam):
    n, p = Xd.shape
    o = _lib.Options()
    L.spmesl_default_options(ctypes.byref(o))
    o.eager = 1
    th = torch.empty((p, p), dtype=torch.float64, device="cuda")
    sg = torch.empty(p, dtype=torch.float64, device="cuda")
    it = torch.empty(p, dtype=torch.int32, device="cuda")
    sw = torch.empty(p, dtype=torch.int32, device="cuda")
    cv = torch.empty(p, dtype=torch.uint8, device="cuda")
    rc = L.spmesl_fit_device(ctypes.c_void_p(Xd.data_ptr()), n, p, lam, 1e-4, 100, ctypes.byref(o),
                             ctypes.c_void_p(th.data_ptr()), ctypes.c_void_p(sg.data_ptr()),
                             ctypes.c_void_p(it.data_ptr()), ctypes.c_void_p(sw.data_ptr()),
                             ctypes.c_void_p(cv.data_ptr()),
                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), None)
    assert rc >= 0
    return th, sg, it, sw


X, _, spec = G.make_config(4, family="hub")
n, p = X.shape
lam = libs[0].spmesl_lambda_ub(n, p, 1.0)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
a = run(libs[0], Xd, lam)
b = run(libs[1], Xd, lam)
d = (a[0] - b[0]).abs()
idx = torch.nonzero(d).cpu().numpy()
print("identical:", [torch.equal(x, y) for x, y in zip(a, b)], "differing entries", len(idx))
for k, j in idx[:10]:
    print(" column", k, "row", j, a[0][k, j].item(), b[0][k, j].item(), "sweeps", a[3][k].item())
