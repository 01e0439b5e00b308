"""Dev: host-API (spmesl_fit_ex) time at config 5 with pinned host buffers."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
X, _, spec = G.make_config(5)
n, p = X.shape
lam = S.lambda_ub(n, p)
Xh = torch.from_numpy(np.ascontiguousarray(X.T)).pin_memory()
Th = torch.empty((p, p), dtype=torch.float64).pin_memory()
sh = torch.empty(p, dtype=torch.float64).pin_memory()
ih = torch.empty(p, dtype=torch.int32).pin_memory()
L = S.load(); o = S.default_options()
for it in range(4):
    t = time.perf_counter()
    rc = L.spmesl_fit_ex(ctypes.c_void_p(Xh.data_ptr()), n, p, lam, 1e-4, 100, ctypes.byref(o),
                         ctypes.c_void_p(Th.data_ptr()), ctypes.c_void_p(sh.data_ptr()),
                         ctypes.c_void_p(ih.data_ptr()), None, None, None)
    print("e2e ms", round(1000 * (time.perf_counter() - t), 2), rc, flush=True)
