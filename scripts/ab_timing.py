"""Development A/B timing: several builds of the library loaded side by side (ctypes, separate
workspaces), eager fits of config 4 band(3)/hub alternated round-robin; median sweep-kernel time
(stats.ms_tail) per build.  Usage: ab_timing.py lib1.so lib2.so ..."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2203_15031_b200 as S
from paper_2203_15031_b200 import _lib
from synth import generators as G

vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
args = [a for a in sys.argv[1:] if not a.startswith("--cases=")]
cases = next((a[8:].split(",") for a in sys.argv[1:] if a.startswith("--cases=")), ["band3", "hub"])
libs = []
for path in args:
    L = ctypes.CDLL(path)
    L.spmesl_fit_device.argtypes = [vp, i64, i64, dbl, dbl, i32, ctypes.POINTER(_lib.Options), vp, vp,
                                    vp, vp, vp, vp, vp]
    L.spmesl_default_options.argtypes = [ctypes.POINTER(_lib.Options)]
    libs.append(L)
rounds = 5
for fam in cases:
    fam_, _, seed = fam.partition("@")    # (e.g. hub@3207: another dataset seed)
    kw = {"seed": int(seed)} if seed else {}
    if fam_ in ("univ5", "ub5"):
        X, _, spec = G.make_config(5, **kw)
    else:
        X, _, spec = G.make_config(4, family=fam_, **kw)
    n, p = X.shape
    lam = S.lambda_univ(n, p) if fam_ == "univ5" else S.lambda_ub(n, p)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()   # (p x n row-major = n x p column-major)
    bufs = [torch.empty((p, p), dtype=torch.float64, device="cuda"), torch.empty(p, dtype=torch.float64, device="cuda")] + \
           [torch.empty(p, dtype=torch.int32, device="cuda") for _ in range(2)] + [torch.empty(p, dtype=torch.uint8, device="cuda")]
    times = [[] for _ in libs]
    sweeps = [None] * len(libs)
    for r in range(rounds + 1):
        for li, L in enumerate(libs):
            o = S._make_opts(eager=True)   # (the binding's defaults)
            st = _lib.Stats()
            rc = L.spmesl_fit_device(vp(Xd.data_ptr()), n, p, lam, 1e-4, 100, ctypes.byref(o),
                                     *[vp(b.data_ptr()) for b in bufs],
                                     vp(torch.cuda.current_stream().cuda_stream), ctypes.byref(st))
            torch.cuda.synchronize()
            assert rc >= 0, rc
            if r > 0:
                times[li].append(st.ms_tail)
            sweeps[li] = int(bufs[3].sum().item())
    for li, path in enumerate(args):
        t = np.array(times[li])
        print(f"{fam:6s} {path:40s} sweep kernel median {np.median(t):.3f} ms (min {t.min():.3f}, max {t.max():.3f}); sweeps {sweeps[li]}")
