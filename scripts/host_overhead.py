"""Where the config-5 step's time outside the kernels goes: CUDA events around (a) the Python
fit_device call, (b) the bare ctypes call with prebuilt arguments, against the device clock's
ms_total (first/last kernel stamps).  Development tool."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15031_b200 as S  # noqa: E402
from paper_2203_15031_b200 import _lib  # noqa: E402
from synth import generators as G  # noqa: E402
from oracle import oracle as O  # noqa: E402

X, _, _ = G.make_config(5)
n, p = X.shape
lam = O.lambda_ub(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
s = torch.cuda.current_stream()
out = dict(theta=torch.empty((p, p), dtype=torch.float64, device="cuda"),
           sigma=torch.empty(p, dtype=torch.float64, device="cuda"),
           iters=torch.empty(p, dtype=torch.int32, device="cuda"),
           sweeps=torch.empty(p, dtype=torch.int32, device="cuda"),
           conv=torch.empty(p, dtype=torch.uint8, device="cuda"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    S.fit_device(Xd, lam, out=out, stream=s)
torch.cuda.synchronize()
L = S.load()
o = S._opts()
st = _lib.Stats()
args = (S._vp(Xd), n, p, float(lam), 1e-4, 100, ctypes.byref(o), S._vp(out["theta"]),
        S._vp(out["sigma"]), S._vp(out["iters"]), S._vp(out["sweeps"]), S._vp(out["conv"]),
        ctypes.c_void_p(s.cuda_stream), ctypes.byref(st))


def timed(fn, reps=20):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(s); b.record(s)
    torch.cuda.synchronize()
    dev, wall, tot = [], [], []
    for a, b in ev:
        flush.fill_(7)
        torch.cuda.synchronize()
        a.record(s)
        t0 = time.perf_counter()
        r = fn()
        t1 = time.perf_counter()
        b.record(s)
        torch.cuda.synchronize()
        wall.append((t1 - t0) * 1e3)
        tot.append(r)
    dev = [a.elapsed_time(b) for a, b in ev]
    return np.median(dev), np.median(wall), np.median(tot)


def py():
    r = S.fit_device(Xd, lam, out=out, stream=s)
    return r.stats["ms_total"]


def bare():
    rc = L.spmesl_fit_device(*args)
    assert rc >= 0
    return st.ms_total


for name, fn in (("python fit_device", py), ("bare ctypes", bare), ("python fit_device", py)):
    d, w, t = timed(fn)
    print(f"{name:20s}: events {d:.4f} ms, host wall {w:.4f} ms, device ms_total {t:.4f} ms,"
          f" outside kernels {d - t:.4f} ms")
