"""Per-phase cycle counters of the sweep kernel (development build, scripts/tail_prof_build.sh):
one eager fit per workload, counters summed over CTAs (tid 0's clock64)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_15031_b200 import _lib
_lib.LIB_PATH = "scripts/_prof/libspmesl.so"
import paper_2203_15031_b200 as S
from synth import generators as G

lib = S.load()
buf = (ctypes.c_ulonglong * 32)()
names = ["multi_chain", "spec_pass", "commit", "single_seg", "refit", "ok", "fail", "ok_sweeps",
         "fail_sstar", "single_cnt", "column_total", "multi_K", "fail_Msw"]
for which in (sys.argv[1:] or ["band3", "hub"]):
    fam, _, seed = which.partition("@")     # (e.g. hub@3207: another dataset seed)
    kw = {"seed": int(seed)} if seed else {}
    if fam == "univ5":
        X, _, spec = G.make_config(5, **kw)
    else:
        X, _, spec = G.make_config(4, family=fam, **kw)
    n, p = X.shape
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    lam = S.lambda_univ(n, p) if fam == "univ5" else S.lambda_ub(n, p)
    lib.spmesl_dev_tail_prof(buf, 1)
    S.fit_device(Xd, lam, eager=True)
    torch.cuda.synchronize()
    lib.spmesl_dev_tail_prof(buf, 1)
    r = S.fit_device(Xd, lam, eager=True)
    torch.cuda.synchronize()
    lib.spmesl_dev_tail_prof(buf, 1)
    v = list(buf)
    print(which, {k: r.stats[k] for k in ("ms_tail", "tail_columns", "tail_passes", "tail_changes")})
    tot = v[10] or 1
    for i, nm in enumerate(names):
        extra = f"  ({100 * v[i] / tot:.1f}% of column cycles)" if i in (0, 1, 2, 3, 4) else ""
        print(f"  {nm:14s} {v[i]:>16d}{extra}")
    m = v[13]
    print(f"  slowest column: {m >> 24} cycles, {(m >> 12) & 4095} passes, {m & 4095} sweeps; columns over 4e6 cycles: {v[14]}")
    print(f"  slowest column: final nnz {(v[28] >> 8) & 255}, failures {v[28] & 255}; mean final nnz of the columns over 4e6 cycles: {v[29] / max(v[14], 1):.1f}")
    if v[30] and v[30] != 2**64 - 1:
        print(f"  kernel span {(v[27] - v[30]) / 1e3:.0f} us; latest start of a column over 4e6 cycles: {(v[31] - v[30]) / 1e3:.0f} us after the first")
    if v[16]:
        print(f"  stragglers (>200 sweeps): {v[16]} columns, {v[25]} sweeps, {v[24]} cycles; multi ok {v[17]} "
              f"({v[20]} sweeps), fail {v[18]}, single segments {v[19]}; cycles: spec {v[21]}, chain {v[22]}, "
              f"single {v[23]}")
