"""Fit times of the multi-sweep workloads (config 4 band(3)/hub, config 5 at lambda_univ and
lambda_ub): device time per fit (CUDA-graph replays) and, from an eager fit, the sweep
kernel's own time.  Development timing aid; bench.py's per_config block is the record."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
if len(sys.argv) > 1:   # (development: time another build of the library)
    from paper_2203_15031_b200 import _lib
    _lib.LIB_PATH = sys.argv[1]
import paper_2203_15031_b200 as S
from synth import generators as G

cases = [(4, dict(family="band3"), "ub"), (4, dict(family="hub"), "ub"), (5, {}, "univ"),
         (5, {}, "ub")]
for cfg, over, rule in cases:
    X, _, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = S.lambda_ub(n, p) if rule == "ub" else S.lambda_univ(n, p)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    out = dict(theta=torch.empty((p, p), dtype=torch.float64, device="cuda"),
               sigma=torch.empty(p, dtype=torch.float64, device="cuda"),
               iters=torch.empty(p, dtype=torch.int32, device="cuda"),
               sweeps=torch.empty(p, dtype=torch.int32, device="cuda"),
               conv=torch.empty(p, dtype=torch.uint8, device="cuda"))
    e = S.fit_device(Xd, lam, out=out, eager=True)
    tail = [S.fit_device(Xd, lam, out=out, eager=True).stats["ms_tail"] for _ in range(3)]
    for _ in range(3):
        S.fit_device(Xd, lam, out=out)
    tot = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = S.fit_device(Xd, lam, out=out)
        tot.append(r.stats["ms_total"])
    st = e.stats
    print(f"config {cfg} {over} {rule}: fit {np.median(tot):.3f} ms (device), sweep kernel "
          f"{np.median(tail):.3f} ms, columns {st['tail_columns']}, sweeps {st['total_sweeps']}, "
          f"max sweeps {st['max_sweeps']}, nnz {st['nnz']}, changes {st['tail_changes']}, "
          f"passes {st['tail_passes']}", flush=True)
