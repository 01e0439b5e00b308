"""Dev: sparse-output fit (no dense Theta) time at config 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
X, _, spec = G.make_config(5)
n, p = X.shape
lam = S.lambda_ub(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
out = dict(col_ptr=torch.empty(p + 1, dtype=torch.int64, device="cuda"),
           rows=torch.empty(65 * p, dtype=torch.int32, device="cuda"),
           vals=torch.empty(65 * p, dtype=torch.float64, device="cuda"),
           sigma=torch.empty(p, dtype=torch.float64, device="cuda"),
           iters=torch.empty(p, dtype=torch.int32, device="cuda"),
           sweeps=torch.empty(p, dtype=torch.int32, device="cuda"),
           conv=torch.empty(p, dtype=torch.uint8, device="cuda"))
for mode in ("per_column", "joint"):
    ts = []
    for it in range(6):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        r = S.fit_sparse_device(Xd, lam, mode=mode, out=out)
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(mode, "sparse fit ms", [round(t, 3) for t in ts], "nnz", r["stats"]["nnz"], "device total", round(r["stats"]["ms_total"], 3), "replay", r["stats"]["graph_replay"])
