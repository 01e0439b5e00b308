"""Dev: every entry point once at small sizes (ragged n, p); exits non-zero on any library error
(compute-sanitizer is not available on this pool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G

X, gt, spec = G.make_config(4, p=333, n=150)
n, p = X.shape
lam = S.lambda_ub(n, p)
for solver in ("residual", "gram", "gram16"):
    S.fit(X, lam, solver=solver)
    S.fit(X, lam, solver=solver, mode="joint")
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
for _ in range(3):                               # eager, capture, replay
    S.fit_device(Xd, lam)
S.fit_sparse_device(Xd, lam)
S.fit_path_device(Xd, [S.lambda_pb(n, p), S.lambda_univ(n, p), lam])
S.fit_columns_device(Xd, 40, 200, lam, solver="residual")
torch.cuda.synchronize()
print("entry_points_smoke ok", n, p)
