"""Dev: one CD sweep wave of 148 x m columns at config 5 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
m = int(sys.argv[1]); T = int(sys.argv[2]) if len(sys.argv) > 2 else 32
X, gt, spec = G.make_config(5)
n, p = X.shape
lam = S.lambda_ub(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
for it in range(3):
    r = S.fit_columns_device(Xd, 0, 148 * m, lam, tile_cols=T)
    print(r["stats"]["ms_cd"])
