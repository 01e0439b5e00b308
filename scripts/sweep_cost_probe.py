"""Dev probe: CD-kernel time for one sweep wave of 148 x m columns (m = 1..32) at config 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
X, gt, spec = G.make_config(5)
n, p = X.shape
lam = S.lambda_ub(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
T = int(os.environ.get("PROBE_T", "32"))
for m in [1, 2, 4, 8, 16, 24, 32, 64, 128]:
    cols = 148 * m
    ts = []
    for it in range(4):
        r = S.fit_columns_device(Xd, 0, cols, lam, tile_cols=T)
        ts.append(r["stats"]["ms_cd"])
    print(f"m={m:3d} cols={cols:6d} cd_ms={min(ts):.3f}  per-step-us={1000*min(ts)/ (p/32) / max(1, m/T):.3f}", flush=True)
