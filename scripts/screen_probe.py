"""Dev: screen-only Gram kernel (no G stores) over all tiles at config 5 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
X, gt, spec = G.make_config(5)
n, p = X.shape
lam = S.lambda_ub(n, p)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
nt = S.gram_tile_count(p)
for it in range(3):
    hit = torch.zeros(p, dtype=torch.uint8, device="cuda")
    st = S.gram_screen_device(Xd, lam, 0, nt, hit)
    print("screen ms", st["ms_gram"], "hits", int(hit.sum()))
