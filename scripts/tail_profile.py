"""One eager fit of a multi-sweep workload (for ncu on tail_sweep_kernel).
    python scripts/tail_profile.py band3|hub|univ5"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2203_15031_b200 as S
from synth import generators as G
which = sys.argv[1] if len(sys.argv) > 1 else "band3"
if which == "univ5":
    X, _, spec = G.make_config(5)
else:
    X, _, spec = G.make_config(4, family=which)
n, p = X.shape
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
lam = S.lambda_univ(n, p) if which == "univ5" else S.lambda_ub(n, p)
for _ in range(2):
    r = S.fit_device(Xd, lam, eager=True)
print({k: r.stats[k] for k in ("ms_total", "ms_tail", "ms_gram", "tail_columns", "tail_passes", "tail_changes", "screen_candidates", "gram_fallback")})
