import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_15031_b200 as S
from synth import generators as G
for cfg, kw in [(5, dict(p=8000, n=500)), (5, dict(p=8000, n=300)), (5, dict(p=6000, n=200)), (3, dict(p=6000, n=200)),
                (5, dict(p=20000, n=500))]:
    X, _, spec = G.make_config(cfg, **kw)
    n, p = X.shape
    for lam, nm in [(S.lambda_ub(n, p), "ub"), (0.5 * (S.lambda_ub(n, p) + S.lambda_univ(n, p)), "mid")]:
        r = S.fit(X, lam)
        print(cfg, kw, nm, "tail", r.stats["tail_columns"], "ondemand", r.stats["tail_gram_ondemand"], "sweeps max", r.stats["max_sweeps"], flush=True)
