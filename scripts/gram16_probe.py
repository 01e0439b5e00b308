"""Dev: config timings and stats for solver gram (FP64 S) vs gram16 (certified f16 screening)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
for cfg, kw in [(5, {}), (4, {}), (4, dict(family="hub")), (3, {}), (2, {})]:
    X, _, spec = G.make_config(cfg, **kw)
    n, p = X.shape
    lam = S.lambda_ub(n, p) if spec["rule"] == "ub" else S.lambda_univ(n, p)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    res = {}
    for solver in ("gram", "gram16"):
        ts = []
        for it in range(4):
            r = S.fit_device(Xd, lam, solver=solver)
            torch.cuda.synchronize()
            ts.append(r.stats["ms_total"])
        res[solver] = r
        print(cfg, kw, solver, "ms_total %.3f" % min(ts), "screen %.3f" % r.stats["ms_gram"],
              "sweeps-kernel %.3f" % r.stats["ms_tail"], "cand", r.stats["screen_candidates"],
              "tail cols", r.stats["tail_columns"], flush=True)
    a, b = res["gram"], res["gram16"]
    print("   identical:", torch.equal(a.Theta, b.Theta), torch.equal(a.sweeps, b.sweeps),
          "max|dTheta|", float((a.Theta - b.Theta).abs().max()), flush=True)
