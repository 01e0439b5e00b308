"""Ad-hoc GPU check used during development: prints parity reports for a few configs."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from oracle import oracle as O
from synth import generators as G
from tests.parity import compare
import paper_2203_15031_b200 as S

for cfg, over, rule in [(1, {}, "univ"), (2, {}, "univ"), (3, {}, "ub"), (4, dict(p=1000, family="hub"), "ub"),
                        (4, dict(p=777, n=203), "univ")]:
    X, gt, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = O.lambda_univ(n, p) if rule == "univ" else O.lambda_ub(n, p)
    t = time.time(); ora = O.spmesl_fit(X, lam); to = time.time() - t
    t = time.time(); r = S.fit(X, lam); tg = time.time() - t
    rep = compare(r.Theta, r.sigma, r.iters, r.sweeps, ora)
    print(cfg, over, rule, f"oracle {to:.2f}s gpu {tg:.3f}s", {k: (v if not isinstance(v, list) else v[:5]) for k, v in rep.items()},
          r.stats, flush=True)
