"""Dev: the tail solver's lazy mode must be bit-identical to the eager update (run twice,
with SPMESL_TAIL_EAGER=1 and without, compare the saved outputs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_15031_b200 as S
from synth import generators as G
tag = "eager" if os.environ.get("SPMESL_TAIL_EAGER") == "1" else "lazy"  # eager = no prefetch
out = {}
for name, cfg, kw, solver in [("hub", 4, dict(family="hub"), "gram"), ("band", 4, {}, "gram"),
                              ("ar", 2, {}, "gram"), ("hubres", 4, dict(p=1500, family="hub"), "residual"),
                              ("c5", 5, dict(p=8000), "residual")]:
    X, _, spec = G.make_config(cfg, **kw)
    n, p = X.shape
    lam = S.lambda_ub(n, p) if spec["rule"] == "ub" else S.lambda_univ(n, p)
    r = S.fit(X, lam, solver=solver)
    out[name + "_theta"] = r.Theta
    out[name + "_sweeps"] = r.sweeps
    print(tag, name, r.stats["ms_tail"], r.stats["tail_columns"], r.stats["max_sweeps"], flush=True)
np.savez(f"/tmp/lazy_{tag}.npz", **out)
if tag == "lazy" and os.path.exists("/tmp/lazy_eager.npz"):
    e = np.load("/tmp/lazy_eager.npz")
    for k in out:
        print(k, "identical" if np.array_equal(out[k], e[k]) else "DIFFERENT")
