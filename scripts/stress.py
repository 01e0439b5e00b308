"""Dev stress: many seeds / shapes — solver 3 == solver 2 bit for bit, mode 1 Gram == mode 1
residual within parity, sparse == dense, graph replay == eager."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from synth import generators as G
from oracle import oracle as O
from tests.parity import compare, assert_parity
bad = 0
cases = []
for seed in range(12):
    cases.append((3, dict(seed=seed)))
    cases.append((4, dict(seed=seed, p=int(600 + 97 * seed), n=int(150 + 13 * seed))))
    cases.append((4, dict(seed=seed, p=500, n=120, family="hub")))
    cases.append((2, dict(seed=seed, p=int(301 + 50 * seed))))
for cfg, kw in cases:
    X, _, spec = G.make_config(cfg, **kw)
    n, p = X.shape
    lam = S.lambda_univ(n, p)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    a = S.fit_device(Xd, lam, solver="gram", eager=True)
    b = S.fit_device(Xd, lam, solver="gram16", eager=True)
    ok = torch.equal(a.Theta, b.Theta) and torch.equal(a.sweeps, b.sweeps)
    sp = S.fit_sparse_device(Xd, lam)
    ok2 = torch.equal(S.sparse_to_dense(sp["col_ptr"], sp["rows"], sp["vals"], p), b.Theta)
    ora = O.spmesl_fit(X, lam, delta=1e-4)
    rep = compare(b.Theta.cpu().numpy(), b.sigma.cpu().numpy(), b.iters.cpu().numpy(), b.sweeps.cpu().numpy(), ora)
    try:
        assert_parity(rep); ok3 = True
    except AssertionError as e:
        ok3 = False
    jg = S.fit_device(Xd, lam, mode="joint", eager=True)
    jo = O.spmesl_fit_joint(X, lam, delta=1e-4)
    repj = compare(jg.Theta.cpu().numpy(), jg.sigma.cpu().numpy(), jg.iters.cpu().numpy(), jg.sweeps.cpu().numpy(), jo)
    try:
        assert_parity(repj); ok4 = True
    except AssertionError:
        ok4 = False
    flag = "" if (ok and ok2 and ok3 and ok4) else "  <-- FAIL"
    bad += bool(flag)
    print(cfg, kw, "n,p", n, p, "gram==gram16", ok, "sparse==dense", ok2, "oracle", ok3, "joint", ok4,
          "cand", b.stats["screen_candidates"], flag, flush=True)
print("failures:", bad)
