"""Dev stress: unusual shapes (tiny / ragged / n > 1024) — solver 3 == solver 2 bit for bit,
oracle parity, sparse == dense, graph replay == eager."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_15031_b200 as S
from oracle import oracle as O
from tests.parity import compare, assert_parity
rng = np.random.default_rng(5)
bad = 0
for n, p in [(2, 5), (3, 40), (7, 129), (33, 255), (64, 257), (129, 513), (1100, 300), (1500, 700), (2100, 130), (97, 2049)]:
    X = rng.standard_normal((n, p))
    X[:, 1::3] += 0.5 * X[:, ::3][:, : X[:, 1::3].shape[1]]
    lam = float(O.lambda_univ(n, p)) if n > 2 else 0.5
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    try:
        a = S.fit_device(Xd, lam, solver="gram", eager=True)
        b = S.fit_device(Xd, lam, solver="gram16", eager=True)
        ok1 = torch.equal(a.Theta, b.Theta) and torch.equal(a.sweeps, b.sweeps)
        sp = S.fit_sparse_device(Xd, lam)
        ok2 = torch.equal(S.sparse_to_dense(sp["col_ptr"], sp["rows"], sp["vals"], p), b.Theta)
        out = dict(theta=torch.empty((p, p), dtype=torch.float64, device="cuda"),
                   sigma=torch.empty(p, dtype=torch.float64, device="cuda"),
                   iters=torch.empty(p, dtype=torch.int32, device="cuda"),
                   sweeps=torch.empty(p, dtype=torch.int32, device="cuda"),
                   conv=torch.empty(p, dtype=torch.uint8, device="cuda"))
        for _ in range(3):
            g = S.fit_device(Xd, lam, out=out)
        ok3 = torch.equal(g.Theta, b.Theta) and g.stats["graph_replay"] == 1
        ora = O.spmesl_fit(X, lam, delta=1e-4)
        rep = compare(b.Theta.cpu().numpy(), b.sigma.cpu().numpy(), b.iters.cpu().numpy(), b.sweeps.cpu().numpy(), ora)
        try:
            assert_parity(rep); ok4 = True
        except AssertionError as e:
            ok4 = False; print("   parity:", e)
        res = "ok" if (ok1 and ok2 and ok3 and ok4) else "FAIL"
        print(n, p, "gram==gram16", ok1, "sparse", ok2, "graph", ok3, "oracle", ok4, res, flush=True)
        bad += res != "ok"
    except Exception as e:
        print(n, p, "EXC", repr(e)[:200]); bad += 1
print("failures:", bad)
