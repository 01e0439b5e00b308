"""The auto solver's screening history: a repeat of a device fit whose certified
f16 screening fell back to the full FP64 Gram kernel runs the full-Gram path (solver 2) directly
— bit-identical, since solvers 2 and 3 compute the same iterates — and new data in the same
buffers with few hit columns hands the choice back to the screening.  Every result is checked
against the oracle (Algorithm 2)."""
import numpy as np
import pytest

from synth import generators as G
from tests.parity import assert_parity, compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_15031_b200 as S
    S.load()
    return S


def _buffers(torch, p):
    return dict(theta=torch.empty((p, p), dtype=torch.float64, device="cuda"),
                sigma=torch.empty(p, dtype=torch.float64, device="cuda"),
                iters=torch.empty(p, dtype=torch.int32, device="cuda"),
                sweeps=torch.empty(p, dtype=torch.int32, device="cuda"),
                conv=torch.empty(p, dtype=torch.uint8, device="cuda"))


def _check(r, ora):
    assert_parity(compare(r.Theta.cpu().numpy(), r.sigma.cpu().numpy(), r.iters.cpu().numpy(),
                          r.sweeps.cpu().numpy(), ora))


def test_auto_history_full_gram_and_back(S, oracle):
    import torch
    X, _, _ = G.make_config(4, p=1200, family="hub")     # most columns are candidates
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    ora = oracle.spmesl_fit(X, lam)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    out = _buffers(torch, p)
    solvers, replays, thetas = [], [], []
    for _ in range(5):
        r = S.fit_device(Xd, lam, out=out)
        torch.cuda.synchronize()
        solvers.append(r.stats["solver"])
        replays.append(r.stats["graph_replay"])
        assert r.stats["gram_fallback"] == 1
        thetas.append(r.Theta.clone())
        _check(r, ora)
    assert solvers[0] == 3 and solvers[-1] == 2, solvers
    assert replays[-1] == 1, replays
    for t in thetas[1:]:
        assert torch.equal(t, thetas[0])
    # new data in the same buffers (same pointers, shape and penalty): few hit columns
    X2, _, _ = G.make_config(5, n=n, p=p)
    ora2 = oracle.spmesl_fit(X2, lam)
    Xd.copy_(torch.from_numpy(np.ascontiguousarray(X2.T)).cuda().t())
    solvers2 = []
    for _ in range(4):
        r = S.fit_device(Xd, lam, out=out)
        torch.cuda.synchronize()
        solvers2.append(r.stats["solver"])
        _check(r, ora2)
    assert solvers2[0] == 2 and solvers2[-1] == 3, solvers2
    # an eager fit shares the history and is bit-identical to the replayed ones
    r = S.fit_device(Xd, lam, out=out, eager=True)
    t_e = r.Theta.clone()
    r = S.fit_device(Xd, lam, out=out)
    assert torch.equal(r.Theta, t_e)
