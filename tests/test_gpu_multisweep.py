"""GPU parity of the sweep kernel's multi-sweep mode against the oracle, on the
cases that exercise its branches: the chain's sigma refits reaching the inner cap (flags) and
the outer cap (retire) inside a multi-sweep, the sigma floor binding there, new rows ending a
multi-sweep (rollback + per-segment continuation), supports of more than 16 rows (the 1-row-
per-thread pass, 16 sweeps per pass), odd p, the most-hits-first work order (hub: skewed hit
counts, more columns than CTAs) and the second z buffer in global memory (p too large for
two z buffers on chip).  Every column is compared (tests/parity.py criteria)."""
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


def _check(S, oracle, X, lam, solver="gram16", **kw):
    okw = {k: v for k, v in kw.items() if k in ("max_inner", "sigma_floor")}
    mo = kw.get("max_iter", 100)
    ora = oracle.spmesl_fit(X, lam, max_outer=mo, **okw)
    r = S.fit(X, lam, max_iter=mo, solver=solver, **okw)
    rep = compare(r.Theta, r.sigma, r.iters, r.sweeps, ora)
    assert_parity(rep)
    assert np.array_equal(r.converged, ora.converged)
    return r, ora


@pytest.mark.parametrize("family,p", [("hub", 1000), ("hub", 999), ("band3", 1001)])
def test_multisweep_columns_every_column(S, oracle, family, p):
    """hub: slow columns (hundreds of sweeps), new rows entering mid-batch, skewed hit counts
    (the work order is used: more columns than CTAs); odd p (no 16-byte row pairs)."""
    X, _, _ = G.make_config(4, p=p, family=family)
    n = X.shape[0]
    r, ora = _check(S, oracle, X, oracle.lambda_ub(n, p))
    assert r.stats["tail_columns"] > 296          # (more columns than CTAs)
    if family == "hub":
        assert int(ora.sweeps.max()) > 32          # (several multi-sweep passes per column)


@pytest.mark.parametrize("max_inner", [2, 5])
def test_inner_cap_inside_the_chain(S, oracle, max_inner):
    """The chain ends inner loops at the cap (flag 2: not converged) and refits sigma there."""
    X, _, _ = G.make_config(4, p=1000, family="hub")
    n, p = X.shape
    r, ora = _check(S, oracle, X, oracle.lambda_ub(n, p), max_inner=max_inner)
    assert not ora.converged.all()


@pytest.mark.parametrize("max_iter", [2, 3])
def test_outer_cap_inside_the_chain(S, oracle, max_iter):
    """The chain retires a column at the outer cap in the middle of a multi-sweep."""
    X, _, _ = G.make_config(4, p=1000, family="hub")
    n, p = X.shape
    r, ora = _check(S, oracle, X, oracle.lambda_ub(n, p), max_iter=max_iter)
    assert (ora.outer == max_iter).any()


def test_sigma_floor_inside_the_chain(S, oracle):
    X, _, _ = G.make_config(4, p=1000, family="band3")
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    base = oracle.spmesl_fit(X, lam)
    floor = float(np.quantile(base.sigma / X.std(0), 0.5))   # binds for about half the columns
    _check(S, oracle, X, lam, sigma_floor=floor)


def test_large_supports(S, oracle):
    """A small penalty: supports beyond 16 rows (the 1-row-per-thread pass, 16 sweeps per
    multi-sweep) and beyond 31 (the per-segment mode)."""
    X, _, _ = G.make_config(4, p=600, n=400, family="hub")
    n, p = X.shape
    lam = 0.5 * oracle.lambda_univ(n, p)
    r, ora = _check(S, oracle, X, lam)
    nnz = (np.abs(ora.Theta) > 0).sum(0) - 1
    assert nnz.max() > 16


def test_global_second_z_buffer(S, oracle):
    """p too large for two z buffers on chip: the multi-sweep mode writes z + changes to global
    scratch (checked on every column whose GPU fit took more than one sweep, and a sample)."""
    X, _, _ = G.make_config(4, p=7000, n=200, family="band3")
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    r = S.fit(X, lam, solver="gram16")
    sw = np.asarray(r.sweeps)
    rng = np.random.default_rng(1)
    cols = np.unique(np.concatenate([np.nonzero(sw > 1)[0][:600], rng.choice(p, 200, replace=False)]))
    Xs, mu, s = oracle.standardize(X)
    oc = oracle.spmesl_columns(Xs, cols, lam, delta=1e-4, want_margin=True)
    assert np.array_equal(sw[cols], oc.sweeps)
    assert np.array_equal(np.asarray(r.iters)[cols], oc.outer)
    sg = np.asarray(r.sigma)[cols]
    assert np.max(np.abs(sg - oc.sigma * s[cols]) / (oc.sigma * s[cols])) <= 1e-10
