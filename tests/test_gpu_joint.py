"""GPU parity of mode 1 (Algorithm 3, joint stop) against the joint oracle."""
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


JCASES = [
    (1, {}),
    (2, {}),
    (4, dict(p=150, n=120, family="hub")),
    (4, dict(p=777, n=203)),          # ragged p and n
    (5, dict(p=1200)),
]


@pytest.mark.parametrize("cfg,over", JCASES)
@pytest.mark.parametrize("delta", [1e-4, 1e-10])
@pytest.mark.parametrize("solver", ["auto", "gram", "residual"])
def test_joint_parity(S, oracle, cfg, over, delta, solver):
    # auto / gram: Algorithm 3 on the Gram form (certified f16 or FP64 screening for the first
    # joint sweep, sweep slots for the columns with a hit); residual: the CD kernel per sweep
    X, _, _ = G.make_config(cfg, **over)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    ora = oracle.spmesl_fit_joint(X, lam, delta=delta)
    res = S.fit(X, lam, tol=delta, max_iter=100, mode="joint", solver=solver)
    assert res.stats["solver"] == {"auto": 3, "gram": 2, "residual": 1}[solver]
    rep = compare(res.Theta, res.sigma, res.iters, res.sweeps, ora)
    print(cfg, over, delta, rep, res.stats["kernel_launches"])
    assert_parity(rep)
    assert np.array_equal(res.converged, ora.converged)
    assert np.array_equal(res.Theta, res.Theta.T)


@pytest.mark.parametrize("T", [8, 16, 32])
def test_joint_bit_identical_across_tile_sizes(S, oracle, T):
    X, _, _ = G.make_config(2)
    lam = oracle.lambda_univ(*X.shape)
    ref = S.fit(X, lam, tol=1e-4, mode="joint", tile_cols=32, solver="residual")
    r = S.fit(X, lam, tol=1e-4, mode="joint", tile_cols=T, solver="residual")
    assert np.array_equal(r.Theta, ref.Theta) and np.array_equal(r.sweeps, ref.sweeps)


def test_joint_caps(S, oracle):
    # max_inner = 2 and max_iter = 3: the inner-cap flag and the outer cap (reading g16)
    X, _, _ = G.make_config(4, p=200, n=100)
    lam = oracle.lambda_univ(*X.shape)
    ora = oracle.spmesl_fit_joint(X, lam, delta=1e-10, max_outer=3, max_inner=2)
    res = S.fit(X, lam, tol=1e-10, max_iter=3, max_inner=2, mode="joint")
    assert res.code == 1 and not res.converged.any()
    rep = compare(res.Theta, res.sigma, res.iters, res.sweeps, ora)
    assert_parity(rep)


def test_joint_device_api(S, oracle):
    import torch
    X, _, _ = G.make_config(1)
    lam = oracle.lambda_univ(*X.shape)
    ora = oracle.spmesl_fit_joint(X, lam, delta=1e-4)
    r = S.fit_device(torch.from_numpy(X).cuda(), lam, tol=1e-4, mode="joint")
    rep = compare(r.Theta.cpu().numpy(), r.sigma.cpu().numpy(), r.iters.cpu().numpy(),
                  r.sweeps.cpu().numpy(), ora)
    assert_parity(rep)


def test_joint_columns_api_rejects_partial_range(S):
    import torch
    X, _, _ = G.make_config(1)
    with pytest.raises(S.SpmeslError):
        S.fit_columns_device(torch.from_numpy(X).cuda(), 0, X.shape[1] // 2, 0.1, mode="joint")


def test_joint_gram_forms_identical_and_unstandardized(S, oracle):
    """Mode 1 on the Gram form: the certified f16 and the FP64 screening give bit-identical
    fits; with standardize = 0 and column norms ||x_k||^2 / n in [0.64, 1.44] the columns
    without a first-sweep hit refit sigma != 1 and stay active (they get sweep slots then), and
    the result still matches the joint oracle."""
    X, _, _ = G.make_config(4, p=400, n=200, family="hub")
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    a = S.fit(X, lam, tol=1e-4, mode="joint", solver="gram")
    b = S.fit(X, lam, tol=1e-4, mode="joint", solver="gram16")
    assert np.array_equal(a.Theta, b.Theta) and np.array_equal(a.sweeps, b.sweeps)
    Xs, _, _ = oracle.standardize(X)
    Xs = Xs * np.linspace(0.8, 1.2, p)[None, :]
    ora = oracle.spmesl_fit_joint(Xs, lam, delta=1e-4, standardize=False)
    for solver in ("auto", "residual"):
        res = S.fit(Xs, lam, tol=1e-4, mode="joint", standardize=False, solver=solver)
        rep = compare(res.Theta, res.sigma, res.iters, res.sweeps, ora)
        print(solver, rep)
        assert_parity(rep)
