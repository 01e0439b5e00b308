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
def test_joint_parity(S, oracle, cfg, over, delta):
    X, _, _ = G.make_config(cfg, **over)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    ora = oracle.spmesl_fit_joint(X, lam, delta=delta)
    res = S.fit(X, lam, tol=delta, max_iter=100, mode="joint")
    rep = compare(res.Theta, res.sigma, res.iters, res.sweeps, ora)
    print(cfg, over, delta, rep, res.stats["kernel_launches"])
    assert_parity(rep)
    assert np.array_equal(res.converged, ora.converged)
    assert np.array_equal(res.Theta, res.Theta.T)


@pytest.mark.parametrize("T", [8, 16, 32])
def test_joint_bit_identical_across_tile_sizes(S, oracle, T):
    X, _, _ = G.make_config(2)
    lam = oracle.lambda_univ(*X.shape)
    ref = S.fit(X, lam, tol=1e-4, mode="joint", tile_cols=32)
    r = S.fit(X, lam, tol=1e-4, mode="joint", tile_cols=T)
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
