"""Cross-implementation check: a second, independent, literal NumPy transcription of
Algorithm 1 / Algorithm 2 against the C oracle on small inputs.
(This is the weakest kind of pin — agreement of two readings of the same text — and is
used alongside the closed-form / brute-force / sklearn pins of test_oracle_pins.py.)"""
import math

import numpy as np
import pytest

from synth import generators as G


def alg1_numpy(Xs, k, lambda0, delta, max_outer=100, max_inner=10000):
    n, p = Xs.shape
    y = Xs[:, k]
    beta = np.zeros(p)
    sigma = 1.0
    outer = sweeps = 0
    while True:
        lam = sigma * lambda0
        inner = 0
        while True:
            cur = beta.copy()
            for j in range(p):
                if j == k:
                    continue
                e = y - Xs @ beta                  # full current residual (reading g22)
                a = Xs[:, j] @ e / n + beta[j]
                beta[j] = math.copysign(max(abs(a) - lam, 0.0), a) if abs(a) > lam else 0.0
            sweeps += 1
            inner += 1
            if np.abs(beta - cur).max() < delta or inner >= max_inner:
                break
        r = y - Xs @ beta
        sn = max(math.sqrt(r @ r) / math.sqrt(n), 1e-8)
        outer += 1
        done = abs(sn - sigma) < delta
        sigma = sn
        if done or outer >= max_outer:
            return beta, sigma, outer, sweeps


@pytest.mark.parametrize("delta", [1e-4, 1e-10])
def test_numpy_alg1_matches_c_oracle(oracle, delta):
    X, _, _ = G.make_config(1)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    r = oracle.spmesl_fit(X, lam, delta=delta)
    Xs, mu, s = oracle.standardize(X)
    for k in range(p):
        b, sig, outer, sweeps = alg1_numpy(Xs, k, lam, delta)
        assert outer == r.outer[k] and sweeps == r.sweeps[k]
        assert np.abs(b - r.B[:, k]).max() < 1e-12
        assert abs(sig * s[k] - r.sigma[k]) < 1e-12 * r.sigma[k]
    # Alg. 2 assembly + symmetrization by hand
    T1 = np.zeros((p, p))
    for k in range(p):
        sk = r.sigma[k] / s[k]
        T1[:, k] = -r.B[:, k] * (1 / (sk * sk))
        T1[k, k] = 1 / (sk * sk)
    T1 = T1 / np.outer(s, s)
    np.testing.assert_allclose(T1, r.Theta1, rtol=1e-14, atol=0)
    T = r.Theta1.copy()
    for j in range(p):
        for k in range(j + 1, p):
            if abs(T[j, k]) > abs(T[k, j]):
                T[j, k] = T[k, j]
            else:
                T[k, j] = T[j, k]
    np.testing.assert_array_equal(T, r.Theta)
