"""Pin of the certified f16 screening on the DEVICE (screen16.cu header).

The certification assumes |R_hat_jc - R_jc| <= eps(n_pad) = 2.1 u + n_pad 2^-22 + 2^-23 + 2^-20
for the f32 accumulators of tcgen05.mma kind::f16, where the n_pad 2^-22 term is the
accumulation model "every f32 accumulation step has relative error <= 2^-23 (of a partial sum
bounded by sum_i |y_ij y_ic| <= n), with a factor-2 margin".  NVIDIA does not document the
tcgen05 accumulation, so these tests read the real accumulators back
(spmesl_screen_accumulators_device) and measure, for every covered pair:
  (1) the accumulation error alone: acc_jc - sum_i fp16(y_ij) fp16(y_ic), the sum formed exactly
      (float64 of products of f16 values) from the GPU's own f16 operands, against the
      accumulation term n_pad 2^-22 n of the bound;
  (2) the whole bound: |acc_jc / n - R_jc| <= eps with R = Y^T Y / n from float64 data.
Inputs stress the bound: near-collinear pairs (|R| ~ 1), heavy tails (large |y_i|), mass
concentrated on two samples, random signs, and — without standardization — column norms
N_k in [0.25, 4].  The observed worst ratios are printed (DESIGN.md §6 records them)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_15031_b200 as S
    S.load()
    return S


def eps_bound(n_pad):
    return 2.1 * 2.0 ** -11 + n_pad * 2.0 ** -22 + 2.0 ** -23 + 2.0 ** -20


def adversarial(n, p, seed, scaled):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, p))
    q = p // 8
    X[:, q:2 * q] = X[:, :q] + 1e-3 * rng.standard_normal((n, q))        # |R| close to 1
    X[:, 2 * q:3 * q] = X[:, :q] * -1.0 + 1e-4 * rng.standard_normal((n, q))   # close to -1
    X[:, 3 * q:4 * q] = rng.standard_normal((n, q)) ** 3                  # heavy tails
    X[:, 4 * q:5 * q] = rng.standard_t(2.5, (n, q)) * 0.3                 # heavier tails
    conc = np.full((n, q), 1e-3)
    conc[:2] = 30.0 * rng.choice([-1.0, 1.0], (2, q))                     # concentrated mass
    X[:, 5 * q:6 * q] = conc
    X[:, 6 * q:7 * q] = np.sign(rng.standard_normal((n, q)))              # +-1 (exact in f16)
    X -= X.mean(0)
    X /= np.sqrt((X ** 2).mean(0))
    if scaled:   # N_k in [0.25, 4] (the case standardize = 0 leaves to the bound's sqrt(N) terms)
        X *= np.sqrt(rng.uniform(0.25, 4.0, p))
    return X


@pytest.mark.parametrize("n,p,scaled", [(500, 640, False), (1000, 384, False), (250, 520, True),
                                        (77, 300, True)])
def test_tcgen05_accumulation_within_certified_bound(S, n, p, scaled):
    import torch
    X = adversarial(n, p, seed=n + p, scaled=scaled)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    acc, cand, Y = S.screen_accumulators_device(Xd, standardize=not scaled, solver="gram16")
    acc = acc.cpu().numpy().astype(np.float64)            # acc[c, j]
    Y16 = Y.cpu().numpy()[:p, :n].astype(np.float64)      # the GPU's f16 operands, exactly
    # the data as the GPU standardizes it (float64; no standardization when scaled)
    Xs = X if scaled else (X - X.mean(0)) / np.sqrt(((X - X.mean(0)) ** 2).mean(0))
    N = (Xs ** 2).sum(0) / n
    Yx = Xs / np.sqrt(N)
    R = (Yx.T @ Yx) / n                                   # float64 reference correlation
    exact = Y16 @ Y16.T                                   # sum_i fp16 * fp16 (exact enough: < 2^-40 rel)
    n_pad = -(-n // 32) * 32
    eps = eps_bound(n_pad)
    jj, cc = np.triu_indices(p)                           # every pair j <= c is covered
    a = acc[cc, jj]
    assert np.all(np.isfinite(a)), "a covered pair was not written"
    acc_err = np.abs(a - exact[jj, cc])
    acc_term = n_pad * 2.0 ** -22 * n                     # the bound's accumulation term (acc units)
    tot_err = np.abs(a / n - R[jj, cc])
    print(f"n={n} p={p} scaled={scaled}: max accumulation error {acc_err.max():.3e} "
          f"= {acc_err.max() / acc_term:.4f} of the bound's term; max |R_hat - R| "
          f"{tot_err.max():.3e} = {tot_err.max() / eps:.4f} of eps")
    assert acc_err.max() <= acc_term
    assert tot_err.max() <= eps
    # the f32 accumulation keeps (at least) f32 precision relative to the sum of |terms|: the
    # model the bound's n_pad 2^-22 term stands on, with its factor-2 margin unused
    absum = np.abs(Y16) @ np.abs(Y16).T
    rel = acc_err / np.maximum(absum[jj, cc], 1e-300)
    assert rel.max() <= n_pad * 2.0 ** -23, rel.max()
