"""CPU pins of the certified f16 screening (screen16.cu header).

The GPU decides "|S_jc| <= lambda0 for all j != c" from R_hat = Y16^T Y16 (f16 operands,
f32 accumulation) and the bound |R_hat_jc - R_jc| <= eps(n_pad).  These tests check that bound
with numpy's IEEE float16 / float32 arithmetic against the exact float64 correlation (in several
accumulation orders, including adversarial columns), and that the epilogue's f32 threshold —
every factor rounded downwards, n eps upwards, one downward-rounded fma — never exceeds the
exact certification threshold n (lambda0 / sqrt(N_j N_c) - eps).  No GPU is used."""
import numpy as np
import pytest


def eps_bound(n_pad):
    # screen16_eps (screen16.cu): 2.1 u + n_pad 2^-22 + 2^-23 + 2^-20, u = 2^-11
    return 2.1 * 2.0 ** -11 + n_pad * 2.0 ** -22 + 2.0 ** -23 + 2.0 ** -20


def f32_accumulate(a16, b16, order):
    """sum_i a_i b_i in float32, products exact (f16 x f16 fits in f32), adds in `order`."""
    prod = a16.astype(np.float32) * b16.astype(np.float32)
    acc = np.float32(0.0)
    for i in order:
        acc = np.float32(acc + prod[i])
    return acc


@pytest.mark.parametrize("n", [50, 250, 500, 1000])
def test_f16_correlation_error_within_bound(n):
    rng = np.random.default_rng(n)
    p = 24
    X = rng.standard_normal((n, p))
    X[:, 1] = X[:, 0] + 1e-3 * rng.standard_normal(n)          # |R| close to 1
    X[:, 2] = rng.standard_normal(n) ** 3                       # heavy tails (large |y_i|)
    X[:, 3] = np.where(np.arange(n) < 2, 30.0, 1e-3)            # concentrated mass
    X -= X.mean(0)
    X /= np.sqrt((X ** 2).mean(0))                              # x~^T x~ = n (standardized)
    N = (X ** 2).sum(0) / n
    Y = X / np.sqrt(N)                                          # y^T y = n
    Y16 = Y.astype(np.float16)
    R = (Y.T @ Y) / n
    n_pad = -(-n // 64) * 64
    eps = eps_bound(n_pad)
    orders = [np.arange(n), np.arange(n)[::-1], rng.permutation(n)]
    worst = 0.0
    for j in range(p):
        for c in range(p):
            for order in orders:
                acc = f32_accumulate(Y16[:, j], Y16[:, c], order)
                worst = max(worst, abs(float(acc) / n - R[j, c]))
    assert worst <= eps, (worst, eps)
    assert worst > 0.0


def rd32(x):
    """float64 -> float32 rounded towards -inf."""
    f = np.float32(x)
    return f if float(f) <= x else np.nextafter(f, np.float32(-np.inf))


def ru32(x):
    f = np.float32(x)
    return f if float(f) >= x else np.nextafter(f, np.float32(np.inf))


def fma_rd32(a, b, c):
    """fma in float32 rounded towards -inf (exact product + sum in float64 for f32 inputs)."""
    exact = float(a) * float(b) + float(c)   # f32 x f32 is exact in f64; the add may round
    return rd32(exact * (1.0 - 2.0 ** -52) if exact > 0 else exact * (1.0 + 2.0 ** -52))


def test_epilogue_threshold_never_exceeds_exact():
    rng = np.random.default_rng(7)
    for _ in range(20000):
        n = int(rng.integers(2, 5000))
        n_pad = -(-n // 64) * 64
        lam = float(rng.uniform(0.01, 1.5))
        Nj, Nc = rng.uniform(0.25, 4.0, 2)
        qj, qc = np.sqrt(Nj), np.sqrt(Nc)
        eps = eps_bound(n_pad)
        # the factors as the standardization writes them (directed roundings, 2^-40 margin)
        lam_n = rd32(n * lam / qj * (1.0 - 2.0 ** -40))
        inv_c = rd32(1.0 / qc * (1.0 - 2.0 ** -40))
        epsn = ru32(n * eps * (1.0 + 2.0 ** -40))
        thr = fma_rd32(lam_n, inv_c, -epsn)
        exact = n * (lam / (qj * qc) - eps)
        assert float(thr) <= exact, (n, lam, Nj, Nc, float(thr), exact)


def test_certification_implies_no_hit():
    """End to end on the emulated arithmetic: a pair the f32 test certifies has |S_jc| <= lam."""
    rng = np.random.default_rng(3)
    n, p = 300, 60
    n_pad = 320
    X = rng.standard_normal((n, p))
    X[:, 1::2] += 0.6 * X[:, ::2]                                 # correlated pairs
    X -= X.mean(0)
    X /= np.sqrt((X ** 2).mean(0))
    X *= rng.uniform(0.9, 1.1, p)                                # N_k != 1
    N = (X ** 2).sum(0) / n
    S = X.T @ X / n
    Y16 = (X / np.sqrt(N)).astype(np.float16)
    eps = eps_bound(n_pad)
    epsn = ru32(n * eps * (1.0 + 2.0 ** -40))
    lam = 0.25
    certified = hits = 0
    for j in range(p):
        lam_n = rd32(n * lam / np.sqrt(N[j]) * (1.0 - 2.0 ** -40))
        for c in range(p):
            if c == j:
                continue
            acc = f32_accumulate(Y16[:, j], Y16[:, c], rng.permutation(n))
            inv_c = rd32(1.0 / np.sqrt(N[c]) * (1.0 - 2.0 ** -40))
            if abs(float(acc)) <= float(fma_rd32(lam_n, inv_c, -epsn)):
                certified += 1
                assert abs(S[j, c]) <= lam
            hits += abs(S[j, c]) > lam
    assert certified > 0 and hits > 0


def _trunc_to(x, ulp):
    """Truncate x towards zero to a multiple of ulp (exact in float64 for these magnitudes)."""
    return np.trunc(x / ulp) * ulp


def blockfma_accumulate(a16, b16, K=16, bits=24):
    """A pessimistic model of a tensor-core f32 accumulation: products of f16 values are exact;
    every group of K products is added to the accumulator in one step that aligns all K + 1
    addends to the largest exponent among them and TRUNCATES each to `bits` significant bits of
    that exponent, then truncates the sum to an f32 (24-bit) significand.  (The certification
    bound must hold for this model when bits >= 24, i.e. when no addend loses more than an f32
    ulp of the block maximum.)"""
    prod = a16.astype(np.float64) * b16.astype(np.float64)
    acc = 0.0
    for k0 in range(0, len(prod), K):
        terms = np.concatenate([[acc], prod[k0:k0 + K]])
        m = np.max(np.abs(terms))
        if m == 0.0:
            continue
        e = np.floor(np.log2(m))
        ulp = 2.0 ** (e - (bits - 1))
        s = float(np.sum(_trunc_to(terms, ulp)))        # exact: aligned integers * ulp
        if s != 0.0:
            es = np.floor(np.log2(abs(s)))
            s = float(_trunc_to(s, 2.0 ** (es - 23)))   # f32 significand, truncated
        acc = s
    return acc


@pytest.mark.parametrize("n", [64, 500, 1000])
def test_blockfma_truncation_model_within_bound(n):
    """The bound's accumulation term n_pad 2^-22 (factor 2 over the per-step model) also covers
    block-FMA accumulation with alignment to the block maximum and truncation (K = 16, 24 kept
    bits), on the adversarial columns; a model keeping only 13 bits (what Hopper's FP8 path is
    reported to keep) exceeds it — so the device test (tests/test_gpu_screen_pin.py) that
    measures the real accumulators is what pins the hardware."""
    rng = np.random.default_rng(100 + n)
    p = 16
    X = rng.standard_normal((n, p))
    X[:, 1] = X[:, 0] + 1e-3 * rng.standard_normal(n)
    X[:, 2] = -X[:, 0] + 1e-4 * rng.standard_normal(n)
    X[:, 3] = rng.standard_normal(n) ** 3
    X[:, 4] = np.where(np.arange(n) < 2, 30.0, 1e-3)
    X[:, 5] = np.sign(rng.standard_normal(n))
    X -= X.mean(0)
    X /= np.sqrt((X ** 2).mean(0))
    N = (X ** 2).sum(0) / n
    Y16 = (X / np.sqrt(N)).astype(np.float16)
    R = (X / np.sqrt(N)).T @ (X / np.sqrt(N)) / n
    n_pad = -(-n // 32) * 32
    eps = eps_bound(n_pad)
    term = n_pad * 2.0 ** -22
    worst, worst_acc, worst13 = 0.0, 0.0, 0.0
    for j in range(p):
        for c in range(j, p):
            exact = float(np.dot(Y16[:, j].astype(np.float64), Y16[:, c].astype(np.float64)))
            acc = blockfma_accumulate(Y16[:, j], Y16[:, c])
            worst_acc = max(worst_acc, abs(acc - exact) / n)
            worst = max(worst, abs(acc / n - R[j, c]))
            acc13 = blockfma_accumulate(Y16[:, j], Y16[:, c], bits=13)
            worst13 = max(worst13, abs(acc13 - exact) / n)
    assert worst_acc <= term, (worst_acc, term)
    assert worst <= eps, (worst, eps)
    if n >= 500:
        assert worst13 > term       # the bound does NOT cover a 13-bit accumulator
