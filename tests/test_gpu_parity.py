"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
on the same seeded inputs.  Needs a B200 (marker gpu)."""
import math

import numpy as np
import pytest

from synth import generators as G
from tests.parity import assert_parity, compare
from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_15031_b200 as S
    S.load()
    return S


def _lam(oracle, rule, n, p):
    return {"univ": oracle.lambda_univ, "ub": oracle.lambda_ub}[rule](n, p)


CASES = [
    # (config, overrides, rule)
    (1, {}, "univ"),
    (1, {}, "ub"),
    (2, {}, "univ"),
    (2, {}, "ub"),
    (3, {}, "ub"),
    (3, {}, "univ"),
    (4, dict(p=1000), "ub"),
    (4, dict(p=1000, family="hub"), "ub"),
    (4, dict(p=777, n=203), "univ"),          # ragged p and n (not multiples of 32)
    (5, dict(p=1500), "ub"),
]


@pytest.mark.parametrize("cfg,over,rule", CASES)
@pytest.mark.parametrize("delta", [1e-4, 1e-10])
@pytest.mark.parametrize("solver", ["residual", "gram", "gram16"])
def test_parity_host_api(S, oracle, cfg, over, rule, delta, solver):
    X, gt, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = _lam(oracle, rule, n, p)
    ora = oracle.spmesl_fit(X, lam, delta=delta)
    res = S.fit(X, lam, tol=delta, max_iter=100, solver=solver)
    assert res.stats["solver"] == {"residual": 1, "gram": 2, "gram16": 3}[solver]
    rep = compare(res.Theta, res.sigma, res.iters, res.sweeps, ora)
    print(cfg, over, rule, delta, rep)
    assert_parity(rep)
    assert np.array_equal(res.converged, ora.converged)
    assert np.array_equal(res.Theta, res.Theta.T)
    st = res.stats
    assert st["coord_updates"] == int(ora.sweeps.sum()) * (p - 1)


@pytest.mark.parametrize("T", [8, 16, 32])
def test_bit_identical_across_tile_sizes(S, oracle, T):
    X, _, _ = G.make_config(4, p=600, family="hub")
    lam = oracle.lambda_ub(*X.shape)
    ref = S.fit(X, lam, tile_cols=8, solver="residual")
    r = S.fit(X, lam, tile_cols=T, solver="residual")
    assert np.array_equal(r.Theta, ref.Theta)
    assert np.array_equal(r.sigma, ref.sigma)
    assert np.array_equal(r.sweeps, ref.sweeps)


@pytest.mark.parametrize("solver", ["residual", "gram", "gram16", "auto"])
def test_theta1_unsymmetrized_and_unstandardized(S, oracle, solver):
    X, _, _ = G.make_config(2)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    ora = oracle.spmesl_fit(X, lam)
    r = S.fit(X, lam, symmetrize=False, solver=solver)
    d = np.abs(r.Theta - ora.Theta1)
    assert np.all(d <= 1e-8 * np.abs(ora.Theta1) + 1e-12 * ora.Theta1.diagonal().max())
    Xs, mu, s = oracle.standardize(X)
    ora2 = oracle.spmesl_fit(Xs, lam, standardize=False)
    r2 = S.fit(Xs, lam, standardize=False, solver=solver)
    assert_parity(compare(r2.Theta, r2.sigma, r2.iters, r2.sweeps, ora2))


def test_device_api_and_stream(S, oracle):
    import torch
    X, _, _ = G.make_config(3)
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    ora = oracle.spmesl_fit(X, lam)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()   # column-major (n, p)
    s = torch.cuda.Stream()
    r = S.fit_device(Xd, lam, stream=s)
    rep = compare(r.Theta.cpu().numpy(), r.sigma.cpu().numpy(), r.iters.cpu().numpy(),
                  r.sweeps.cpu().numpy(), ora)
    assert_parity(rep)
    # a row-major tensor is accepted too (copied to column-major)
    r2 = S.fit_device(torch.from_numpy(np.ascontiguousarray(X)).cuda(), lam)
    assert torch.equal(r2.Theta, r.Theta)


def test_column_blocks_reproduce_full_fit(S, oracle):
    """The multi-GPU building blocks: CSC of column blocks + assembly == single fit, bitwise."""
    import torch
    X, _, _ = G.make_config(4, p=900, family="hub")
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    full = S.fit(X, lam, solver="residual")
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    bounds = [0, 250, 251, 600, 900]
    parts = [S.fit_columns_device(Xd, a, b, lam) for a, b in zip(bounds[:-1], bounds[1:])]
    counts = torch.cat([q["counts"] for q in parts]).long()
    col_ptr = torch.zeros(p + 1, dtype=torch.int64, device="cuda")
    col_ptr[1:] = torch.cumsum(counts, 0)
    rows = torch.cat([q["rows"] for q in parts])
    vals = torch.cat([q["vals"] for q in parts])
    sig = torch.cat([q["sigma_std"] for q in parts])
    scale = parts[0]["scale"]
    th, so = S.assemble_device(p, 0, p, col_ptr, rows, vals, sig, scale)
    assert np.array_equal(th.cpu().numpy(), full.Theta)
    assert np.array_equal(so.cpu().numpy(), full.sigma)
    th2, so2 = S.assemble_device(p, 300, 700, col_ptr, rows, vals, sig, scale)
    assert np.array_equal(th2.cpu().numpy(), full.Theta[:, 300:700])


@pytest.mark.parametrize("solver", ["residual", "gram", "gram16", "auto"])
def test_null_case_and_small_p(S, oracle, solver):
    rng = np.random.default_rng(5)
    for (n, p) in [(7, 2), (33, 3), (64, 31), (65, 33), (40, 129)]:
        X = rng.standard_normal((n, p)) * rng.uniform(0.5, 2, p)
        for lam in (0.05, 0.3, 5.0):
            ora = oracle.spmesl_fit(X, lam)
            r = S.fit(X, lam, solver=solver)
            assert_parity(compare(r.Theta, r.sigma, r.iters, r.sweeps, ora))


@pytest.mark.parametrize("solver", ["residual", "gram", "gram16", "auto"])
def test_errors(S, solver):
    X = np.random.default_rng(1).standard_normal((20, 40))
    X[:, 17] = 2.5
    with pytest.raises(S.SpmeslError) as e:
        S.fit(X, 0.3, solver=solver)
    assert e.value.code == -2 and e.value.bad_column == 17
    X[:, 17] = np.arange(20)
    X[3, 30] = np.inf
    X[0, 35] = np.nan
    with pytest.raises(S.SpmeslError) as e:
        S.fit(X, 0.3, solver=solver)
    assert e.value.code == -3 and e.value.bad_column == 30
    # the library recovers after an error
    X[3, 30] = 1.0
    X[0, 35] = 1.0
    S.fit(X, 0.3, solver=solver)


@pytest.mark.parametrize("solver", ["residual", "gram", "gram16", "auto"])
def test_max_iter_cap_flags_columns(S, oracle, solver):
    X, _, _ = G.make_config(2)
    lam = oracle.lambda_univ(*X.shape)
    ora = oracle.spmesl_fit(X, lam, max_outer=2)
    r = S.fit(X, lam, max_iter=2, solver=solver)
    assert r.code == 1 and not r.converged.all()
    assert np.array_equal(r.converged, ora.converged)
    assert_parity(compare(r.Theta, r.sigma, r.iters, r.sweeps, ora))


@pytest.mark.parametrize("solver", ["residual", "gram", "gram16"])
def test_full_size_config5_sampled_columns(S, oracle, solver):
    """BASELINE config 5 at full size (n=500, p=20000) in the bench's launch configuration;
    the oracle solves a sample of columns one by one (each column is independent): random
    columns plus every column that needed more than one sweep (at most 40 of them)."""
    X, _, spec = G.make_config(5)
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    r = S.fit(X, lam, symmetrize=False, solver=solver)   # Theta1: column k depends on k only
    rng = np.random.default_rng(0)
    multi = np.nonzero(r.sweeps > 1)[0][:40]
    cols = np.unique(np.concatenate([rng.choice(p, 48, replace=False), multi]))
    Xs, mu, s = oracle.standardize(X)
    oc = oracle.spmesl_columns(Xs, cols, lam, want_margin=False)
    assert np.array_equal(r.iters[cols], oc.outer) and np.array_equal(r.sweeps[cols], oc.sweeps)
    np.testing.assert_allclose(r.sigma[cols], oc.sigma * s[cols], rtol=1e-10)
    for c, k in enumerate(cols):
        want = np.zeros(p)
        want[:] = -oc.B[:, c] * (1.0 / (oc.sigma[c] * oc.sigma[c]))
        want[k] = 1.0 / (oc.sigma[c] * oc.sigma[c])
        want = want / (s * s[k])
        got = r.Theta[:, k]
        assert np.all(np.abs(got - want) <= 1e-8 * np.abs(want) + 1e-12 * abs(want[k])), k


def _rank_worker(rank, world, port, X, lam, q, solver):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2203_15031_b200.distributed import fit_distributed
        Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
        r = fit_distributed(Xd, lam, solver=solver)
        q.put((rank, r["col_range"], r["theta"].cpu().numpy(), r["sigma"].cpu().numpy(),
               r["iters"].cpu().numpy(), r["sweeps"].cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("solver", ["residual", "gram", "auto"])
def test_two_ranks_sharing_one_gpu_match_single_fit(S, oracle, solver):
    """fit_distributed (column blocks + CSC all-gather + per-rank assembly; for the Gram solver
    also the tile-share screening + flag all-reduce) on 2 ranks that share cuda:0 over gloo
    must reproduce the single-GPU fit bit for bit."""
    import socket
    import torch.multiprocessing as mp
    X, _, _ = G.make_config(4, p=1200, family="hub")
    lam = oracle.lambda_ub(*X.shape)
    full = S.fit(X, lam, solver=solver)
    sk = socket.socket(); sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]; sk.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, port, X, lam, q, solver))
             for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    ora = oracle.spmesl_fit(X, lam)
    for rank, (c0, c1), th, sg, it, sw in res:
        assert np.array_equal(th, full.Theta[:, c0:c1])
        assert np.array_equal(sg, full.sigma[c0:c1])
        assert np.array_equal(it, full.iters[c0:c1]) and np.array_equal(sw, full.sweeps[c0:c1])
        # each rank's column block against the oracle directly
        cols = np.arange(c0, c1)
        rep = compare(np.concatenate([np.zeros((th.shape[0], c0)), th,
                                      np.zeros((th.shape[0], X.shape[1] - c1))], axis=1),
                      np.concatenate([ora.sigma[:c0], sg, ora.sigma[c1:]]),
                      np.concatenate([ora.outer[:c0], it, ora.outer[c1:]]),
                      np.concatenate([ora.sweeps[:c0], sw, ora.sweeps[c1:]]), ora, cols=cols)
        assert_parity(rep)


@pytest.mark.parametrize("tail_after", [0, 1, 3])
def test_tail_solver_handoff_points(S, oracle, tail_after):
    """Columns needing several sweeps are finished by the covariance-update tail solver after
    `tail_after` sweeps (0: never); every hand-off point must reproduce the oracle."""
    X, _, _ = G.make_config(4, p=700, n=300, family="hub")
    lam = oracle.lambda_ub(*X.shape)
    ora = oracle.spmesl_fit(X, lam)
    r = S.fit(X, lam, tail_after=tail_after, solver="residual")
    assert_parity(compare(r.Theta, r.sigma, r.iters, r.sweeps, ora))
    if tail_after == 0:
        assert r.stats["tail_columns"] == 0
    else:
        assert r.stats["tail_columns"] > 0


def test_tail_solver_on_demand_gram_columns(S, oracle):
    """Few handed-over columns -> only their active variables get precomputed Gram columns;
    a variable entering later is computed on first use (same DMMA routine).  Config 5 family at
    p = 8000: the columns that needed more than one sweep (the tail) are checked one by one
    against the oracle."""
    X, _, _ = G.make_config(5, p=8000)
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    r = S.fit(X, lam, symmetrize=False, solver="residual")
    assert r.stats["tail_columns"] > 0 and r.stats["tail_gram_ondemand"] > 0
    cols = np.nonzero(r.sweeps > 1)[0]
    assert len(cols) == r.stats["tail_columns"]
    Xs, mu, s = oracle.standardize(X)
    oc = oracle.spmesl_columns(Xs, cols, lam, want_margin=False)
    assert np.array_equal(r.iters[cols], oc.outer) and np.array_equal(r.sweeps[cols], oc.sweeps)
    np.testing.assert_allclose(r.sigma[cols], oc.sigma * s[cols], rtol=1e-10)
    for c, k in enumerate(cols):
        w = 1.0 / (oc.sigma[c] * oc.sigma[c])
        want = -oc.B[:, c] * w
        want[k] = w
        want = want / (s * s[k])
        got = r.Theta[:, k]
        assert np.array_equal(got != 0, want != 0), k
        assert np.all(np.abs(got - want) <= 1e-8 * np.abs(want) + 1e-12 * abs(want[k])), k


@pytest.mark.parametrize("solver", ["residual", "gram", "gram16", "auto"])
@pytest.mark.parametrize("mi", [1, 100])
def test_unstandardized_scaled_columns_and_caps(S, oracle, solver, mi):
    # standardize = 0 with column norms ||x_k||^2 / n in [0.64, 1.44] (sigma of a column whose
    # first sweep changes nothing is then not 1, so it continues) and max_iter = 1.  (Unit-step
    # CD assumes x_j^T x_j = n; norms far from that make both sides diverge alike.)
    X, gt, spec = G.make_config(2)
    n, p = X.shape
    Xs, _, _ = oracle.standardize(X)
    Xs = Xs * np.linspace(0.8, 1.2, p)[None, :]
    lam = oracle.lambda_univ(n, p)
    if True:
        ora = oracle.spmesl_fit(Xs, lam, delta=1e-4, max_outer=mi, standardize=False)
        res = S.fit(Xs, lam, tol=1e-4, max_iter=mi, standardize=False, solver=solver)
        rep = compare(res.Theta, res.sigma, res.iters, res.sweeps, ora)
        print(solver, mi, rep)
        assert_parity(rep)
        assert np.array_equal(res.converged, ora.converged)


@pytest.mark.parametrize("solver", ["gram", "gram16"])
def test_gram_building_blocks_reproduce_full_fit(S, oracle, solver):
    """Screening in tile shares + Gram column blocks + assembly == the single Gram fit (gram16:
    the shares flag candidates, each column block decides its own exactly)."""
    import torch
    X, _, _ = G.make_config(4, p=900, family="hub")
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    full = S.fit(X, lam, solver="gram")
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    nt = S.gram_tile_count(p, solver=solver)
    hit = torch.zeros(p, dtype=torch.uint8, device="cuda")
    for a, b in [(0, nt // 3), (nt // 3, nt // 3), (nt // 3, nt)]:
        S.gram_screen_device(Xd, lam, a, b, hit, solver=solver)
    if solver == "gram16":   # candidates: a superset of the exact hits of the FP64 screening
        exact = torch.zeros(p, dtype=torch.uint8, device="cuda")
        S.gram_screen_device(Xd, lam, 0, S.gram_tile_count(p), exact, solver="gram")
        assert bool(((exact == 1) <= (hit == 1)).all())
    bounds = [0, 250, 251, 600, 900]
    parts = [S.fit_columns_gram_device(Xd, a, b, lam, hit, solver=solver)
             for a, b in zip(bounds[:-1], bounds[1:])]
    counts = torch.cat([q["counts"] for q in parts]).long()
    col_ptr = torch.zeros(p + 1, dtype=torch.int64, device="cuda")
    col_ptr[1:] = torch.cumsum(counts, 0)
    rows = torch.cat([q["rows"] for q in parts])
    vals = torch.cat([q["vals"] for q in parts])
    sig = torch.cat([q["sigma_std"] for q in parts])
    th, so = S.assemble_device(p, 0, p, col_ptr, rows, vals, sig, parts[0]["scale"])
    it = torch.cat([q["iters"] for q in parts]).cpu().numpy()
    sw = torch.cat([q["sweeps"] for q in parts]).cpu().numpy()
    assert np.array_equal(it, full.iters) and np.array_equal(sw, full.sweeps)
    assert np.array_equal(so.cpu().numpy(), full.sigma)
    assert np.array_equal(th.cpu().numpy(), full.Theta)


@pytest.mark.parametrize("solver", ["gram", "residual"])
def test_penalty_path_equals_single_fits(S, oracle, solver):
    """spmesl_fit_path_device: lambda_pb, lambda_univ, lambda_ub (SPMESL-P/-2/-4) in
    one call; every level equals its own single fit (bit for bit with the Gram solver) and the
    oracle."""
    import torch
    X, _, _ = G.make_config(2, p=300, n=150)
    n, p = X.shape
    lams = [oracle.lambda_pb(n, p), oracle.lambda_univ(n, p), oracle.lambda_ub(n, p)]
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    res = S.fit_path_device(Xd, lams, solver=solver)
    for lam, r in zip(lams, res):
        one = S.fit_device(Xd, lam, solver=solver)
        assert torch.equal(r.Theta, one.Theta) and torch.equal(r.sigma, one.sigma)
        assert torch.equal(r.sweeps, one.sweeps) and torch.equal(r.iters, one.iters)
        ora = oracle.spmesl_fit(X, lam)
        assert_parity(compare(r.Theta.cpu().numpy(), r.sigma.cpu().numpy(),
                              r.iters.cpu().numpy(), r.sweeps.cpu().numpy(), ora))
    # levels are independent of their order in the call
    rev = S.fit_path_device(Xd, lams[::-1], solver=solver)
    for a, b in zip(res, rev[::-1]):
        assert torch.equal(a.Theta, b.Theta)


def test_estimation_workload_ar1_matches_paper_band(S):
    """f4: the estimation workload (one penalty-path fit per dataset, three levels) on the
    paper's AR(1) setting (p = 500, n = 250): SPMESL-4 recovers every edge with FDR near the
    paper's 1.07 % (Table 3); SPMESL-P has the most false discoveries."""
    from workloads.estimation import run
    r = run(reps=2, networks=["ar1_paper"])["ar1_paper"]
    assert r["SPMESL-4"]["SEN"] == 100.0 and r["SPMESL-4"]["FDR"] <= 4.0
    assert r["SPMESL-P"]["FDR"] > r["SPMESL-2"]["FDR"] > r["SPMESL-4"]["FDR"]
    assert r["SPMESL-P"]["Frob"] < r["SPMESL-4"]["Frob"]


@pytest.mark.parametrize("family", ["band3", "hub"])
def test_full_size_config4_slowest_columns(S, oracle, family):
    """BASELINE config 4 at full size (n = 400, p = 5000; band(3) and hub): the 6 columns that
    needed the most sweeps (the stragglers, up to ~490 sweeps for hub graphs) and 10 random ones
    are solved one by one by the oracle; counts identical, sigma and Theta_1 within tolerance."""
    X, _, spec = G.make_config(4, family=family)
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    r = S.fit(X, lam, symmetrize=False)
    rng = np.random.default_rng(1)
    slow = np.argsort(-r.sweeps)[:6]
    cols = np.unique(np.concatenate([slow, rng.choice(p, 10, replace=False)]))
    Xs, mu, s = oracle.standardize(X)
    oc = oracle.spmesl_columns(Xs, cols, lam, want_margin=False)
    assert r.sweeps[slow].max() == oc.sweeps.max() and r.sweeps[slow].min() > 10
    assert np.array_equal(r.iters[cols], oc.outer) and np.array_equal(r.sweeps[cols], oc.sweeps)
    np.testing.assert_allclose(r.sigma[cols], oc.sigma * s[cols], rtol=1e-10)
    for c, k in enumerate(cols):
        w = 1.0 / (oc.sigma[c] * oc.sigma[c])
        want = -oc.B[:, c] * w
        want[k] = w
        want = want / (s * s[k])
        got = r.Theta[:, k]
        assert np.all(np.abs(got - want) <= 1e-8 * np.abs(want) + 1e-12 * abs(want[k])), k


def test_certified_screening_equals_full_gram(S):
    """solver 3 (f16 screening certified by an error bound + exact FP64 Gram columns of the
    candidates) gives bit-identical results to solver 2 (the full FP64 S) — the low-precision
    pass only decides which columns need no exact work — on screening-dominated (ER) and
    multi-sweep (band, hub) workloads, including the penalty path."""
    import torch
    for cfg, over in [(5, dict(p=6000)), (4, dict(p=1500)), (4, dict(p=1500, family="hub")),
                      (3, {})]:
        X, _, spec = G.make_config(cfg, **over)
        n, p = X.shape
        Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
        lam = S.lambda_ub(n, p)
        a = S.fit_device(Xd, lam, solver="gram")
        b = S.fit_device(Xd, lam, solver="gram16")
        assert b.stats["solver"] == 3 and b.stats["screen_candidates"] >= b.stats["tail_columns"] - 0
        assert torch.equal(a.Theta, b.Theta) and torch.equal(a.sweeps, b.sweeps)
        # the fallback to the full FP64 Gram kernel is taken on the device above p/4 or 1024
        # candidates; the screening kernel zero-fills all of Theta (default split)
        nc = b.stats["screen_candidates"]
        assert b.stats["gram_fallback"] == int(4 * nc > p or nc > 1024)
        assert b.stats["screen_fill_bytes"] == 8 * p * p and b.stats["ms_screen"] > 0
        lams = [S.lambda_pb(n, p), S.lambda_univ(n, p), lam]
        pa = S.fit_path_device(Xd, lams, solver="gram")
        pb = S.fit_path_device(Xd, lams, solver="gram16")
        for x, y in zip(pa, pb):
            assert torch.equal(x.Theta, y.Theta) and torch.equal(x.sweeps, y.sweeps)


def test_graph_replay_matches_eager(S, oracle):
    """spmesl_fit_device with the same arguments: the second call captures the enqueued fit as
    a CUDA graph and later calls replay it; every replay equals the eager fit bit for bit, and
    a replay reads the current contents of X (new data at the same address -> new result)."""
    import torch
    X, _, _ = G.make_config(5, p=3000)
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()

    def outs():
        return dict(theta=torch.empty((p, p), dtype=torch.float64, device="cuda"),
                    sigma=torch.empty(p, dtype=torch.float64, device="cuda"),
                    iters=torch.empty(p, dtype=torch.int32, device="cuda"),
                    sweeps=torch.empty(p, dtype=torch.int32, device="cuda"),
                    conv=torch.empty(p, dtype=torch.uint8, device="cuda"))

    ref = S.fit_device(Xd, lam, out=outs(), eager=True)
    ref = [t.clone() for t in (ref.Theta, ref.sigma, ref.iters, ref.sweeps)]
    out = outs()
    flags = []
    for _ in range(4):
        r = S.fit_device(Xd, lam, out=out)
        flags.append(r.stats["graph_replay"])
        got = (r.Theta, r.sigma, r.iters, r.sweeps)
        assert all(torch.equal(a, b) for a, b in zip(got, ref))
        assert r.stats["ms_total"] > 0 and r.stats["ms_screen"] > 0
    assert flags == [0, 1, 1, 1]
    # new data in the same buffer: the replay must see it
    X2, _, _ = G.make_config(5, p=3000, seed=7)
    Xd.copy_(torch.from_numpy(np.ascontiguousarray(X2.T)).cuda().t())
    r = S.fit_device(Xd, lam, out=out)
    assert r.stats["graph_replay"] == 1
    e = S.fit_device(Xd, lam, out=outs(), eager=True)
    assert torch.equal(r.Theta, e.Theta) and torch.equal(r.sweeps, e.sweeps)


@pytest.mark.parametrize("solver,mode,cfg,over,sym", [
    ("auto", "per_column", 5, dict(p=3000), True),
    ("auto", "per_column", 4, dict(p=777, n=203), True),     # ragged, multi-sweep
    ("residual", "per_column", 2, {}, True),
    ("auto", "per_column", 2, {}, False),                    # Theta_1 (unsymmetrized)
    ("auto", "joint", 4, dict(p=300, n=150, family="hub"), True),
])
def test_sparse_output_equals_dense(S, oracle, solver, mode, cfg, over, sym):
    """spmesl_fit_sparse_device (§8(f) f3): Theta as CSC without the dense array equals the
    dense device fit entry for entry (bit for bit), rows ascending, diagonal present."""
    import torch
    X, _, _ = G.make_config(cfg, **over)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda().t()
    dense = S.fit_device(Xd, lam, solver=solver, mode=mode, symmetrize=sym, eager=True)
    sp = S.fit_sparse_device(Xd, lam, solver=solver, mode=mode, symmetrize=sym, cap=p + 4)
    cp, rows, vals = sp["col_ptr"].cpu().numpy(), sp["rows"].cpu().numpy(), sp["vals"].cpu().numpy()
    assert cp[0] == 0 and cp[-1] == len(rows)
    for k in range(p):
        r = rows[cp[k]:cp[k + 1]]
        assert np.all(np.diff(r) > 0) and k in r
    T = S.sparse_to_dense(sp["col_ptr"], sp["rows"], sp["vals"], p)
    assert torch.equal(T, dense.Theta)
    assert torch.equal(sp["sigma"], dense.sigma) and torch.equal(sp["sweeps"], dense.sweeps)
    assert sp["stats"]["nnz"] == len(rows) - p


@pytest.mark.parametrize("solver", ["residual", "gram", "gram16"])
def test_degenerate_penalties_closed_forms(S, oracle, solver):
    """lambda0 = 0 (allowed: S:42-44 rejects only lambda0 < 0): every column regression is plain
    least squares, so at convergence Theta_1 = S_n^{-1}, the inverse sample covariance with
    divisor n (Eq. relation P:268-272 with sigma_k^2 = RSS_k/n; Prop. 1 P:312-365 for the
    original scale) — symmetric already, so the symmetrization keeps it.  lambda0 above every
    |x~_j^T x~_k|/n: B = 0, sigma = 1 on the standardized scale, Theta = diag(1/s_k^2)."""
    rng = np.random.default_rng(11)
    n, p = 400, 24
    X = rng.standard_normal((n, p)) @ (np.eye(p) + 0.1 * rng.standard_normal((p, p))) \
        * rng.uniform(0.5, 2.0, p)
    Xc = X - X.mean(axis=0)
    Sn = Xc.T @ Xc / n
    r = S.fit(X, 0.0, tol=1e-10, max_iter=100, solver=solver)
    assert np.all(r.converged)
    inv = np.linalg.inv(Sn)              # (condition number of the correlation matrix ~ 3)
    assert np.abs(r.Theta - inv).max() <= 1e-8 * np.abs(inv).max()
    ora = oracle.spmesl_fit(X, 0.0, delta=1e-10)
    assert_parity(compare(r.Theta, r.sigma, r.iters, r.sweeps, ora))
    big = 1.5 * np.abs(np.corrcoef(X, rowvar=False) - np.eye(p)).max()
    r = S.fit(X, big, solver=solver)
    np.testing.assert_allclose(r.Theta, np.diag(1.0 / Sn.diagonal()), rtol=1e-12, atol=0)
    assert np.all(r.iters <= 2)


@pytest.mark.parametrize("solver", ["residual", "gram", "gram16", "auto"])
def test_sigma_floor_binds(S, oracle, solver):
    """The sigma floor (reading g5) applied identically on both sides where it binds:
    sigma_floor = 0.9 on config 2 at lambda_univ clamps the columns whose residual scale
    ||r||/sqrt(n) falls below 0.9 (their lambda is then 0.9 lambda0)."""
    X, _, _ = G.make_config(2)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    ora = oracle.spmesl_fit(X, lam, sigma_floor=0.9)
    Xs, mu, s = oracle.standardize(X)
    clamped = np.isclose(ora.sigma / s, 0.9, rtol=0, atol=1e-15)
    assert clamped.sum() > 10, clamped.sum()          # the floor really binds
    r = S.fit(X, lam, sigma_floor=0.9, solver=solver)
    assert_parity(compare(r.Theta, r.sigma, r.iters, r.sweeps, ora))
    # and the unclamped fit differs on those columns (the branch changes the result)
    free = oracle.spmesl_fit(X, lam)
    assert np.any(free.sigma[clamped] < ora.sigma[clamped])


@pytest.mark.parametrize("solver", ["residual", "gram16"])
def test_near_constant_column_rule(S, oracle, solver):
    """The constant-column rule s_k <= 1e-13 max_i |x_ik| (reading g15) on both sides: a
    column 10x below the threshold is an error (the same column on both sides), one 10x above
    is fitted without error by both."""
    rng = np.random.default_rng(3)
    n, p = 100, 40
    X = rng.standard_normal((n, p))
    for a, constant in ((1e-14, True), (1e-12, False)):
        Y = X.copy()
        Y[:, 13] = 1.0 + a * rng.standard_normal(n)
        if constant:
            with pytest.raises(oracle.OracleError) as eo:
                oracle.spmesl_fit(Y, 0.3)
            with pytest.raises(S.SpmeslError) as eg:
                S.fit(Y, 0.3, solver=solver)
            assert eo.value.code == -2 and eg.value.code == -2
            assert eo.value.bad_col == 13 and eg.value.bad_column == 13
        else:
            ora = oracle.spmesl_fit(Y, 0.3)
            r = S.fit(Y, 0.3, solver=solver)
            assert ora.code >= 0 and r.code >= 0
            assert np.all(np.isfinite(r.Theta)) and np.all(np.isfinite(r.sigma))


def _bare_fit(S, X, lam, tol=1e-4, max_iter=100):
    """spmesl_fit (the BASELINE.json signature) through ctypes with host buffers."""
    import ctypes
    X = np.asfortranarray(X, dtype=np.float64)
    n, p = X.shape
    Theta = np.empty((p, p), order="F")
    sigma = np.empty(p)
    iters = np.empty(p, np.int32)
    rc = S.load().spmesl_fit(ctypes.c_void_p(X.ctypes.data), n, p, float(lam), float(tol),
                             int(max_iter), ctypes.c_void_p(Theta.ctypes.data),
                             ctypes.c_void_p(sigma.ctypes.data), ctypes.c_void_p(iters.ctypes.data))
    return rc, Theta, sigma, iters


@pytest.mark.parametrize("cfg,over", [(2, {}), (5, dict(p=3000))])
def test_bare_spmesl_fit_signature(S, oracle, cfg, over):
    X, _, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p) if spec["rule"] == "univ" else oracle.lambda_ub(n, p)
    ora = oracle.spmesl_fit(X, lam)
    rc, Theta, sigma, iters = _bare_fit(S, X, lam)
    assert rc == (1 if not ora.converged.all() else 0)
    assert np.array_equal(iters, ora.outer)
    # (sweeps are not returned by the bare signature: iters + Theta + sigma are compared)
    rep = compare(Theta, sigma, iters, ora.sweeps, ora)
    rep["sweeps_mismatch"] = []
    assert_parity(rep)


def test_bare_spmesl_fit_status_codes(S, oracle):
    """Every status code the BASELINE-signature entry point can return on this path."""
    X, _, _ = G.make_config(2)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    assert _bare_fit(S, X, lam)[0] == 0                               # SPMESL_OK
    rc, _, _, iters = _bare_fit(S, X, lam, max_iter=1)                # outer cap hit
    assert rc == 1 and iters.max() == 1                               # SPMESL_WARN_NOT_CONVERGED
    assert _bare_fit(S, X, -1.0)[0] == -1                             # SPMESL_ERR_ARG
    assert _bare_fit(S, X, lam, tol=0.0)[0] == -1
    assert _bare_fit(S, X, lam, max_iter=0)[0] == -1
    assert _bare_fit(S, X[:1], lam)[0] == -1                          # n < 2
    Y = X.copy()
    Y[:, 7] = 3.0
    assert _bare_fit(S, Y, lam)[0] == -2                              # SPMESL_ERR_CONSTANT_COLUMN
    Y = X.copy()
    Y[5, 9] = np.nan
    assert _bare_fit(S, Y, lam)[0] == -3                              # SPMESL_ERR_NONFINITE
    assert _bare_fit(S, X, lam)[0] == 0                               # and it recovers


@pytest.mark.parametrize("cfg,over", [(2, {}), (5, dict(p=3000))])
def test_host_sparse_entry_point(S, oracle, cfg, over):
    """spmesl_fit_sparse (host X, Theta as host CSC): every entry equals the dense host fit's,
    which the oracle checks; a capacity that is too small reports the count needed."""
    X, _, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = oracle.lambda_univ(n, p)
    dense = S.fit(X, lam)
    sp = S.fit_sparse(X, lam, cap=p + 4)       # (retried with the count needed)
    cp, rows, vals = sp["col_ptr"], sp["rows"], sp["vals"]
    assert cp[0] == 0 and cp[-1] == len(rows)
    T = np.zeros((p, p))
    for k in range(p):
        r = rows[cp[k]:cp[k + 1]]
        assert np.all(np.diff(r) > 0) and k in r
        T[r, k] = vals[cp[k]:cp[k + 1]]
    assert np.array_equal(T, dense.Theta)
    assert np.array_equal(sp["sigma"], dense.sigma) and np.array_equal(sp["iters"], dense.iters)
    assert np.array_equal(sp["sweeps"], dense.sweeps)
    ora = oracle.spmesl_fit(X, lam)
    assert_parity(compare(T, sp["sigma"], sp["iters"], sp["sweeps"], ora))
