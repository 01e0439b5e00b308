"""Column-block sharding host logic on CPU: world_size 2 over gloo (127.0.0.1).

Each rank fits its contiguous block of columns (with the oracle here — these CPU tests
check the partition and the CSC all-gather, not the kernels) and all-gathers the
nonzeros; the gathered CSC must equal the CSC of a single full fit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_15031_b200.distributed import column_range, gather_csc


def test_column_range_partition():
    for p in (2, 3, 7, 20, 1000, 20001):
        for world in (1, 2, 3, 4, 8):
            if world > p:
                continue
            blocks = [column_range(p, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == p
            for (a0, a1), (b0, b1) in zip(blocks[:-1], blocks[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def _csc_of(B):
    counts, rows, vals = [], [], []
    for c in range(B.shape[1]):
        nz = np.nonzero(B[:, c])[0]
        counts.append(len(nz))
        rows.extend(nz.tolist())
        vals.extend(B[nz, c].tolist())
    return (np.array(counts, np.int32), np.array(rows, np.int32), np.array(vals, np.float64))


def _worker(rank, world, port, Xs, lam, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        p = Xs.shape[1]
        c0, c1 = column_range(p, rank, world)
        r = O.spmesl_columns(Xs, np.arange(c0, c1), lam, want_margin=False)
        cnt, rows, vals = _csc_of(r.B)
        col_ptr, grows, gvals, gsig = gather_csc(
            p, torch.from_numpy(cnt), torch.from_numpy(rows), torch.from_numpy(vals),
            torch.from_numpy(r.sigma), None)
        out_q.put((rank, col_ptr.numpy(), grows.numpy(), gvals.numpy(), gsig.numpy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_gather_csc_matches_single_fit(oracle, world):
    from synth import generators as G
    X, _, _ = G.make_config(4, p=157, n=120, family="hub")
    Xs, mu, s = oracle.standardize(X)
    lam = oracle.lambda_univ(*X.shape)
    full = oracle.spmesl_columns(Xs, np.arange(X.shape[1]), lam, want_margin=False)
    cnt, rows, vals = _csc_of(full.B)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, Xs, lam, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    want_ptr = np.concatenate([[0], np.cumsum(cnt)])
    assert rows.size > 0
    for rank, col_ptr, grows, gvals, gsig in res:
        np.testing.assert_array_equal(col_ptr, want_ptr)
        np.testing.assert_array_equal(grows, rows)
        np.testing.assert_array_equal(gvals, vals)
        np.testing.assert_array_equal(gsig, full.sigma)


def _hits_worker(rank, world, port, Xs, lam, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_15031_b200.distributed import allreduce_hits, tile_range
        n, p = Xs.shape
        S = Xs.T @ Xs / n
        np.fill_diagonal(S, 0.0)
        # this rank's share of the (column-pair) work: a contiguous block of rows of S
        r0, r1 = tile_range(p, rank, world)
        hit = np.zeros(p, np.uint8)
        blk = np.abs(S[r0:r1, :]) > lam          # (j in share, c): S is symmetric
        hit[np.any(blk, axis=0)] = 1              # column c hit through row j
        hit[r0:r1][np.any(blk, axis=1)] = 1       # the mirror entries (c, j)
        t = torch.from_numpy(hit)
        allreduce_hits(t, None)
        out_q.put((rank, t.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allreduce_hits_is_the_global_screen(oracle, world):
    """The max-all-reduce of per-rank screening flags equals the screening of the full S."""
    from synth import generators as G
    X, _, _ = G.make_config(3, p=300, n=150)
    Xs, mu, s = oracle.standardize(X)
    lam = oracle.lambda_univ(*X.shape)
    S = Xs.T @ Xs / X.shape[0]
    np.fill_diagonal(S, 0.0)
    want = np.any(np.abs(S) > lam, axis=0).astype(np.uint8)
    assert 0 < want.sum() < want.size
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hits_worker, args=(r, world, port, Xs, lam, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, hit in res:
        np.testing.assert_array_equal(hit, want)
