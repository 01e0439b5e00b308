"""Multi-device paths on the GPU (one B200 per call here): the C-ABI multi-device fit
(options.num_devices) with one device under both exchanges — NCCL (loaded at run time: the flag
all-reduce and CSC all-gather really execute) and peer-to-peer — the peer-to-peer exchange with
2-5 column blocks sharing the one device (device ids repeat: every block reads its partners'
coefficients and flags from the other blocks' buffers exactly as it would from a peer GPU's
memory; the host meets the blocks between the steps, no kernel waits on another), and
fit_distributed under an NCCL process group of world size 1.  All must equal the single-device
fit bit for bit and the oracle within the parity tolerance (
DESIGN.md §8)."""
import os
import socket

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


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
@pytest.mark.parametrize("cfg,over,solver", [(4, dict(p=1000, family="hub"), "auto"),
                                             (2, {}, "gram"), (2, {}, "residual"),
                                             (5, dict(p=3000), "auto")])
def test_c_abi_multi_device_one_gpu(S, oracle, cfg, over, solver, exchange):
    X, _, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    one = S.fit(X, lam, solver=solver)
    multi = S.fit(X, lam, solver=solver, num_devices=1, exchange=exchange)
    assert multi.stats["num_devices"] == 1 and one.stats["num_devices"] == 0
    assert multi.stats["exchange"] == (1 if exchange == "nccl" else 2)
    assert multi.stats["ms_comm"] > 0.0
    assert np.array_equal(multi.Theta, one.Theta) and np.array_equal(multi.sigma, one.sigma)
    assert np.array_equal(multi.iters, one.iters) and np.array_equal(multi.sweeps, one.sweeps)
    assert np.array_equal(multi.converged, one.converged)
    ora = oracle.spmesl_fit(X, lam)
    assert_parity(compare(multi.Theta, multi.sigma, multi.iters, multi.sweeps, ora))


def test_c_abi_multi_device_errors(S):
    X, _, _ = G.make_config(2)
    with pytest.raises(S.SpmeslError) as e:          # duplicate device ids under NCCL
        S.fit(X, 0.3, num_devices=2, device_ids=[0, 0], exchange="nccl")
    assert e.value.code == -1
    with pytest.raises(S.SpmeslError) as e:          # peer-to-peer: at most 16 blocks
        S.fit(X, 0.3, num_devices=17, device_ids=[0] * 17, exchange="p2p")
    assert e.value.code == -7
    with pytest.raises(S.SpmeslError) as e:          # not a device
        S.fit(X, 0.3, num_devices=1, device_ids=[4096])
    assert e.value.code == -1
    with pytest.raises(S.SpmeslError) as e:          # joint stop: one device only
        S.fit(X, 0.3, num_devices=1, mode="joint")
    assert e.value.code == -7
    S.fit(X, 0.3, num_devices=1)                     # and the library recovers


@pytest.mark.parametrize("cfg,over,solver,nb,kw", [
    (4, dict(p=1000, family="hub"), "auto", 2, {}),
    (4, dict(p=1003, family="band3"), "auto", 3, {}),                 # p % G != 0
    (5, dict(p=3001), "auto", 4, {}),
    (2, {}, "gram", 5, {}),
    (2, {}, "residual", 3, {}),                                      # no screening flags
    (4, dict(p=600, family="hub"), "auto", 2, dict(symmetrize=False)),  # Theta1
    (2, {}, "auto", 3, dict(standardize=False)),                     # no rescale
])
def test_c_abi_p2p_blocks_share_one_gpu(S, oracle, cfg, over, solver, nb, kw):
    """Peer-to-peer exchange with nb column blocks on the one device: the flag max over the
    blocks' screening shares and the symmetrizing assembly that reads each partner b_kj and
    sigma_j from the block owning column j — bit-identical to the single-device fit."""
    X, _, _ = G.make_config(cfg, **over)
    n, p = X.shape
    if not kw.get("standardize", True):
        X = oracle.standardize(X)[0]
    lam = oracle.lambda_ub(n, p)
    one = S.fit(X, lam, solver=solver, **kw)
    multi = S.fit(X, lam, solver=solver, num_devices=nb, device_ids=[0] * nb, exchange="p2p", **kw)
    assert multi.stats["num_devices"] == nb and multi.stats["exchange"] == 2
    assert np.array_equal(multi.Theta, one.Theta) and np.array_equal(multi.sigma, one.sigma)
    assert np.array_equal(multi.iters, one.iters) and np.array_equal(multi.sweeps, one.sweeps)
    assert np.array_equal(multi.converged, one.converged)
    assert multi.stats["nnz"] == one.stats["nnz"]
    ora = oracle.spmesl_fit(X, lam, standardize=kw.get("standardize", True))
    if kw.get("symmetrize", True):
        assert_parity(compare(multi.Theta, multi.sigma, multi.iters, multi.sweeps, ora))
    else:
        d = np.abs(multi.Theta - ora.Theta1)
        assert np.all(d <= 1e-8 * np.abs(ora.Theta1) + 1e-12 * ora.Theta1.diagonal().max())
        assert not np.array_equal(multi.Theta, multi.Theta.T)   # (really unsymmetrized)


def _nccl_worker(port, X, lam, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2203_15031_b200.distributed import fit_distributed
        Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
        s = torch.cuda.Stream()
        r = fit_distributed(Xd, lam, stream=s)
        torch.cuda.synchronize()
        q.put((r["theta"].cpu().numpy(), r["sigma"].cpu().numpy(), r["iters"].cpu().numpy(),
               r["sweeps"].cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_fit_distributed_nccl_world_one(S, oracle):
    """fit_distributed under an NCCL process group (world size 1, on a side stream): the flag
    all-reduce and the CSC all-gather run through NCCL on the B200."""
    import torch.multiprocessing as mp
    X, _, _ = G.make_config(4, p=1200, family="hub")
    lam = oracle.lambda_ub(*X.shape)
    full = S.fit(X, lam)
    sk = socket.socket(); sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]; sk.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_worker, args=(port, X, lam, q))
    pr.start()
    th, sg, it, sw = q.get(timeout=300)
    pr.join(timeout=60)
    assert pr.exitcode == 0
    assert np.array_equal(th, full.Theta) and np.array_equal(sg, full.sigma)
    assert np.array_equal(it, full.iters) and np.array_equal(sw, full.sweeps)
    ora = oracle.spmesl_fit(X, lam)
    assert_parity(compare(th, sg, it, sw, ora))
