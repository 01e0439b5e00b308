"""Multi-device paths on the GPU (one B200 per call here): the C-ABI multi-device fit
(options.num_devices, NCCL loaded at run time) with one device — so the NCCL data path (flag
all-reduce, CSC all-gather) really executes — and fit_distributed under an NCCL process group of
world size 1.  Both must equal the single-device fit bit for bit and the oracle within the
parity tolerance."""
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


@pytest.mark.parametrize("cfg,over,solver", [(4, dict(p=1000, family="hub"), "auto"),
                                             (2, {}, "gram"), (2, {}, "residual"),
                                             (5, dict(p=3000), "auto")])
def test_c_abi_multi_device_one_gpu(S, oracle, cfg, over, solver):
    X, _, spec = G.make_config(cfg, **over)
    n, p = X.shape
    lam = oracle.lambda_ub(n, p)
    one = S.fit(X, lam, solver=solver)
    multi = S.fit(X, lam, solver=solver, num_devices=1)
    assert multi.stats["num_devices"] == 1 and one.stats["num_devices"] == 0
    assert multi.stats["ms_comm"] > 0.0
    assert np.array_equal(multi.Theta, one.Theta) and np.array_equal(multi.sigma, one.sigma)
    assert np.array_equal(multi.iters, one.iters) and np.array_equal(multi.sweeps, one.sweeps)
    assert np.array_equal(multi.converged, one.converged)
    ora = oracle.spmesl_fit(X, lam)
    assert_parity(compare(multi.Theta, multi.sigma, multi.iters, multi.sweeps, ora))


def test_c_abi_multi_device_errors(S):
    X, _, _ = G.make_config(2)
    with pytest.raises(S.SpmeslError) as e:          # duplicate device ids
        S.fit(X, 0.3, num_devices=2, device_ids=[0, 0])
    assert e.value.code == -1
    with pytest.raises(S.SpmeslError) as e:          # not a device
        S.fit(X, 0.3, num_devices=1, device_ids=[4096])
    assert e.value.code == -1
    with pytest.raises(S.SpmeslError) as e:          # joint stop: one device only
        S.fit(X, 0.3, num_devices=1, mode="joint")
    assert e.value.code == -7
    S.fit(X, 0.3, num_devices=1)                     # and the library recovers


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
