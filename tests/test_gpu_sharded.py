"""Row-sharded MAPI (NEXT-4) on the one available GPU: the NCCL path with a world of 1
(init, all-gather, normalise) and the library kernels, vs the oracle (T2) and the single-GPU path."""
import os
import socket

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _t2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    a, b = a / np.linalg.norm(a), b / np.linalg.norm(b)
    assert abs(float(a @ b)) >= 1 - 1e-6 and np.max(np.abs(a - b)) <= 1e-4


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [256, 4096])
def test_sharded_world1_vs_oracle(mapi_lib, orc, nccl_world1, n):
    from paper_2110_12065_b200.sharded import iterate_sharded

    m = mapi_lib
    r = np.random.default_rng(n)
    A = (r.standard_normal((n, n)) + np.eye(n) * 3).astype(np.float32)
    b0 = np.full(n, 1 / np.sqrt(n), np.float32)
    res = iterate_sharded(torch.from_numpy(A).cuda(), n, torch.from_numpy(b0).cuda(), 25)
    ref = orc.mapi(A, b0, 25)
    _t2(res.w.cpu().numpy(), ref.w)
    np.testing.assert_allclose(res.norms.cpu().numpy(), ref.norms, rtol=1e-5)
    single = m.iterate(torch.from_numpy(A).cuda(), torch.from_numpy(b0).cuda(), 25)
    _t2(res.w.cpu().numpy(), single.w.cpu().numpy())


def test_sharded_tol_and_rows_generator(mapi_lib, orc, nccl_world1):
    from paper_2110_12065_b200.sharded import iterate_sharded

    n = 8192
    cfg = synth.cfg3_rows(0, n, device="cuda", n=n, rank=64)
    res = iterate_sharded(cfg["A"], n, torch.from_numpy(cfg["b0"]).cuda(), 200, tol=5e-3)
    d = res.deltas.cpu().numpy()
    assert res.iters_done < 200 and d[-1] < 5e-3 and np.all(d[:-1] >= 5e-3)  # stops at the first delta < tol
    A_full = synth.cfg3(device="cuda", n=n, rank=64)["A"]
    assert torch.equal(A_full, cfg["A"])  # the row-block generator reproduces the full matrix
