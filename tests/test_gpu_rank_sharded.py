"""GPU parity of the row-sharded MAPI ranking (K3n, mapi_rank_csr_shard_*, Eq. 13)
against the oracle's rank_csr.  A pool box has ONE GPU, so worlds of 1-4 ranks are run as that many sessions
on the one device, stepped in lockstep by the HOST (rows of every rank, then the exchange as device copies of
the owners' e_t blocks, then every rank's normalisation): no kernel waits on another rank, and every rank's
kernels, partition and state are exactly those of a real N-rank run.  Checked: every rank ends with bitwise
the same w / deltas / iteration count, T2 + T3 against the oracle, and against the single-GPU mapi_rank_csr.
"""
import numpy as np
import pytest
import torch

import synth
from test_gpu_rank import _dev, _t2, _t3

pytestmark = pytest.mark.gpu


def _run_world(m, n, row_ptr, col_idx, b0, iters, tol, world, starts=None, alpha=0.85, check_every=4):
    from paper_2110_12065_b200 import sharded

    rp = _dev(row_ptr, torch.int32)
    ci = _dev(col_idx.astype(np.int32)) if col_idx.size else torch.empty(0, dtype=torch.int32, device="cuda")
    cap, bg = m.csr_prepare(n, rp, ci, alpha)
    b0d = _dev(b0.astype(np.float32))
    starts = starts or sharded.csr_row_partition(row_ptr, world)
    rp_host = torch.from_numpy(np.ascontiguousarray(row_ptr)).to(torch.int32)
    ses = []
    for r in range(world):
        r0, r1 = starts[r], starts[r + 1]
        lo, hi = int(rp_host[r0]), int(rp_host[r1])
        rpl = (rp[r0:r1 + 1] - lo).contiguous()
        cil = ci[lo:hi].contiguous()
        ses.append(sharded.CsrShardSession(n, r0, rpl, cil, cap, bg, b0d, iters, tol))
    for s in ses:
        s.begin()
    for t in range(iters):
        for s in ses:
            s.rows(t)
        for q, dst in enumerate(ses):  # the all-gather: every rank receives every owner's block
            ev = dst.e_view(t)
            for r, src in enumerate(ses):
                if r != q and starts[r + 1] > starts[r]:
                    ev[starts[r]:starts[r + 1]].copy_(src.e_view(t)[starts[r]:starts[r + 1]])
        for s in ses:
            s.normalize(t)
        if tol > 0 and (t + 1) % check_every == 0:
            polls = [s.poll() for s in ses]
            assert len(set(polls)) == 1  # the same stop decision everywhere
            if polls[0][1]:
                break
    res = [s.finish() for s in ses]
    for r in res[1:]:  # every rank holds the same bits
        assert r.iters_done == res[0].iters_done
        assert torch.equal(r.w, res[0].w) and torch.equal(r.w_l2, res[0].w_l2)
        assert torch.equal(r.deltas, res[0].deltas)
    single = m.rank_csr(n, rp, ci, cap, bg, b0d, iters, tol)
    return res[0], single, starts


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("trial", range(4))
def test_sharded_random_graphs(mapi_lib, orc, world, trial):
    r = np.random.default_rng(100 + trial)
    n = int(r.integers(5, 500))
    edges, row_ptr, col_idx = synth.random_graph(n, float(r.uniform(0.005, 0.1)), seed=trial,
                                                 n_dangling=int(r.integers(0, n // 3 + 1)))
    b0 = np.full(n, 1.0 / n)
    res, single, starts = _run_world(mapi_lib, n, row_ptr, col_idx, b0, 15, 0.0, world)
    ref = orc.rank_csr(n, row_ptr, col_idx, b0=b0.astype(np.float32), max_iters=15, tol=0.0)
    assert res.iters_done == ref.iters_done == 15
    _t2(res.w_l2.cpu().numpy(), ref.w)
    np.testing.assert_allclose(res.w.cpu().numpy(), ref.w, rtol=2e-5, atol=1e-9)
    np.testing.assert_allclose(res.deltas.cpu().numpy(), ref.deltas, rtol=1e-2, atol=2e-7)
    _t3(orc, res.w.cpu().numpy(), ref.w, k=min(20, n))
    # vs the single-GPU path: same method, the sum of e is taken in another fixed order
    np.testing.assert_allclose(res.w.cpu().numpy(), single.w.cpu().numpy(), rtol=1e-6, atol=1e-12)


def test_sharded_uneven_and_empty_blocks(mapi_lib, orc):
    """Hand-made partitions: an empty block in the middle, a one-row block, a rank owning everything."""
    n = 300
    edges, row_ptr, col_idx = synth.random_graph(n, 0.05, seed=7, n_dangling=30)
    b0 = np.full(n, 1.0 / n)
    ref = orc.rank_csr(n, row_ptr, col_idx, b0=b0.astype(np.float32), max_iters=12, tol=0.0)
    for starts in ([0, 120, 120, 121, 300], [0, 0, 300], [0, 299, 300]):
        res, _, _ = _run_world(mapi_lib, n, row_ptr, col_idx, b0, 12, 0.0, len(starts) - 1, starts=list(starts))
        _t2(res.w_l2.cpu().numpy(), ref.w)
        np.testing.assert_allclose(res.w.cpu().numpy(), ref.w, rtol=2e-5, atol=1e-9)


def test_sharded_tol_stop_gnutella_like(mapi_lib, orc):
    g = synth.gnutella_like()
    n = g["n"]
    res, single, _ = _run_world(mapi_lib, n, g["row_ptr"], g["col_idx"], g["b0"], 200, 1e-7, 3)
    ref = orc.rank_csr(n, g["row_ptr"], g["col_idx"], b0=g["b0"], max_iters=200, tol=1e-7)
    assert abs(res.iters_done - ref.iters_done) <= 1
    assert res.iters_done == single.iters_done
    _t2(res.w_l2.cpu().numpy(), ref.w)
    _t3(orc, res.w.cpu().numpy(), ref.w)


def test_sharded_negative_start_and_hub_rows(mapi_lib, orc):
    m = mapi_lib
    n = 64
    edges, row_ptr, col_idx = synth.random_graph(n, 0.1, seed=1)
    b0 = np.full(n, 1.0 / n)
    b0[5] = -0.1
    with pytest.raises(m.MapiError) as ei:
        _run_world(m, n, row_ptr, col_idx, b0, 3, 0.0, 2)
    assert ei.value.status == 5
    # a star: one row with n - 1 in-edges spans several merge tiles of its owner
    n = 6000
    src = np.arange(1, n, dtype=np.int64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr[1:] = n - 1
    col_idx = src
    b0 = np.full(n, 1.0 / n)
    res, _, starts = _run_world(m, n, row_ptr, col_idx, b0, 6, 0.0, 3)
    ref = orc.rank_csr(n, row_ptr, col_idx, b0=b0.astype(np.float32), max_iters=6, tol=0.0)
    _t2(res.w_l2.cpu().numpy(), ref.w)
    assert int(np.argmax(res.w.cpu().numpy())) == 0


def test_sharded_cfg5_world4(mapi_lib, orc):
    """BASELINE configs[4] at full size over a world of 4 (10 fixed iterations, T2 + T3), the partition
    balanced by rows + in-edges."""
    c = synth.cfg5()
    n = c["n"]
    res, single, starts = _run_world(mapi_lib, n, c["row_ptr"], c["col_idx"], c["b0"], 10, 0.0, 4)
    items = [(starts[r + 1] - starts[r]) + int(c["row_ptr"][starts[r + 1]] - c["row_ptr"][starts[r]]) for r in range(4)]
    assert max(items) <= 1.02 * min(items) + 1e5
    ref = orc.rank_csr(n, c["row_ptr"], c["col_idx"], b0=c["b0"], max_iters=10, tol=0.0)
    _t2(res.w_l2.cpu().numpy(), ref.w)
    _t3(orc, res.w.cpu().numpy(), ref.w)
    _t2(res.w_l2.cpu().numpy(), single.w_l2.cpu().numpy())


def test_rank_csr_sharded_world1_product_call(mapi_lib, orc):
    """The product entry point (sharded.rank_csr_sharded) without a process group: a world of one."""
    from paper_2110_12065_b200 import sharded

    m = mapi_lib
    g = synth.gnutella_like()
    n = g["n"]
    rp, ci = _dev(g["row_ptr"], torch.int32), _dev(g["col_idx"].astype(np.int32))
    cap, bg = m.csr_prepare(n, rp, ci, 0.85)
    res = sharded.rank_csr_sharded(n, [0, n], rp, ci, cap, bg, _dev(g["b0"].astype(np.float32)), 200, 1e-7)
    ref = orc.rank_csr(n, g["row_ptr"], g["col_idx"], b0=g["b0"], max_iters=200, tol=1e-7)
    assert abs(res.iters_done - ref.iters_done) <= 1
    _t2(res.w_l2.cpu().numpy(), ref.w)
    _t3(orc, res.w.cpu().numpy(), ref.w)
