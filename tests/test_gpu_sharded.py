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


# ------------------------------------------------------------------ fused P2P exchange (K2p)


def _p2p_exchange(n):
    from paper_2110_12065_b200.sharded import P2PExchange

    return P2PExchange(n, 0, 1, device="cuda")


def test_p2p_world1_bitwise_vs_coop(mapi_lib, monkeypatch):
    """With one rank the fused kernel runs the exchange through its own buffer (local stores, own
    flag as the grid barrier); its rows, partial order and s order are K2c's, so the iterates, norms
    and deltas are bitwise identical to mapi_iterate on the cooperative path."""
    from paper_2110_12065_b200.sharded import iterate_sharded_p2p

    m = mapi_lib
    n = 8192
    r = np.random.default_rng(11)
    A = torch.from_numpy((r.standard_normal((n, n)) + np.eye(n) * 4).astype(np.float32)).cuda()
    b0 = torch.full((n,), 1 / np.sqrt(n), device="cuda")
    ex = _p2p_exchange(n)
    try:
        res = iterate_sharded_p2p(A, n, 0, b0, 30, ex)
        monkeypatch.setenv("MAPI_DENSE_PATH", "coop")
        ref = m.iterate(A, b0, 30)
        assert torch.equal(res.w, ref.w) and torch.equal(res.norms, ref.norms) and torch.equal(res.deltas, ref.deltas)
        assert ex.epoch == 30
    finally:
        ex.close()


def test_p2p_world1_calls_continue_epoch_and_parity(mapi_lib, orc):
    """Consecutive calls on one exchange buffer (odd iteration counts flip the buffer parity between
    calls; the flag keeps counting) give the same results as fresh buffers; ragged n (n % 256 != 0)
    and min2 / dot operators against the oracle (T2)."""
    from paper_2110_12065_b200.sharded import iterate_sharded_p2p

    m = mapi_lib
    n = 4104
    r = np.random.default_rng(5)
    A_h = (r.standard_normal((n, n)) + np.eye(n) * 3).astype(np.float32)
    A = torch.from_numpy(A_h).cuda()
    b0_h = np.full(n, 1 / np.sqrt(n), np.float32)
    b0 = torch.from_numpy(b0_h).cuda()
    ex = _p2p_exchange(n)
    try:
        outs = [iterate_sharded_p2p(A, n, 0, b0, k, ex) for k in (7, 8, 5)]
        assert ex.epoch == 20
        for k, o in zip((7, 8, 5), outs):
            fresh_ex = _p2p_exchange(n)
            try:
                fresh = iterate_sharded_p2p(A, n, 0, b0, k, fresh_ex)
            finally:
                fresh_ex.close()
            assert torch.equal(o.w, fresh.w) and torch.equal(o.deltas, fresh.deltas)
        for op, name in ((m.MIN2, "min2"), (m.DOT, None)):
            res = iterate_sharded_p2p(A, n, 0, b0, 20, ex, op=op)
            ref = orc.mapi(A_h, b0_h, 20, op=name) if name else orc.rpi(A_h, b0_h, 20)
            _t2(res.w.cpu().numpy(), ref.w)
            np.testing.assert_allclose(res.norms.cpu().numpy(), ref.norms, rtol=1e-5)
    finally:
        ex.close()


def test_p2p_world1_tol_stop_and_degenerate(mapi_lib):
    """Early stop by tol and a degenerate run advance the exchange epoch by the iterations that
    reached the exchange; a following normal call is unaffected."""
    from paper_2110_12065_b200.sharded import iterate_sharded_p2p

    m = mapi_lib
    n = 2048
    r = np.random.default_rng(2)
    A = torch.from_numpy(((r.standard_normal((n, n)) / 8) + np.diag(np.linspace(4, 1, n))).astype(np.float32)).cuda()
    b0 = torch.full((n,), 1 / np.sqrt(n), device="cuda")
    ex = _p2p_exchange(n)
    try:
        full = iterate_sharded_p2p(A, n, 0, b0, 100, ex)
        d = full.deltas.cpu().numpy()
        tol = float(d[30]) * 1.0001
        first = int(np.nonzero(d < tol)[0][0])
        e0 = ex.epoch
        res = iterate_sharded_p2p(A, n, 0, b0, 100, ex, tol=tol)
        assert res.iters_done == first + 1 and ex.epoch == e0 + first + 1
        assert torch.equal(res.deltas, full.deltas[: first + 1])
        e1 = ex.epoch
        with pytest.raises(m.MapiError) as ei:
            iterate_sharded_p2p(torch.zeros(n, n, device="cuda"), n, 0, b0, 10, ex)
        assert ei.value.name == "MAPI_ERR_DEGENERATE" and ex.epoch == e1 + 1
        again = iterate_sharded_p2p(A, n, 0, b0, 100, ex)
        assert torch.equal(again.w, full.w)
    finally:
        ex.close()


# ------------------------------------------------------------ sharded symmetric K2s (K2sp)


def _sym(n, seed):
    r = np.random.default_rng(seed)
    G = r.standard_normal((n, n)).astype(np.float32) / 16
    S = np.triu(G) + np.triu(G, 1).T
    S[np.diag_indices(n)] += np.linspace(4.0, 1.0, n).astype(np.float32)
    return S.astype(np.float32)


@pytest.mark.parametrize("n,op", [(8192, 0), (2056, 0), (2056, 1), (2056, 2)])
def test_sym_sharded_world1_bitwise_vs_k2s(mapi_lib, monkeypatch, n, op):
    """With one rank K2sp runs K2s's whole task list, exchanges its partial y through its own buffer and sums
    one partial: the iterates, norms and deltas are bitwise mapi_iterate_sym's (K2s).  The lower triangle is
    NaN (never read); consecutive calls continue the exchange epoch."""
    from paper_2110_12065_b200.sharded import iterate_sym_sharded_p2p, sym_shard

    m = mapi_lib
    monkeypatch.setenv("MAPI_SYM_PATH", "sym")
    S = _sym(n, n)
    dev = np.triu(S) + np.tril(np.full((n, n), np.nan, np.float32), -1)
    A = torch.from_numpy(dev).cuda()
    b0 = torch.full((n,), 1 / np.sqrt(n), device="cuda")
    lo, hi, tlo, thi = sym_shard(n, 0, 1)
    assert (lo, hi, tlo) == (0, n, 0)
    ex = _p2p_exchange(n)
    try:
        res = iterate_sym_sharded_p2p(A[lo:hi], lo, hi, n, b0, 25, ex, op=op)
        ref = m.iterate_sym(A, b0, 25, op=op)
        assert res.iters_done == 25 and ex.epoch == 25
        assert torch.equal(res.w, ref.w) and torch.equal(res.norms, ref.norms) and torch.equal(res.deltas, ref.deltas)
        again = iterate_sym_sharded_p2p(A[lo:hi], lo, hi, n, b0, 25, ex, op=op)  # odd epoch parity now
        assert torch.equal(again.w, ref.w) and ex.epoch == 50
    finally:
        ex.close()


def test_sym_sharded_world1_tol_and_degenerate(mapi_lib, monkeypatch, orc):
    """Tol stop (lagged one task phase, same outputs as K2s), the epoch advances by the published iterations,
    a degenerate matrix stops with MAPI_ERR_DEGENERATE at iteration 0 (one published), T2 vs the oracle."""
    from paper_2110_12065_b200.sharded import iterate_sym_sharded_p2p

    m = mapi_lib
    monkeypatch.setenv("MAPI_SYM_PATH", "sym")
    n = 2048
    S = _sym(n, 9)
    A = torch.from_numpy(S).cuda()
    b0_h = np.full(n, 1 / np.sqrt(n), np.float32)
    b0 = torch.from_numpy(b0_h).cuda()
    ex = _p2p_exchange(n)
    try:
        full = iterate_sym_sharded_p2p(A, 0, n, n, b0, 120, ex)
        d = full.deltas.cpu().numpy()
        tol = float(d[40]) * 1.0001
        first = int(np.nonzero(d < tol)[0][0])
        e0 = ex.epoch
        res = iterate_sym_sharded_p2p(A, 0, n, n, b0, 120, ex, tol=tol)
        ref = m.iterate_sym(A, b0, 120, tol=tol)
        assert res.iters_done == ref.iters_done == first + 1 and ex.epoch == e0 + first + 1
        assert torch.equal(res.w, ref.w) and torch.equal(res.deltas, full.deltas[: first + 1])
        o = orc.mapi(S, b0_h, first + 1)
        w = res.w.cpu().numpy().astype(np.float64)
        _t2(w, o.w)
        e1 = ex.epoch
        with pytest.raises(m.MapiError) as ei:
            iterate_sym_sharded_p2p(torch.zeros(n, n, device="cuda"), 0, n, n, b0, 10, ex)
        assert ei.value.name == "MAPI_ERR_DEGENERATE" and ex.epoch == e1 + 1
        again = iterate_sym_sharded_p2p(A, 0, n, n, b0, 120, ex)
        assert torch.equal(again.w, full.w)
    finally:
        ex.close()
