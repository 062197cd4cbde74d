"""GPU parity of the segmented ranking path (mapi_csr_plan + mapi_rank_csr_plan, K3s) against the
fp64 oracle (Eq. 13; RPI arm reading R13), through the C ABI.

T2: on the l2-normalised final vectors |cos| >= 1 - 1e-6 and max|diff| <= 1e-4.
T3: every id in the symmetric difference of the top-100 sets is within 1e-6 (relative) of the oracle's 100th.
"""
import functools

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _t2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    a, b = a / np.linalg.norm(a), b / np.linalg.norm(b)
    assert abs(float(a @ b)) >= 1 - 1e-6
    assert np.max(np.abs(a - b)) <= 1e-4


def _t3(orc, w_gpu, w_orc, k=100):
    k = min(k, w_orc.size)
    O = orc.rank_order(w_orc)[:k]
    G = orc.rank_order(np.asarray(w_gpu, np.float64))[:k]
    kth = w_orc[O[-1]]
    for i in set(O.tolist()) ^ set(G.tolist()):
        assert abs(w_orc[i] - kth) <= 1e-6 * kth, f"id {i}: {w_orc[i]} vs 100th {kth}"


def _plan_run(m, n, row_ptr, col_idx, b0, iters, tol, op=0, alpha=0.85):
    rp = _dev(row_ptr, torch.int32)
    ci = _dev(col_idx.astype(np.int32), torch.int32) if col_idx.size else torch.empty(0, dtype=torch.int32,
                                                                                       device="cuda")
    cap, bg = m.csr_prepare(n, rp, ci, alpha)
    plan = m.csr_plan(n, rp, ci)
    res = m.rank_csr_plan(plan, cap, bg, _dev(np.asarray(b0, np.float32)), iters, tol, op=op)
    return res, plan, (rp, ci, cap, bg)


@functools.lru_cache(maxsize=None)
def _graphs():
    out = {}
    g = synth.gnutella_like()
    out["gnutella"] = (g["n"], g["row_ptr"], g["col_idx"])
    r = np.random.default_rng(11)
    n = 60000
    src = np.minimum((r.pareto(1.2, 400000) * 50).astype(np.int64), n - 1)
    dst = r.integers(0, n, 400000)
    out["skewed60k"] = (n, *synth.csr_by_destination(n, src, dst))
    # many sources: 7 segments of 32,767, uniform sources, dangling nodes, ragged
    n = 230001
    src = r.integers(0, n - 5000, 900000)
    dst = r.integers(0, n, 900000)
    out["uniform230k"] = (n, *synth.csr_by_destination(n, src, dst))
    # hub rows with thousands of in-edges (pieces split at 256) + a long tail
    n = 70000
    src = np.concatenate([np.arange(1, 9000), r.integers(0, n, 200000), np.arange(2, 40000)])
    dst = np.concatenate([np.zeros(8999, np.int64), r.integers(0, n, 200000), np.ones(39998, np.int64)])
    out["hubs70k"] = (n, *synth.csr_by_destination(n, src, dst))
    edges, rp, ci = synth.random_graph(150, 0.05, seed=3, n_dangling=20)
    out["random150"] = (150, rp, ci)
    return out


NAMES = ["gnutella", "hubs70k", "random150", "skewed60k", "uniform230k"]


@pytest.mark.parametrize("name", NAMES)
def test_plan_matches_oracle(mapi_lib, orc, name):
    """Fixed-iteration runs (T2 + T3 + the per-iteration l1 changes) on graphs spanning one to seven segments,
    hub rows split into many pieces, dangling and empty rows, and ragged sizes."""
    m = mapi_lib
    n, rp, ci = _graphs()[name]
    b0 = np.full(n, 1.0 / n)
    res, plan, _ = _plan_run(m, n, rp, ci, b0, 25, 0.0)
    ref = orc.rank_csr(n, rp, ci, b0=b0, max_iters=25, tol=0.0)
    assert res.iters_done == 25
    _t2(res.w_l2.cpu().numpy(), ref.w)
    _t3(orc, res.w.cpu().numpy(), ref.w)
    np.testing.assert_allclose(res.w.cpu().numpy(), ref.w, rtol=2e-5, atol=1e-12)
    d = res.deltas.cpu().numpy().astype(np.float64)
    big = ref.deltas > 1e-5
    np.testing.assert_allclose(d[big], ref.deltas[big], rtol=1e-3)
    info = plan.info
    assert info.n == n and info.nnz == ci.size
    assert info.nsrc == np.count_nonzero(np.bincount(ci, minlength=n))
    assert info.nseg == max(1, -(-info.nsrc // 32767))
    assert info.npieces >= 1 and info.nwords % 16 == 0


@pytest.mark.parametrize("name", ["gnutella", "hubs70k", "random150"])
def test_plan_rpi_matches_oracle(mapi_lib, orc, name):
    """op = DOT: the PageRank power iteration G w (reading R13) against the oracle's RPI arm."""
    m = mapi_lib
    n, rp, ci = _graphs()[name]
    b0 = np.full(n, 1.0 / n)
    res, _, _ = _plan_run(m, n, rp, ci, b0, 30, 0.0, op=m.DOT)
    ref = orc.rank_csr(n, rp, ci, b0=b0, max_iters=30, tol=0.0, op="dot")
    _t2(res.w_l2.cpu().numpy(), ref.w)
    _t3(orc, res.w.cpu().numpy(), ref.w)
    np.testing.assert_allclose(res.w.cpu().numpy(), ref.w, rtol=2e-5, atol=1e-12)


def test_plan_min2_equals_min1_bitwise(mapi_lib):
    m = mapi_lib
    n, rp, ci = _graphs()["skewed60k"]
    b0 = np.full(n, 1.0 / n)
    a, _, _ = _plan_run(m, n, rp, ci, b0, 12, 0.0, op=m.MIN1)
    b, _, _ = _plan_run(m, n, rp, ci, b0, 12, 0.0, op=m.MIN2)
    assert torch.equal(a.w, b.w) and torch.equal(a.deltas, b.deltas)


def test_plan_deterministic_and_tol_stop(mapi_lib, orc):
    """Bitwise repeatable; a tol stop ends on the device at the first delta_t < tol (the prefix of the
    fixed run's trace), matching the oracle's stopping iteration within one."""
    m = mapi_lib
    n, rp, ci = _graphs()["uniform230k"]
    b0 = np.full(n, 1.0 / n)
    a, plan, (rpd, cid, cap, bg) = _plan_run(m, n, rp, ci, b0, 40, 0.0)
    b = m.rank_csr_plan(plan, cap, bg, _dev(b0.astype(np.float32)), 40, 0.0)
    assert torch.equal(a.w, b.w) and torch.equal(a.deltas, b.deltas)
    d = a.deltas.cpu().numpy()
    tol = float(d[1]) * 1.0001  # (MAPI settles in a few iterations here: later deltas may be exactly 0)
    assert tol > 0
    first = int(np.nonzero(d < tol)[0][0])
    c = m.rank_csr_plan(plan, cap, bg, _dev(b0.astype(np.float32)), 40, tol)
    assert c.iters_done == first + 1
    assert torch.equal(c.deltas, a.deltas[: first + 1])
    ref = orc.rank_csr(n, rp, ci, b0=b0, max_iters=40, tol=tol)
    assert abs(ref.iters_done - c.iters_done) <= 1


def test_plan_vs_csr_path(mapi_lib):
    """The planned kernel and the plan-free K3 path compute the same iteration (different summation order):
    agreement at fp32 level."""
    m = mapi_lib
    n, rp, ci = _graphs()["hubs70k"]
    b0 = np.full(n, 1.0 / n)
    a, _, (rpd, cid, cap, bg) = _plan_run(m, n, rp, ci, b0, 20, 0.0)
    k3 = m.rank_csr(n, rpd, cid, cap, bg, _dev(b0.astype(np.float32)), 20, 0.0)
    np.testing.assert_allclose(a.w.cpu().numpy(), k3.w.cpu().numpy(), rtol=2e-5, atol=1e-12)


@pytest.mark.parametrize("name", ["hubs70k", "skewed60k", "uniform230k"])
def test_plan_word_order_only_reorders_sums(mapi_lib, monkeypatch, name):
    """The plan-time bank-conflict-aware word order (kp_deconflict, K3s 3c) only permutes the source
    offsets inside a (lane chunk, fragment) group: with it (default passes, and 5 passes) and without it
    (MAPI_PLAN_DECONFLICT=0) the plan has the same sizes and the run gives the same iteration count and the same
    scores up to the fp32 addition order inside a fragment."""
    m = mapi_lib
    n, row_ptr, col_idx = _graphs()[name]
    b0 = np.full(n, 1.0 / n, np.float32)
    runs = {}
    for passes in ("0", None, "5"):
        if passes is None:
            monkeypatch.delenv("MAPI_PLAN_DECONFLICT", raising=False)
        else:
            monkeypatch.setenv("MAPI_PLAN_DECONFLICT", passes)
        res, plan, _ = _plan_run(m, n, row_ptr, col_idx, b0, 12, 0.0)
        runs[passes] = (res.w.cpu().numpy().astype(np.float64), res.deltas.cpu().numpy(), res.iters_done,
                        (plan.info.npieces, plan.info.nwords, plan.info.nseg, plan.info.nunits))
    w0, d0, k0, sz0 = runs["0"]
    for key in (None, "5"):
        w, d, k, sz = runs[key]
        assert k == k0 == 12 and sz == sz0
        np.testing.assert_allclose(w, w0, rtol=2e-6, atol=1e-12)
        np.testing.assert_allclose(d, d0, rtol=1e-3, atol=1e-8)

def test_plan_edge_cases(mapi_lib, orc):
    m = mapi_lib
    # no edges at all: every column dangling, w stays uniform
    n = 100
    res, plan, _ = _plan_run(m, n, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.full(n, 1.0 / n), 3, 0.0)
    assert plan.info.npieces == 0 and plan.info.nsrc == 0
    np.testing.assert_allclose(res.w.cpu().numpy(), np.full(n, 1.0 / n), rtol=1e-6)
    # a single node with a self-loop; two nodes
    for n, src, dst in ((1, [0], [0]), (2, [0, 1], [1, 1]), (3, [2], [0])):
        rp, ci = synth.csr_by_destination(n, np.array(src), np.array(dst))
        b0 = np.full(n, 1.0 / n)
        res, _, _ = _plan_run(m, n, rp, ci, b0, 7, 0.0)
        ref = orc.rank_csr(n, rp, ci, b0=b0, max_iters=7, tol=0.0)
        np.testing.assert_allclose(res.w.cpu().numpy(), ref.w, rtol=1e-6)
    # a non-uniform start and a negative start
    n, rp, ci = _graphs()["random150"]
    r = np.random.default_rng(5)
    b0 = r.random(n)
    b0 /= b0.sum()
    res, _, (rpd, cid, cap, bg) = _plan_run(m, n, rp, ci, b0, 9, 0.0)
    ref = orc.rank_csr(n, rp, ci, b0=b0, max_iters=9, tol=0.0)
    _t2(res.w_l2.cpu().numpy(), ref.w)
    bad = b0.copy()
    bad[3] = -1e-3
    with pytest.raises(m.MapiError) as ei:
        _plan_run(m, n, rp, ci, bad, 5, 0.0)
    assert ei.value.name == "MAPI_ERR_NEGATIVE"


@pytest.fixture(scope="module")
def cfg5():
    return synth.cfg5()


def test_cfg5_plan_full_size(mapi_lib, orc, cfg5):
    """BASELINE configs[4] through the planned path exactly as bench.py times it: 200 fixed iterations
    (T2 + T3 + deltas) and the tol 1e-7 / 200 run as specified (T3, stop within one iteration)."""
    m = mapi_lib
    n = cfg5["n"]
    b0 = cfg5["b0"].astype(np.float64)
    res, plan, (rpd, cid, cap, bg) = _plan_run(m, n, cfg5["row_ptr"], cfg5["col_idx"], b0, 200, 0.0)
    ref = orc.rank_csr(n, cfg5["row_ptr"], cfg5["col_idx"], b0=b0, max_iters=200, tol=0.0)
    assert res.iters_done == 200
    _t2(res.w_l2.cpu().numpy(), ref.w)
    _t3(orc, res.w.cpu().numpy(), ref.w)
    d_gpu, d_orc = res.deltas.cpu().numpy().astype(np.float64), ref.deltas
    big = d_orc > 1e-6
    np.testing.assert_allclose(d_gpu[big], d_orc[big], rtol=1e-3)
    tol_run = m.rank_csr_plan(plan, cap, bg, _dev(cfg5["b0"]), 200, 1e-7)
    ref_tol = orc.rank_csr(n, cfg5["row_ptr"], cfg5["col_idx"], b0=b0, max_iters=200, tol=1e-7)
    assert abs(tol_run.iters_done - ref_tol.iters_done) <= 1
    _t3(orc, tol_run.w.cpu().numpy(), ref_tol.w)
    rpi = m.rank_csr_plan(plan, cap, bg, _dev(cfg5["b0"]), 30, 0.0, op=m.DOT)
    ref_rpi = orc.rank_csr(n, cfg5["row_ptr"], cfg5["col_idx"], b0=b0, max_iters=30, tol=0.0, op="dot")
    _t2(rpi.w_l2.cpu().numpy(), ref_rpi.w)
    _t3(orc, rpi.w.cpu().numpy(), ref_rpi.w)
