"""GPU parity of mapi_iterate_batched (k independent MAPI runs on one A; BASELINE configs[3])
against the oracle's single-vector MAPI, per vector (T2: |cos| >= 1 - 1e-6, max|diff| <= 1e-4 on
the l2-normalised vectors; norms relative <= 1e-5)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _t2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    a, b = a / np.linalg.norm(a), b / np.linalg.norm(b)
    cos = float(a @ b)
    assert abs(cos) >= 1 - 1e-6, f"|cos| {abs(cos)!r}"
    assert np.max(np.abs(a - b)) <= 1e-4, f"max abs {np.max(np.abs(a - b))}"


@pytest.mark.parametrize("n,k", [(1, 1), (7, 3), (129, 70), (300, 5), (1000, 64), (2051, 9)])
@pytest.mark.parametrize("op", ["min1", "min2"])
def test_batched_small(mapi_lib, orc, n, k, op):
    m = mapi_lib
    r = np.random.default_rng(n * 100 + k)
    A = r.standard_normal((n, n)).astype(np.float32)
    if op == "min2":
        A = np.abs(A) + np.eye(n, dtype=np.float32)
    B0 = np.abs(r.standard_normal((k, n))) + 0.05 if op == "min2" else r.standard_normal((k, n))
    B0 = (B0 / np.linalg.norm(B0, axis=1, keepdims=True)).astype(np.float32)
    T = 20
    res = m.iterate_batched(torch.from_numpy(A).cuda(), torch.from_numpy(B0).cuda(), T,
                            op=m.MIN1 if op == "min1" else m.MIN2)
    W = res.W.cpu().numpy()
    norms = res.norms.cpu().numpy()
    for v in sorted({0, k // 2, k - 1}):
        ref = orc.mapi(A, B0[v], T, op=op)
        assert res.iters_done[v] == ref.iters_done == T
        _t2(W[v], ref.w)
        np.testing.assert_allclose(norms[:, v], ref.norms, rtol=1e-5)


@pytest.mark.parametrize("n,k", [(300, 5), (1000, 64), (4100, 9)])
def test_batched_rpi_matches_oracle(mapi_lib, orc, monkeypatch, n, k):
    """op = DOT on the batched kernels (stream-K v2 and the split-K v1): k independent RPI runs (Eq. 1, l2
    normalisation) against the oracle's RPI per vector (T2, norms = ||A w_t||_2 at 1e-5)."""
    m = mapi_lib
    r = np.random.default_rng(n + k)
    G = r.standard_normal((n, n)).astype(np.float32) / np.sqrt(n)
    A = ((G + G.T) / 2 + np.diag(np.linspace(3.0, 1.0, n))).astype(np.float32)
    B0 = r.standard_normal((k, n))
    B0 = (B0 / np.linalg.norm(B0, axis=1, keepdims=True)).astype(np.float32)
    T = 15
    for path in ("v2", "v1"):
        if path == "v1":
            monkeypatch.setenv("MAPI_BATCHED_PATH", "v1")
        res = m.iterate_batched(torch.from_numpy(A).cuda(), torch.from_numpy(B0).cuda(), T, op=m.DOT)
        W, norms = res.W.cpu().numpy(), res.norms.cpu().numpy()
        for v in sorted({0, k // 2, k - 1}):
            ref = orc.rpi(A, B0[v], T)
            assert res.iters_done[v] == T
            _t2(W[v], ref.w)
            np.testing.assert_allclose(np.linalg.norm(W[v]), 1.0, rtol=1e-5)
            np.testing.assert_allclose(norms[:, v], ref.norms, rtol=1e-5)


def test_batched_tol_per_vector_and_identity(mapi_lib):
    m = mapi_lib
    n, k = 96, 4
    A = np.eye(n, dtype=np.float32)
    r = np.random.default_rng(0)
    B0 = r.random((k, n)).astype(np.float32) + 0.1
    B0 /= np.linalg.norm(B0, axis=1, keepdims=True)
    res = m.iterate_batched(torch.from_numpy(A).cuda(), torch.from_numpy(B0).cuda(), 30, tol=1e-6)
    assert res.iters_done == [2] * k
    np.testing.assert_allclose(res.W.cpu().numpy(), B0 / B0.sum(axis=1, keepdims=True), rtol=2e-7)


def test_batched_degenerate(mapi_lib):
    m = mapi_lib
    A = torch.zeros(50, 50, device="cuda")
    B0 = torch.full((3, 50), 0.1, device="cuda")
    with pytest.raises(m.MapiError) as ei:
        m.iterate_batched(A, B0, 5)
    assert ei.value.name == "MAPI_ERR_DEGENERATE"


def test_batched_matches_single_vector_runs(mapi_lib):
    m = mapi_lib
    cfg = synth.cfg1()
    A = torch.from_numpy(cfg["A"]).cuda()
    r = np.random.default_rng(2)
    B0 = r.standard_normal((16, 256))
    B0 = torch.from_numpy((B0 / np.linalg.norm(B0, axis=1, keepdims=True)).astype(np.float32)).cuda()
    res = m.iterate_batched(A, B0, 50)
    for v in range(16):
        single = m.iterate(A, B0[v].contiguous(), 50)
        _t2(res.W[v].cpu().numpy(), single.w.cpu().numpy())


@pytest.fixture(scope="module")
def cfg4():
    return synth.cfg4(device="cuda")


def test_cfg4_full_size(mapi_lib, orc, cfg4):
    """BASELINE configs[3] at full size (16384^2, k = 64, 100 iterations): every vector vs the GPU
    single-vector path (itself oracle-checked), vectors {0, 1, 31, 63} (both ends, a neighbour pair and the
    middle of the 64-vector tile) vs the fp64 oracle."""
    m = mapi_lib
    A = cfg4["A"]
    B0 = torch.from_numpy(cfg4["B0"]).cuda()
    T = cfg4["iters"]
    res = m.iterate_batched(A, B0, T)
    W = res.W.cpu().numpy()
    for v in range(64):
        single = m.iterate(A, B0[v].contiguous(), T)
        _t2(W[v], single.w.cpu().numpy())
    A_host = A.cpu().numpy()
    norms = res.norms.cpu().numpy()
    for v in (0, 1, 31, 63):
        ref = orc.mapi(A_host, cfg4["B0"][v], T)
        _t2(W[v], ref.w)
        np.testing.assert_allclose(norms[:, v], ref.norms, rtol=1e-5)


@pytest.mark.parametrize("path", ["v1", "v2", "v3"])
@pytest.mark.parametrize("n,k", [(300, 64), (1028, 70), (2048, 5)])
def test_batched_every_kernel(mapi_lib, orc, monkeypatch, path, n, k):
    """Each batched kernel (v1 split-K, v2 stream-K 8x8, v3 stream-K 8x4 + smem fold) vs the oracle."""
    m = mapi_lib
    r = np.random.default_rng(n + k)
    A = (r.standard_normal((n, n)) + np.eye(n) * 3).astype(np.float32)
    B0 = r.standard_normal((k, n))
    B0 = (B0 / np.linalg.norm(B0, axis=1, keepdims=True)).astype(np.float32)
    monkeypatch.setenv("MAPI_BATCHED_PATH", path)
    res = m.iterate_batched(torch.from_numpy(A).cuda(), torch.from_numpy(B0).cuda(), 15)
    W = res.W.cpu().numpy()
    for v in sorted({0, k - 1}):
        ref = orc.mapi(A, B0[v], 15)
        _t2(W[v], ref.w)
        np.testing.assert_allclose(res.norms.cpu().numpy()[:, v], ref.norms, rtol=1e-5)
