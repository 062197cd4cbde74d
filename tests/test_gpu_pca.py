"""GPU parity of mapi_pca_topk (MAPI + L2 deflation; BASELINE configs[1]) vs the oracle.

T2 per principal vector: |cos| >= 1 - 1e-6 and max|diff| <= 1e-4 on the l2-unit vectors; the
per-iteration norms relative <= 1e-5 for every vector, deflated ones included (measured at cfg2 with the
fp32-rounded D_i: max 5.3e-6 for vector 8, profiles/r02_cfg2_norms.log; reading R8 in DESIGN.md).  cfg2 is checked end-to-end and
conditioned (the GPU iteration fed the oracle's own D_i, rounded once to fp32) to localise error.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _t2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    a = a / np.linalg.norm(a)
    b = b / np.linalg.norm(b)
    cos = float(a @ b)
    assert abs(cos) >= 1 - 1e-6, f"|cos| {abs(cos)!r}"
    assert np.max(np.abs(a - b)) <= 1e-4, f"max abs {np.max(np.abs(a - b))}"


@pytest.mark.parametrize("n,k", [(64, 4), (257, 3), (1000, 5)])
def test_pca_small(mapi_lib, orc, n, k):
    m = mapi_lib
    r = np.random.default_rng(n)
    X = r.standard_normal((n, 2 * n))
    X[r.random(X.shape) < 0.05] = 10.0
    X -= X.mean(axis=1, keepdims=True)
    C = synth.covariance_like(X, 1.0 / (2 * n))
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    res = m.pca_topk(torch.from_numpy(C).cuda(), k, 40, torch.from_numpy(b0).cuda())
    ref = orc.pca_topk(C, k, 40, b0)
    assert ref.status == orc.OK
    P = res.P.cpu().numpy()
    np.testing.assert_allclose(np.linalg.norm(P, axis=1), 1.0, rtol=1e-6)
    for i in range(k):
        _t2(P[i], ref.P[i])
        np.testing.assert_allclose(res.norms[i].cpu().numpy(), ref.norms[i], rtol=1e-5)


def test_pca_k1_equals_iterate(mapi_lib):
    m = mapi_lib
    cfg = synth.cfg1()
    C = torch.from_numpy(cfg["A"]).cuda()
    b0 = torch.from_numpy(cfg["b0"]).cuda()
    res = m.pca_topk(C, 1, 50, b0)
    it = m.iterate(C, b0, 50)
    w = it.w.double()
    np.testing.assert_allclose(res.P[0].cpu().numpy(), (w / w.norm()).float().cpu().numpy(), rtol=1e-6,
                               atol=1e-8)
    assert torch.equal(res.norms[0], it.norms)


@pytest.mark.parametrize("n,k,pad", [(1500, 3, 0), (3001, 4, 5), (4096, 8, 0)])
def test_pca_fused_deflation_bitwise(mapi_lib, monkeypatch, n, k, pad):
    """K2r stages D_i = fp32(C - sum p_m r_m^T) itself when MAPI_PCA_FUSE=1 (no D_i written to memory): P,
    norms and deltas are bitwise those of the separate build kernel, ragged n and padded ldc included."""
    m = mapi_lib
    r = np.random.default_rng(n + k)
    X = r.standard_normal((n, 2 * n // 3)).astype(np.float32)
    Cf = np.full((n, n + pad), np.nan, np.float32)
    Cf[:, :n] = (X @ X.T / X.shape[1]).astype(np.float32)
    C = torch.from_numpy(Cf).cuda()[:, :n]
    b0 = torch.full((n,), 1 / np.sqrt(n), device="cuda")
    monkeypatch.setenv("MAPI_PCA_FUSE", "1")
    fused = m.pca_topk(C, k, 30, b0)
    monkeypatch.setenv("MAPI_PCA_FUSE", "0")
    sep = m.pca_topk(C, k, 30, b0)
    assert torch.equal(fused.P, sep.P) and torch.equal(fused.norms, sep.norms) and torch.equal(fused.deltas, sep.deltas)


@pytest.mark.parametrize("n", [64, 300, 4096])
def test_pca_degenerate_reports_vector(mapi_lib, n):
    """The per-vector status words are read back once after the last vector: a degenerate first vector
    (C = 0) still reports MAPI_ERR_DEGENERATE with its index, and the stream stays usable."""
    m = mapi_lib
    b0 = torch.full((n,), 1 / np.sqrt(n), device="cuda")
    with pytest.raises(m.MapiError) as ei:
        m.pca_topk(torch.zeros(n, n, device="cuda"), 3, 10, b0)
    assert ei.value.name == "MAPI_ERR_DEGENERATE" and "vector 0" in str(ei.value)
    C = torch.eye(n, device="cuda") * 2
    ok = m.pca_topk(C, 1, 5, b0)
    assert torch.isfinite(ok.P).all()


@pytest.fixture(scope="module")
def cfg2():
    cfg = synth.cfg2(device="cuda")
    cfg["A_host"] = cfg["A"].cpu().numpy()
    return cfg


def test_cfg2_end_to_end(mapi_lib, orc, cfg2):
    m = mapi_lib
    k, T = cfg2["k"], cfg2["iters"]
    res = m.pca_topk(cfg2["A"], k, T, torch.from_numpy(cfg2["b0"]).cuda())
    ref = orc.pca_topk(cfg2["A_host"], k, T, cfg2["b0"])
    assert ref.status == orc.OK
    P = res.P.cpu().numpy()
    for i in range(k):
        _t2(P[i], ref.P[i])
        np.testing.assert_allclose(res.norms[i].cpu().numpy(), ref.norms[i], rtol=1e-5)
    cfg2["oracle_P"] = ref.P


def test_cfg2_conditioned(mapi_lib, orc, cfg2):
    """Stage i of the GPU pipeline fed the oracle's D_i (fp64, rounded once to fp32)."""
    m = mapi_lib
    T = cfg2["iters"]
    P_orc = cfg2.get("oracle_P")
    if P_orc is None:
        P_orc = orc.pca_topk(cfg2["A_host"], cfg2["k"], T, cfg2["b0"]).P
    b0 = torch.from_numpy(cfg2["b0"]).cuda()
    for i in (1, 4, 7):
        D = orc.deflate(cfg2["A_host"], P_orc, i)
        D32 = torch.from_numpy(D.astype(np.float32)).cuda()
        res = m.iterate(D32, b0, T)
        _t2(res.w_l2.cpu().numpy(), P_orc[i])
