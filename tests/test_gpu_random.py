"""Seeded random sweeps over the on-chip / symmetric dense kernels added in round 1 (K2s, K2r, K6t): random
sizes (ragged against every tile shape), random lda padding filled with NaN, random operator, random
starting vectors (positive and mixed-sign), each against the fp64 oracle (T2 after 12 iterations; the RPI
limit for dot).  Complements the hand-picked shapes in test_gpu_dense.py."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

OPS = ["min1", "min2", "dot"]


def _t2(w_gpu, w_orc, norms_gpu, norms_orc):
    a = np.asarray(w_gpu, np.float64)
    b = np.asarray(w_orc, np.float64)
    b = b / np.linalg.norm(b)
    a = a / np.linalg.norm(a)
    assert abs(float(a @ b)) >= 1 - 1e-6
    assert np.max(np.abs(a - b)) <= 1e-4
    np.testing.assert_allclose(np.asarray(norms_gpu, np.float64), norms_orc, rtol=1e-5)


def _case(seed, lo, hi, mult=1, sym=False):
    r = np.random.default_rng(seed)
    n = int(r.integers(lo, hi + 1))
    n = max(mult, n - n % mult)
    op = OPS[int(r.integers(0, 3))]
    G = r.standard_normal((n, n)).astype(np.float32)
    A = (np.triu(G) + np.triu(G, 1).T) if sym else G
    A = A + np.diag(np.abs(r.standard_normal(n)) * 4).astype(np.float32)
    if op == "dot":
        A = ((A + A.T) / (2 * np.sqrt(n))).astype(np.float32)  # symmetric: a real dominant eigenvector
    A = A.astype(np.float32)
    b0 = (np.abs(r.standard_normal(n)) + 0.1) if r.random() < 0.5 else r.standard_normal(n)
    b0 = (b0 / np.linalg.norm(b0)).astype(np.float32)
    pad = int(r.choice([0, 8, 16])) if sym else int(r.integers(0, 9))
    return n, op, A, b0, pad


def _device(A, n, pad, lower_nan=False):
    dev = np.full((n, n + pad), np.nan, np.float32)
    dev[:, :n] = A
    if lower_nan:
        dev[np.tril_indices(n, -1)] = np.nan
    return torch.from_numpy(dev).cuda()[:, :n]


def _check(m, orc, res, A, b0, op):
    ref = orc.rpi(A, b0, 12) if op == "dot" else orc.mapi(A, b0, 12, op=op)
    assert res.iters_done == 12
    got = res.w.cpu().numpy() if op == "dot" else res.w_l2.cpu().numpy()
    _t2(got, ref.w, res.norms.cpu().numpy(), ref.norms)


@pytest.mark.parametrize("seed", range(16))
def test_random_symmetric_k2s(mapi_lib, orc, monkeypatch, seed):
    m = mapi_lib
    n, op, A, b0, pad = _case(1000 + seed, 8, 3000, mult=8, sym=True)
    monkeypatch.setenv("MAPI_SYM_PATH", "sym")
    opc = {"min1": m.MIN1, "min2": m.MIN2, "dot": m.DOT}[op]
    res = m.iterate_sym(_device(A, n, pad, lower_nan=True), torch.from_numpy(b0).cuda(), 12, op=opc)
    _check(m, orc, res, A, b0, op)


@pytest.mark.parametrize("seed", range(16))
def test_random_resident_k2r(mapi_lib, orc, monkeypatch, seed):
    m = mapi_lib
    n, op, A, b0, pad = _case(2000 + seed, 300, 4096)
    monkeypatch.setenv("MAPI_DENSE_PATH", "resident")
    opc = {"min1": m.MIN1, "min2": m.MIN2, "dot": m.DOT}[op]
    res = m.iterate(_device(A, n, pad), torch.from_numpy(b0).cuda(), 12, op=opc)
    _check(m, orc, res, A, b0, op)


@pytest.mark.parametrize("seed", range(16))
def test_random_single_cta_k6t(mapi_lib, orc, monkeypatch, seed):
    m = mapi_lib
    n, op, A, b0, pad = _case(3000 + seed, 2, 256)
    monkeypatch.setenv("MAPI_DENSE_PATH", "single")
    opc = {"min1": m.MIN1, "min2": m.MIN2, "dot": m.DOT}[op]
    res = m.iterate(_device(A, n, pad), torch.from_numpy(b0).cuda(), 12, op=opc)
    _check(m, orc, res, A, b0, op)
