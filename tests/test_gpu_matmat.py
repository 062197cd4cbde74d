"""GPU parity of mapi_mavp_matmat (matrix extension P:69-70) and min-covariance (Eq. 5, Alg. 2 step 4)
against the oracle's matmat: per element |C_gpu - C_orc| <= 1e-5 * sum_k |term| / d (T1 scaled)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _check(C_gpu, A, B, d, orc, op="min1"):
    ref = orc.matmat(A, B, op, d)
    mag = orc.matmat(np.abs(A), np.abs(B), "min1", d)  # sum_k min(|a|,|b|) / d  >=  sum |term| / d
    err = np.abs(np.asarray(C_gpu, np.float64) - ref)
    assert np.all(err <= 1e-5 * mag + 1e-30), float(np.max(err / (mag + 1e-30)))


@pytest.mark.parametrize("m,p,K", [(1, 1, 1), (5, 3, 7), (64, 256, 32), (65, 257, 33), (130, 600, 100),
                                   (300, 70, 1000), (17, 1000, 10)])
@pytest.mark.parametrize("aligned", [True, False])
@pytest.mark.parametrize("op", ["min1", "min2"])
def test_matmat_vs_oracle(mapi_lib, orc, m, p, K, aligned, op):
    mm = mapi_lib
    r = np.random.default_rng(m * 7 + p * 3 + K)
    lda = K + (0 if aligned else 1)
    if aligned:
        lda = (K + 3) // 4 * 4
    A = np.full((m, lda), np.nan, np.float32)
    B = np.full((p, lda), np.nan, np.float32)
    A[:, :K] = r.standard_normal((m, K))
    B[:, :K] = r.standard_normal((p, K))
    A[:, :K][r.random((m, K)) < 0.05] = 0.0
    Ad = torch.from_numpy(A).cuda()[:, :K]
    Bd = torch.from_numpy(B).cuda()[:, :K]
    C = mm.mavp_matmat(Ad, Bd, divisor=3.0, op=mm.MIN1 if op == "min1" else mm.MIN2).cpu().numpy()
    _check(C, np.ascontiguousarray(A[:, :K]), np.ascontiguousarray(B[:, :K]), 3.0, orc, op)


def test_matmat_edge_cases(mapi_lib):
    mm = mapi_lib
    C = torch.full((3, 4), 7.0, device="cuda")
    mm.mavp_matmat(torch.empty(3, 0, device="cuda"), torch.empty(4, 0, device="cuda"), C=C)
    torch.cuda.synchronize()
    assert C.abs().sum().item() == 0.0  # K = 0 -> C = 0
    out = mm.mavp_matmat(torch.empty(0, 5, device="cuda"), torch.ones(2, 5, device="cuda"))
    assert tuple(out.shape) == (0, 2)
    with pytest.raises(mm.MapiError):
        mm.mavp_matmat(torch.ones(2, 5, device="cuda"), torch.ones(2, 5, device="cuda"), divisor=0.0)
    v = torch.tensor([[1.0, -2.0]], device="cuda")
    assert mm.mavp_matmat(v, v).tolist() == [[3.0]]


def test_min_covariance_paper_shape(mapi_lib, orc):
    """Alg. 2 step 4 on the paper's image shape (128x128 pixels, N = 10 occluded copies): the full
    16384^2 min-covariance, bitwise symmetric, diagonal = ||v_i||_1/(N-1), 2048 sampled rows vs oracle."""
    mm = mapi_lib
    V, _ = synth.occluded_images()
    Vd = torch.from_numpy(V).cuda()
    C = mm.min_covariance(Vd)
    torch.cuda.synchronize()
    assert tuple(C.shape) == (16384, 16384)
    assert torch.equal(C, C.T)
    r = np.random.default_rng(0)
    rows = np.sort(r.choice(16384, 2048, replace=False))
    Crow = C[torch.from_numpy(rows).cuda()].cpu().numpy()
    ref = orc.matmat(np.ascontiguousarray(V[rows]), V, "min1", 9.0)
    mag = orc.matmat(np.ascontiguousarray(np.abs(V[rows])), np.abs(V), "min1", 9.0)
    assert np.all(np.abs(Crow - ref) <= 1e-5 * mag + 1e-30)
    np.testing.assert_allclose(np.diag(Crow[:, rows]) if False else Crow[np.arange(2048), rows],
                               np.abs(V[rows].astype(np.float64)).sum(axis=1) / 9.0, rtol=2e-6)


def test_min_covariance_large_K_symmetric(mapi_lib, orc):
    """Large inner dimension (ALU-bound regime): 1024 x 4096 samples, cp.async path."""
    mm = mapi_lib
    r = np.random.default_rng(3)
    V = r.standard_normal((1024, 4096)).astype(np.float32)
    C = mm.min_covariance(torch.from_numpy(V).cuda(), divisor=4096.0)
    assert torch.equal(C, C.T)
    rows = np.arange(0, 1024, 97)
    Crow = C[torch.from_numpy(rows).cuda()].cpu().numpy()
    ref = orc.matmat(np.ascontiguousarray(V[rows]), V, "min1", 4096.0)
    mag = orc.matmat(np.ascontiguousarray(np.abs(V[rows])), np.abs(V), "min1", 4096.0)
    assert np.all(np.abs(Crow - ref) <= 1e-5 * mag + 1e-30)


@pytest.mark.parametrize("m,p,K", [(1, 1, 1), (33, 257, 3), (64, 256, 4), (100, 300, 10), (97, 513, 12), (300, 70, 8)])
@pytest.mark.parametrize("op", ["min1", "min2"])
def test_small_k_kernel_bitwise_vs_tiled(mapi_lib, orc, monkeypatch, m, p, K, op):
    """K8s (B columns in registers, K <= 12) accumulates every element in ascending k from 0, as K8
    does for K <= 32: bitwise-identical C; both within T1 of the oracle; divisor applied."""
    mm = mapi_lib
    r = np.random.default_rng(m * 1000 + p + K)
    A = r.standard_normal((m, K)).astype(np.float32)
    B = r.standard_normal((p, K)).astype(np.float32)
    opc = mm.MIN1 if op == "min1" else mm.MIN2
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    small = mm.mavp_matmat(Ad, Bd, 9.0, op=opc)
    monkeypatch.setenv("MAPI_MATMAT_PATH", "tiled")
    tiled = mm.mavp_matmat(Ad, Bd, 9.0, op=opc)
    torch.cuda.synchronize()
    assert torch.equal(small, tiled)
    _check(small.cpu().numpy(), A, B, 9.0, orc, op)
