"""GPU parity of Alg. 2's MAVP deflation (step 6) and reconstruction (steps 3 + 8)
against the oracle's literal Q materialisation, and the end-to-end image
reconstruction pipeline on the paper's image shape (synthetic stand-in images)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
OPS = {"min1": 0, "min2": 1, "dot": 2}


def _mag(orc, W, X, rows=None):
    """|X| + sum_j |Q_ij| |X_jk| >= every partial sum's magnitude (tolerance scale)."""
    Wa = np.abs(np.asarray(W, np.float32))
    Xa = np.abs(np.asarray(X, np.float32))
    if rows is None:
        return Xa + orc.outer_apply(Wa, Xa, "min1") * (Wa.shape[1] if Wa.ndim > 1 else 1)
    return Xa[rows] + orc.outer_apply_rows(Wa, Xa, rows, "min1") * (Wa.shape[1] if Wa.ndim > 1 else 1)


def _close(gpu, ref, mag):
    err = np.abs(np.asarray(gpu, np.float64) - ref)
    tol = 1e-6 * mag + 1.2e-7 * np.abs(ref) + 1e-30
    assert np.all(err <= tol), float(np.max(err / tol))


@pytest.mark.parametrize("M", [1, 7, 300, 1000, 2049])
@pytest.mark.parametrize("op", ["min1", "min2", "dot"])
def test_mavp_deflate_vs_oracle(mapi_lib, orc, M, op):
    m = mapi_lib
    r = np.random.default_rng(M)
    X = r.standard_normal((M, M + 40))  # a covariance-like symmetric C
    C = (X @ X.T / (M + 40)).astype(np.float32)
    w = r.standard_normal(M)
    w[r.random(M) < 0.1] = 0.0
    w[: min(M, 5)] = w[0]  # ties in |w|
    w = (w / max(np.linalg.norm(w), 1e-30)).astype(np.float32)
    D = m.mavp_deflate(torch.from_numpy(C).cuda(), torch.from_numpy(w).cuda(), op=OPS[op]).cpu().numpy()
    ref = orc.mavp_deflate(C, w, op)
    _close(D, ref, _mag(orc, w[:, None], C))


def test_mavp_deflate_spec_e1_exact(mapi_lib):
    m = mapi_lib
    C = torch.randn(50, 50, device="cuda")
    w = torch.zeros(50, device="cuda")
    w[0] = 1.0
    D = m.mavp_deflate(C, w)
    assert torch.all(D[0] == 0) and torch.equal(D[1:], C[1:])


@pytest.mark.parametrize("op", ["min1", "min2", "dot"])
def test_reconstruct_vs_oracle(mapi_lib, orc, op):
    m = mapi_lib
    V, _ = synth.occluded_copies(D=64, N=10, seed=9, tile=16)  # raw 4096 x 10 (centred inside, step 3)
    r = np.random.default_rng(1)
    W = r.standard_normal((4096, 2))
    W = (W / np.linalg.norm(W, axis=0)).astype(np.float32)
    Vh, mean = m.mavp_reconstruct(torch.from_numpy(W).cuda(), torch.from_numpy(V).cuda(), op=OPS[op])
    ref, m_ref = orc.reconstruct(W, V, op)
    np.testing.assert_allclose(mean.cpu().numpy(), m_ref, rtol=1e-6, atol=1e-7)
    Xc = (V.astype(np.float64) - m_ref[:, None]).astype(np.float32)
    _close(Vh.cpu().numpy(), ref, _mag(orc, W, Xc) + np.abs(m_ref)[:, None])


def test_alg2_pipeline_paper_shape(mapi_lib, orc):
    """Alg. 2 on 128x128 images, N = 10 occluded copies (3 of 16 tiles of U[0,1] noise): every step on
    the GPU; the deflated matrix checked on sampled rows against the oracle's literal product, and the
    reconstruction must beat the occluded inputs in PSNR (S:283-287 property)."""
    m = mapi_lib
    V_raw, img = synth.occluded_copies()  # steps 1-2: 10 occluded 128x128 copies as columns
    Vd = torch.from_numpy(V_raw).cuda()
    Vc, mean = m.center_rows(Vd)
    C = m.min_covariance(Vc)  # step 4, divisor N-1
    b0 = torch.full((16384,), 1.0 / 128.0, device="cuda")
    # steps 5-7 use the l1-unit MAPI outputs (reading R11: w (+) w = ||w||_1, so ||w||_1 = 1 makes the MAVP
    # outer product the analogue of the projector u u^T; with l2-unit w it is ~sqrt(M) too large)
    w1 = m.iterate(C, b0, 100).w  # step 5
    D = m.mavp_deflate(C, w1)  # step 6
    w2 = m.iterate(D, b0, 100).w
    W = torch.stack([w1, w2], dim=1).contiguous()  # step 7
    Vhat, _ = m.mavp_reconstruct(W, Vd)  # step 8
    torch.cuda.synchronize()
    # deflation on 8 sampled rows vs the oracle's literal (w1 (+) w1^T) C
    rows = np.array([0, 1, 4097, 8191, 8192, 12000, 16000, 16383])
    C_h = C.cpu().numpy()
    w1_h = w1.cpu().numpy()
    ref = orc.outer_apply_rows(w1_h[:, None], C_h, rows, "min1", subtract=True)
    mag = np.abs(C_h[rows]) + orc.outer_apply_rows(np.abs(w1_h)[:, None], np.abs(C_h), rows, "min1")
    _close(D.cpu().numpy()[rows], ref, mag)
    # reconstruction quality (clamped to [0,1]): better than the occluded copies on average
    Vh = np.clip(Vhat.cpu().numpy(), 0, 1)
    Vo = Vd.cpu().numpy()
    p_rec = np.mean([orc.psnr(img.reshape(-1), Vh[:, i]) for i in range(10)])
    p_occ = np.mean([orc.psnr(img.reshape(-1), Vo[:, i]) for i in range(10)])
    assert p_rec > p_occ + 5.0, (p_rec, p_occ)  # paper, Table 1: 16.31 -> 24.05 dB (min1)
