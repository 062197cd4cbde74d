"""GPU parity of Algorithm 3, mini-batch MAPI with momentum (mapi_minibatch, K10, readings R14 /
R15) against the fp64 oracle's step-by-step Algorithm 3 on the same fp32 samples and the same batch draws."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
GRAM = {"min1": 0, "dot": 2}


def _run(m, X, idx, beta, w0, gram):
    res = m.minibatch(torch.from_numpy(X).cuda(), torch.from_numpy(idx).cuda(), beta,
                      torch.from_numpy(w0).cuda(), gram=GRAM[gram])
    return res.w.cpu().numpy(), res.w_l2.cpu().numpy(), res.norms.cpu().numpy(), res.iters_done


def _t2(orc, X, idx, beta, w0, gram, got, norm_rtol=1e-5):
    w, wl2, norms, done = got
    ref = orc.minibatch_mapi(X.astype(np.float64), idx.astype(np.int64), beta, w0.astype(np.float64), gram=gram)
    assert ref.status == 0 and done == ref.iters_done == idx.shape[0]
    cos = abs(float(np.dot(wl2.astype(np.float64), ref.w_l2)))
    assert cos >= 1 - 1e-6, cos
    assert np.max(np.abs(wl2 - ref.w_l2)) <= 1e-4
    np.testing.assert_allclose(norms, ref.norms, rtol=norm_rtol)
    assert abs(np.sum(np.abs(w.astype(np.float64))) - 1) < 1e-5  # l1-unit iterate (step 5)


def _w0(D, seed):
    w = np.random.default_rng(seed).standard_normal(D)
    return (w / np.linalg.norm(w)).astype(np.float32)


def _paper_data():
    """The paper's experiment shape: D = 10, the eigen-gap dataset (N = 10^5 here), entries rescaled
    by sqrt(N) so |x| is comparable to |w| (with the literal 1/sqrt(N) scale every term is |M_jk|)."""
    X, _ = synth.stochastic_pca(N=100_000, D=10, seed=7)
    return (X * np.float32(np.sqrt(X.shape[0]))).astype(np.float32)


@pytest.mark.parametrize("gram", ["min1", "dot"])
@pytest.mark.parametrize("beta", [0.0, 0.225])
def test_paper_shape_s1024(mapi_lib, orc, gram, beta):
    """T = 100 end to end at s = 1024, where the stochastic iteration does not amplify rounding differences
    (measured: per-iteration norm error <= 1e-7 throughout, K10)."""
    X = _paper_data()
    idx = synth.batch_draws(X.shape[0], 100, 1024, seed=8)
    w0 = _w0(10, 1)
    _t2(orc, X, idx, beta, w0, gram, _run(mapi_lib, X, idx, beta, w0, gram))


@pytest.mark.parametrize("gram", ["min1", "dot"])
@pytest.mark.parametrize("beta", [0.0, 0.225])
def test_paper_shape_s128(mapi_lib, orc, gram, beta):
    """s = 128 (the small-batch regime): the iteration is a noisy map that is NOT contractive, so an fp32
    rounding difference of 5e-8 at t = 0 grows to ~1e-3 by t = 100 (scripts/probe_alg3_gpu.py).  End-to-end
    parity is therefore taken over a short horizon (T = 8), and at T = 100 every step is checked
    CONDITIONED on the GPU's own state: the oracle continues from the GPU's (w_t, w_prev_t) for 4 steps."""
    m = mapi_lib
    X = _paper_data()
    idx = synth.batch_draws(X.shape[0], 100, 128, seed=8)
    w0 = _w0(10, 1)
    _t2(orc, X, idx[:8], beta, w0, gram, _run(m, X, idx[:8], beta, w0, gram))
    Xd, w0d = torch.from_numpy(X).cuda(), torch.from_numpy(w0).cuda()
    X64 = X.astype(np.float64)
    for t0 in (1, 17, 60, 96):
        a = m.minibatch(Xd, torch.from_numpy(idx[:t0]).cuda(), beta, w0d, gram=GRAM[gram])
        b = m.minibatch(Xd, torch.from_numpy(idx[t0:t0 + 4]).cuda(), beta, a.w, gram=GRAM[gram], w_prev0=a.deltas)
        ref = orc.minibatch_mapi(X64, idx[t0:t0 + 4].astype(np.int64), beta, a.w.cpu().numpy().astype(np.float64),
                                 gram=gram, w_prev0=a.deltas.cpu().numpy().astype(np.float64))
        assert abs(float(np.dot(b.w_l2.cpu().numpy().astype(np.float64), ref.w_l2))) >= 1 - 1e-6
        assert np.max(np.abs(b.w_l2.cpu().numpy() - ref.w_l2)) <= 1e-4
        np.testing.assert_allclose(b.norms.cpu().numpy(), ref.norms, rtol=1e-5)
        np.testing.assert_allclose(b.deltas.cpu().numpy(), ref.w_prev, rtol=1e-5, atol=1e-7)
    # continuing a run is bitwise the same as running it in one call
    full = m.minibatch(Xd, torch.from_numpy(idx).cuda(), beta, w0d, gram=GRAM[gram])
    a = m.minibatch(Xd, torch.from_numpy(idx[:37]).cuda(), beta, w0d, gram=GRAM[gram])
    b = m.minibatch(Xd, torch.from_numpy(idx[37:]).cuda(), beta, a.w, gram=GRAM[gram], w_prev0=a.deltas)
    assert torch.equal(b.w, full.w) and torch.equal(b.deltas, full.deltas)
    assert torch.equal(torch.cat([a.norms, b.norms]), full.norms)


def test_paper_literal_scale(mapi_lib, orc):
    X, _ = synth.stochastic_pca(N=100_000, D=10, seed=7)  # entries ~ 1/sqrt(N)
    idx = synth.batch_draws(X.shape[0], 100, 1024, seed=9)
    w0 = _w0(10, 2)
    _t2(orc, X, idx, 0.225, w0, "min1", _run(mapi_lib, X, idx, 0.225, w0, "min1"))


@pytest.mark.parametrize("D,s,T", [(1, 1, 1), (2, 3, 5), (7, 129, 9), (31, 300, 12), (33, 257, 6), (64, 200, 8),
                                   (10, 5000, 3), (45, 4097, 2)])
def test_shapes(mapi_lib, orc, D, s, T):
    """Ragged folds (s % 128 != 0), several chunks (s > 4096), D across the pairs-per-thread variants and the
    two-terms-per-lane rows (D > 32), padded rows (ldx > D) with NaN in the padding."""
    r = np.random.default_rng(100 * D + s)
    N = 700
    Xp = np.full((N, D + 3), np.nan, np.float32)
    Xp[:, :D] = (0.4 * r.standard_normal((N, D))).astype(np.float32)
    idx = synth.batch_draws(N, T, s, seed=D + T)
    w0 = _w0(D, D)
    m = mapi_lib
    Xd = torch.from_numpy(Xp).cuda()[:, :D]  # row-major view, stride(0) = D + 3
    res = m.minibatch(Xd, torch.from_numpy(idx).cuda(), 0.1, torch.from_numpy(w0).cuda())
    got = (res.w.cpu().numpy(), res.w_l2.cpu().numpy(), res.norms.cpu().numpy(), res.iters_done)
    _t2(orc, np.ascontiguousarray(Xp[:, :D]), idx, 0.1, w0, "min1", got)


def test_full_batch_no_momentum_is_algorithm_1(mapi_lib):
    """beta = 0 with every batch = all samples once: Alg. 3 is Alg. 1 on M = (1/N) sum_i x_i (.) x_i^T — the
    library's own mapi_iterate on the min-covariance of mapi_mavp_matmat (K8), two independent kernels."""
    m = mapi_lib
    r = np.random.default_rng(5)
    N, D, T = 300, 12, 20
    X = (0.5 * r.standard_normal((N, D))).astype(np.float32)
    idx = np.tile(np.arange(N, dtype=np.int32), (T, 1))
    w0 = _w0(D, 3)
    res = m.minibatch(torch.from_numpy(X).cuda(), torch.from_numpy(idx).cuda(), 0.0, torch.from_numpy(w0).cuda())
    Xt = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    C = m.min_covariance(Xt, divisor=N)  # C_jk = (1/N) sum_i x_ij (.) x_ik
    ref = m.iterate(C, torch.from_numpy(w0).cuda(), T)
    assert abs(float(torch.dot(res.w_l2.double(), ref.w_l2.double()))) >= 1 - 1e-6
    np.testing.assert_allclose(res.norms.cpu().numpy(), ref.norms.cpu().numpy(), rtol=1e-5)


def test_bitwise_repeatable(mapi_lib):
    m = mapi_lib
    X, _ = synth.stochastic_pca(N=20_000, D=10, seed=3)
    X = torch.from_numpy((X * np.float32(140.0)).astype(np.float32)).cuda()
    idx = torch.from_numpy(synth.batch_draws(20_000, 50, 128, seed=4)).cuda()
    w0 = torch.from_numpy(_w0(10, 9)).cuda()
    a = m.minibatch(X, idx, 0.225, w0)
    b = m.minibatch(X, idx, 0.225, w0)
    assert torch.equal(a.w, b.w) and torch.equal(a.norms, b.norms) and torch.equal(a.w_l2, b.w_l2)


def test_errors(mapi_lib):
    m = mapi_lib
    X = torch.zeros(50, 4, device="cuda")
    idx = torch.zeros(3, 8, dtype=torch.int32, device="cuda")
    w0 = torch.full((4,), 0.5, device="cuda")
    with pytest.raises(m.MapiError) as e:  # all-zero samples: ||w_1||_1 = 0 (w_{-1} = 0)
        m.minibatch(X, idx, 0.1, w0)
    assert e.value.status == 4 and e.value.iters_done == 0
    Xn = torch.randn(50, 4, device="cuda")
    Xn[7, 2] = float("inf")
    idx7 = torch.full((3, 8), 7, dtype=torch.int32, device="cuda")
    with pytest.raises(m.MapiError) as e:
        m.minibatch(Xn, idx7, 0.1, torch.full((4,), float("inf"), device="cuda"))
    assert e.value.status == 6
    bad = idx.clone()
    bad[1, 3] = 50
    with pytest.raises(m.MapiError) as e:  # an index outside [0, N)
        m.minibatch(torch.randn(50, 4, device="cuda"), bad, 0.1, w0)
    assert e.value.status == 3
    with pytest.raises(m.MapiError) as e:  # D > 64
        m.minibatch(torch.randn(10, 65, device="cuda"), idx, 0.1, torch.ones(65, device="cuda"))
    assert e.value.status == 2
