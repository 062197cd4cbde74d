"""Host-side checks of the seeded input generators (synth/): determinism, shapes, recipes."""
import numpy as np

import synth


def test_cfg1_recipe_and_determinism():
    a, b = synth.cfg1(), synth.cfg1()
    assert synth.digest(a["A"], a["b0"]) == synth.digest(b["A"], b["b0"])
    C = a["A"]
    assert C.shape == (256, 256) and C.dtype == np.float32
    np.testing.assert_array_equal(C, C.T)  # mirrored blocks: exactly symmetric
    assert np.all(np.diag(C) > 0)
    np.testing.assert_array_equal(a["b0"], np.full(256, 1 / 16, np.float32))
    # recipe: row-centred N(0,1) X, C = X X^T / 1024  ->  diag ~ 1
    assert 0.8 < float(np.mean(np.diag(C))) < 1.2


def test_covariance_like_block_mirroring_matches_direct():
    r = np.random.default_rng(0)
    F = r.standard_normal((70, 9))
    C = synth.covariance_like(F, 0.5, np.arange(70.0), block=16)
    D = (F @ F.T * 0.5 + np.diag(np.arange(70.0))).astype(np.float32)
    np.testing.assert_allclose(C, D, rtol=1e-6, atol=1e-6)
    np.testing.assert_array_equal(C, C.T)


def test_rmat_quadrant_frequencies():
    src, dst = synth.rmat_edges(1, 200000, seed=9)
    q = np.bincount(src * 2 + dst, minlength=4) / src.size  # (0,0) a, (0,1) b, (1,0) c, (1,1) d
    np.testing.assert_allclose(q, [0.57, 0.19, 0.19, 0.05], atol=0.005)
    s2, d2 = synth.rmat_edges(10, 50000, seed=9)
    assert s2.max() < 1024 and d2.max() < 1024 and s2.min() >= 0


def test_csr_by_destination_dedup_keeps_self_loops():
    src = np.array([0, 0, 1, 2, 2, 2, 3])
    dst = np.array([1, 1, 1, 2, 0, 0, 3])
    row_ptr, col_idx = synth.csr_by_destination(4, src, dst)
    assert list(row_ptr) == [0, 1, 3, 4, 5]
    assert list(col_idx) == [2, 0, 1, 2, 3]
    assert col_idx.dtype == np.int32 and row_ptr.dtype == np.int64


def test_gnutella_like_counts():
    g = synth.gnutella_like()
    assert g["n"] == 6301 and int(g["row_ptr"][-1]) == 20777
    assert len({(int(s), int(d)) for s, d in g["edges"]}) == 20777


def test_random_matrix_padding_is_nan():
    M, lda = synth.random_matrix(5, 7, seed=1, lda=9, kind="mixed")
    assert lda == 9 and M.shape == (5, 9)
    assert np.all(np.isnan(M[:, 7:])) and np.all(np.isfinite(M[:, :7]))


def test_covariance_like_rows_is_a_slice_of_the_full_matrix():
    r = np.random.default_rng(5)
    F = r.standard_normal((96, 7))
    d = np.abs(r.standard_normal(96))
    full = synth.covariance_like(F, 0.25, d, block=32)
    for row0, row1 in ((0, 32), (32, 64), (64, 96), (32, 96)):
        np.testing.assert_array_equal(synth.covariance_like_rows(F, 0.25, d, row0, row1, block=32), full[row0:row1])


def test_stochastic_pca_recipe():
    """C = X^T X has eigenvalues {1, 0.9 x 9} (eigen-gap 0.1) and u1 is its dominant eigenvector."""
    X, u1 = synth.stochastic_pca(N=4000, D=10, gap=0.1, seed=7)
    assert X.dtype == np.float32 and X.shape == (4000, 10)
    ev, V = np.linalg.eigh(X.astype(np.float64).T @ X.astype(np.float64))
    np.testing.assert_allclose(ev, [0.9] * 9 + [1.0], rtol=1e-5)
    assert abs(V[:, -1] @ u1) > 1 - 1e-5
    idx = synth.batch_draws(4000, 7, 33, seed=8)
    assert idx.dtype == np.int32 and idx.shape == (7, 33) and idx.min() >= 0 and idx.max() < 4000
    assert np.array_equal(idx, synth.batch_draws(4000, 7, 33, seed=8))
