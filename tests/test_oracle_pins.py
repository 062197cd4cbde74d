"""Pins for the fp64 oracle (oracle/oracle.c) against things other than itself.

Each test checks the oracle against what the paper and mathematics fix: SPEC/paper worked
examples (tests/golden/), the north-star MAVP invariants, literal brute force
(oracle/brute.py, independent pure-Python loops), closed forms, Proposition 1, the RPI
limit vs LAPACK, the deflation identity vs a numpy matrix product, and the CSR ranking
form vs the materialised Google matrix.  Chosen so that a dropped term, a wrong sign or
index, a transposed operand, or the wrong normalisation fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import synth
from oracle import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _seq_sum(v):
    s = 0.0
    for x in v:
        s += float(x)
    return s


# ---------------------------------------------------------------- worked examples


def test_spec_mavp_dot_examples(orc):
    for case in _gold("spec_examples.json")["mavp_dot"]:
        got = orc.mavp_dot(case["w"], case["x"], case["op"])
        assert got == case["expect"], case["cite"]


def test_spec_matvec_examples(orc):
    for case in _gold("spec_examples.json")["matvec"]:
        A = np.asarray(case["A"], dtype=np.float32)
        y = orc.matvec(A, case["x"], case["op"])
        assert list(y) == case["expect"], case["cite"]


def test_spec_diamond_fixed_point(orc):
    case = _gold("spec_examples.json")["diamond_fixed_point"][0]
    A = np.asarray(case["A"], dtype=np.float32)
    r = orc.power_iterate(A, [0.3, 0.7], 2, op="diamond", norm=orc.NORM_L1)
    np.testing.assert_allclose(r.w, case["expect"], rtol=0, atol=1e-15)


def test_spec_rpi_limit(orc):
    case = _gold("spec_examples.json")["rpi"][0]
    A = np.asarray(case["A"], dtype=np.float32)
    r = orc.rpi(A, [0.6, 0.8], case["iters"])
    np.testing.assert_allclose(np.abs(r.w), case["expect_abs"], atol=case["tol"])


# ---------------------------------------------------------------- MAVP invariants (north star)


def _cases(n_cases=300, seed=11):
    r = np.random.default_rng(seed)
    for _ in range(n_cases):
        n = int(r.integers(1, 9))
        x = r.standard_normal(n) * 10.0 ** r.uniform(-3, 3)
        y = r.standard_normal(n) * 10.0 ** r.uniform(-3, 3)
        x[r.random(n) < 0.15] = 0.0
        y[r.random(n) < 0.15] = 0.0
        yield x, y


def test_l1_induction(orc):
    # x (+) x = sum_i min(|x_i|,|x_i|) = ||x||_1, for min1 and min2
    for x, _ in _cases():
        l1 = _seq_sum(np.abs(x))
        assert orc.mavp_dot(x, x, "min1") == l1
        assert orc.mavp_dot(x, x, "min2") == l1


def test_symmetry_oddness_bound(orc):
    for x, y in _cases():
        xy = orc.mavp_dot(x, y, "min1")
        assert xy == orc.mavp_dot(y, x, "min1")  # symmetry, exact
        assert orc.mavp_dot(-x, y, "min1") == -xy  # oddness (-x)(+)y = -(x(+)y), exact
        assert orc.mavp_dot(x, -y, "min1") == -xy
        bound = min(np.abs(x).sum(), np.abs(y).sum())
        assert abs(xy) <= bound * (1 + 1e-15)
        assert orc.mavp_dot(x, y, "min2") >= 0.0
        assert orc.mavp_dot(x, y, "min2") == orc.mavp_dot(y, x, "min2")


def test_joint_homogeneity(orc):
    for i, (x, y) in enumerate(_cases()):
        xy = orc.mavp_dot(x, y, "min1")
        assert orc.mavp_dot(4.0 * x, 4.0 * y, "min1") == 4.0 * xy  # exact for powers of 2
        c = 0.37 + i * 0.01
        assert orc.mavp_dot(c * x, c * y, "min1") == pytest.approx(c * xy, rel=1e-12, abs=1e-300)


def test_not_homogeneous_in_one_argument(orc):
    # min(|a|,|c b|) != c min(|a|,|b|): a product in place of the min would pass this
    x = np.array([1.0, -2.0, 0.5])
    y = np.array([0.3, 0.4, -5.0])
    assert orc.mavp_dot(x, 100 * y, "min1") != pytest.approx(100 * orc.mavp_dot(x, y, "min1"))


def test_min1_equals_min2_when_signs_agree(orc):
    r = np.random.default_rng(3)
    for _ in range(100):
        n = int(r.integers(1, 9))
        x = np.abs(r.standard_normal(n))
        y = np.abs(r.standard_normal(n))
        s = np.where(r.random(n) < 0.5, -1.0, 1.0)
        assert orc.mavp_dot(s * x, s * y, "min1") == orc.mavp_dot(s * x, s * y, "min2")


def test_diamond_positive_vectors(orc):
    r = np.random.default_rng(4)
    for _ in range(50):
        n = int(r.integers(1, 9))
        w, x = r.random(n) + 0.01, r.random(n) + 0.01
        assert orc.mavp_dot(w, x, "diamond") == pytest.approx(w.sum() + x.sum(), rel=1e-14)


# ---------------------------------------------------------------- brute force (independent loops)


@pytest.mark.parametrize("op", ["min1", "min2", "diamond", "dot"])
def test_dot_vs_brute(orc, op):
    f = brute.OPS[op]
    for x, y in _cases(200, seed=12):
        assert orc.mavp_dot(x, y, op) == pytest.approx(f(x, y), rel=1e-14, abs=1e-300)


@pytest.mark.parametrize("op", ["min1", "min2", "diamond", "dot"])
def test_matvec_vs_brute_nonsquare(orc, op):
    r = np.random.default_rng(21)
    for trial in range(60):
        m, n = int(r.integers(1, 9)), int(r.integers(1, 9))
        M, lda = synth.random_matrix(m, n, seed=100 + trial, lda=n + int(r.integers(0, 3)),
                                     kind="mixed" if trial % 2 else "normal")
        x = synth.random_vector(n, seed=200 + trial, kind="mixed")
        y = orc.matvec(M[:, :n], x, op)
        exp = brute.matvec(M[:, :n].astype(np.float64), x.astype(np.float64), op)
        np.testing.assert_allclose(y, exp, rtol=1e-13, atol=1e-300)


def test_matvec_row_orientation(orc):
    # y_j uses ROW j of A (reading Q6): a transposed operand fails this
    A = np.array([[3.0, 0.0], [1.0, 1.0]], np.float32)
    y = orc.matvec(A, [1.0, 0.5])
    assert list(y) == [1.0, 1.5]


def test_mavp_magnitude_scale(orc):
    A = np.array([[1.0, -2.0, 0.0], [-0.5, 0.25, 4.0]], np.float32)
    x = np.array([-1.0, 1.0, 2.0])
    y, mag = orc.matvec(A, x, return_mag=True)
    assert list(y) == [-2.0, 2.75]
    assert list(mag) == [2.0, 2.75]


@pytest.mark.parametrize("op", ["min1", "min2"])
def test_mapi_vs_brute(orc, op):
    r = np.random.default_rng(31)
    for trial in range(40):
        n = int(r.integers(1, 9))
        A = r.standard_normal((n, n)).astype(np.float32)  # non-symmetric on purpose
        if op == "min2":
            A = np.abs(A)
        b0 = np.abs(r.standard_normal(n)) + 0.1
        b0 /= np.linalg.norm(b0)
        res = orc.mapi(A, b0, 6, op=op)
        if res.status != orc.OK:
            continue
        w, norms = brute.mapi(A.astype(np.float64), b0, 6, op)
        np.testing.assert_allclose(res.w, w, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(res.norms, norms, rtol=1e-12)
        assert np.sum(np.abs(res.w)) == pytest.approx(1.0, abs=1e-12)


def test_rpi_vs_brute(orc):
    r = np.random.default_rng(32)
    A = r.standard_normal((6, 6)).astype(np.float32)
    b0 = r.random(6) + 0.1
    res = orc.rpi(A, b0, 7)
    np.testing.assert_allclose(res.w, brute.rpi(A.astype(np.float64), b0, 7), rtol=1e-12)


# ---------------------------------------------------------------- closed forms


def test_identity_fixed_point(orc):
    # A = I, w0 with |w0_k| <= 1 -> w_1 = w0/||w0||_1 and stationary; s_0 = ||w0||_1
    r = np.random.default_rng(41)
    for n in (1, 2, 5, 33):
        b0 = r.standard_normal(n)
        b0 /= np.linalg.norm(b0)
        A = np.eye(n, dtype=np.float32)
        res = orc.mapi(A, b0, 5)
        l1 = np.abs(b0).sum()
        np.testing.assert_allclose(res.w, b0 / l1, rtol=1e-15, atol=1e-17)
        assert res.norms[0] == pytest.approx(l1, rel=1e-15)
        assert res.deltas[0] == pytest.approx(np.abs(b0 / l1 - b0).sum(), rel=1e-13, abs=1e-17)
        assert np.all(res.deltas[1:] <= 1e-15)  # stationary up to fp64 rounding of 1/s
        assert res.norms[1] == pytest.approx(1.0, rel=1e-15)
        np.testing.assert_allclose(res.w_l2, b0, rtol=1e-13, atol=1e-16)


def test_sign_regime_equals_l1_rpi_on_signA(orc):
    # all |a_jk| >= 1 and ||w||_1 = 1  =>  min(|a|,|w|) = |w|  =>  A (+) w = sign(A) w
    r = np.random.default_rng(42)
    n = 24
    S = np.sign(r.standard_normal((n, n)))
    S = np.triu(S) + np.triu(S, 1).T
    A = (S * (1.0 + np.abs(r.standard_normal((n, n))) * 3)).astype(np.float32)
    A = np.triu(A) + np.triu(A, 1).T
    b0 = r.standard_normal(n)
    b0 /= np.linalg.norm(b0)
    T = 400
    res = orc.mapi(A, b0, T)
    w = b0.copy()
    for _ in range(T):  # l1-normalised RPI on sign(A) by numpy matmul
        y = S @ w
        w = y / np.abs(y).sum()
    np.testing.assert_allclose(res.w, w, rtol=1e-9, atol=1e-12)
    evals, evecs = np.linalg.eigh(S)  # LAPACK
    order = np.argsort(np.abs(evals))
    lam1, lam2 = evals[order[-1]], evals[order[-2]]
    assert abs(lam2 / lam1) < 0.95 and lam1 > 0 and abs(evals.min()) < lam1
    u = evecs[:, order[-1]]
    wl2 = res.w_l2 * np.sign(res.w_l2 @ u)
    np.testing.assert_allclose(wl2, u, atol=1e-6)


def test_sign_rank_one_one_step(orc):
    r = np.random.default_rng(43)
    n = 17
    s = np.where(r.random(n) < 0.5, -1.0, 1.0)
    m = 1.0 + r.random((n, n)) * 5
    A = (s[:, None] * s[None, :] * m).astype(np.float32)
    b0 = r.standard_normal(n)
    b0 /= np.linalg.norm(b0)
    res = orc.mapi(A, b0, 1)
    np.testing.assert_allclose(res.w, np.sign(s @ b0) * s / n, rtol=1e-14)


def test_constant_matrix_uniform(orc):
    r = np.random.default_rng(44)
    n = 9
    A = np.full((n, n), 0.05, np.float32)
    b0 = r.random(n) + 0.01
    res = orc.mapi(A, b0 / np.linalg.norm(b0), 1)
    np.testing.assert_allclose(res.w, np.full(n, 1.0 / n), rtol=1e-14)


def test_proposition1_positive_start(orc):
    # diamond-MAPI on positive A reaches [1+||a_i||_1]/sum(1+||a_j||_1) in 2 steps
    r = np.random.default_rng(45)
    for _ in range(20):
        n = int(r.integers(2, 30))
        A = (r.random((n, n)) + 0.01).astype(np.float32)
        b0 = r.random(n) + 0.01
        res = orc.power_iterate(A, b0 / np.linalg.norm(b0), 2, op="diamond", norm=orc.NORM_L1)
        rows = np.abs(A.astype(np.float64)).sum(axis=1)
        expect = (1 + rows) / np.sum(1 + rows)
        np.testing.assert_allclose(res.w, expect, rtol=0, atol=1e-12)


def test_rpi_limit_vs_eigh(orc):
    # Eq.(1): RPI converges to the dominant eigenvector (LAPACK eigh) given an eigen-gap
    r = np.random.default_rng(46)
    n = 30
    Q, _ = np.linalg.qr(r.standard_normal((n, n)))
    lam = np.concatenate([[3.0], np.linspace(1.5, 0.1, n - 1)])
    A = ((Q * lam) @ Q.T).astype(np.float32)
    res = orc.rpi(A, np.ones(n) / np.sqrt(n), 200)
    evals, evecs = np.linalg.eigh(A.astype(np.float64))
    u = evecs[:, -1]
    np.testing.assert_allclose(res.w * np.sign(res.w @ u), u, atol=1e-9)


# ---------------------------------------------------------------- control flow


def test_degenerate_and_tol(orc):
    A = np.zeros((4, 4), np.float32)
    res = orc.mapi(A, np.ones(4) / 2, 5)
    assert res.status == orc.ERR_DEGENERATE and res.iters_done == 0
    np.testing.assert_array_equal(res.w, np.ones(4) / 2)
    A = np.eye(4, dtype=np.float32)
    res = orc.mapi(A, np.array([0.5, 0.5, 0.5, 0.5]), 50, tol=1e-12)
    assert res.status == orc.OK and res.iters_done == 2  # delta_1 == 0 < tol
    res = orc.mapi(A, np.array([0.5, 0.5, 0.5, 0.5]), 50, tol=0.0)
    assert res.iters_done == 50  # tol = 0 never stops


def test_thread_count_independent(orc):
    C = synth.cfg1()["A"]
    b0 = synth.cfg1()["b0"]
    nt = orc.num_threads()
    orc.set_num_threads(1)
    a = orc.mapi(C, b0, 10)
    orc.set_num_threads(max(2, nt))
    b = orc.mapi(C, b0, 10)
    orc.set_num_threads(nt)
    np.testing.assert_array_equal(a.w, b.w)
    np.testing.assert_array_equal(a.norms, b.norms)


# ---------------------------------------------------------------- deflation


def test_deflation_identity_vs_numpy(orc):
    r = np.random.default_rng(51)
    for n, i in ((8, 1), (8, 3), (33, 4)):
        C = r.standard_normal((n, n)).astype(np.float32)  # not symmetric on purpose
        P = r.standard_normal((i, n))
        P /= np.linalg.norm(P, axis=1, keepdims=True)
        D = orc.deflate(C, P, i)
        expect = (np.eye(n) - P.T @ P) @ C.astype(np.float64)  # (I - sum p p^T) C, literal
        np.testing.assert_allclose(D, expect, rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(orc.deflate(C, P, 0), C.astype(np.float64))


def test_pca_topk_composition(orc):
    r = np.random.default_rng(52)
    n = 20
    X = r.standard_normal((n, 60))
    C = (X @ X.T / 60).astype(np.float32)
    b0 = np.ones(n) / np.sqrt(n)
    res = orc.pca_topk(C, 3, 30, b0)
    assert res.status == orc.OK
    P = np.zeros((3, n))
    for i in range(3):
        D = (np.eye(n) - P[:i].T @ P[:i]) @ C.astype(np.float64)
        w, norms = brute.mapi(D, b0, 30)
        w = np.asarray(w)
        P[i] = w / np.linalg.norm(w)
        np.testing.assert_allclose(res.norms[i], norms, rtol=1e-10)
    np.testing.assert_allclose(res.P, P, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(res.P, axis=1), 1.0, rtol=1e-14)


# ---------------------------------------------------------------- ranking (Eq. 13)


def test_google_matrix_column_stochastic():
    edges, _, _ = synth.random_graph(40, 0.1, seed=60, n_dangling=5)
    G = brute.google_matrix(40, edges)
    np.testing.assert_allclose(G.sum(axis=0), 1.0, rtol=1e-14)
    assert np.all(G > 0)


def test_rank_csr_vs_dense_bruteforce(orc):
    # S:550 / F7: the sparse + background form equals the dense G (+) w on <= 200-node graphs
    r = np.random.default_rng(61)
    for trial in range(50):
        n = int(r.integers(2, 201))
        edges, row_ptr, col_idx = synth.random_graph(n, float(r.uniform(0.01, 0.1)),
                                                     seed=1000 + trial,
                                                     n_dangling=int(r.integers(0, max(1, n // 5))))
        w_d, deltas_d = brute.rank_dense(n, edges, iters=6)
        res = orc.rank_csr(n, row_ptr, col_idx, b0=np.full(n, 1.0 / n), max_iters=6, tol=0.0)
        assert res.status == orc.OK and res.iters_done == 6
        np.testing.assert_allclose(res.w, w_d, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(res.deltas, deltas_d, rtol=1e-8, atol=1e-15)
        assert np.all(res.w > 0)  # S:465 positivity


def test_rank_one_step_vs_dense_arbitrary_w(orc):
    # one step from a non-uniform positive w: exercises both branches of each min(G_ij, w_j)
    r = np.random.default_rng(62)
    n = 120
    edges, row_ptr, col_idx = synth.random_graph(n, 0.05, seed=7, n_dangling=10)
    w = r.random(n) * 0.05
    y = brute.google_mavp(n, edges, w)
    res = orc.rank_csr(n, row_ptr, col_idx, b0=w, max_iters=1, tol=0.0)
    np.testing.assert_allclose(res.w, y / y.sum(), rtol=1e-13)


def test_rank_dot_vs_dense_google_product(orc):
    # RPI arm (reading R13): one step of the oracle's sparse + background dot form equals the dense G w of the
    # materialised Google matrix, normalised by its l1 norm, from an arbitrary positive w (no sign or min)
    r = np.random.default_rng(63)
    for trial in range(20):
        n = int(r.integers(2, 150))
        edges, row_ptr, col_idx = synth.random_graph(n, float(r.uniform(0.01, 0.1)), seed=2000 + trial,
                                                     n_dangling=int(r.integers(0, max(1, n // 5))))
        w = r.random(n) + 0.01
        y = brute.google_dot(n, edges, w)
        res = orc.rank_csr(n, row_ptr, col_idx, b0=w, max_iters=1, tol=0.0, op="dot")
        assert res.status == orc.OK
        np.testing.assert_allclose(res.w, y / y.sum(), rtol=1e-13)
        # column-stochastic G preserves the l1 norm of a non-negative vector
        assert abs(y.sum() - w.sum()) <= 1e-12 * w.sum()


def test_rank_dot_converges_to_pagerank_eigenvector(orc):
    # the RPI ranking's fixed point is THE PageRank vector: the eigenvalue-1 eigenvector of the dense G
    # from LAPACK (geev), independent of the iteration
    for seed, n in ((70, 60), (71, 150)):
        edges, row_ptr, col_idx = synth.random_graph(n, 0.05, seed=seed, n_dangling=n // 10)
        pr = brute.pagerank_eig(n, edges)
        res = orc.rank_csr(n, row_ptr, col_idx, max_iters=400, tol=0.0, op="dot")
        np.testing.assert_allclose(res.w, pr, rtol=1e-9, atol=1e-14)
        np.testing.assert_allclose(res.w_l2, pr / np.linalg.norm(pr), rtol=1e-9)


def test_rank_min2_equals_min1(orc):
    # all G_ij > 0 and w >= 0: Eq. (4)'s sign indicator is always 1, so min2 == min1 exactly
    edges, row_ptr, col_idx = synth.random_graph(90, 0.06, seed=72, n_dangling=9)
    a = orc.rank_csr(90, row_ptr, col_idx, max_iters=15, tol=0.0)
    b = orc.rank_csr(90, row_ptr, col_idx, max_iters=15, tol=0.0, op="min2")
    assert np.array_equal(a.w, b.w)


def test_rank_star_graph_hub_first(orc):
    n = 30
    src = np.arange(1, n)
    dst = np.zeros(n - 1, np.int64)
    row_ptr, col_idx = synth.csr_by_destination(n, src, dst)
    res = orc.rank_csr(n, row_ptr, col_idx, max_iters=20, tol=0.0)
    assert orc.rank_order(res.w)[0] == 0


def test_rank_negative_start_rejected(orc):
    row_ptr, col_idx = synth.csr_by_destination(3, [0, 1], [1, 2])
    res = orc.rank_csr(3, row_ptr, col_idx, b0=np.array([0.5, -0.1, 0.6]))
    assert res.status == orc.ERR_NEGATIVE


# ---------------------------------------------------------------- paper-printed rank utilities


def test_paper_printed_rank_orders(orc):
    g = _gold("paper_printed.json")
    sp = g["stochastic_pca_final_vectors"]
    for key in ("rpi", "min1"):
        assert list(orc.rank_order(sp[key]) + 1) == sp["ranks_1based"], sp["cite"]
        assert np.linalg.norm(sp[key]) == pytest.approx(1.0, abs=1e-3)
    pr = g["pagerank_4node"]
    for key in ("rpi", "mapi"):
        assert list(orc.rank_order(pr[key]) + 1) == pr["ranks_1based"], pr["cite"]
    gn = g["gnutella_top10"]
    assert orc.topk_overlap(gn["g08_rpi"], gn["g08_mapi"], 10) == gn["g08_common"]
    assert orc.topk_overlap(gn["g09_rpi"], gn["g09_mapi"], 10) == gn["g09_common"]


def test_rank_order_ties_by_index(orc):
    assert list(orc.rank_order([0.5, 0.7, 0.5, 0.7])) == [1, 3, 0, 2]


# ---------------------------------------------------------------- matrix extension / min-covariance (NEXT-1)


@pytest.mark.parametrize("op", ["min1", "min2", "dot"])
def test_matmat_vs_brute(orc, op):
    r = np.random.default_rng(71)
    for trial in range(25):
        m, p, K = (int(x) for x in r.integers(1, 8, size=3))
        A = r.standard_normal((m, K)).astype(np.float32)
        B = r.standard_normal((p, K)).astype(np.float32)
        A[r.random(A.shape) < 0.1] = 0.0
        C = orc.matmat(A, B, op, d=3.0)
        f = brute.OPS[op]
        for i in range(m):
            for j in range(p):
                assert C[i, j] == pytest.approx(f(A[i], B[j]) / 3.0, rel=1e-14, abs=1e-300)


def test_matmat_spec_examples(orc):
    # W = X = [[1],[-2]] (one column; vectors as rows here: one vector [1,-2]) -> [[3]]
    v = np.array([[1.0, -2.0]], np.float32)
    assert orc.matmat(v, v).tolist() == [[3.0]]
    # empty p -> m x 0
    assert orc.matmat(v, np.zeros((0, 2), np.float32)).shape == (1, 0)


def test_min_covariance_properties(orc):
    r = np.random.default_rng(72)
    V = r.standard_normal((40, 10))
    V -= V.mean(axis=1, keepdims=True)
    V = V.astype(np.float32)
    C = orc.min_covariance(V)
    np.testing.assert_array_equal(C, C.T)  # min1 is symmetric (exact)
    np.testing.assert_allclose(np.diag(C), np.abs(V.astype(np.float64)).sum(axis=1) / 9, rtol=1e-14)
    assert np.all(np.abs(C) <= np.diag(C)[:, None] + 1e-15)  # |a (+) b| <= min(||a||_1, ||b||_1)
    C5 = orc.min_covariance(V, divisor=10)  # Eq. (5) divisor N
    np.testing.assert_allclose(C5 * 10, C * 9, rtol=1e-14)


def test_pca_topk_dot_recovers_lapack_eigenvectors(orc):
    # with the regular product (Eq. 1) and L2 deflation, power iteration + deflation returns the
    # leading eigenvectors of a symmetric matrix with a spectral gap (LAPACK eigh)
    r = np.random.default_rng(53)
    n = 24
    Q, _ = np.linalg.qr(r.standard_normal((n, n)))
    lam = np.array([10.0, 6.0, 3.5] + list(np.linspace(1.0, 0.1, n - 3)))
    C = ((Q * lam) @ Q.T).astype(np.float32)
    res = orc.pca_topk(C, 3, 300, np.ones(n) / np.sqrt(n), op="dot")
    evals, evecs = np.linalg.eigh(C.astype(np.float64))
    for i in range(3):
        u = evecs[:, -1 - i]
        np.testing.assert_allclose(res.P[i] * np.sign(res.P[i] @ u), u, atol=1e-6)


# ---------------------------------------------------------------- Alg. 2 MAVP deflation / reconstruction (NEXT-2)


def test_mavp_deflate_spec_e1(orc):
    # w1 = e1 -> P(1,1) = 1, zeros elsewhere -> the deflation zeroes row 1 of C
    r = np.random.default_rng(81)
    C = r.standard_normal((6, 6)).astype(np.float32)
    w = np.zeros(6, np.float32)
    w[0] = 1.0
    D = orc.mavp_deflate(C, w)
    np.testing.assert_array_equal(D[0], 0.0)
    np.testing.assert_array_equal(D[1:], C[1:].astype(np.float64))


def test_mavp_deflate_dot_is_l2_deflation(orc):
    # with the regular product P = w w^T, matching (I - w w^T) C — vs the numpy product
    r = np.random.default_rng(82)
    C = r.standard_normal((9, 9)).astype(np.float32)
    w = r.standard_normal(9)
    w = (w / np.linalg.norm(w)).astype(np.float32)
    D = orc.mavp_deflate(C, w, op="dot")
    w64 = w.astype(np.float64)
    np.testing.assert_allclose(D, (np.eye(9) - np.outer(w64, w64)) @ C.astype(np.float64), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("op", ["min1", "min2"])
def test_outer_apply_vs_brute(orc, op):
    r = np.random.default_rng(83)
    for trial in range(10):
        M, rr, q = int(r.integers(1, 8)), int(r.integers(1, 3)), int(r.integers(1, 4))
        W = r.standard_normal((M, rr)).astype(np.float32)
        X = r.standard_normal((M, q)).astype(np.float32)
        f = brute.OPS[op]
        Q = np.array([[f(W[i], W[j]) for j in range(M)] for i in range(M)])
        np.testing.assert_allclose(orc.outer_apply(W, X, op), Q @ X.astype(np.float64), rtol=1e-12, atol=1e-13)


def test_reconstruct_identical_copies_returns_image(orc):
    # N identical copies -> zero-centred V = 0 -> v_hat = m = the image
    img = np.random.default_rng(84).random(64)
    V = np.repeat(img[:, None], 5, axis=1).astype(np.float32)
    W = np.random.default_rng(85).standard_normal((64, 2)).astype(np.float32)
    Vh, m = orc.reconstruct(W, V)
    np.testing.assert_allclose(Vh, np.repeat(img[:, None], 5, axis=1), atol=1e-7)


def test_psnr_closed_forms(orc):
    a = np.zeros(100)
    assert orc.psnr(a, np.full(100, 0.1)) == pytest.approx(20.0)  # MSE 0.01 -> 20 dB
    assert orc.psnr(a, np.ones(100)) == pytest.approx(0.0)  # MSE 1 -> 0 dB


def test_outer_apply_rows_matches_full(orc):
    r = np.random.default_rng(86)
    W = r.standard_normal((40, 2)).astype(np.float32)
    X = r.standard_normal((40, 5)).astype(np.float32)
    full = orc.outer_apply(W, X, "min1", subtract=True)
    rows = np.array([0, 7, 39, 7])
    np.testing.assert_array_equal(orc.outer_apply_rows(W, X, rows, "min1", subtract=True), full[rows])


# ------------------------------------------------------------------ Algorithm 3 (mini-batch MAPI with momentum)


@pytest.mark.parametrize("gram", ["min1", "dot"])
@pytest.mark.parametrize("beta", [0.0, 0.225, 0.9])
def test_minibatch_mapi_matches_brute(orc, gram, beta):
    """Alg. 3 against the literal pure-Python statement (brute.minibatch_mapi): random tiny
    datasets, i.i.d. batches with replacement (step 3), momentum (step 4), both iterates rescaled by
    ||w_{t+1}||_1 (step 5 verbatim), the traced norms and the final l2 copy (line 7)."""
    for seed in range(6):
        r = np.random.default_rng(300 + seed)
        N, D, T, s = int(r.integers(1, 9)), int(r.integers(1, 5)), int(r.integers(1, 6)), int(r.integers(1, 5))
        X = r.standard_normal((N, D))
        idx = r.integers(0, N, (T, s))
        w0 = r.standard_normal(D)
        w0 /= np.linalg.norm(w0)
        got = orc.minibatch_mapi(X, idx, beta, w0, gram=gram)
        if got.status != 0:  # a degenerate draw (tiny D): the brute force divides by zero there
            continue
        w, norms = brute.minibatch_mapi(X, idx, beta, w0, gram=gram)
        np.testing.assert_allclose(got.w, w, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(got.norms, norms, rtol=1e-12)
        np.testing.assert_allclose(got.w_l2, w / np.linalg.norm(w), rtol=1e-12, atol=1e-15)


def test_minibatch_mapi_full_batch_no_momentum_is_algorithm_1(orc):
    """beta = 0 and every batch = all N samples: Alg. 3 reduces to Alg. 1 on A = (1/N) X^T (.) X,
    iterate for iterate (the fp64 oracle power iteration on that matrix, the matrix formed by the brute
    force's Eq. (3) on the columns of X)."""
    r = np.random.default_rng(77)
    N, D, T = 40, 6, 12
    X = r.standard_normal((N, D))
    idx = np.tile(np.arange(N), (T, 1))
    w0 = r.standard_normal(D)
    w0 /= np.linalg.norm(w0)
    got = orc.minibatch_mapi(X, idx, 0.0, w0)
    M = np.array([[brute.min1(X[:, j], X[:, k]) / N for k in range(D)] for j in range(D)])
    ref = orc.power_iterate(M, w0, T, op="min1")
    assert got.iters_done == ref.iters_done == T
    np.testing.assert_allclose(got.w, ref.w, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(got.norms, ref.norms, rtol=1e-12)


def test_minibatch_mapi_continuation(orc):
    """The optional (w_prev0, w_prev) state changes no step: T1 steps, then T2 more from the returned
    (w, w_prev), reproduce T1 + T2 steps exactly; and w_prev after one step from w_{-1} = 0 is w_0 / s_0
    (Alg. 3 step 5, verbatim: both vectors divided by ||w_{t+1}||_1, R15)."""
    r = np.random.default_rng(11)
    X = r.standard_normal((40, 5))
    idx = r.integers(0, 40, (9, 6))
    w0 = r.standard_normal(5)
    full = orc.minibatch_mapi(X, idx, 0.3, w0)
    a = orc.minibatch_mapi(X, idx[:4], 0.3, w0)
    b = orc.minibatch_mapi(X, idx[4:], 0.3, a.w, w_prev0=a.w_prev)
    assert np.array_equal(b.w, full.w) and np.array_equal(b.w_prev, full.w_prev)
    assert np.array_equal(np.concatenate([a.norms, b.norms]), full.norms)
    one = orc.minibatch_mapi(X, idx[:1], 0.3, w0)
    np.testing.assert_allclose(one.w_prev, w0 / one.norms[0], rtol=1e-15)


def test_minibatch_mapi_degenerate_and_bad_input(orc):
    X = np.zeros((5, 3))
    res = orc.minibatch_mapi(X, np.zeros((2, 2), np.int64), 0.1, np.ones(3) / np.sqrt(3))
    assert res.status == orc.ERR_DEGENERATE and res.iters_done == 0
    with pytest.raises(ValueError):
        orc.minibatch_mapi(np.ones((5, 3)), np.full((2, 2), 5), 0.1, np.ones(3))  # index out of range
