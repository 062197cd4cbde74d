/*
 * oracle.c — fp64 CPU ORACLE for the MAPI / MAVP hot path (arXiv 2110.12065).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  It shares no code,
 * header, table or helper with the CUDA library under paper_2110_12065_b200/csrc/, and
 * the CUDA library never calls it.
 *
 * Design rules:
 *   - plain loops, fp64 arithmetic on the SAME fp32 input bytes (promoted exactly);
 *   - every row y_j is summed sequentially in index order k = 0..n-1, so the result
 *     does not depend on the OpenMP thread count (threads only split ROWS);
 *   - compiled -O2 -fno-fast-math -ffp-contract=off (no FMA contraction, no reassociation);
 *   - no blocking, fusion or reordering beyond what the paper's definition states.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n (spec of a
 * different CPU program; used only for conventions), Qn = reading n in DESIGN.md §Readings.
 *
 * Parity pins (tests/test_oracle_pins.py, `-m "not gpu"`): SPEC worked examples, the
 * north-star MAVP invariants, literal brute force (oracle/brute.py) on n<=8, closed forms
 * (A=I, |a|>=1 sign regime vs LAPACK eigh, sign-rank-1, constant A), Proposition 1,
 * the RPI limit, the deflation identity vs a numpy matrix product, and the CSR ranking
 * form vs the dense Google matrix on 50 random graphs.  Every function below is pinned;
 * none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Operators.  ORC_MIN1 = Eq.(3), ORC_MIN2 = Eq.(4),
 * ORC_DIAMOND = Eq.(9) (reading y == w, Q-diamond / S:134),
 * ORC_DOT = the Euclidean product of Eq.(1). */
enum { ORC_MIN1 = 0, ORC_MIN2 = 1, ORC_DIAMOND = 2, ORC_DOT = 3 };
/* Normalisation after each step: 1 = l1 (Eq. 8), 2 = l2 (Eq. 1). */
enum { ORC_NORM_L1 = 1, ORC_NORM_L2 = 2 };
/* Status codes (same numeric meaning as the product ABI, defined independently here). */
enum { ORC_OK = 0, ORC_ERR_BAD_PARAM = 3, ORC_ERR_DEGENERATE = 4, ORC_ERR_NEGATIVE = 5,
       ORC_ERR_NONFINITE = 6 };

/* sign(.) with sign(0) = 0 (the paper never defines sign(0); S:119 and reading Q1). */
static double orc_sign(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

/* One summand of w^T (op) x for a single pair (w_i, x_i). */
static double orc_term(int op, double w, double x) {
    switch (op) {
    case ORC_MIN1: /* Eq.(3): sign(w_i x_i) min(|w_i|,|x_i|); sign(w x) = sign(w) sign(x). */
        return orc_sign(w) * orc_sign(x) * fmin(fabs(w), fabs(x));
    case ORC_MIN2: /* Eq.(4): 1(sign w_i = sign x_i) min(|w_i|,|x_i|). */
        return (orc_sign(w) == orc_sign(x)) ? fmin(fabs(w), fabs(x)) : 0.0;
    case ORC_DIAMOND: /* Eq.(9): sign(x_i) y_i + x_i sign(y_i), with y == w. */
        return orc_sign(x) * w + x * orc_sign(w);
    default: /* ORC_DOT: Euclidean product, Eq.(1). */
        return w * x;
    }
}

/* w^T (op) x = sum_i term(w_i, x_i), summed in index order (Eq. 3 / 4 / 9). */
double orc_mavp_dot(int op, const double *w, const double *x, int64_t n) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += orc_term(op, w[i], x[i]);
    return acc;
}

/* Matrix extension (reading Q6/Q7): y_j = a_j^T (op) x where a_j is ROW j of A.
 * A is fp32 row-major with leading dimension lda (fp32 bytes promoted exactly to fp64).
 * mag_j = sum_k |term_jk| (the per-element tolerance scale of T1), may be NULL. */
void orc_matvec_f32(int op, const float *A, int64_t n_rows, int64_t n_cols, int64_t lda,
                    const double *x, double *y, double *mag) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n_rows; ++j) {
        const float *a = A + j * lda;
        double acc = 0.0, m = 0.0;
        for (int64_t k = 0; k < n_cols; ++k) {
            double t = orc_term(op, (double)a[k], x[k]);
            acc += t;
            m += fabs(t);
        }
        y[j] = acc;
        if (mag) mag[j] = m;
    }
}

/* Same, for an fp64 matrix (used for the deflated matrices D_i, which the oracle keeps in fp64). */
void orc_matvec_f64(int op, const double *A, int64_t n_rows, int64_t n_cols, int64_t lda,
                    const double *x, double *y, double *mag) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n_rows; ++j) {
        const double *a = A + j * lda;
        double acc = 0.0, m = 0.0;
        for (int64_t k = 0; k < n_cols; ++k) {
            double t = orc_term(op, a[k], x[k]);
            acc += t;
            m += fabs(t);
        }
        y[j] = acc;
        if (mag) mag[j] = m;
    }
}

static double orc_norm(int norm, const double *v, int64_t n) {
    double s = 0.0;
    if (norm == ORC_NORM_L1) {
        for (int64_t i = 0; i < n; ++i) s += fabs(v[i]);
        return s;
    }
    for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* Power iteration, Algorithm 1 for op in {MIN1, MIN2, DIAMOND} with norm = L1,
 * or regular power iteration Eq.(1) for op = DOT with norm = L2.
 *
 *   w = b0 (used as given; BJ configs pass l2-unit b0, reading Q2)
 *   for t = 0..T-1:
 *       y = A (op) w                         Alg.1 line 3
 *       s = ||y||                            Alg.1 line 4 / Eq.(8)
 *       if s == 0: DEGENERATE at t           (reading Q9 family)
 *       w' = y / s ; delta = ||w' - w||_1    ("||w_t - w_{t-1}||", reading Q9)
 *       norms[t] = s ; deltas[t] = delta ; w = w'
 *       if tol > 0 and delta < tol: stop     (reading Q9: strict <, tol = 0 never stops)
 *   w_l2 = w / ||w||_2                       Alg.1 line 6, optional
 *
 * A is fp32 (a_is_f64 = 0) or fp64 (a_is_f64 = 1), row-major, leading dimension lda.
 * w_out, w_l2_out, norms, deltas may be NULL.  *iters_done = number of completed steps.
 * On DEGENERATE, w_out holds the last good iterate w_t. */
int orc_power_iterate(int op, int norm, const void *A, int a_is_f64, int64_t n, int64_t lda,
                      const double *b0, int32_t T, double tol, double *w_out, double *w_l2_out,
                      double *norms, double *deltas, int32_t *iters_done) {
    if (n < 1 || lda < n || T < 1 || !(tol >= 0.0) || !A || !b0) return ORC_ERR_BAD_PARAM;
    double *w = (double *)malloc(sizeof(double) * (size_t)n);
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    int status = ORC_OK;
    int32_t done = 0;
    memcpy(w, b0, sizeof(double) * (size_t)n);
    for (int32_t t = 0; t < T; ++t) {
        if (a_is_f64)
            orc_matvec_f64(op, (const double *)A, n, n, lda, w, y, NULL);
        else
            orc_matvec_f32(op, (const float *)A, n, n, lda, w, y, NULL);
        double s = orc_norm(norm, y, n);
        if (!isfinite(s)) { status = ORC_ERR_NONFINITE; break; }
        if (s == 0.0) { status = ORC_ERR_DEGENERATE; break; }
        double delta = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double wn = y[j] / s;
            delta += fabs(wn - w[j]);
            w[j] = wn;
        }
        if (norms) norms[t] = s;
        if (deltas) deltas[t] = delta;
        done = t + 1;
        if (tol > 0.0 && delta < tol) break;
    }
    if (w_out) memcpy(w_out, w, sizeof(double) * (size_t)n);
    if (w_l2_out) {
        double l2 = orc_norm(ORC_NORM_L2, w, n);
        for (int64_t j = 0; j < n; ++j) w_l2_out[j] = l2 > 0.0 ? w[j] / l2 : 0.0;
    }
    if (iters_done) *iters_done = done;
    free(w);
    free(y);
    return status;
}

/* MAVP matrix product, the matrix extension (reading Q7: entry (i,j) = w_i^T (op) x_j) with the
 * vectors stored as ROWS:  C[i][j] = ( a_i (op) b_j ) / d,  a_i = row i of A (m x K, lda),
 * b_j = row j of B (p x K, ldb).  With A = B = V (pixels x samples) and d = N-1 this is the
 * min-covariance of Alg. 2 step 4; d = N gives Eq. (5).  fp64, k in index order. */
void orc_matmat_f32(int op, const float *A, int64_t m, int64_t K, int64_t lda, const float *B, int64_t p,
                    int64_t ldb, double d, double *C) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t j = 0; j < p; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k) acc += orc_term(op, (double)A[i * lda + k], (double)B[j * ldb + k]);
            C[i * p + j] = acc / d;
        }
    }
}

/* MAVP outer-product operator of Alg. 2: for W (M x r, ldw; columns w_1..w_r) the M x M
 * matrix Q = W (op) W^T has Q[i][j] = sum_c term(W[i][c], W[j][c])  (row i of W against row j, i.e. the
 * matrix extension P:69-70 with the r-component rows as vectors; r = 1 gives the scalar-MAVP outer
 * product of step 6, r = 2 the W = [w1 w2] of step 8).  Y = X - Q X  (subtract = 1, step 6) or
 * Y = Q X (subtract = 0, step 8), with Q X a REGULAR matrix product.  X: M x q (ldx),
 * Y: M x q (ldy).  Literal: Q is materialised row by row, the product summed over j in index order. */
void orc_outer_apply(int op, const float *W, int64_t M, int64_t r, int64_t ldw, const float *X, int64_t q,
                     int64_t ldx, int subtract, double *Y, int64_t ldy) {
#pragma omp parallel
    {
        double *Qi = (double *)malloc(sizeof(double) * (size_t)M);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < M; ++i) {
            for (int64_t j = 0; j < M; ++j) {
                double t = 0.0;
                for (int64_t c = 0; c < r; ++c) t += orc_term(op, (double)W[i * ldw + c], (double)W[j * ldw + c]);
                Qi[j] = t;
            }
            for (int64_t k = 0; k < q; ++k) {
                double acc = 0.0;
                for (int64_t j = 0; j < M; ++j) acc += Qi[j] * (double)X[j * ldx + k];
                Y[i * ldy + k] = subtract ? (double)X[i * ldx + k] - acc : acc;
            }
        }
        free(Qi);
    }
}

/* orc_outer_apply restricted to the rows listed in `rows` (nrows of them): Y is nrows x q (ldy).
 * Same arithmetic, used to check full-size GPU results on sampled rows. */
void orc_outer_apply_rows(int op, const float *W, int64_t M, int64_t r, int64_t ldw, const float *X, int64_t q,
                          int64_t ldx, int subtract, const int64_t *rows, int64_t nrows, double *Y, int64_t ldy) {
#pragma omp parallel
    {
        double *Qi = (double *)malloc(sizeof(double) * (size_t)M);
#pragma omp for schedule(static)
        for (int64_t ri = 0; ri < nrows; ++ri) {
            const int64_t i = rows[ri];
            for (int64_t j = 0; j < M; ++j) {
                double t = 0.0;
                for (int64_t c = 0; c < r; ++c) t += orc_term(op, (double)W[i * ldw + c], (double)W[j * ldw + c]);
                Qi[j] = t;
            }
            for (int64_t k = 0; k < q; ++k) {
                double acc = 0.0;
                for (int64_t j = 0; j < M; ++j) acc += Qi[j] * (double)X[j * ldx + k];
                Y[ri * ldy + k] = subtract ? (double)X[i * ldx + k] - acc : acc;
            }
        }
        free(Qi);
    }
}

/* L2 deflation: the i-th principal vector is extracted by power iteration on
 *     D_i = (I - sum_{m<i} p_m p_m^T) C,
 * with p_m the l2-normalised MAPI outputs.  Expanded entry-wise:
 *     D_i[r][c] = C[r][c] - sum_{m<i} p_m[r] * (p_m^T C)[c]
 * (only associativity of the matrix product; no symmetry of C is assumed).
 * C is fp32 n x n (ldc), D is an fp64 n x n output (leading dimension n). P is k x n fp64,
 * the first `i` rows are used. */
void orc_deflate(const float *C, int64_t n, int64_t ldc, const double *P, int32_t i, double *D) {
    double *r = (double *)calloc((size_t)n * (size_t)(i > 0 ? i : 1), sizeof(double));
    /* r_m = p_m^T C  (row vector), for m < i. */
    for (int32_t m = 0; m < i; ++m) {
        const double *p = P + (int64_t)m * n;
        double *rm = r + (int64_t)m * n;
#pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) {
            double acc = 0.0;
            for (int64_t l = 0; l < n; ++l) acc += p[l] * (double)C[l * ldc + c];
            rm[c] = acc;
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < n; ++row) {
        for (int64_t c = 0; c < n; ++c) {
            double v = (double)C[row * ldc + c];
            for (int32_t m = 0; m < i; ++m) v -= P[(int64_t)m * n + row] * r[(int64_t)m * n + c];
            D[row * n + c] = v;
        }
    }
    free(r);
}

/* Top-k principal vectors by MAPI with L2 deflation (BJ configs[1]).
 * For i = 0..k-1: D_i = (I - sum_{m<i} p_m p_m^T) C ; w = MAPI(D_i, b0, T, tol=0) ;
 * p_i = w / ||w||_2.  Outputs P (k x n), norms/deltas (k x T), iters_done (k). */
int orc_pca_topk(int op, const float *C, int64_t n, int64_t ldc, int32_t k, int32_t T,
                 const double *b0, double *P, double *norms, double *deltas, int32_t *iters_done) {
    if (n < 1 || ldc < n || k < 1 || k > n || T < 1 || !C || !b0 || !P) return ORC_ERR_BAD_PARAM;
    double *D = (double *)malloc(sizeof(double) * (size_t)n * (size_t)n);
    int status = ORC_OK;
    for (int32_t i = 0; i < k; ++i) {
        orc_deflate(C, n, ldc, P, i, D);
        int32_t done = 0;
        /* MAVP operators use the l1 normalisation of Eq. (8); the regular product (RPI comparator)
         * the l2 normalisation of Eq. (1) */
        status = orc_power_iterate(op, op == ORC_DOT ? ORC_NORM_L2 : ORC_NORM_L1, D, 1, n, n, b0, T, 0.0, NULL,
                                   P + (int64_t)i * n, norms ? norms + (int64_t)i * T : NULL,
                                   deltas ? deltas + (int64_t)i * T : NULL, &done);
        if (iters_done) iters_done[i] = done;
        if (status != ORC_OK) break;
    }
    free(D);
    return status;
}

/* MAPI ranking on the Google matrix, Eq.(13), reading Q10:
 *   G = alpha M + (1-alpha)/n 1,  M_ij = 1/outdeg(j) for each (deduplicated) edge j -> i,
 *   dangling columns (outdeg 0) of M are uniform 1/n, so G_ij = 1/n there.
 * The graph is given by destination: row i of (row_ptr, col_idx) lists the sources j of
 * the edges j -> i.  w >= 0 throughout (positive start, positive G), so every min1 term is
 * min(G_ij, w_j).  The oracle evaluates  y_i = sum_j min(G_ij, w_j)  exactly rewritten as
 *     y_i = S + sum_{j in in(i)} [ min(c_j + alpha/outdeg(j), w_j) - min(c_j, w_j) ],
 *     S   = sum_j min(c_j, w_j),  c_j = (1-alpha)/n  (1/n if j dangling),
 * i.e. the background term plus the per-edge difference of mins (a literal re-grouping of
 * the sum, not the GPU's clamp form).  Pinned to the dense brute force (oracle/brute.py)
 * on random graphs.  Then Algorithm 1 steps: l1 normalise, delta = ||w'-w||_1,
 * stop when tol > 0 and delta < tol, final l2 copy.
 * op = ORC_DOT is the regular PageRank power iteration y = G w (Eq. 1 on the G of P:307; the paper's
 * RPI arm of Sec. 3.3), written the same way:  y_i = S + sum_{j in in(i)} (alpha/outdeg(j)) w_j,
 * S = sum_j c_j w_j  (distributivity over G_ij = c_j + [j->i] alpha/outdeg(j)); reading R13: the iterate is
 * l1-normalised every iteration (G is column-stochastic, so ||Gw||_1 = ||w||_1 for w >= 0 and the step is
 * the textbook PageRank update), with the final l2 copy of P:322.  Pinned to the dense G w brute force and
 * to the PageRank vector from a dense eigen-solve.  ORC_MIN2 equals ORC_MIN1 here (all terms >= 0). */
int orc_rank_csr_op(int op, int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                    double alpha, const double *b0, int32_t max_iters, double tol, double *w_out,
                    double *w_l2_out, double *deltas, int32_t *iters_done) {
    if (op != ORC_MIN1 && op != ORC_MIN2 && op != ORC_DOT) return ORC_ERR_BAD_PARAM;
    if (n < 1 || nnz < 0 || !row_ptr || (nnz > 0 && !col_idx) || !b0 || max_iters < 1 ||
        !(alpha > 0.0 && alpha < 1.0) || !(tol >= 0.0))
        return ORC_ERR_BAD_PARAM;
    for (int64_t j = 0; j < n; ++j)
        if (b0[j] < 0.0) return ORC_ERR_NEGATIVE;
    int64_t *outdeg = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    double *c = (double *)malloc(sizeof(double) * (size_t)n);
    double *w = (double *)malloc(sizeof(double) * (size_t)n);
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t e = 0; e < nnz; ++e) outdeg[col_idx[e]] += 1;
    for (int64_t j = 0; j < n; ++j) c[j] = outdeg[j] == 0 ? 1.0 / (double)n : (1.0 - alpha) / (double)n;
    memcpy(w, b0, sizeof(double) * (size_t)n);
    int status = ORC_OK;
    int32_t done = 0;
    for (int32_t t = 0; t < max_iters; ++t) {
        double S = 0.0;
        if (op == ORC_DOT)
            for (int64_t j = 0; j < n; ++j) S += c[j] * w[j];
        else
            for (int64_t j = 0; j < n; ++j) S += fmin(c[j], w[j]);
#pragma omp parallel for schedule(dynamic, 1024)
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
                int32_t j = col_idx[e];
                if (op == ORC_DOT) {
                    acc += (alpha / (double)outdeg[j]) * w[j];
                } else {
                    double g = c[j] + alpha / (double)outdeg[j];
                    acc += fmin(g, w[j]) - fmin(c[j], w[j]);
                }
            }
            y[i] = S + acc;
        }
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s += fabs(y[i]);
        if (!isfinite(s)) { status = ORC_ERR_NONFINITE; break; }
        if (s == 0.0) { status = ORC_ERR_DEGENERATE; break; }
        double delta = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double wn = y[i] / s;
            delta += fabs(wn - w[i]);
            w[i] = wn;
        }
        if (deltas) deltas[t] = delta;
        done = t + 1;
        if (tol > 0.0 && delta < tol) break;
    }
    if (w_out) memcpy(w_out, w, sizeof(double) * (size_t)n);
    if (w_l2_out) {
        double l2 = 0.0;
        for (int64_t i = 0; i < n; ++i) l2 += w[i] * w[i];
        l2 = sqrt(l2);
        for (int64_t i = 0; i < n; ++i) w_l2_out[i] = w[i] / l2;
    }
    if (iters_done) *iters_done = done;
    free(outdeg);
    free(c);
    free(w);
    free(y);
    return status;
}

/* Number of OpenMP threads the oracle will use (reported beside every oracle timing). */
/* Algorithm 3 (§3.2): mini-batch MAPI with momentum, in the paper's step order.
 *   X: N x D fp64 samples (rows, ldx); batch: T x s row indices (the i.i.d. draws of step 3 are INPUTS,
 *   drawn by the caller); beta: momentum; w0: D (step 1; used as given);
 *   gram_op: the product forming each sample's matrix A~_i (reading R14): ORC_MIN1 (the paper, P:266:
 *   "we apply MAPI on A = X^T (.) X", A~_i[j][k] = x_ij (.) x_ik) or ORC_DOT (x_ij x_ik).
 *   t = 0 .. T-1:
 *     step 3/4: M = (1/s) sum_{i in batch t} A~_i   (entries summed over the batch in batch order, then / s)
 *               y_j = sum_k term_min1(M[j][k], w_t[k]) - beta w_{t-1}[j]    (w_{-1} = 0; row j of M, Q6)
 *     step 5:   s_t = ||y||_1;  w_{t-1} <- w_t / s_t;  w_t <- y / s_t       (both by ||w_{t+1}||_1, verbatim)
 *   optional final l2 copy (Alg. 3 line 7).  norms[t] = s_t.  DEGENERATE if s_t == 0, NONFINITE if not finite
 *   (w_out then holds the last good iterate).
 *   wprev0 (nullable): the momentum vector to start from instead of w_{-1} = 0, and wprev_out (nullable): the
 *   momentum vector after the last step (w_{T-1} / s_{T-1}) — the state a run needs to be continued; they
 *   change nothing in the steps above. */
int orc_minibatch_mapi(const double *X, int64_t N, int64_t D, int64_t ldx, const int64_t *batch, int32_t s,
                       int32_t T, double beta, const double *w0, int gram_op, double *w_out, double *w_l2_out,
                       double *norms, int32_t *iters_done, const double *wprev0, double *wprev_out) {
    if (N < 1 || D < 1 || ldx < D || s < 1 || T < 1 || !X || !batch || !w0) return ORC_ERR_BAD_PARAM;
    for (int64_t q = 0; q < (int64_t)T * s; ++q)
        if (batch[q] < 0 || batch[q] >= N) return ORC_ERR_BAD_PARAM;
    double *M = (double *)malloc(sizeof(double) * (size_t)(D * D));
    double *w = (double *)malloc(sizeof(double) * (size_t)D);
    double *wp = (double *)calloc((size_t)D, sizeof(double));
    double *y = (double *)malloc(sizeof(double) * (size_t)D);
    memcpy(w, w0, sizeof(double) * (size_t)D);
    if (wprev0) memcpy(wp, wprev0, sizeof(double) * (size_t)D);
    int status = ORC_OK;
    int32_t done = 0;
    for (int32_t t = 0; t < T; ++t) {
        for (int64_t e = 0; e < D * D; ++e) M[e] = 0.0;
        for (int32_t i = 0; i < s; ++i) {
            const double *x = X + batch[(int64_t)t * s + i] * ldx;
            for (int64_t j = 0; j < D; ++j)
                for (int64_t k = 0; k < D; ++k) M[j * D + k] += orc_term(gram_op, x[j], x[k]);
        }
        for (int64_t e = 0; e < D * D; ++e) M[e] /= (double)s;
        for (int64_t j = 0; j < D; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < D; ++k) acc += orc_term(ORC_MIN1, M[j * D + k], w[k]);
            y[j] = acc - beta * wp[j];
        }
        double st = 0.0;
        for (int64_t j = 0; j < D; ++j) st += fabs(y[j]);
        if (!isfinite(st)) { status = ORC_ERR_NONFINITE; break; }
        if (st == 0.0) { status = ORC_ERR_DEGENERATE; break; }
        for (int64_t j = 0; j < D; ++j) {
            wp[j] = w[j] / st;
            w[j] = y[j] / st;
        }
        if (norms) norms[t] = st;
        done = t + 1;
    }
    if (w_out) memcpy(w_out, w, sizeof(double) * (size_t)D);
    if (wprev_out) memcpy(wprev_out, wp, sizeof(double) * (size_t)D);
    if (w_l2_out) {
        double l2 = orc_norm(ORC_NORM_L2, w, D);
        for (int64_t j = 0; j < D; ++j) w_l2_out[j] = l2 > 0.0 ? w[j] / l2 : 0.0;
    }
    if (iters_done) *iters_done = done;
    free(M);
    free(w);
    free(wp);
    free(y);
    return status;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* The min1 ranking (the original entry point): orc_rank_csr_op with ORC_MIN1. */
int orc_rank_csr(int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                 double alpha, const double *b0, int32_t max_iters, double tol, double *w_out,
                 double *w_l2_out, double *deltas, int32_t *iters_done) {
    return orc_rank_csr_op(ORC_MIN1, n, nnz, row_ptr, col_idx, alpha, b0, max_iters, tol, w_out, w_l2_out,
                           deltas, iters_done);
}
