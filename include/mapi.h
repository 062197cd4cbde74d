/*
 * mapi.h — C ABI of libmapi.so, the B200 (sm_100a) hot path of multiplication-avoiding power
 * iteration (MAPI, arXiv 2110.12065).
 *
 * Citation keys: P:n = PAPER.md line n (the paper's LaTeX source), S:n = SPEC.md line n,
 * Qn = reading n of the paper listed in DESIGN.md §Readings.
 *
 * CONVENTIONS (all entry points)
 *  - Pointers are DEVICE pointers owned by the caller unless the parameter is marked (host).
 *    The library never allocates, frees or retains caller memory; scratch comes from a
 *    caller-provided device workspace `ws` of at least mapi_workspace_size(...) bytes
 *    (any alignment >= 256 B; torch/cudaMalloc allocations qualify).  mapi_iterate_host is
 *    the one exception that takes host buffers (it copies through the workspace).
 *  - Matrices are fp32 row-major with leading dimension (row stride, in elements) >= #cols.
 *    Vectors are fp32, contiguous.  Sizes are int64_t; graph indices are int32_t.
 *  - `stream` is a cudaStream_t (CUstream) passed as void*; NULL = the legacy default stream.
 *    Work is stream-ordered.  mapi_mavp_matvec and mapi_csr_prepare are asynchronous; every
 *    call that returns an iteration count or a device-detected status (iterate, batched,
 *    pca, rank) synchronises `stream` before returning.
 *  - Errors: a non-MAPI_OK status; mapi_last_error_message() (thread-local) explains it,
 *    e.g. "lda (100) < n_cols (128)".  Argument validation happens before any launch, so a
 *    validation error leaves all outputs untouched.  MAPI_ERR_CUDA wraps a CUDA runtime
 *    error (message = cudaGetErrorString).
 *  - Operator `op`: MAPI_OP_MIN1 = Eq.(3), MAPI_OP_MIN2 = Eq.(4);
 *    MAPI_OP_DOT = Eq.(1) (RPI comparator, see mapi_op).
 *  - Arithmetic: fp32, IEEE round-to-nearest adds, div.rn for the l1 normalisation (P:146
 *    "N divisions"), no FTZ, no fast-math; the MAVP loops contain no multiplication (P:5).
 *  - Determinism: every reduction has a fixed order for a given device and shape, so repeated
 *    calls are bitwise identical.
 */
#ifndef MAPI_H
#define MAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *mapi_stream_t;

typedef enum {
    MAPI_OK = 0,
    MAPI_ERR_NULL = 1,       /* a required pointer is NULL */
    MAPI_ERR_SHAPE = 2,      /* inconsistent sizes; the message carries both values */
    MAPI_ERR_BAD_PARAM = 3,  /* iters < 1, tol < 0, alpha not in (0,1), k < 1 or k > n, bad op */
    MAPI_ERR_DEGENERATE = 4, /* ||A (+) w_t||_1 == 0 at iteration *iters_done */
    MAPI_ERR_NEGATIVE = 5,   /* ranking: b0 has a negative entry */
    MAPI_ERR_NONFINITE = 6,  /* the l1 norm became Inf/NaN (non-finite input) */
    MAPI_ERR_WORKSPACE = 7,  /* ws is NULL or ws_bytes < mapi_workspace_size(...) */
    MAPI_ERR_CUDA = 8        /* CUDA runtime error, or no sm_100 device */
} mapi_status;

/* MAPI_OP_MIN1: Eq.(3); MAPI_OP_MIN2: Eq.(4); MAPI_OP_DOT: the regular product of
 * Eq.(1), the RPI comparator: accepted by mapi_mavp_matvec, mapi_iterate(_host,
 * _sym, _sharded), mapi_iterate_batched and mapi_pca_topk, where it also switches the normalisation to l2
 * (b <- Ab/||Ab||_2, norms[t] = ||A w_t||_2), and by mapi_rank_csr_plan (PageRank G w with the l1
 * normalisation, reading R13); mapi_mavp_matmat and mapi_rank_csr take MIN1/MIN2 only. */
typedef enum { MAPI_OP_MIN1 = 0, MAPI_OP_MIN2 = 1, MAPI_OP_DOT = 2 } mapi_op;

/* Workspace query ids (first argument of mapi_workspace_size). */
typedef enum {
    MAPI_WS_MATVEC = 0,
    MAPI_WS_ITERATE = 1,
    MAPI_WS_ITERATE_BATCHED = 2,
    MAPI_WS_PCA_TOPK = 3,
    MAPI_WS_CSR_PREPARE = 4,
    MAPI_WS_RANK_CSR = 5,
    MAPI_WS_ITERATE_HOST = 6,
    MAPI_WS_MAVP_DEFLATE = 7, /* n = M */
    MAPI_WS_RECONSTRUCT = 8,  /* n = M, nnz = N (images), k = r (components) */
    MAPI_WS_ITERATE_SHARDED = 9,
    MAPI_WS_ITERATE_HOST_MANY = 10, /* n, nnz = lda, k = iters; add 8 bytes per problem beyond 2 */
    MAPI_WS_ITERATE_HOST_MANY_PACKED = 11, /* n, k = iters; add 8 bytes per problem beyond 2 */
    MAPI_WS_ITERATE_SYM = 12,             /* n */
    MAPI_WS_CSR_REORDER = 13,             /* n */
    MAPI_WS_CSR_PLAN = 14,                /* n, nnz: bytes of the plan buffer of mapi_csr_plan (an upper bound) */
    MAPI_WS_CSR_PLAN_BUILD = 15,          /* n, nnz: temporary workspace of mapi_csr_plan */
    MAPI_WS_RANK_CSR_PLAN = 16,           /* n, nnz: workspace of mapi_rank_csr_plan */
    MAPI_WS_ITERATE_HOST_MANY_SYM = 17,   /* n, k = iters; add 8 bytes per problem beyond 2 */
    MAPI_WS_MINIBATCH = 18,               /* n = D, nnz = s (batch size), k = T (iterations) */
    MAPI_WS_RANK_CSR_SHARD = 19           /* n nodes, nnz = the rank's edges, k = m (the rank's rows) */
} mapi_ws_op;

/* y = A (op) x — the matrix extension of the MAVP (reading Q6: y_j uses ROW j):
 *     y_j = sum_k sign(A[j*lda+k] * x_k) * min(|A[j*lda+k]|, |x_k|)      (op = MIN1, Eq. 3)
 * A: n_rows x n_cols (lda >= n_cols), x: n_cols, y: n_rows (must not alias A or x).
 * n_rows == 0 or n_cols == 0 is allowed (y = 0 for n_cols == 0).  Asynchronous. */
mapi_status mapi_mavp_matvec(int32_t op, const float *A, int64_t n_rows, int64_t n_cols,
                             int64_t lda, const float *x, float *y, mapi_stream_t stream);

/* MAVP matrix product — the matrix extension of P:69-70 with the vectors as rows (reading Q7):
 *     C[i*ldc + j] = (1/divisor) * ( sum_k A[i*lda + k] (op) B[j*ldb + k] )
 * (the scalar factor of Eq. 5 is applied as one fp32 multiply by fp32(1/divisor) per element)
 * A: m x K (lda >= K), B: p x K (ldb >= K), C: m x p (ldc >= p), divisor > 0 (1 for the plain product).
 * With B = A = V (pixels x N mean-removed samples) this is the min-covariance: divisor N-1 as in
 * Alg. 2 step 4, N as in Eq. (5).  C must not alias A or B.  K == 0 gives C = 0;
 * m == 0 or p == 0 is a no-op.  Asynchronous. */
mapi_status mapi_mavp_matmat(int32_t op, const float *A, int64_t m, int64_t K, int64_t lda, const float *B,
                             int64_t p, int64_t ldb, float divisor, float *C, int64_t ldc,
                             mapi_stream_t stream);

/* MAPI, Eq.(8) / Algorithm 1:
 *     w_0 = b0 (used as given; Q2)
 *     for t = 0..iters-1:  y = A (op) w_t;  s_t = ||y||_1;  w_{t+1} = y / s_t;
 *                          delta_t = ||w_{t+1} - w_t||_1;  stop early iff tol > 0 && delta_t < tol (Q9)
 *     optional final l2 copy w / ||w||_2 (Alg.1 line 6).
 * A: n x n (lda >= n). b0: n. Outputs: w_out (n, l1-unit final iterate), w_l2_out (n, or NULL),
 * norms[t] = s_t and deltas[t] = delta_t for t < *iters_done (arrays of `iters`, or NULL),
 * *iters_done (host, may be NULL).  On MAPI_ERR_DEGENERATE / NONFINITE, w_out = the last good
 * iterate and *iters_done = the iteration that failed.  Synchronises `stream`. */
mapi_status mapi_iterate(int32_t op, const float *A, int64_t n, int64_t lda, const float *b0,
                         int32_t iters, float tol, float *w_out, float *w_l2_out, float *norms,
                         float *deltas, int32_t *iters_done, void *ws, size_t ws_bytes,
                         mapi_stream_t stream);

/* mapi_iterate for a SYMMETRIC A (the covariance matrices of Eq. 2 / Eq. 5; A[j][k] == A[k][j]),
 * reading only its upper triangle (k >= j): every stored element a_jk, k > j, yields both MAVP terms
 * term(a_jk, w_k) -> y_j and term(a_jk, w_j) -> y_k (the same n^2 terms, no multiply, half the HBM bytes).
 * Used when n >= 8192, n % 8 == 0, lda % 8 == 0 and A is 32 B-aligned; otherwise the full-matrix path of
 * mapi_iterate runs (A must then hold the full symmetric matrix; the library never checks symmetry: it is
 * the caller's declaration by choosing this entry point).  Same outputs, errors and synchronisation as
 * mapi_iterate; results differ from it only by the fp32 summation order.
 * ws: mapi_workspace_size(MAPI_WS_ITERATE_SYM, n, 0, 0) bytes (includes n (n/64 + n/256) floats of partials). */
mapi_status mapi_iterate_sym(int32_t op, const float *A, int64_t n, int64_t lda, const float *b0,
                             int32_t iters, float tol, float *w_out, float *w_l2_out, float *norms,
                             float *deltas, int32_t *iters_done, void *ws, size_t ws_bytes,
                             mapi_stream_t stream);

/* One normalisation step of Algorithm 1 on a full y (used by the row-sharded multi-GPU path after
 * the all-gather of y):  s = ||y|| (l1 for MIN1/MIN2, l2 for DOT; fp64, fixed order),
 * w_new = fp32(y / s), delta = ||w_new - w||_1;  w (n, in/out), *s_out and *delta_out (device, float,
 * nullable), status_out (device int32[1], nullable): 0, MAPI_ERR_DEGENERATE or MAPI_ERR_NONFINITE (w is
 * left unchanged then).  One CTA, deterministic; every rank computes the same bits.  Asynchronous. */
mapi_status mapi_normalize(int32_t op, const float *y, int64_t n, float *w, float *s_out, float *delta_out,
                           int32_t *status_out, mapi_stream_t stream);

/* One fused Algorithm 1 step for a block of rows given the previous FULL y (row-sharded path,
 * DESIGN.md §8): x = y_prev / ||y_prev|| (l1; l2 for DOT), y_out = A (op) x for the n_rows rows of A
 * (n_cols = length of y_prev), and w_next = x, *s_out = ||y_prev||, *delta_out = ||x - w_prev||_1,
 * *status_out as in mapi_normalize (device pointers, nullable).  Every CTA derives x itself in the same
 * fixed order, so no separate normalisation launch is needed.  n_cols * 4 bytes must fit in shared
 * memory (n_cols <= 51200).  Asynchronous. */
mapi_status mapi_matvec_normalized(int32_t op, const float *A, int64_t n_rows, int64_t n_cols, int64_t lda,
                                   const float *y_prev, const float *w_prev, float *w_next, float *y_out,
                                   float *s_out, float *delta_out, int32_t *status_out, mapi_stream_t stream);

/* ---- Multi-GPU MAPI with the exchange fused into the kernel.
 * Every rank allocates one EXCHANGE buffer with mapi_p2p_alloc (device memory, zeroed; layout in p2p.cuh: a
 * u64 arrival flag, world x n floats of exchanged y per iteration parity, world rank totals per parity),
 * publishes its 64-byte CUDA IPC handle (mapi_ipc_get_handle), opens every peer's (mapi_ipc_open_handle; the
 * own buffer is used directly), and passes the device array `peers` (world x u64 base addresses,
 * peers[rank] = own) to mapi_iterate_sharded / mapi_iterate_sym_sharded.  Protocol: per iteration each rank
 * stores its share into every rank's buffer (NVLink P2P, coalesced), fences at system scope, passes a local
 * grid barrier, and ONE thread release-adds 1 to every rank's flag; every CTA waits for world arrivals.
 * epoch0 / flag_base: the global iteration index and own flag value at the start of a call (0 / 0 for a
 * fresh buffer; afterwards advance by *published_out and *published_out x world); identical on every rank.
 * grid: the CTAs per rank, IDENTICAL on every rank (it fixes the row ownership and the summation orders):
 * agree on it before the first call (e.g. the minimum SM count over the ranks); 0 = the device's SM count,
 * allowed only for world == 1.  Ownership: the caller frees with mapi_p2p_free / closes with
 * mapi_ipc_close_handle. */
size_t mapi_p2p_exchange_bytes(int64_t n, int32_t world);
mapi_status mapi_p2p_alloc(size_t bytes, void **ptr_out);
mapi_status mapi_p2p_free(void *ptr);
mapi_status mapi_ipc_get_handle(const void *ptr, void *handle_out /* 64 bytes, host */);
mapi_status mapi_ipc_open_handle(const void *handle /* 64 bytes, host */, void **ptr_out);
mapi_status mapi_ipc_close_handle(void *ptr);

/* K2p: Algorithm 1 on a row-sharded A in ONE cooperative launch per rank: rank `rank` of `world`
 * holds rows [row0, row0 + m) of the n x n matrix (A_local: m x n, lda; 32 B-aligned rows, lda % 8 == 0,
 * n >= 256); b0 is the full start vector (n).  Per iteration every CTA computes its rows into the own buffer,
 * the rank copies its row block and its |y| total to every peer, then s_t = the rank totals in rank order,
 * w_{t+1} and delta_t are formed in the same fixed order on every rank (identical bits, identical stop
 * decision; on one rank bitwise mapi_iterate's cooperative kernel).  Outputs: w_out (full n, l1-unit;
 * l2-unit for DOT), norms / deltas (iters, nullable), host *iters_done, *published_out (iterations that
 * reached the exchange), *grid_out.  ws: mapi_workspace_size(MAPI_WS_ITERATE_SHARDED, 0, 0, 0) bytes.
 * Synchronises `stream`. */
mapi_status mapi_iterate_sharded(int32_t op, const float *A_local, int64_t m, int64_t n, int64_t lda, int64_t row0,
                                 const float *b0, int32_t iters, float tol, int32_t rank, int32_t world,
                                 const uint64_t *peers, uint64_t epoch0, uint64_t flag_base, int32_t grid,
                                 float *w_out, float *norms, float *deltas, int32_t *iters_done,
                                 int32_t *published_out, int32_t *grid_out, void *ws, size_t ws_bytes,
                                 mapi_stream_t stream);

/* K2sp: Algorithm 1 on a SYMMETRIC A (Eq. 2 / 5 covariances) over `world` ranks: K2s's upper-
 * triangle task list (mapi_iterate_sym) is split into equal contiguous ranges; rank r holds only the rows its
 * tasks read, [row_lo, row_hi) as given by mapi_sym_shard_rows (A_local: (row_hi - row_lo) x n, lda, full
 * rows; only their upper-triangle part is read).  Per iteration each rank reduces the partials of its own
 * tasks into a partial y, stores it (fp32) into every rank's buffer, and after the arrivals every rank sums
 * the world partials in rank order (fp64, one rounding): identical y, s_t, w and stop decision everywhere; on
 * one rank bitwise mapi_iterate_sym.  Outputs, epoch / flag / grid as mapi_iterate_sharded.  ws:
 * mapi_workspace_size(MAPI_WS_ITERATE_SYM, n, 0, 0).  Synchronises `stream`. */
mapi_status mapi_iterate_sym_sharded(int32_t op, const float *A_local, int64_t row_lo, int64_t row_hi, int64_t n,
                                     int64_t lda, const float *b0, int32_t iters, float tol, int32_t rank,
                                     int32_t world, const uint64_t *peers, uint64_t epoch0, uint64_t flag_base,
                                     int32_t grid, float *w_out, float *norms, float *deltas, int32_t *iters_done,
                                     int32_t *published_out, int32_t *grid_out, void *ws, size_t ws_bytes,
                                     mapi_stream_t stream);
/* Host-only helpers of K2sp (no device calls): the rows [*row_lo, *row_hi) and tasks [*task_lo, *task_hi) of
 * rank `rank`; and, for row j, the rank's valid partial ranges out4 = {first chunk, end chunk, first row
 * block, end row block} (for tests of the partition). */
mapi_status mapi_sym_shard_rows(int64_t n, int32_t rank, int32_t world, int64_t *row_lo, int64_t *row_hi,
                                int64_t *task_lo, int64_t *task_hi);
mapi_status mapi_sym_shard_valid(int64_t n, int32_t rank, int32_t world, int64_t j, int64_t *out4);

/* mapi_iterate with HOST buffers (end-to-end path): A_host (n x lda), b0_host, w_out_host,
 * w_l2_out_host / norms_host / deltas_host (nullable), iters_done (host).  The call copies A and
 * b0 host->device into the device workspace `ws` (mapi_workspace_size(MAPI_WS_ITERATE_HOST,
 * n, lda, 0) bytes), runs mapi_iterate on the copies, and copies the results device->host, all
 * on `stream`.  Pinned host memory gives full PCIe bandwidth.  Synchronises `stream`. */
mapi_status mapi_iterate_host(int32_t op, const float *A_host, int64_t n, int64_t lda,
                              const float *b0_host, int32_t iters, float tol, float *w_out_host,
                              float *w_l2_out_host, float *norms_host, float *deltas_host,
                              int32_t *iters_done, void *ws, size_t ws_bytes, mapi_stream_t stream);

/* `count` independent mapi_iterate problems with HOST buffers, pipelined (end-to-end serving path):
 * problem i+1's A_hosts[i+1] / b0_hosts[i+1] host->device copies run on an internal copy stream while
 * problem i iterates on `stream` (two device slots alternate), and each result is copied back to
 * w_out_hosts[i] (norms_hosts / deltas_hosts: nullable arrays of nullable pointers).  Host buffers must
 * be PINNED for the copies to overlap.  iters_done: host int32[count] (nullable).  ws:
 * mapi_workspace_size(MAPI_WS_ITERATE_HOST_MANY, n, lda, iters) + 8 * max(0, count - 2) bytes.  Returns the
 * first problem's error, if any.  Synchronises `stream`. */
mapi_status mapi_iterate_host_many(int32_t op, int32_t count, const float *const *A_hosts, int64_t n, int64_t lda,
                                   const float *const *b0_hosts, int32_t iters, float tol,
                                   float *const *w_out_hosts, float *const *norms_hosts,
                                   float *const *deltas_hosts, int32_t *iters_done, void *ws, size_t ws_bytes,
                                   mapi_stream_t stream);

/* mapi_iterate_host_many for SYMMETRIC matrices (the covariance inputs of Eq. 2 / Eq. 5) sent in
 * packed upper-triangular form: Ap_hosts[i] holds n(n+1)/2 floats, row j = A[j][j..n-1] at offset
 * j*n - j*(j-1)/2 (LAPACK "packed" storage, row-major).  Half the host->device bytes of the full matrix;
 * the device rebuilds the full row-major matrix bitwise (A[k][j] = A[j][k]) before iterating, so results are
 * bitwise those of mapi_iterate_host_many on the full matrix.  The library does not check symmetry: it is
 * the caller's declaration by choosing this entry point.  ws: mapi_workspace_size(
 * MAPI_WS_ITERATE_HOST_MANY_PACKED, n, 0, iters) + 8 * max(0, count - 2) bytes.  Synchronises `stream`. */
mapi_status mapi_iterate_host_many_packed(int32_t op, int32_t count, const float *const *Ap_hosts, int64_t n,
                                          const float *const *b0_hosts, int32_t iters, float tol,
                                          float *const *w_out_hosts, float *const *norms_hosts,
                                          float *const *deltas_hosts, int32_t *iters_done, void *ws,
                                          size_t ws_bytes, mapi_stream_t stream);

/* mapi_iterate_host_many for SYMMETRIC matrices given as FULL host matrices (n x lda, pinned for overlap):
 * only the upper-triangle block rows are copied host->device (one 2-D copy per 128-row block: columns
 * [128 b, n) of rows [128 b, 128 b + 128)), half the PCIe bytes and no host-side packing, and K2s
 * (mapi_iterate_sym) iterates on them; the strictly-lower part of the device copy is never read.  Results
 * bitwise those of mapi_iterate_sym on the device matrix.  ws: mapi_workspace_size(
 * MAPI_WS_ITERATE_HOST_MANY_SYM, n, 0, iters) + 8 * max(0, count - 2) bytes.  Synchronises `stream`. */
mapi_status mapi_iterate_host_many_sym(int32_t op, int32_t count, const float *const *A_hosts, int64_t n, int64_t lda,
                                       const float *const *b0_hosts, int32_t iters, float tol,
                                       float *const *w_out_hosts, float *const *norms_hosts,
                                       float *const *deltas_hosts, int32_t *iters_done, void *ws, size_t ws_bytes,
                                       mapi_stream_t stream);

/* Host-side input preparation for mapi_iterate_host_many_packed: the upper triangle of the n x lda host
 * matrix A in LAPACK packed row-major order (row j = A[j, j:], n(n+1)/2 floats into `out`), copied by
 * `threads` host threads (0 = all hardware threads).  Pure data movement; synchronous. */
mapi_status mapi_pack_upper_host(const float *A, int64_t n, int64_t lda, float *out, int32_t threads);

/* Batched MAPI: k independent runs of mapi_iterate on the same A ("multiple independent
 * runs"; matrix extension P:69-70 with p = k columns), Y = A (op) W each iteration.
 * B0, W_out: k x n, vector-major (vector v at B0 + v*n).  norms, deltas: iters x k
 * (entry [t*k + v]), nullable.  iters_done (host, k entries, nullable): per-vector count; a
 * vector stops individually when its own delta < tol (tol > 0).  op MAPI_OP_DOT: k independent RPI runs
 * (Eq. 1, l2 normalisation).  The call returns the worst status over vectors.  Synchronises `stream`. */
mapi_status mapi_iterate_batched(int32_t op, const float *A, int64_t n, int64_t lda,
                                 const float *B0, int32_t k, int32_t iters, float tol, float *W_out,
                                 float *norms, float *deltas, int32_t *iters_done, void *ws,
                                 size_t ws_bytes, mapi_stream_t stream);

/* Top-k principal vectors by MAPI with L2 deflation (BASELINE configs[1]):
 *     for i = 0..k-1:  D_i = (I - sum_{m<i} p_m p_m^T) C ;  w = MAPI(D_i, b0, iters, tol = 0) ;
 *                      p_i = w / ||w||_2
 * D_i is formed as C - sum_m p_m r_m^T with r_m = p_m^T C, accumulated in fp64 and rounded
 * once to fp32 (K5).  C: n x n (ldc >= n).  b0: n.  P_out: k x n (l2-unit rows).
 * norms, deltas: k x iters (row i = vector i), nullable.  Synchronises `stream`. */
mapi_status mapi_pca_topk(int32_t op, const float *C, int64_t n, int64_t ldc, int32_t k,
                          int32_t iters, const float *b0, float *P_out, float *norms, float *deltas,
                          void *ws, size_t ws_bytes, mapi_stream_t stream);

/* Alg. 2 step 3: mean over the N columns of each row of V (M x N, ldv; the images as columns),
 * mean_out[i] = m_i (fp64 sum, rounded once), Vc = V - m (M x N, ldvc; may alias V).  Asynchronous. */
mapi_status mapi_center_rows(const float *V, int64_t M, int64_t N, int64_t ldv, float *Vc, int64_t ldvc,
                             float *mean_out, mapi_stream_t stream);

/* Alg. 2 step 6: D = C - (w (op) w^T) C, where (w (op) w^T)[i][j] = term(w_i, w_j) is
 * the scalar-MAVP outer product and the product with C is a REGULAR matrix product.  Evaluated exactly
 * in O(M^2) through the sorted prefix-sum regrouping of DESIGN.md R10 (fp64 scans, one fp32 rounding).
 * C: M x M (ldc >= M), w: M (normally the l2-unit MAPI output, Alg. 1 line 6), D: M x M (ldd >= M, must
 * not alias C).  op: MIN1, MIN2 or DOT (DOT gives the L2 deflation (I - w w^T) C of P:26).
 * M <= 16384.  Workspace: mapi_workspace_size(MAPI_WS_MAVP_DEFLATE, M, 0, 0).  Asynchronous. */
mapi_status mapi_mavp_deflate(int32_t op, const float *C, int64_t M, int64_t ldc, const float *w, float *D,
                              int64_t ldd, void *ws, size_t ws_bytes, mapi_stream_t stream);

/* Alg. 2 steps 3 and 8: for the N images stored as the columns of V (M x N, ldv),
 * m = mean over the columns, and every column j of Vhat (M x N, ldvh) is
 *     v_hat_j = (W (op) W^T)(v_j - m) + m,   (W (op) W^T)[i][i'] = sum_c term(W[i][c], W[i'][c]),
 * W: M x r (ldw >= r; normally [w1 w2], r = 2).  mean_out (M, required).  Same exact O(M r N) regrouping
 * as mapi_mavp_deflate; M <= 16384.  Workspace: mapi_workspace_size(MAPI_WS_RECONSTRUCT, M, N, r).
 * No clamping (the paper is silent; callers clamp to [0, 1] for display / PSNR).  Asynchronous. */
mapi_status mapi_mavp_reconstruct(int32_t op, const float *W, int64_t M, int32_t r, int64_t ldw, const float *V,
                                  int64_t N, int64_t ldv, float *Vhat, int64_t ldvh, float *mean_out, void *ws,
                                  size_t ws_bytes, mapi_stream_t stream);

/* Google-matrix preparation for MAPI ranking (Eq. 13; reading Q10):
 * the graph is CSR by DESTINATION (row i lists the sources j of the distinct edges j -> i);
 * row_ptr: n+1 int32 (nnz < 2^31), col_idx: nnz int32 in [0, n).
 * Outputs per column j:  cap_out[j] = alpha / outdeg(j) (0 if dangling),
 *                        bg_out[j]  = (1 - alpha)/n, or 1/n if j is dangling (outdeg 0).
 * outdeg is counted from col_idx on the device.  Asynchronous. */
mapi_status mapi_csr_prepare(int64_t n, int64_t nnz, const int32_t *row_ptr, const int32_t *col_idx,
                             float alpha, float *cap_out, float *bg_out, void *ws, size_t ws_bytes,
                             mapi_stream_t stream);

/* MAPI ranking: w <- (G (min1) w) / ||G (min1) w||_1 with G = alpha M + (1-alpha)/n 1 never
 * materialised.  For w >= 0 the min1 row product equals exactly (K3)
 *     y_i = S + sum_{e in row i} min(max(w_j - bg_j, 0), cap_j),  j = col_idx[e],
 *     S   = sum_j min(bg_j, w_j).
 * cap, bg: from mapi_csr_prepare.  b0: n, >= 0 (else MAPI_ERR_NEGATIVE).  Stops when
 * tol > 0 && delta_t < tol or after max_iters.  w_out: n (l1-unit), w_l2_out (n or NULL,
 * final l2 copy P:322), deltas (max_iters, nullable), *iters_done (host).  Synchronises. */
mapi_status mapi_rank_csr(int64_t n, int64_t nnz, const int32_t *row_ptr, const int32_t *col_idx,
                          const float *cap, const float *bg, const float *b0, int32_t max_iters,
                          float tol, float *w_out, float *w_l2_out, float *deltas,
                          int32_t *iters_done, void *ws, size_t ws_bytes, mapi_stream_t stream);

/* Segmented ranking plan (K3s): a one-time, per-graph layout of the same CSR graph for the
 * planned ranking kernel.  Nodes are put in "plan order": sources (out-degree >= 1) by DESCENDING out-degree,
 * then dangling nodes with in-edges, then isolated nodes (ties by ascending id).  The sources are cut into
 * segments of 32,767; the edges are stored segment-major, then by the plan position of their destination
 * row, as 16-bit words (local source offset | end-of-fragment flag), where a "fragment" is a run of one row
 * inside one segment and one 512-word tile.  Per iteration every CTA gathers the v values of one segment at
 * a time from SHARED memory instead of scattered L2 reads and writes one partial per fragment; the node pass
 * collects each batch of rows' fragments through a precomputed (batch, fragment)-ordered list and sums each
 * row's fragments in a fixed (segment, position) order.  The graph and its semantics are those of
 * mapi_rank_csr (row_ptr / col_idx by destination, int32, nnz < 2^31).
 * plan: device buffer of mapi_workspace_size(MAPI_WS_CSR_PLAN, n, nnz, 0) bytes (an upper bound); info
 * (host) receives the sizes the run needs (keep it with the plan).  ws: MAPI_WS_CSR_PLAN_BUILD bytes of
 * temporary device workspace.  The plan is tied to the device's SM count (info->grid).  Deterministic.
 * MAPI_ERR_SHAPE if one row has so many fragments that a node batch exceeds the kernel's shared memory
 * (> 49,152 fragment sums in a batch of up to 32,768 + one row's; not reachable below ~2^23 in-edges per row): use mapi_rank_csr then.
 * Synchronises `stream` (small read-backs size the later steps). */
typedef struct mapi_csr_plan_info {
    int64_t n, nnz;      /* the graph */
    int64_t nsrc;        /* sources with out-degree >= 1 */
    int64_t npieces;     /* fragments (= partial sums per iteration) */
    int64_t nwords;      /* 16-bit edge words incl. segment padding (a multiple of 512) */
    int32_t nseg;        /* segments of 32,767 sources */
    int32_t grid;        /* CTAs of the planned kernel (one per SM) */
    int64_t nlive;       /* non-isolated nodes (plan positions [0, nlive)) */
    int64_t nbatch;      /* node-pass batches */
    int64_t nunits;      /* edge-pass work units */
} mapi_csr_plan_info;
mapi_status mapi_csr_plan(int64_t n, int64_t nnz, const int32_t *row_ptr, const int32_t *col_idx, void *plan,
                          size_t plan_bytes, mapi_csr_plan_info *info, void *ws, size_t ws_bytes,
                          mapi_stream_t stream);

/* MAPI ranking (Eq. 13) through a plan of mapi_csr_plan: the same iteration, stop rule and
 * outputs as mapi_rank_csr, run as ONE persistent cooperative launch (two grid barriers per iteration; a
 * tol stop ends it on the device, no per-iteration launches).  op: MAPI_OP_MIN1 / MAPI_OP_MIN2 (identical
 * here: G >= 0 and w >= 0) or MAPI_OP_DOT — the PageRank power iteration G w (Eq. 1 with G of P:307,
 * reading R13: y_i = sum_j bg_j w_j + sum_{j -> i} cap_j w_j, normalised by its l1 norm each iteration
 * (the column-stochastic G preserves it), final l2 copy P:322).  cap, bg, b0 as mapi_rank_csr.
 * ws: mapi_workspace_size(MAPI_WS_RANK_CSR_PLAN, n, nnz, 0).  Synchronises `stream`. */
mapi_status mapi_rank_csr_plan(int32_t op, const void *plan, const mapi_csr_plan_info *info, const float *cap,
                               const float *bg, const float *b0, int32_t max_iters, float tol, float *w_out,
                               float *w_l2_out, float *deltas, int32_t *iters_done, void *ws, size_t ws_bytes,
                               mapi_stream_t stream);

/* MAPI ranking with the destination rows PARTITIONED OVER RANKS (K3n; the ranking
 * update of Eq. 13, exactly as mapi_rank_csr computes it).  Rank r owns the rows [row0, row0 + m):
 * row_ptr_local (m + 1 int32, rebased so that row_ptr_local[0] == 0) and col_idx_local (nnz_local int32 GLOBAL
 * source ids in [0, n)) are its part of the CSR-by-destination graph.  cap, bg (mapi_csr_prepare on the WHOLE
 * graph) and b0 are full n-vectors on every rank; every rank keeps the full node state in its workspace and runs
 * the same fixed-order node kernels on it, so s_t, w_t, delta_t and the stop decision are bitwise identical on
 * all ranks.  One iteration t (t = 0, 1, ... in order) is three steps on ONE stream:
 *   mapi_rank_csr_shard_rows(t):      e_t[row0, row0 + m) = the gather-sum over the rank's edges; *e_out
 *                                     (host pointer, may be NULL) receives the DEVICE address of e_t (n floats);
 *   the caller's collective:          all-gather the ranks' blocks of e_t in place (n * 4 bytes in total);
 *   mapi_rank_csr_shard_normalize(t): sum_i e_i over all n (fixed order), s_t = n S_t + sum e, w_{t+1},
 *                                     v_{t+1}, S_{t+1}, delta_t -> deltas[t] (device, nullable), iteration
 *                                     count, stop flag (tol > 0 && delta_t < tol), DEGENERATE / NONFINITE.
 * All three are ASYNCHRONOUS; once the stop flag or an error status is set every later step returns at once on
 * the device.  mapi_rank_csr_shard_begin starts a run (state in ws; w_0 = b0 >= 0 else MAPI_ERR_NEGATIVE at
 * finish).  mapi_rank_csr_shard_finish writes w_out (n, l1-unit; NULL: only read the status — the host's
 * periodic stop check) and w_l2_out (nullable), *iters_done and *stopped (host, nullable), SYNCHRONISES
 * `stream` and returns the run's status.  ws: mapi_workspace_size(MAPI_WS_RANK_CSR_SHARD, n, nnz_local, m),
 * the same buffer for every call of a run.  m == 0 (a rank without rows) is valid. */
mapi_status mapi_rank_csr_shard_begin(int64_t n, int64_t m, int64_t nnz_local, const int32_t *row_ptr_local,
                                      const float *cap, const float *bg, const float *b0, void *ws, size_t ws_bytes,
                                      mapi_stream_t stream);
mapi_status mapi_rank_csr_shard_rows(int64_t n, int64_t m, int64_t row0, int64_t nnz_local,
                                     const int32_t *row_ptr_local, const int32_t *col_idx_local, int32_t t,
                                     float **e_out, void *ws, size_t ws_bytes, mapi_stream_t stream);
mapi_status mapi_rank_csr_shard_normalize(int64_t n, int64_t m, int64_t nnz_local, const float *cap, const float *bg,
                                          const float *b0, int32_t t, float tol, float *deltas, void *ws,
                                          size_t ws_bytes, mapi_stream_t stream);
mapi_status mapi_rank_csr_shard_finish(int64_t n, int64_t m, int64_t nnz_local, const float *b0, float *w_out,
                                       float *w_l2_out, int32_t *iters_done, int32_t *stopped, void *ws,
                                       size_t ws_bytes, mapi_stream_t stream);

/* Optional preparation for the ranking path: relabel the nodes by DESCENDING out-degree (ties by ascending
 * id), so the most gathered sources get the lowest ids, which the gather kernel keeps in shared memory
 * (K3h).  perm_out[old] = new (n).  row_ptr_out (n+1) / col_idx_out (nnz): the same graph in the
 * new ids (new row i' = the in-edges of the old node with perm = i', sources renamed, in their original
 * order).  Rank the relabelled graph (mapi_csr_prepare + mapi_rank_csr with b0 permuted by
 * mapi_csr_permute) and map the result back with mapi_csr_permute(to_new = 0).  Deterministic (stable
 * radix sort).  ws: mapi_workspace_size(MAPI_WS_CSR_REORDER, n, 0, 0).  Asynchronous. */
mapi_status mapi_csr_reorder(int64_t n, int64_t nnz, const int32_t *row_ptr, const int32_t *col_idx,
                             int32_t *perm_out, int32_t *row_ptr_out, int32_t *col_idx_out, void *ws,
                             size_t ws_bytes, mapi_stream_t stream);
/* out[perm[j]] = x[j] (to_new != 0: original ids -> relabelled) or out[j] = x[perm[j]] (to_new == 0:
 * relabelled -> original).  x and out must not alias.  Asynchronous. */
mapi_status mapi_csr_permute(int64_t n, const int32_t *perm, const float *x, float *out, int32_t to_new,
                             mapi_stream_t stream);

/* Algorithm 3, mini-batch MAPI with momentum (Section 3.2; K10, readings R14 / R15):
 *   for t = 0 .. T-1:  M_t = (1/s) sum_{i in batch t} A~_i,  A~_i[j][k] = x_ij (gram_op) x_ik   (steps 3-4)
 *                      y_j = sum_k min1-term(M_t[j][k], w_t[k]) - beta w_{t-1}[j]   (w_{-1} = 0)   (step 4)
 *                      s_t = ||y||_1;  w_{t-1} <- w_t / s_t;  w_t <- y / s_t                     (step 5)
 * X: N x D samples (device, fp32, row-major, leading dimension ldx >= D), 1 <= D <= 64 (MAPI_ERR_SHAPE
 * beyond).  batch: T x s int32 row indices in [0, N) (device) — the i.i.d. draws of step 3 are the caller's;
 * an index outside [0, N) is detected on the device (it is read as a zero sample) and the call returns
 * MAPI_ERR_BAD_PARAM after the run.  gram_op: MAPI_OP_MIN1 (the paper's A = X^T (.) X) or
 * MAPI_OP_DOT (x_i x_i^T).  w0: D (used as given, step 1).  w_prev0 (D or NULL): the momentum vector to
 * continue a run from (NULL: the paper's w_{-1} = 0).  Outputs: w_out D (l1-unit w_T), w_l2_out (D or NULL,
 * Alg. 3 line 7), w_prev_out (D or NULL: w_{T-1} / s_{T-1}, the state a continued run needs), norms (T or
 * NULL: s_t), *iters_done (host, may be NULL).  MAPI_ERR_DEGENERATE /
 * MAPI_ERR_NONFINITE as for mapi_iterate (w_out = the last good iterate).  Because the draws are inputs,
 * all M_t are formed in parallel before the T dependent steps.  T <= 65535.
 * ws: mapi_workspace_size(MAPI_WS_MINIBATCH, D, s, T).  Synchronises `stream`. */
mapi_status mapi_minibatch(int32_t gram_op, const float *X, int64_t N, int64_t D, int64_t ldx,
                           const int32_t *batch, int32_t s, int32_t T, float beta, const float *w0,
                           const float *w_prev0, float *w_out, float *w_l2_out, float *w_prev_out,
                           float *norms, int32_t *iters_done, void *ws, size_t ws_bytes,
                           mapi_stream_t stream);

/* Bytes of device workspace the call `op` needs for the given sizes (0 if none).
 *   MAPI_WS_MATVEC: 0.  MAPI_WS_ITERATE: n.  MAPI_WS_ITERATE_BATCHED: n, k.
 *   MAPI_WS_PCA_TOPK: n, k.  MAPI_WS_CSR_PREPARE / MAPI_WS_RANK_CSR: n, nnz.
 *   MAPI_WS_ITERATE_HOST: n, and nnz = lda (the device copy of A is n*lda floats), k = iters.
 *   MAPI_WS_MAVP_DEFLATE: n = M.  MAPI_WS_RECONSTRUCT: n = M, nnz = N, k = r.
 *   MAPI_WS_ITERATE_SHARDED: 256 (status words).
 *   MAPI_WS_ITERATE_HOST_MANY: n, nnz = lda, k = iters (two slots; + 8 bytes per problem beyond 2).
 *   MAPI_WS_ITERATE_HOST_MANY_PACKED: n, k = iters (same, plus a packed buffer per slot).
 *   MAPI_WS_CSR_PLAN / MAPI_WS_CSR_PLAN_BUILD / MAPI_WS_RANK_CSR_PLAN: n, nnz.
 *   MAPI_WS_MINIBATCH: n = D, nnz = s, k = T.
 *   MAPI_WS_RANK_CSR_SHARD: n nodes, nnz = the rank's edges, k = m (the rank's rows). */
size_t mapi_workspace_size(int32_t op, int64_t n, int64_t nnz, int32_t k);

const char *mapi_status_string(mapi_status status);
const char *mapi_last_error_message(void);

/* Instrumentation (bench.py): number of kernels this library has launched in the process, and
 * the device time (CUDA events on the launching stream) of the most recent launch of the
 * dominant kernel of the last iterate / batched / pca / rank call when profiling is on. */
uint64_t mapi_launch_count(void);
void mapi_set_profiling(int32_t enable);
float mapi_last_kernel_ms(void);

#ifdef __cplusplus
}
#endif
#endif /* MAPI_H */
