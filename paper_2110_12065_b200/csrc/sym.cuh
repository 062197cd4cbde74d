// sym.cuh — K2s: persistent MAPI iteration for SYMMETRIC matrices reading only the upper triangle.
//
// MAPI's dense inputs are covariance matrices (Eq. 2 / Eq. 5: C = X X^T / N), symmetric by
// construction, and at n = 32768 (BASELINE configs[2]) an iteration is bound by the 4 GiB read of A.  A
// stored element a_jk (k > j) appears in two MAVP terms of y = A (+) w (Eq. 3, matrix extension
// P:69-70): term(a_jk, w_k) in y_j and term(a_kj, w_j) = term(a_jk, w_j) in y_k.  K2s reads each
// upper-triangle element once (half the HBM bytes) and forms BOTH terms — still one FMNMX.XORSIGN per term
// and no multiply, n^2 terms per iteration, exactly the same sum as the full read:
//     y_j = sum_{k >= j} term(a_jk, w_k)  [row terms]  +  sum_{k < j} term(a_kj, w_k)  [column terms].
//
// Tasks: (row block b of kSymRB = 64 rows, column chunk c of kSymCC = 256 columns = 1 KB per row) with
// chunk end > block start, i.e. chunks c >= b / 4; tasks are dealt round-robin to the grid's warps (~14
// per warp at n = 32768: balanced to 0.4%).  A warp streams its task row by row (lane l holds columns
// c0 + 8l .. +8 of the row: one 256-bit evict-first load; two 4-row batches in flight): the row term of the
// lane's 8 elements against w_k (registers, loaded once per task) is summed in a tree and across the warp
// by a butterfly -> P_row[c][j]; the column terms against w_j (a shared-memory broadcast) accumulate per
// lane in 8 registers over the task's 64 rows (64-term chains) -> P_col[b][k].  On the diagonal tasks
// the row term keeps k >= j and the column term k > j; everything below the diagonal is skipped.
//
// Per iteration: tasks -> grid barrier -> every CTA sums its rows' partials in fp64 (4 threads per row,
// interleaved, fixed combine order): y_j = sum_{c >= c(j)} P_row[c][j] + sum_{b <= b(j)} P_col[b][j]
// (fp32 chains <= 256 terms inside the partials, fp64 across them: within T1) -> fp64 |y|
// partial per CTA -> grid barrier -> s_t, w_{t+1} = fp32(y / s_t), delta_t exactly as K2c.  Deterministic
// for a given (n, grid).  Requirements: n % 8 == 0, lda % 8 == 0, 32 B-aligned A (the caller falls back to
// the full-matrix kernels otherwise), w (n floats) in shared memory.
#pragma once
#include "dense.cuh"
#include "mapi_common.cuh"

namespace mapi {

constexpr int kSymRB = 64;         // rows per task (column-partial chain length)
constexpr int kSymCC = 256;        // columns per task (one 1 KB row chunk per warp row)
constexpr int kSymNW = 16;         // warps per CTA
constexpr int kSymThreads = kSymNW * 32;

struct SymArgs {
    IterArgs it;
    float* prow;  // [nc][n] row partials
    float* pcol;  // [nb][n] column partials
};

__host__ __device__ inline int64_t sym_nb(int64_t n) { return (n + kSymRB - 1) / kSymRB; }
__host__ __device__ inline int64_t sym_nc(int64_t n) { return (n + kSymCC - 1) / kSymCC; }
// first task of row block b: sum_{b' < b} (nc - b' / 4)   (kSymCC / kSymRB = 4)
__host__ __device__ inline int64_t sym_task_start(int64_t b, int64_t nc) {
    const int64_t q = b / 4, r = b % 4;
    return b * nc - (2 * q * (q - 1) + r * q);
}
inline size_t sym_partials_bytes(int64_t n) {
    return sizeof(float) * (size_t)n * (size_t)(sym_nb(n) + sym_nc(n));
}
inline size_t sym_smem_bytes(int64_t n) { return sizeof(float) * (size_t)((n + 3) & ~int64_t(3)) + sizeof(double) * 40; }

template <int OP>
__device__ __forceinline__ float sym_tree8(const float (&a)[8], const float (&w)[8]) {
    float t[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) t[e] = mavp_term<OP>(a[e], w[e]);
    return tree_sum(t);
}

template <int OP>
__global__ void __launch_bounds__(kSymThreads, 1) k_iterate_sym(SymArgs sa) {
    extern __shared__ __align__(16) float w_s[];
    const IterArgs& p = sa.it;
    const int64_t n = p.n;
    double* red = reinterpret_cast<double*>(w_s + ((n + 3) & ~int64_t(3)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nb = sym_nb(n), nc = sym_nc(n), ntasks = sym_task_start(nb, nc);
    const int64_t gw = (int64_t)blockIdx.x * kSymNW + warp, W = (int64_t)gridDim.x * kSymNW;
    const int64_t r0 = (int64_t)blockIdx.x * n / gridDim.x, r1 = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
    for (int64_t k = tid; k < n; k += blockDim.x) w_s[k] = p.b0[k];
    __syncthreads();

    int32_t done = 0, status = kStOk;
    double* slots = reinterpret_cast<double*>(p.slots);
    for (int32_t t = 0; t < p.iters; ++t) {
        float* y = p.y + (t & 1) * n;
        // ---- phase 1: upper-triangle tasks
        for (int64_t task = gw; task < ntasks; task += W) {
            int64_t lo = 0, hi = nb - 1;  // row block: last b with start(b) <= task
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (sym_task_start(mid, nc) <= task) lo = mid;
                else hi = mid - 1;
            }
            const int64_t b = lo, c = b / 4 + (task - sym_task_start(b, nc));
            const int64_t j0 = b * kSymRB, j1 = min(n, j0 + kSymRB), c0 = c * kSymCC;
            const int64_t kl = c0 + 8 * lane;  // this lane's first column
            const bool live = kl < n;          // n % 8 == 0: a lane is all in or all out
            const bool diag = c0 < j1;         // some element with k <= j: masked path
            float wk[8], col[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                wk[e] = live ? w_s[kl + e] : 0.0f;
                col[e] = 0.0f;
            }
            float keep0 = 0.0f, keep1 = 0.0f;  // row partials of rows j0 + lane, j0 + 32 + lane
            const float* base = p.A + j0 * p.lda + kl;
            const int rows = (int)(j1 - j0);
            float a[2][4][8];
            auto load = [&](float (&buf)[4][8], int rb) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (live && rb + r < rows) ld_stream<8, 0>(base + (int64_t)(rb + r) * p.lda, buf[r]);
                    else
#pragma unroll
                        for (int e = 0; e < 8; ++e) buf[r][e] = 0.0f;
                }
            };
            auto consume = [&](const float (&buf)[4][8], int rb) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int jr = rb + r;
                    if (jr >= rows) break;  // warp-uniform
                    const int64_t j = j0 + jr;
                    const float wj = w_s[j];
                    float rs;
                    if (!diag) {
                        rs = sym_tree8<OP>(buf[r], wk);
#pragma unroll
                        for (int e = 0; e < 8; ++e) col[e] += mavp_term<OP>(buf[r][e], wj);
                    } else {
                        float tr[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int64_t k = kl + e;
                            tr[e] = k >= j ? mavp_term<OP>(buf[r][e], wk[e]) : 0.0f;
                            if (k > j) col[e] += mavp_term<OP>(buf[r][e], wj);
                        }
                        rs = tree_sum(tr);
                    }
                    rs = warp_sum(rs);
                    if (lane == (jr & 31)) {
                        if (jr < 32) keep0 = rs;
                        else keep1 = rs;
                    }
                }
            };
            load(a[0], 0);
            for (int rb = 0; rb < rows; rb += 8) {
                load(a[1], rb + 4);
                consume(a[0], rb);
                if (rb + 8 < rows) load(a[0], rb + 8);
                consume(a[1], rb + 4);
            }
            float* prow = sa.prow + c * n;
            if (j0 + lane < j1) prow[j0 + lane] = keep0;
            if (j0 + 32 + lane < j1) prow[j0 + 32 + lane] = keep1;
            if (live) {
                float4* pc = reinterpret_cast<float4*>(sa.pcol + b * n + kl);
                pc[0] = make_float4(col[0], col[1], col[2], col[3]);
                pc[1] = make_float4(col[4], col[5], col[6], col[7]);
            }
        }
        grid_barrier(p.bar, (unsigned int)(2 * t + 1) * gridDim.x);
        // ---- phase 2: y_j of this CTA's rows; 4 threads per row take every 4th partial, fp64
        double abs_part = 0.0;
        for (int64_t rbase = r0; rbase < r1; rbase += kSymThreads / 4) {
            const int64_t j = rbase + tid / 4;
            const int sub = tid & 3;
            double acc = 0.0;
            if (j < r1) {
                const int64_t cj = j / kSymCC, bj = j / kSymRB;
                const int64_t nrow = nc - cj, ntot = nrow + bj + 1;
                for (int64_t q = sub; q < ntot; q += 4)
                    acc += (double)(q < nrow ? __ldcg(sa.prow + (cj + q) * n + j) : __ldcg(sa.pcol + (q - nrow) * n + j));
            }
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            if (sub == 0 && j < r1) {
                const float v = (float)acc;
                y[j] = v;
                abs_part += norm_part<OP>(v);
            }
        }
        const double cta_abs = block_sum(abs_part, red);
        if (tid == 0) slots[(t & 1) * gridDim.x + blockIdx.x] = cta_abs;
        grid_barrier(p.bar, (unsigned int)(2 * t + 2) * gridDim.x);
        // ---- s_t: the same fixed-order fp64 sum in every CTA
        double sd;
        {
            if (warp == 0) {
                double pp = 0.0;
                for (int cc = lane; cc < (int)gridDim.x; cc += 32) pp += __ldcg(slots + (t & 1) * gridDim.x + cc);
                pp = warp_sum(pp);
                if (lane == 0) red[32] = pp;
            }
            __syncthreads();
            sd = norm_final<OP>(red[32]);
            __syncthreads();
        }
        if (!(sd > 0.0) || isinf(sd)) {  // uniform across the grid
            status = (sd == 0.0) ? kStDegenerate : kStNonfinite;
            break;
        }
        // ---- w_{t+1} = y / s_t, delta_t, into this CTA's shared memory (as K2c)
        double dpart = 0.0;
        for (int64_t k = tid; k < n; k += blockDim.x) {
            const float wn = (float)((double)ld_cg(y + k) / sd);
            dpart += (double)fabsf(wn - w_s[k]);
            w_s[k] = wn;
        }
        const double delta = block_sum(dpart, red);  // its barriers also publish w_s
        if (blockIdx.x == 0 && tid == 0) {
            if (p.norms) p.norms[t] = (float)sd;
            if (p.deltas) p.deltas[t] = (float)delta;
        }
        done = t + 1;
        if (p.tol > 0.0f && delta < (double)p.tol) break;
    }
    for (int64_t k = r0 + tid; k < r1; k += blockDim.x) p.w_out[k] = w_s[k];
    if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
}

}  // namespace mapi
