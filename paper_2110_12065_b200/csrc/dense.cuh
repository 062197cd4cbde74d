// dense.cuh — K1 (streaming MAVP mat-vec) and K2 (persistent MAPI iteration) for sm_100a.
//
// K1: y_j = sum_k A[j,k] (+) w_k  (matrix extension P:69-70, Eq. 3).  One warp owns a row;
//     each lane streams 32-byte vectors (LDG.E.NA.EFL2.256) of the row, the iterate w is read
//     from shared memory (LDS.128) or global/L1.  Per lane VEC independent fp32 chains of at
//     most kFold = 128 terms each (then folded), a fixed pairwise tree over the VEC slots and a
//     warp butterfly: a fixed summation order with the error bound of DESIGN.md §a2.
// K2: Algorithm 1 as ONE cooperative persistent kernel: per iteration
//     {rows -> y, per-CTA sum |y|} -> grid barrier -> every CTA reduces the per-CTA partials in
//     the same fixed order to s_t, divides y by s_t (IEEE div.rn) while re-staging w_{t+1} into
//     its own shared memory and accumulating delta_t = ||w_{t+1} - w_t||_1 in the same fixed
//     order -> identical s_t, delta_t and stop decision in every CTA with ONE barrier/iteration.
#pragma once
#include "mapi_common.cuh"

namespace mapi {

constexpr int kFold = 128;  // max fp32 terms per accumulator chain before folding

// status codes (mirror mapi_status)
constexpr int kStOk = 0, kStDegenerate = 4, kStNonfinite = 6;

// L2 bulk prefetch of `bytes` (multiple of 16) starting at 16 B-aligned `p` (no register cost).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Row MAVP: sum_k a[k] (+) w[k] for k < n, by one warp. Returns the same value in all lanes.
// a must be VEC*4-byte aligned; w (smem or global) likewise.  U = warp-wide loads in flight per
// lane; PF > 0: lane 0 also bulk-prefetches into L2 the U-step group PF groups ahead (same row).
// Summation order: per lane VEC chains of <= kFold terms, pairwise tree over the VEC slots, the
// blocks of kFold steps added in order, the scalar tail, then the warp butterfly.
template <int OP, int VEC, int POL, bool WG, int U, int PF = 0>
__device__ __forceinline__ float row_mavp(const float* __restrict__ a, const float* __restrict__ w,
                                          int64_t n, int lane) {
    constexpr int STEP = kWarp * VEC;
    const int64_t n_main = (n / STEP) * STEP;
    float tot = 0.0f;

    for (int64_t blk = 0; blk < n_main; blk += (int64_t)kFold * STEP) {
        const int64_t blk_end = min(n_main, blk + (int64_t)kFold * STEP);
        float acc[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc[i] = 0.0f;
        int64_t c = blk + lane * VEC;
        const int64_t base_end = blk_end - (int64_t)(U - 1) * STEP;  // warp-uniform bound
        for (; c - lane * VEC < base_end; c += (int64_t)U * STEP) {
            if constexpr (PF > 0) {
                const int64_t pf = c - lane * VEC + (int64_t)PF * U * STEP;
                if (lane == 0 && pf + (int64_t)U * STEP <= n_main)
                    prefetch_l2(a + pf, (uint32_t)(U * STEP * sizeof(float)));
            }
            float v[U][VEC];
#pragma unroll
            for (int u = 0; u < U; ++u) ld_stream<VEC, POL>(a + c + u * STEP, v[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float x[VEC];
                ld_vec<VEC, WG>(w + c + u * STEP, x);
#pragma unroll
                for (int i = 0; i < VEC; ++i) acc[i] += mavp_term<OP>(v[u][i], x[i]);
            }
        }
        for (; c < blk_end; c += STEP) {
            float v[VEC], x[VEC];
            ld_stream<VEC, POL>(a + c, v);
            ld_vec<VEC, WG>(w + c, x);
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc[i] += mavp_term<OP>(v[i], x[i]);
        }
        tot += tree_sum(acc);
    }
    // ragged tail (< STEP elements): scalar loads, at most VEC terms per lane
    float tail = 0.0f;
    for (int64_t k = n_main + lane; k < n; k += kWarp) {
        float v[1];
        ld_stream<1, POL>(a + k, v);
        tail += mavp_term<OP>(v[0], WG ? __ldg(w + k) : w[k]);
    }
    return warp_sum(tot + tail);
}

// ---------------------------------------------------------------------------------------------
// K1 standalone mat-vec: y = A (+) x.  Grid-stride over rows, one warp per row.
// WG = false: x staged in dynamic shared memory (n_cols floats); WG = true: x read via L1.
template <int OP, int VEC, int POL, bool WG, int U>
__global__ void __launch_bounds__(512, 1) k_matvec(const float* __restrict__ A, int64_t n_rows,
                                                int64_t n_cols, int64_t lda,
                                                const float* __restrict__ x, float* __restrict__ y) {
    extern __shared__ __align__(16) float xs[];
    const float* w = x;
    if constexpr (!WG) {
        for (int64_t k = threadIdx.x; k < n_cols; k += blockDim.x) xs[k] = x[k];
        __syncthreads();
        w = xs;
    }
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n_rows;
         row += warps) {
        float v = row_mavp<OP, VEC, POL, WG, U>(A + row * lda, w, n_cols, lane);
        if (lane == 0) y[row] = v;
    }
}

// ---------------------------------------------------------------------------------------------
// K1n: one fused Algorithm 1 step for a row block, given the previous FULL y (row-sharded path):
//   s = ||y_prev|| (l1; l2 for DOT; fp64, the same fixed order in every CTA and on every rank),
//   x = fp32(y_prev / s) staged into shared memory,  y_out = A_rows (op) x  (as K1),
//   CTA 0 also writes w_next = x, s_out, delta_out = ||x - w_prev||_1 and the status word.
template <int OP, int VEC, int POL, int U>
__global__ void __launch_bounds__(512, 1) k_matvec_norm(const float* __restrict__ A, int64_t n_rows, int64_t n_cols,
                                                        int64_t lda, const float* __restrict__ y_prev,
                                                        const float* __restrict__ w_prev, float* __restrict__ w_next,
                                                        float* __restrict__ y, float* s_out, float* delta_out,
                                                        int32_t* status) {
    extern __shared__ __align__(16) float xs[];
    __shared__ double red[33];
    double part = 0.0;
    for (int64_t k = threadIdx.x; k < n_cols; k += blockDim.x) part += norm_part<OP>(y_prev[k]);
    const double sd = norm_final<OP>(block_sum(part, red));
    if (!(sd > 0.0) || isinf(sd)) {  // uniform in every CTA
        if (blockIdx.x == 0 && threadIdx.x == 0 && status) *status = (sd == 0.0) ? kStDegenerate : kStNonfinite;
        return;
    }
    double dp = 0.0;
    for (int64_t k = threadIdx.x; k < n_cols; k += blockDim.x) {
        const float x = (float)((double)y_prev[k] / sd);
        xs[k] = x;
        if (blockIdx.x == 0) {
            dp += (double)fabsf(x - w_prev[k]);
            w_next[k] = x;
        }
    }
    if (blockIdx.x == 0) {
        const double d = block_sum(dp, red);
        if (threadIdx.x == 0) {
            if (s_out) *s_out = (float)sd;
            if (delta_out) *delta_out = (float)d;
            if (status) *status = kStOk;
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n_rows; row += warps) {
        const float v = row_mavp<OP, VEC, POL, false, U>(A + row * lda, xs, n_cols, lane);
        if (lane == 0) y[row] = v;
    }
}

// ---------------------------------------------------------------------------------------------
// K2 persistent MAPI iteration.
struct IterArgs {
    const float* A;
    int64_t n, lda;
    const float* b0;
    int32_t iters;
    float tol;
    float* w_out;      // n
    float* norms;      // iters or null
    float* deltas;     // iters or null
    float* y;          // 2*n (double-buffered by iteration parity)
    float* slots;      // 2*gridDim.x
    unsigned int* bar; // grid barrier counter (zeroed before launch)
    int32_t* status;   // [0] status, [1] iters_done
    // fused L2 deflation (K2r staging only; dk = 0 elsewhere): A_eff = C - sum_{m<dk} dP[m] dR[m]^T
    const double* dP = nullptr;  // dk x n
    const double* dR = nullptr;  // dk x n
    int32_t dk = 0;
    float* w_l2 = nullptr;       // K6t only: the final l2 copy written in-kernel (else k_l2_copy runs)
};


template <int OP, int VEC, int POL, int U, int PF = 0, int PH = 0, int MINB = 1>
__global__ void __launch_bounds__(512, MINB) k_iterate_persistent(IterArgs p) {
    extern __shared__ __align__(16) float ws_[];
    float* w_s = ws_;                                                    // n floats (w_t)
    double* red = reinterpret_cast<double*>(ws_ + ((p.n + 3) & ~int64_t(3)));  // 33 doubles
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int64_t n = p.n;

    for (int64_t k = tid; k < n; k += blockDim.x) w_s[k] = p.b0[k];
    __syncthreads();

    const int64_t gwarp = (int64_t)blockIdx.x * nw + warp;
    const int64_t total_warps = (int64_t)gridDim.x * nw;
    int32_t done = 0, status = kStOk;

    for (int32_t t = 0; t < p.iters; ++t) {
        float* y = p.y + (t & 1) * n;
        // ---- rows -> y, |y| partial (a1, a2)
        double abs_part = 0.0;
        for (int64_t row = gwarp; row < n; row += total_warps) {
            if constexpr (PH > 0) {  // warm L2 with the head of this warp's next row
                const int64_t nxt = row + total_warps;
                if (lane == 0 && nxt < n)
                    prefetch_l2(p.A + nxt * p.lda, (uint32_t)min((int64_t)PH * 1024, (n * 4) & ~int64_t(15)));
            }
            const float v = row_mavp<OP, VEC, POL, false, U, PF>(p.A + row * p.lda, w_s, n, lane);
            if (lane == 0) y[row] = v;
            abs_part += norm_part<OP>(v);
        }
        const double cta_abs = block_sum(lane == 0 ? abs_part : 0.0, red);
        double* slots = reinterpret_cast<double*>(p.slots);
        if (tid == 0) slots[(t & 1) * gridDim.x + blockIdx.x] = cta_abs;
        grid_barrier(p.bar, (unsigned int)(t + 1) * gridDim.x);

        // ---- s_t = ||y||_1 from the per-CTA partials, same fixed fp64 order in every CTA (a3)
        double s;
        {
            if (warp == 0) {
                double part = 0.0;
                for (int c = lane; c < (int)gridDim.x; c += 32) part += __ldcg(slots + (t & 1) * gridDim.x + c);
                part = warp_sum(part);
                if (lane == 0) red[32] = part;
            }
            __syncthreads();
            s = norm_final<OP>(red[32]);
            __syncthreads();
        }
        if (!(s > 0.0) || isinf(s)) {  // uniform across the grid (same s everywhere)
            status = (s == 0.0) ? kStDegenerate : kStNonfinite;
            break;
        }
        // ---- w_{t+1} = fp32(y / s_t) (division in fp64, a4), delta_t in fp64 (a5)
        double dpart = 0.0;
        for (int64_t k = tid; k < n; k += blockDim.x) {
            const float wn = (float)((double)ld_cg(y + k) / s);
            dpart += (double)fabsf(wn - w_s[k]);
            w_s[k] = wn;
        }
        const double delta = block_sum(dpart, red);  // also orders the w_s writes before reuse
        if (blockIdx.x == 0 && tid == 0) {
            if (p.norms) p.norms[t] = (float)s;
            if (p.deltas) p.deltas[t] = (float)delta;
        }
        done = t + 1;
        if (p.tol > 0.0f && delta < (double)p.tol) break;
    }
    // ---- final iterate out: CTA c writes its slice of its (identical) copy
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t k0 = (int64_t)blockIdx.x * per, k1 = min(n, k0 + per);
    for (int64_t k = k0 + tid; k < k1; k += blockDim.x) p.w_out[k] = w_s[k];
    if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
}

// ---------------------------------------------------------------------------------------------
// K2c: CTA-cooperative persistent MAPI iteration (the default dense path; K2).
//
// Rows are dealt to CTAs round-robin (row = cta + k*grid) and the NW warps of a CTA split every row
// into NW contiguous runs of 1 KB chunks, so at any moment the grid streams a compact window of
// ~grid consecutive rows (measured: 7.22 TB/s read ceiling for this pattern vs 7.00 TB/s for one
// row per warp scattered over the matrix).  Each warp's chunk loads (one LDG.256 per lane) are
// software-pipelined over its (row, chunk) sequence with a register double buffer, so row ends
// never drain the load queue, and the first load of iteration t+1 is issued before the grid
// barrier of iteration t (A does not depend on w).  Per row the NW warp partials go to shared
// memory and are summed in warp order after the rows loop.  The n % 256 ragged tail of each row is
// handled by the last warp with scalar loads.  Requires a 32 B-aligned A and lda % 8 == 0.
//
// Numerics: fp32 MAVP terms and row sums (per lane 8 chains of <= ceil(C/NW) terms, tree, butterfly,
// NW warp partials in order); s_t and delta_t are accumulated in fp64 (fixed order), and
// w_{t+1} = fp32(y / s_t) with the division in fp64, so w carries no common-mode rounding of s_t.
template <int OP, int POL, int NW, int D = 2>
__global__ void __launch_bounds__(NW * 32, 1) k_iterate_coop(IterArgs p) {
    constexpr int STEP = 256;  // floats per warp-wide LDG.256 (one 1 KB chunk)
    extern __shared__ __align__(16) float ws_[];
    const int64_t n = p.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t rows_cta = (n - blockIdx.x + gridDim.x - 1) / gridDim.x;  // rows c, c+G, ...
    float* w_s = ws_;                                                        // n (+pad) floats
    float* part = ws_ + ((n + 7) & ~int64_t(7));                             // rows_cta * NW
    double* red = reinterpret_cast<double*>(part + ((rows_cta * NW + 1) & ~int64_t(1)));  // 33 doubles
    const int64_t cfull = n / STEP;                     // full chunks per row
    const int c0 = (int)(warp * cfull / NW), c1 = (int)((warp + 1) * cfull / NW);
    const int spr = c1 - c0;                            // this warp's chunks per row
    const int nsteps = (int)rows_cta * spr;
    const int64_t tail0 = cfull * STEP;                 // ragged tail [tail0, n), last warp
    const bool has_tail = tail0 < n && warp == NW - 1;
    const int64_t rstride = (int64_t)gridDim.x * p.lda;
    const float* abase = p.A + (int64_t)blockIdx.x * p.lda + (int64_t)c0 * STEP + lane * 8;

    for (int64_t k = tid; k < n; k += blockDim.x) w_s[k] = p.b0[k];

    float buf[D][8], acc[8];  // register ring: D chunk loads in flight per warp
    int lr = 0, lq = 0;        // (row, chunk) of the next load
    auto load = [&](float (&b)[8]) {
        ld_stream<8, POL>(abase + lr * rstride + (int64_t)lq * STEP, b);
        if (++lq == spr) { lq = 0; ++lr; }
    };
    constexpr int D0 = D == 2 ? 1 : D;  // chunks pre-loaded ahead of the rows loop
#pragma unroll
    for (int j = 0; j < D0; ++j)
        if (j < nsteps) load(buf[j]);  // first loads of iteration 0 (overlap the w staging)
    __syncthreads();
    int32_t done = 0, status = kStOk;

    for (int32_t t = 0; t < p.iters; ++t) {
        float* y = p.y + (t & 1) * n;
        int cr = 0, cq = 0;  // (row, chunk) of the next consume
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        auto finish_row = [&]() {
            float v = tree_sum(acc);
            if (has_tail) {  // n % 256 elements of row (blockIdx.x + cr*G), scalar
                const float* a = p.A + ((int64_t)blockIdx.x + (int64_t)cr * gridDim.x) * p.lda;
                for (int64_t k = tail0 + lane; k < n; k += 32) {
                    float x[1];
                    ld_stream<1, POL>(a + k, x);
                    v += mavp_term<OP>(x[0], w_s[k]);
                }
            }
            v = warp_sum(v);
            if (lane == 0) part[cr * NW + warp] = v;
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        };
        auto consume = [&](const float (&b)[8]) {
            float x[8];
            ld_vec<8, false>(w_s + (int64_t)(c0 + cq) * STEP + lane * 8, x);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] += mavp_term<OP>(b[i], x[i]);
            if (++cq == spr) {
                finish_row();
                cq = 0;
                ++cr;
            }
        };
        // ---- rows (a1, a2): buf[0..D) already hold steps 0..D-1; step s lives in buf[s % D]
        if constexpr (D == 2) {  // explicit double buffer (measured faster than the generic ring)
            // here only buf[0] holds step 0; buf[1] is loaded just ahead of each consume
            int s = 0;
            for (; s + 1 < nsteps; s += 2) {
                load(buf[1]);
                consume(buf[0]);
                if (s + 2 < nsteps) load(buf[0]);
                consume(buf[1]);
            }
            if (s < nsteps) consume(buf[0]);
        } else {
            for (int s = 0; s < nsteps; s += D) {
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    if (s + j < nsteps) {
                        consume(buf[j]);
                        if (s + j + D < nsteps) load(buf[j]);
                    }
                }
            }
        }
        if (spr == 0)  // no full chunk for this warp: zero partials (+ the tail if it owns it)
            for (cr = 0; cr < (int)rows_cta; ++cr) finish_row();
        lr = 0;
        lq = 0;
        if (t + 1 < p.iters)  // next iteration's first chunks, in flight across the barrier
#pragma unroll
            for (int j = 0; j < D0; ++j)
                if (j < nsteps) load(buf[j]);
        __syncthreads();
        // ---- y rows of this CTA (NW partials in warp order), fp64 |y| partial (a3)
        double abs_part = 0.0;
        for (int64_t r = tid; r < rows_cta; r += blockDim.x) {
            float v = 0.0f;
#pragma unroll 8
            for (int q = 0; q < NW; ++q) v += part[r * NW + q];
            y[blockIdx.x + r * gridDim.x] = v;
            abs_part += norm_part<OP>(v);
        }
        const double cta_abs = block_sum(abs_part, red);
        double* slots = reinterpret_cast<double*>(p.slots);
        if (tid == 0) slots[(t & 1) * gridDim.x + blockIdx.x] = cta_abs;
        grid_barrier(p.bar, (unsigned int)(t + 1) * gridDim.x);
        // ---- s_t: the same fixed-order fp64 sum in every CTA
        double sd;
        {
            if (warp == 0) {
                double pp = 0.0;
                for (int c = lane; c < (int)gridDim.x; c += 32) pp += __ldcg(slots + (t & 1) * gridDim.x + c);
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
        // ---- w_{t+1} = y / s_t (a4), delta_t (a5), staged into this CTA's shared memory
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
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t k0 = (int64_t)blockIdx.x * per, k1 = min(n, k0 + per);
    for (int64_t k = k0 + tid; k < k1; k += blockDim.x) p.w_out[k] = w_s[k];
    if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
}

inline size_t coop_smem_bytes(int64_t n, int grid, int nw) {
    const int64_t rows_cta = (n + grid - 1) / grid;
    return sizeof(float) * (size_t)(((n + 7) & ~int64_t(7)) + ((rows_cta * nw + 1) & ~int64_t(1))) +
           sizeof(double) * 33;
}

// ---------------------------------------------------------------------------------------------
// K6: small-n MAPI in ONE thread-block cluster of kClusterCtas CTAs (latency-bound case, cfg1).
// CTA r of the cluster stages rows [r*R, (r+1)*R) of A into its shared memory once; every iteration
// each CTA computes its y rows (warp per row, lane-strided columns, butterfly), pushes each y_j into
// the y buffer of every CTA of the cluster with DSMEM stores (st.shared::cluster), and one cluster
// barrier (release/acquire) publishes them.  Each CTA then forms s_t, w_{t+1} = fp32(y/s_t) and
// delta_t in the same fixed fp64 order (identical in all CTAs).  y is double-buffered by parity.
constexpr int kClusterCtas = 8;
constexpr int kClusterThreads = 1024;

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store v to the same shared-memory offset as `local` in CTA `rank` of this cluster
__device__ __forceinline__ void st_cluster(float* local, uint32_t rank, float v) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
}

__host__ __device__ inline int64_t cluster_rows_per_cta(int64_t n) { return (n + kClusterCtas - 1) / kClusterCtas; }
__host__ __device__ inline int64_t cluster_ld(int64_t n) { return (n + 255) & ~int64_t(255); }  // zero-padded rows
inline size_t cluster_smem_bytes(int64_t n) {
    const int64_t R = cluster_rows_per_cta(n), np = cluster_ld(n);
    return sizeof(float) * (size_t)(R * np + 3 * np);
}

// Row r of this CTA against w: lane-contiguous 8-column chunks (LDS.128 x 2 each), tree, butterfly.
template <int OP>
__device__ __forceinline__ float cluster_row(const float* __restrict__ a, const float* __restrict__ w, int64_t np,
                                             int lane) {
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
    for (int64_t c = lane * 8; c < np; c += 256) {
        float x[8], v[8];
        ld_vec<8, false>(a + c, v);
        ld_vec<8, false>(w + c, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += mavp_term<OP>(v[i], x[i]);
    }
    return warp_sum(tree_sum(acc));
}

template <int OP>
__global__ void __launch_bounds__(kClusterThreads, 1) k_iterate_cluster(IterArgs p) {
    extern __shared__ __align__(16) float sm[];
    const int64_t n = p.n, np = cluster_ld(n);
    const int64_t R = cluster_rows_per_cta(n);
    float* As = sm;              // R x np, zero padded (padding terms are exactly 0)
    float* w_s = sm + R * np;    // np, zero padded
    float* ybuf = w_s + np;      // 2 x np
    const uint32_t rank = cluster_ctarank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kClusterThreads / 32;
    const int64_t r0 = (int64_t)rank * R, r1 = min(n, r0 + R);
    for (int64_t q = tid; q < R * np; q += kClusterThreads) {
        const int64_t r = q / np, c = q - r * np;
        As[q] = (r0 + r < n && c < n) ? p.A[(r0 + r) * p.lda + c] : 0.0f;
    }
    for (int64_t k = tid; k < np; k += kClusterThreads) w_s[k] = k < n ? p.b0[k] : 0.0f;
    cluster_sync_all();  // every CTA resident and staged before any DSMEM store
    int32_t done = 0, status = kStOk;
    __shared__ int32_t s_flag[2];
    for (int32_t t = 0; t < p.iters; ++t) {
        float* yb = ybuf + (t & 1) * np;
        for (int64_t r = r0 + warp; r < r1; r += nw) {
            const float v = cluster_row<OP>(As + (r - r0) * np, w_s, np, lane);
            if (lane < kClusterCtas) st_cluster(yb + r, (uint32_t)lane, v);
        }
        cluster_sync_all();
        // epilogue by warp 0 (fixed order, identical in every CTA): s_t, w_{t+1}, delta_t
        if (warp == 0) {
            double ap = 0.0;
            for (int64_t k = lane; k < n; k += 32) ap += norm_part<OP>(yb[k]);
            const double sd = norm_final<OP>(warp_sum(ap));
            int st = kStOk;
            if (!(sd > 0.0) || isinf(sd)) st = (sd == 0.0) ? kStDegenerate : kStNonfinite;
            double dp = 0.0;
            if (st == kStOk)
                for (int64_t k = lane; k < n; k += 32) {
                    const float wn = (float)((double)yb[k] / sd);
                    dp += (double)fabsf(wn - w_s[k]);
                    w_s[k] = wn;
                }
            const double delta = warp_sum(dp);
            if (lane == 0) {
                s_flag[0] = st;
                s_flag[1] = (st == kStOk && p.tol > 0.0f && delta < (double)p.tol) ? 1 : 0;
                if (rank == 0 && st == kStOk) {
                    if (p.norms) p.norms[t] = (float)sd;
                    if (p.deltas) p.deltas[t] = (float)delta;
                }
            }
        }
        __syncthreads();
        if (s_flag[0] != kStOk) {
            status = s_flag[0];
            break;
        }
        done = t + 1;
        if (s_flag[1]) break;
    }
    for (int64_t k = r0 + tid; k < r1; k += kClusterThreads) p.w_out[k] = w_s[k];
    if (rank == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
    cluster_sync_all();  // keep every CTA's shared memory alive until all DSMEM stores landed
}

// K6r: the same cluster iteration with the CTA's rows held in REGISTERS (n <= 512: a warp owns
// RW = NPT rows, a lane 8 * NPT columns of each — 8 or 32 registers), so an iteration reads only w
// from shared memory (the smem version spent ~1700 of its ~5500 cycles per iteration queueing the
// 64 KB of A + w reads on the shared-memory pipe; scripts/probe_k6.cu).  The epilogue is spread
// over the CTA instead of warp 0 (which spent ~2300 cycles on 8 dependent fp64 divisions per lane):
// every warp forms s_t itself from the broadcast y (same fixed order everywhere), thread k forms
// w_k = fp32(y_k / s_t) and its |delta| term, the warps' delta partials meet in shared memory, and
// after the one __syncthreads every warp sums them in warp order -> the stop decision is uniform
// without a second barrier.  Same per-row summation order as K6 (bitwise-identical w; the fp64
// delta is summed in a different order).
// Alternative y hand-off, off by default (measured slower: 2.42 vs 2.03 us/iteration at n = 256,
// 4.19 vs 3.68 at n = 500): instead of a full cluster barrier (MAPI_K6_MBAR=1), each warp, after its DSMEM stores of
// y, arrives (release.cluster, lane L -> CTA L) on the destination CTA's mbarrier for this iteration
// parity; a CTA waits (acquire.cluster) for the 8 x 32 warp arrivals.  Two barriers alternate by
// iteration, so arrivals of iteration t+1 never mix with t (a CTA can only be one iteration ahead
// of the slowest one: it needs that CTA's arrivals to leave the current iteration).
#ifndef MAPI_K6_MBAR
#define MAPI_K6_MBAR 0
#endif
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* local_bar, uint32_t rank) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(local_bar);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}

template <int OP, int NPT>
__global__ void __launch_bounds__(kClusterThreads, 1) k_iterate_cluster_reg(IterArgs p) {
    constexpr int NP = 256 * NPT, RW = NPT, CPL = 8 * NPT;
    __shared__ __align__(16) float w_s[NP];
    __shared__ __align__(16) float ybuf[2][NP];
    __shared__ double dpart[kClusterThreads / 32];
    __shared__ __align__(8) uint64_t ybar[2];
    const int64_t n = p.n;
    const int64_t R = cluster_rows_per_cta(n);
    const uint32_t rank = cluster_ctarank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = (int64_t)rank * R, r1 = min(n, r0 + R);
    const int nwd = (int)((n + 31) / 32);  // warps holding a delta partial
    float a[RW][CPL];
#pragma unroll
    for (int j = 0; j < RW; ++j) {
        const int64_t r = r0 + warp + 32 * j;
#pragma unroll
        for (int k = 0; k < NPT; ++k)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t c = (int64_t)lane * 8 + 256 * k + i;
                a[j][8 * k + i] = (r < r1 && c < n) ? p.A[r * p.lda + c] : 0.0f;
            }
    }
    for (int k = tid; k < NP; k += kClusterThreads) w_s[k] = k < n ? p.b0[k] : 0.0f;
    for (int k = tid; k < 2 * NP; k += kClusterThreads) (&ybuf[0][0])[k] = 0.0f;
    if (MAPI_K6_MBAR && tid == 0) {
        const uint32_t b0a = (uint32_t)__cvta_generic_to_shared(&ybar[0]);
        const uint32_t b1a = (uint32_t)__cvta_generic_to_shared(&ybar[1]);
        const uint32_t cnt = kClusterCtas * (kClusterThreads / 32);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b0a), "r"(cnt) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b1a), "r"(cnt) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync_all();  // every CTA resident and staged before any DSMEM store
    int32_t done = 0, status = kStOk;
    for (int32_t t = 0; t < p.iters; ++t) {
        float* yb = ybuf[t & 1];
#pragma unroll
        for (int j = 0; j < RW; ++j) {
            const int64_t r = r0 + warp + 32 * j;
            float acc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                float x[8];
                ld_vec<8, false>(w_s + lane * 8 + 256 * k, x);
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] += mavp_term<OP>(a[j][8 * k + i], x[i]);
            }
            const float v = warp_sum(tree_sum(acc));
            if (r < r1 && lane < kClusterCtas) st_cluster(yb + r, (uint32_t)lane, v);
        }
#if MAPI_K6_MBAR
        if (lane < kClusterCtas) mbar_arrive_remote(&ybar[t & 1], (uint32_t)lane);
        mbar_wait_cluster(&ybar[t & 1], (uint32_t)((t >> 1) & 1));
#else
        cluster_sync_all();
#endif
        // s_t: every warp, same fixed order (lane-strided fp64 partials, butterfly)
        double ap = 0.0;
        for (int64_t k = lane; k < n; k += 32) ap += norm_part<OP>(yb[k]);
        const double sd = norm_final<OP>(warp_sum(ap));
        if (!(sd > 0.0) || isinf(sd)) {  // uniform across the cluster
            status = (sd == 0.0) ? kStDegenerate : kStNonfinite;
            break;
        }
        // w_{t+1} = fp32(y / s_t) (fp64 division), one element per thread; delta partial per warp
        double dp = 0.0;
        if (tid < n) {
            const float wn = (float)((double)yb[tid] / sd);
            dp = (double)fabsf(wn - w_s[tid]);
            w_s[tid] = wn;
        }
        dp = warp_sum(dp);
        if (lane == 0 && warp < nwd) dpart[warp] = dp;
        __syncthreads();
        double delta = 0.0;
        for (int q = 0; q < nwd; ++q) delta += dpart[q];
        if (rank == 0 && tid == 0) {
            if (p.norms) p.norms[t] = (float)sd;
            if (p.deltas) p.deltas[t] = (float)delta;
        }
        done = t + 1;
        if (p.tol > 0.0f && delta < (double)p.tol) break;
    }
    for (int64_t k = r0 + tid; k < r1; k += kClusterThreads) p.w_out[k] = w_s[k];
    if (rank == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
    cluster_sync_all();  // keep every CTA's shared memory alive until all DSMEM stores landed
}

// ---------------------------------------------------------------------------------------------
// Multi-launch path (any n; also the CUDA-graph-style comparator): per iteration
//   k_rows_partial: y = A (+) w (w in global, L1-cached), per-CTA sum|y| -> slots
//   k_normalize   : 1 CTA; s = sum slots; w = y/s; delta; trace; stop flag
// Both kernels return immediately once the device stop flag is set.
template <int OP, int VEC, int POL, int U>
__global__ void __launch_bounds__(512, 1) k_rows_partial(const float* __restrict__ A, int64_t n,
                                                      int64_t lda, const float* __restrict__ w,
                                                      float* __restrict__ y, float* __restrict__ slots,
                                                      const int32_t* __restrict__ stop) {
    __shared__ double red[33];
    if (*(volatile const int32_t*)stop) return;
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int64_t total_warps = (int64_t)gridDim.x * nw;
    double abs_part = 0.0;
    for (int64_t row = (int64_t)blockIdx.x * nw + (threadIdx.x >> 5); row < n; row += total_warps) {
        const float v = row_mavp<OP, VEC, POL, true, U>(A + row * lda, w, n, lane);
        if (lane == 0) y[row] = v;
        abs_part += norm_part<OP>(v);
    }
    const double cta_abs = block_sum(lane == 0 ? abs_part : 0.0, red);
    if (threadIdx.x == 0) reinterpret_cast<double*>(slots)[blockIdx.x] = cta_abs;
}

__global__ void __launch_bounds__(1024) k_normalize(int64_t n, const float* __restrict__ y,
                                                    const float* __restrict__ slots, int n_slots,
                                                    float* __restrict__ w, int32_t t, float tol,
                                                    float* norms, float* deltas, int32_t* status,
                                                    int32_t* stop, int l2) {
    __shared__ double red[33];
    if (*(volatile int32_t*)stop) return;
    const double* dslots = reinterpret_cast<const double*>(slots);
    if (threadIdx.x < 32) {
        double part = 0.0;
        for (int c = threadIdx.x; c < n_slots; c += 32) part += dslots[c];
        part = warp_sum(part);
        if (threadIdx.x == 0) red[32] = part;
    }
    __syncthreads();
    const double s = l2 ? sqrt(red[32]) : red[32];
    __syncthreads();
    if (!(s > 0.0) || isinf(s)) {
        if (threadIdx.x == 0) {
            status[0] = (s == 0.0) ? kStDegenerate : kStNonfinite;
            status[1] = t;
            *stop = 1;
        }
        return;
    }
    double dpart = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const float wn = (float)((double)y[k] / s);
        dpart += (double)fabsf(wn - w[k]);
        w[k] = wn;
    }
    const double delta = block_sum(dpart, red);
    if (threadIdx.x == 0) {
        if (norms) norms[t] = (float)s;
        if (deltas) deltas[t] = (float)delta;
        status[1] = t + 1;
        if (tol > 0.0f && delta < (double)tol) *stop = 1;
    }
}

// ---------------------------------------------------------------------------------------------
// Stand-alone normalisation step (row-sharded path): one CTA, fixed order, fp64 reductions.
__global__ void __launch_bounds__(1024) k_normalize_full(int64_t n, const float* __restrict__ y, float* __restrict__ w,
                                                         int l2, float* s_out, float* delta_out, int32_t* status) {
    __shared__ double red[33];
    double part = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const double v = (double)y[k];
        part += l2 ? v * v : fabs(v);
    }
    double s = block_sum(part, red);
    if (l2) s = sqrt(s);
    if (!(s > 0.0) || isinf(s)) {
        if (threadIdx.x == 0) {
            if (status) *status = (s == 0.0) ? kStDegenerate : kStNonfinite;
            if (s_out) *s_out = (float)s;
        }
        return;
    }
    double dp = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const float wn = (float)((double)y[k] / s);
        dp += (double)fabsf(wn - w[k]);
        w[k] = wn;
    }
    const double d = block_sum(dp, red);
    if (threadIdx.x == 0) {
        if (status) *status = kStOk;
        if (s_out) *s_out = (float)s;
        if (delta_out) *delta_out = (float)d;
    }
}

// ---------------------------------------------------------------------------------------------
// Optional final l2 copy (Alg. 1 line 6): the n multiplies of the whole run, once.
// One CTA, fixed order.  Works on `rows` independent vectors of length n (vector-major).
__global__ void __launch_bounds__(1024) k_l2_copy(int64_t n, const float* __restrict__ w,
                                                  float* __restrict__ out) {
    __shared__ float red[33];
    const float* wv = w + (int64_t)blockIdx.x * n;
    float* ov = out + (int64_t)blockIdx.x * n;
    float part = 0.0f;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) part += wv[k] * wv[k];
    const float l2 = sqrtf(block_sum(part, red));
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) ov[k] = l2 > 0.0f ? wv[k] / l2 : 0.0f;
}

}  // namespace mapi
