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

// Row MAVP: sum_k a[k] (+) w[k] for k < n, by one warp. Returns the same value in all lanes.
// a must be VEC*4-byte aligned; w (smem or global) likewise.
template <int OP, int VEC, int POL, bool WG, int U>
__device__ __forceinline__ float row_mavp(const float* __restrict__ a, const float* __restrict__ w,
                                          int64_t n, int lane) {
    constexpr int STEP = kWarp * VEC;
    const int64_t n_main = (n / STEP) * STEP;
    float tot[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) tot[i] = 0.0f;

    for (int64_t blk = 0; blk < n_main; blk += (int64_t)kFold * STEP) {
        const int64_t blk_end = min(n_main, blk + (int64_t)kFold * STEP);
        float acc[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc[i] = 0.0f;
        int64_t c = blk + lane * VEC;
        const int64_t base_end = blk_end - (int64_t)(U - 1) * STEP;  // warp-uniform bound
        for (; c - lane * VEC < base_end; c += (int64_t)U * STEP) {
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
#pragma unroll
        for (int i = 0; i < VEC; ++i) tot[i] += acc[i];
    }
    // ragged tail (< STEP elements): scalar loads, at most VEC terms per lane
    float tail = 0.0f;
    for (int64_t k = n_main + lane; k < n; k += kWarp) {
        float v[1];
        ld_stream<1, POL>(a + k, v);
        tail += mavp_term<OP>(v[0], WG ? __ldg(w + k) : w[k]);
    }
    return warp_sum(tree_sum(tot) + tail);
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
};

// status codes (mirror mapi_status)
constexpr int kStOk = 0, kStDegenerate = 4, kStNonfinite = 6;

template <int OP, int VEC, int POL, int U>
__global__ void __launch_bounds__(512, 1) k_iterate_persistent(IterArgs p) {
    extern __shared__ __align__(16) float ws_[];
    float* w_s = ws_;                                // n floats (the current iterate w_t)
    float* red = ws_ + ((p.n + 3) & ~int64_t(3));    // 33 floats of reduction scratch
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
        float abs_part = 0.0f;
        for (int64_t row = gwarp; row < n; row += total_warps) {
            const float v = row_mavp<OP, VEC, POL, false, U>(p.A + row * p.lda, w_s, n, lane);
            if (lane == 0) y[row] = v;
            abs_part += fabsf(v);
        }
        const float cta_abs = block_sum(lane == 0 ? abs_part : 0.0f, red);
        if (tid == 0) p.slots[(t & 1) * gridDim.x + blockIdx.x] = cta_abs;
        grid_barrier(p.bar, (unsigned int)(t + 1) * gridDim.x);

        // ---- s_t = ||y||_1 from the per-CTA partials, same fixed order in every CTA (a3)
        float s;
        {
            float part = 0.0f;
            if (warp == 0)
                for (int c = lane; c < (int)gridDim.x; c += 32)
                    part += ld_cg(p.slots + (t & 1) * gridDim.x + c);
            if (warp == 0) {
                part = warp_sum(part);
                if (lane == 0) red[32] = part;
            }
            __syncthreads();
            s = red[32];
            __syncthreads();
        }
        if (!(s > 0.0f) || isinf(s)) {  // uniform across the grid (same s everywhere)
            status = (s == 0.0f) ? kStDegenerate : kStNonfinite;
            break;
        }
        // ---- w_{t+1} = y / s_t (IEEE division, a4), delta_t (a5)
        float dpart = 0.0f;
        for (int64_t k = tid; k < n; k += blockDim.x) {
            const float wn = ld_cg(y + k) / s;
            dpart += fabsf(wn - w_s[k]);
            w_s[k] = wn;
        }
        const float delta = block_sum(dpart, red);  // also orders the w_s writes before reuse
        if (blockIdx.x == 0 && tid == 0) {
            if (p.norms) p.norms[t] = s;
            if (p.deltas) p.deltas[t] = delta;
        }
        done = t + 1;
        if (p.tol > 0.0f && delta < p.tol) break;
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
// Multi-launch path (any n; also the CUDA-graph-style comparator): per iteration
//   k_rows_partial: y = A (+) w (w in global, L1-cached), per-CTA sum|y| -> slots
//   k_normalize   : 1 CTA; s = sum slots; w = y/s; delta; trace; stop flag
// Both kernels return immediately once the device stop flag is set.
template <int OP, int VEC, int POL, int U>
__global__ void __launch_bounds__(512, 1) k_rows_partial(const float* __restrict__ A, int64_t n,
                                                      int64_t lda, const float* __restrict__ w,
                                                      float* __restrict__ y, float* __restrict__ slots,
                                                      const int32_t* __restrict__ stop) {
    __shared__ float red[33];
    if (*(volatile const int32_t*)stop) return;
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int64_t total_warps = (int64_t)gridDim.x * nw;
    float abs_part = 0.0f;
    for (int64_t row = (int64_t)blockIdx.x * nw + (threadIdx.x >> 5); row < n; row += total_warps) {
        const float v = row_mavp<OP, VEC, POL, true, U>(A + row * lda, w, n, lane);
        if (lane == 0) y[row] = v;
        abs_part += fabsf(v);
    }
    const float cta_abs = block_sum(lane == 0 ? abs_part : 0.0f, red);
    if (threadIdx.x == 0) slots[blockIdx.x] = cta_abs;
}

__global__ void __launch_bounds__(1024) k_normalize(int64_t n, const float* __restrict__ y,
                                                    const float* __restrict__ slots, int n_slots,
                                                    float* __restrict__ w, int32_t t, float tol,
                                                    float* norms, float* deltas, int32_t* status,
                                                    int32_t* stop) {
    __shared__ float red[33];
    if (*(volatile int32_t*)stop) return;
    float part = 0.0f;
    if (threadIdx.x < 32)
        for (int c = threadIdx.x; c < n_slots; c += 32) part += slots[c];
    if (threadIdx.x < 32) {
        part = warp_sum(part);
        if (threadIdx.x == 0) red[32] = part;
    }
    __syncthreads();
    const float s = red[32];
    __syncthreads();
    if (!(s > 0.0f) || isinf(s)) {
        if (threadIdx.x == 0) {
            status[0] = (s == 0.0f) ? kStDegenerate : kStNonfinite;
            status[1] = t;
            *stop = 1;
        }
        return;
    }
    float dpart = 0.0f;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const float wn = y[k] / s;
        dpart += fabsf(wn - w[k]);
        w[k] = wn;
    }
    const float delta = block_sum(dpart, red);
    if (threadIdx.x == 0) {
        if (norms) norms[t] = s;
        if (deltas) deltas[t] = delta;
        status[1] = t + 1;
        if (tol > 0.0f && delta < tol) *stop = 1;
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
