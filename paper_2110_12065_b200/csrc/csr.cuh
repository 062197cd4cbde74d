// csr.cuh — K7 (Google-matrix preparation) and K3 (CSR MAPI ranking step) for sm_100a.
//
// Eq.(13), reading Q10: G = alpha M + (1-alpha)/n 1, M_ij = 1/outdeg(j) for each
// distinct edge j -> i, dangling columns of M uniform 1/n.  The iterate stays w >= 0, so every
// min1 term is min(G_ij, w_j).  Writing G_ij = bg_j + [j -> i] cap_j with
//     bg_j  = (1-alpha)/n (1/n if j dangling),   cap_j = alpha/outdeg(j)  (0 if dangling),
// the row product is EXACTLY (real arithmetic, pinned in the oracle tests)
//     y_i = S + sum_{j -> i} v_j,   S = sum_j min(bg_j, w_j),   v_j = min(max(w_j - bg_j, 0), cap_j)
// because min(bg + cap, w) - min(bg, w) = min(max(w - bg, 0), cap).  Per iteration that is
//   K3a (columns, n):  v_j, per-CTA partials of S            (fused into the previous normalise)
//   K3b (rows, nnz):   y_i = S + gather-sum of v over row i, per-CTA partials of sum y
//   K3c (columns, n):  s = ||y||_1, w = y / s, delta partials, next v_j and S partials
//   K3d (1 CTA):       delta_t, trace, stop flag
// No multiplication anywhere in the step; the only divisions are w = y / s.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdio>
#include "../../include/mapi.h"
#include "mapi_common.cuh"

namespace mapi {

constexpr int kCsrThreads = 256;
constexpr int kCsrMaxGrid = 2048;

inline size_t cal256(size_t b) { return (b + 255) & ~size_t(255); }

static thread_local char g_csr_err[256] = "";
inline const char* csr_last_error() { return g_csr_err; }
inline mapi_status csr_cuda_fail(cudaError_t e, const char* what) {
    snprintf(g_csr_err, sizeof(g_csr_err), "%s: %s", what, cudaGetErrorString(e));
    return MAPI_ERR_CUDA;
}

// ------------------------------------------------------------------------------- K7 prepare
inline size_t csr_prepare_ws_bytes(int64_t n, int64_t /*nnz*/) { return cal256(4 * (size_t)n); }

__global__ void k_outdeg(int64_t nnz, const int32_t* __restrict__ col_idx, int32_t* __restrict__ outdeg) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(outdeg + col_idx[e], 1);  // integer histogram: order-independent
}

__global__ void k_cap_bg(int64_t n, float alpha, const int32_t* __restrict__ outdeg, float* __restrict__ cap,
                         float* __restrict__ bg) {
    const float bg_link = (1.0f - alpha) / (float)n, bg_dangling = 1.0f / (float)n;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int32_t d = outdeg[j];
        cap[j] = d > 0 ? alpha / (float)d : 0.0f;
        bg[j] = d > 0 ? bg_link : bg_dangling;
    }
}

inline mapi_status csr_prepare_run(int64_t n, int64_t nnz, const int32_t* /*row_ptr*/, const int32_t* col_idx,
                                   float alpha, float* cap, float* bg, void* ws, int sms, cudaStream_t s,
                                   std::atomic<uint64_t>& launches) {
    int32_t* outdeg = static_cast<int32_t*>(ws);
    cudaError_t e = cudaMemsetAsync(outdeg, 0, 4 * (size_t)n, s);
    if (e != cudaSuccess) return csr_cuda_fail(e, "memset");
    if (nnz > 0) {
        k_outdeg<<<4 * sms, 512, 0, s>>>(nnz, col_idx, outdeg);
        launches.fetch_add(1, std::memory_order_relaxed);
    }
    k_cap_bg<<<4 * sms, 512, 0, s>>>(n, alpha, outdeg, cap, bg);
    launches.fetch_add(1, std::memory_order_relaxed);
    if ((e = cudaGetLastError()) != cudaSuccess) return csr_cuda_fail(e, "prepare launch");
    return MAPI_OK;
}

// ------------------------------------------------------------------------------- K3 rank
// Numerics (K3): the per-edge gather e_i = sum v_j runs in fp32; the per-node state
// (w, S, y_i = S + e_i, s = ||y||_1, w = y / s, delta) is fp64.  Reason: at n = 2^22 the iterate
// entries are ~2.4e-7 and y_i = S + e_i is dominated by the common background S ~ 0.6, so an fp32
// state has a delta noise floor of ~1e-7 (the BASELINE tol) and would decide the stopping iteration
// by rounding noise; the paper computes in double (MATLAB).  Cost: +~70 MB/iteration of node traffic.
//
// workspace: [hdr 256: status[2] @0, stop @8][w n f64][e n f32][v n f32]
//            [slotS 2*G f64][slotY G f64][slotD G f64]
struct CsrWs {
    int32_t* status;
    int32_t* stop;
    double* w;
    float *e, *v;
    double *slotS, *slotY, *slotD;
};

inline size_t csr_rank_ws_bytes(int64_t n, int64_t /*nnz*/) {
    return 256 + cal256(8 * (size_t)n) + 2 * cal256(4 * (size_t)n) + 4 * cal256(8 * (size_t)kCsrMaxGrid);
}

inline CsrWs carve_csr(void* ws, int64_t n) {
    char* p = static_cast<char*>(ws);
    CsrWs c;
    c.status = reinterpret_cast<int32_t*>(p);
    c.stop = reinterpret_cast<int32_t*>(p + 8);
    p += 256;
    c.w = reinterpret_cast<double*>(p);
    p += cal256(8 * (size_t)n);
    c.e = reinterpret_cast<float*>(p);
    p += cal256(4 * (size_t)n);
    c.v = reinterpret_cast<float*>(p);
    p += cal256(4 * (size_t)n);
    c.slotS = reinterpret_cast<double*>(p);
    p += 2 * cal256(8 * (size_t)kCsrMaxGrid);
    c.slotY = reinterpret_cast<double*>(p);
    p += cal256(8 * (size_t)kCsrMaxGrid);
    c.slotD = reinterpret_cast<double*>(p);
    return c;
}

// v_j = min(max(w_j - bg_j, 0), cap_j) = min(bg+cap, w) - min(bg, w)   (exact identity, F7)
__device__ __forceinline__ float csr_v(double w, float bg, float cap) {
    return (float)fmin(fmax(w - (double)bg, 0.0), (double)cap);
}

// sum of the first `count` fp64 slots in a fixed order (warp 0 lane-strided, then butterfly)
__device__ __forceinline__ double slots_sum(const double* slots, int count, double* red) {
    if (threadIdx.x < 32) {
        double part = 0.0;
        for (int c = threadIdx.x; c < count; c += 32) part += slots[c];
        part = warp_sum(part);
        if (threadIdx.x == 0) red[32] = part;
    }
    __syncthreads();
    const double r = red[32];
    __syncthreads();
    return r;
}

// K3a at t = 0: w = b0 (checked >= 0), v_j, S partials (slot parity 0).
__global__ void __launch_bounds__(kCsrThreads) k_rank_init(int64_t n, const float* __restrict__ b0,
                                                           const float* __restrict__ bg, const float* __restrict__ cap,
                                                           double* __restrict__ w, float* __restrict__ v,
                                                           double* __restrict__ slotS, int32_t* status, int32_t* stop) {
    __shared__ double red[33];
    double sp = 0.0;
    bool neg = false;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double wj = (double)b0[j];
        neg |= wj < 0.0;
        w[j] = wj;
        const float b = bg[j];
        v[j] = csr_v(wj, b, cap[j]);
        sp += fmin((double)b, wj);
    }
    if (neg) {
        status[0] = 5;
        *stop = 1;
    }
    const double S = block_sum(sp, red);
    if (threadIdx.x == 0) slotS[blockIdx.x] = S;
}

// K3b: e_i = sum_{e in row i} v[col_idx[e]] (fp32 gather, one warp per row); fp64 partials of
// sum_i y_i = sum_i (S + e_i) (= ||y||_1, all terms >= 0).
__global__ void __launch_bounds__(kCsrThreads) k_rank_rows(int64_t n, const int32_t* __restrict__ row_ptr,
                                                           const int32_t* __restrict__ col_idx,
                                                           const float* __restrict__ v, const double* __restrict__ slotS,
                                                           int nslots, float* __restrict__ e, double* __restrict__ slotY,
                                                           const int32_t* stop) {
    __shared__ double red[33];
    if (*(volatile const int32_t*)stop) return;
    const double S = slots_sum(slotS, nslots, red);
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    double ypart = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
        const int32_t e0 = row_ptr[i], e1 = row_ptr[i + 1];
        float acc = 0.0f;
        for (int32_t k = e0 + lane; k < e1; k += 32) acc += __ldg(v + col_idx[k]);
        acc = warp_sum(acc);
        if (lane == 0) {
            e[i] = acc;
            ypart += S + (double)acc;
        }
    }
    const double Y = block_sum(ypart, red);
    if (threadIdx.x == 0) slotY[blockIdx.x] = Y;
}

// K3c: s = ||y||_1, w_new = (S + e_j) / s (fp64), delta partials; next v_j and S partials.
__global__ void __launch_bounds__(kCsrThreads) k_rank_normalize(int64_t n, const float* __restrict__ e,
                                                                const double* __restrict__ slotS_cur,
                                                                double* __restrict__ slotS_next, int nS,
                                                                const double* __restrict__ slotY, int nY,
                                                                const float* __restrict__ bg,
                                                                const float* __restrict__ cap, double* __restrict__ w,
                                                                float* __restrict__ v, double* __restrict__ slotD,
                                                                const int32_t* stop) {
    __shared__ double red[33];
    if (*(volatile const int32_t*)stop) return;
    const double S = slots_sum(slotS_cur, nS, red);
    const double s = slots_sum(slotY, nY, red);
    double dp = 0.0, sp = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double wn = (S + (double)e[j]) / s;
        dp += fabs(wn - w[j]);
        w[j] = wn;
        const float b = bg[j];
        v[j] = csr_v(wn, b, cap[j]);
        sp += fmin((double)b, wn);
    }
    const double D = block_sum(dp, red);
    const double Sn = block_sum(sp, red);
    if (threadIdx.x == 0) {
        slotD[blockIdx.x] = D;
        slotS_next[blockIdx.x] = Sn;
    }
}

// K3d: delta_t, trace, status, stop.
__global__ void k_rank_step_end(const double* __restrict__ slotY, int ny, const double* __restrict__ slotD, int nd,
                                int32_t t, float tol, float* deltas, int32_t* status, int32_t* stop) {
    __shared__ double red[33];
    if (*(volatile int32_t*)stop) return;
    const double s = slots_sum(slotY, ny, red);
    const double d = slots_sum(slotD, nd, red);
    if (threadIdx.x == 0) {
        if (!(s > 0.0) || isinf(s)) {
            status[0] = (s == 0.0) ? 4 : 6;
            *stop = 1;
            return;
        }
        if (deltas) deltas[t] = (float)d;
        status[1] = t + 1;
        if (tol > 0.0f && d < (double)tol) *stop = 1;
    }
}

// Final outputs from the fp64 state: w_out = fp32(w), optional l2 copy, one CTA.
__global__ void __launch_bounds__(1024) k_rank_output(int64_t n, const double* __restrict__ w, float* __restrict__ w_out,
                                                      float* __restrict__ w_l2) {
    __shared__ double red[33];
    double part = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double x = w[j];
        w_out[j] = (float)x;
        part = fma(x, x, part);
    }
    if (!w_l2) return;
    const double l2 = sqrt(block_sum(part, red));
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) w_l2[j] = l2 > 0.0 ? (float)(w[j] / l2) : 0.0f;
}

inline mapi_status csr_rank_run(int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* col_idx,
                                const float* cap, const float* bg, const float* b0, int32_t max_iters, float tol,
                                float* w_out, float* w_l2_out, float* deltas, void* ws, int sms, cudaStream_t s,
                                cudaEvent_t* ev_a, cudaEvent_t* ev_b, std::atomic<uint64_t>& launches) {
    (void)nnz;
    CsrWs W = carve_csr(ws, n);
    cudaError_t err = cudaMemsetAsync(ws, 0, 256, s);
    if (err != cudaSuccess) return csr_cuda_fail(err, "memset");
    const int gcol = (int)std::min<int64_t>({(n + kCsrThreads - 1) / kCsrThreads, (int64_t)4 * sms, (int64_t)kCsrMaxGrid});
    const int grow = (int)std::min<int64_t>({(n + 7) / 8, (int64_t)8 * sms, (int64_t)kCsrMaxGrid});
    if (ev_a) cudaEventRecord(*ev_a, s);
    k_rank_init<<<gcol, kCsrThreads, 0, s>>>(n, b0, bg, cap, W.w, W.v, W.slotS, W.status, W.stop);
    launches.fetch_add(1, std::memory_order_relaxed);
    for (int32_t t = 0; t < max_iters; ++t) {
        double* S_cur = W.slotS + (t & 1) * kCsrMaxGrid;
        double* S_next = W.slotS + ((t + 1) & 1) * kCsrMaxGrid;
        k_rank_rows<<<grow, kCsrThreads, 0, s>>>(n, row_ptr, col_idx, W.v, S_cur, gcol, W.e, W.slotY, W.stop);
        k_rank_normalize<<<gcol, kCsrThreads, 0, s>>>(n, W.e, S_cur, S_next, gcol, W.slotY, grow, bg, cap, W.w, W.v,
                                                       W.slotD, W.stop);
        k_rank_step_end<<<1, 32, 0, s>>>(W.slotY, grow, W.slotD, gcol, t, tol, deltas, W.status, W.stop);
        launches.fetch_add(3, std::memory_order_relaxed);
        if ((err = cudaGetLastError()) != cudaSuccess) return csr_cuda_fail(err, "rank launch");
    }
    if (ev_b) cudaEventRecord(*ev_b, s);
    k_rank_output<<<1, 1024, 0, s>>>(n, W.w, w_out, w_l2_out);
    launches.fetch_add(1, std::memory_order_relaxed);
    if ((err = cudaGetLastError()) != cudaSuccess) return csr_cuda_fail(err, "rank output");
    return MAPI_OK;
}

inline mapi_status csr_rank_finish(void* ws, int64_t /*n*/, int64_t /*nnz*/, cudaStream_t s, int32_t* iters_done) {
    int32_t h[2] = {0, 0};
    cudaError_t e = cudaMemcpyAsync(h, ws, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return csr_cuda_fail(e, "status read-back");
    if (iters_done) *iters_done = h[1];
    return (mapi_status)h[0];
}

}  // namespace mapi
