// batched.cuh — K4: batched multi-vector MAPI (BASELINE configs[3]; matrix extension P:69-70
// with p = k columns; "multiple independent runs").
//
//   Y[v][j] = sum_k A[j][k] (+) W[v][k]     for all rows j and vectors v, every iteration
//   then per vector v: s_v = ||Y[v]||_1, W[v] = Y[v] / s_v, delta_v, stop_v (Algorithm 1 per run).
//
// Register micro-tiles: each thread owns TM rows x TV vectors of accumulators; each A element is
// loaded once from shared memory per k and reused across TV vectors in registers, each W element
// across TM rows, so the kernel is bound by the FMNMX.XORSIGN issue rate (ALU pipe), not HBM.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdio>
#include "../../include/mapi.h"
#include "mapi_common.cuh"

namespace mapi {

constexpr int kBM = 64;       // rows per CTA tile
constexpr int kBV = 64;       // vectors per CTA tile
constexpr int kBK = 32;       // k per smem stage
constexpr int kTM = 8;        // rows per thread
constexpr int kTV = 8;        // vectors per thread
constexpr int kBThreads = (kBM / kTM) * (kBV / kTV);  // 64 threads
constexpr int kBStages = 2;

inline size_t bal256(size_t b) { return (b + 255) & ~size_t(255); }

inline int batched_ksplit(int64_t n, int32_t k, int sms) {
    const int64_t tiles = ((n + kBM - 1) / kBM) * ((k + kBV - 1) / kBV);
    int64_t ks = (4 * (int64_t)sms + tiles - 1) / tiles;  // >= ~4 CTAs per SM
    const int64_t kmax = std::max<int64_t>(1, (n + 255) / 256);
    ks = std::min<int64_t>(std::max<int64_t>(ks, 1), std::min<int64_t>(kmax, 64));
    return (int)ks;
}

// workspace: [hdr 256: unused][status 2k i32][stop k i32][W k*n][Y k*n][part KS*k*n][colpart k*RB]
inline size_t batched_ws_bytes(int64_t n, int32_t k) {
    const int64_t rb = (n + 255) / 256;
    return 256 + bal256(8 * (size_t)k) + bal256(4 * (size_t)k) + 2 * bal256(4 * (size_t)k * n) +
           bal256(4 * (size_t)64 * k * n) + bal256(4 * (size_t)k * rb);
}

struct BatchedWs {
    int32_t* status;  // [2v] = status, [2v+1] = iters_done
    int32_t* stop;
    float *W, *Y, *part, *colpart;
    int64_t rb;
};

inline BatchedWs carve_batched(void* ws, int64_t n, int32_t k) {
    char* p = static_cast<char*>(ws) + 256;
    BatchedWs b;
    b.status = reinterpret_cast<int32_t*>(p);
    p += bal256(8 * (size_t)k);
    b.stop = reinterpret_cast<int32_t*>(p);
    p += bal256(4 * (size_t)k);
    b.W = reinterpret_cast<float*>(p);
    p += bal256(4 * (size_t)k * n);
    b.Y = reinterpret_cast<float*>(p);
    p += bal256(4 * (size_t)k * n);
    b.part = reinterpret_cast<float*>(p);
    p += bal256(4 * (size_t)64 * k * n);
    b.colpart = reinterpret_cast<float*>(p);
    b.rb = (n + 255) / 256;
    return b;
}

// Partial products over one k-slice: part[s][v][j] = sum_{k in slice s} A[j][k] (+) W[v][k].
// grid = (row tiles, vector tiles, KS).  smem: As[k][row] and Ws[k][vec] (k-major) so that a
// thread's TM rows / TV vectors for one k are contiguous (LDS.128 x 2 each).
template <int OP>
__global__ void __launch_bounds__(kBThreads) k_batched_partial(const float* __restrict__ A, int64_t n,
                                                              int64_t lda, const float* __restrict__ W,
                                                              int32_t kv, int64_t kslice,
                                                              float* __restrict__ part) {
    __shared__ __align__(16) float As[kBStages][kBK][kBM + 4];
    __shared__ __align__(16) float Ws[kBStages][kBK][kBV + 4];
    const int tid = threadIdx.x;
    const int tr = tid / (kBV / kTV);  // 0..7  -> rows tr*TM ..
    const int tv = tid % (kBV / kTV);  // 0..7  -> vecs tv*TV ..
    const int64_t row0 = (int64_t)blockIdx.x * kBM;
    const int v0 = blockIdx.y * kBV;
    const int64_t k_begin = (int64_t)blockIdx.z * kslice;
    const int64_t k_end = min(n, k_begin + kslice);

    float acc[kTM][kTV];
#pragma unroll
    for (int i = 0; i < kTM; ++i)
#pragma unroll
        for (int j = 0; j < kTV; ++j) acc[i][j] = 0.0f;

    // global -> smem staging: each thread loads (kBM*kBK)/64 = 32 A values and 32 W values
    auto stage = [&](int buf, int64_t k0) {
#pragma unroll 4
        for (int e = tid; e < kBM * kBK; e += kBThreads) {
            const int r = e / kBK, kk = e % kBK;
            const int64_t row = row0 + r, kc = k0 + kk;
            As[buf][kk][r] = (row < n && kc < k_end) ? __ldg(A + row * lda + kc) : 0.0f;
        }
#pragma unroll 4
        for (int e = tid; e < kBV * kBK; e += kBThreads) {
            const int v = e / kBK, kk = e % kBK;
            const int64_t kc = k0 + kk;
            Ws[buf][kk][v] = (v0 + v < kv && kc < k_end) ? __ldg(W + (int64_t)(v0 + v) * n + kc) : 0.0f;
        }
    };

    int buf = 0;
    stage(0, k_begin);
    __syncthreads();
    for (int64_t k0 = k_begin; k0 < k_end; k0 += kBK) {
        if (k0 + kBK < k_end) stage(buf ^ 1, k0 + kBK);
#pragma unroll 4
        for (int kk = 0; kk < kBK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][tr * kTM]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][tr * kTM + 4]);
            const float4 w0 = *reinterpret_cast<const float4*>(&Ws[buf][kk][tv * kTV]);
            const float4 w1 = *reinterpret_cast<const float4*>(&Ws[buf][kk][tv * kTV + 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
            for (int i = 0; i < kTM; ++i)
#pragma unroll
                for (int j = 0; j < kTV; ++j) acc[i][j] += mavp_term<OP>(a[i], w[j]);
        }
        __syncthreads();
        buf ^= 1;
    }
    float* out = part + (int64_t)blockIdx.z * kv * n;
#pragma unroll
    for (int j = 0; j < kTV; ++j) {
        const int v = v0 + tv * kTV + j;
        if (v >= kv) continue;
#pragma unroll
        for (int i = 0; i < kTM; ++i) {
            const int64_t row = row0 + tr * kTM + i;
            if (row < n) out[(int64_t)v * n + row] = acc[i][j];
        }
    }
}

// Y[v][j] = sum_s part[s][v][j] (s ascending); colpart[v][blk] = sum_{j in blk} |Y[v][j]|.
__global__ void __launch_bounds__(256) k_batched_reduce(int64_t n, int32_t kv, int ks,
                                                        const float* __restrict__ part, float* __restrict__ Y,
                                                        float* __restrict__ colpart, int64_t rb) {
    __shared__ float red[33];
    const int v = blockIdx.y;
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    float y = 0.0f;
    if (j < n) {
        for (int s = 0; s < ks; ++s) y += part[((int64_t)s * kv + v) * n + j];
        Y[(int64_t)v * n + j] = y;
    }
    const float a = block_sum(fabsf(y), red);
    if (threadIdx.x == 0) colpart[(int64_t)v * rb + blockIdx.x] = a;
}

// Per vector v (one CTA each): s = sum colpart (fixed order), W = Y / s, delta, trace, stop.
__global__ void __launch_bounds__(1024) k_batched_normalize(int64_t n, int32_t kv, int32_t t, float tol,
                                                            const float* __restrict__ Y,
                                                            const float* __restrict__ colpart, int64_t rb,
                                                            float* __restrict__ W, float* norms, float* deltas,
                                                            int32_t* status, int32_t* stop) {
    __shared__ float red[33];
    const int v = blockIdx.x;
    if (stop[v]) return;
    float part = 0.0f;
    if (threadIdx.x < 32) {
        for (int64_t b = threadIdx.x; b < rb; b += 32) part += colpart[(int64_t)v * rb + b];
        part = warp_sum(part);
        if (threadIdx.x == 0) red[32] = part;
    }
    __syncthreads();
    const float s = red[32];
    __syncthreads();
    if (!(s > 0.0f) || isinf(s)) {
        if (threadIdx.x == 0) {
            status[2 * v] = (s == 0.0f) ? 4 : 6;
            stop[v] = 1;
        }
        return;
    }
    float dpart = 0.0f;
    float* wv = W + (int64_t)v * n;
    const float* yv = Y + (int64_t)v * n;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const float wn = yv[k] / s;
        dpart += fabsf(wn - wv[k]);
        wv[k] = wn;
    }
    const float delta = block_sum(dpart, red);
    if (threadIdx.x == 0) {
        if (norms) norms[(int64_t)t * kv + v] = s;
        if (deltas) deltas[(int64_t)t * kv + v] = delta;
        status[2 * v + 1] = t + 1;
        if (tol > 0.0f && delta < tol) stop[v] = 1;
    }
}

static thread_local char g_batched_err[256] = "";
inline const char* batched_last_error() { return g_batched_err; }

inline mapi_status batched_cuda_fail(cudaError_t e, const char* what) {
    snprintf(g_batched_err, sizeof(g_batched_err), "%s: %s", what, cudaGetErrorString(e));
    return MAPI_ERR_CUDA;
}

// Launch the whole batched run (no sync).  Events (if timing) bracket the iteration loop.
inline mapi_status batched_run(int32_t op, const float* A, int64_t n, int64_t lda, const float* B0, int32_t k,
                               int32_t iters, float tol, float* W_out, float* norms, float* deltas, void* ws,
                               int sms, cudaStream_t s, cudaEvent_t* ev_a, cudaEvent_t* ev_b, bool timing,
                               std::atomic<uint64_t>& launches) {
    BatchedWs B = carve_batched(ws, n, k);
    cudaError_t e;
    if ((e = cudaMemsetAsync(B.status, 0, 8 * (size_t)k, s)) != cudaSuccess) return batched_cuda_fail(e, "memset");
    if ((e = cudaMemsetAsync(B.stop, 0, 4 * (size_t)k, s)) != cudaSuccess) return batched_cuda_fail(e, "memset");
    if ((e = cudaMemcpyAsync(B.W, B0, 4 * (size_t)k * n, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return batched_cuda_fail(e, "copy B0");
    const int ks0 = batched_ksplit(n, k, sms);
    int64_t kslice = (n + ks0 - 1) / ks0;
    kslice = (kslice + kBK - 1) / kBK * kBK;
    const int ks = (int)((n + kslice - 1) / kslice);
    const dim3 gp((unsigned)((n + kBM - 1) / kBM), (unsigned)((k + kBV - 1) / kBV), (unsigned)ks);
    const dim3 gr((unsigned)B.rb, (unsigned)k);
    if (timing) cudaEventRecord(*ev_a, s);
    for (int32_t t = 0; t < iters; ++t) {
        if (op == 1)
            k_batched_partial<1><<<gp, kBThreads, 0, s>>>(A, n, lda, B.W, k, kslice, B.part);
        else
            k_batched_partial<0><<<gp, kBThreads, 0, s>>>(A, n, lda, B.W, k, kslice, B.part);
        k_batched_reduce<<<gr, 256, 0, s>>>(n, k, ks, B.part, B.Y, B.colpart, B.rb);
        k_batched_normalize<<<k, 1024, 0, s>>>(n, k, t, tol, B.Y, B.colpart, B.rb, B.W, norms, deltas, B.status,
                                               B.stop);
        launches.fetch_add(3, std::memory_order_relaxed);
        if ((e = cudaGetLastError()) != cudaSuccess) return batched_cuda_fail(e, "batched launch");
    }
    if (timing) cudaEventRecord(*ev_b, s);
    if ((e = cudaMemcpyAsync(W_out, B.W, 4 * (size_t)k * n, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return batched_cuda_fail(e, "copy W");
    return MAPI_OK;
}

// Sync, read per-vector status / iteration counts; returns the worst status.
inline mapi_status batched_finish(void* ws, int64_t n, int32_t k, cudaStream_t s, int32_t* iters_done) {
    BatchedWs B = carve_batched(ws, n, k);
    int32_t* h = static_cast<int32_t*>(malloc(8 * (size_t)k));
    cudaError_t e = cudaMemcpyAsync(h, B.status, 8 * (size_t)k, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        free(h);
        return batched_cuda_fail(e, "status read-back");
    }
    mapi_status worst = MAPI_OK;
    for (int32_t v = 0; v < k; ++v) {
        if (iters_done) iters_done[v] = h[2 * v + 1];
        if (h[2 * v] != 0 && worst == MAPI_OK) worst = (mapi_status)h[2 * v];
    }
    free(h);
    return worst;
}

}  // namespace mapi
