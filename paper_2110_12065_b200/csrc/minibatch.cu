// minibatch.cu — K10: Algorithm 3, mini-batch MAPI with momentum (§3.2; readings R14 / R15) for sm_100a.
//
//   for t = 0 .. T-1:   M_t = (1/s) sum_{i in batch t} A~_i,   A~_i[j][k] = x_ij (gram) x_ik        (steps 3, 4)
//                       y_j = sum_k term_min1(M_t[j][k], w_t[k]) - beta w_{t-1}[j]                    (step 4)
//                       s_t = ||y||_1;  w_{t-1} <- w_t / s_t;  w_t <- y / s_t                        (step 5, verbatim)
//
// The batch draws are INPUTS (step 3's i.i.d. indices come from the caller), so no M_t depends on an iterate:
// the s D^2 terms per iteration that dominate the work are formed for ALL iterations at once, in parallel
// (k_minibatch_gram: one CTA per (iteration, chunk of 4096 samples), sample rows staged in shared memory,
// fp32 chains of <= 128 terms folded in fp64, chunk partials summed in chunk order); only the D^2-term step 4
// and the normalisation stay on the dependent chain, which one CTA runs for all T iterations
// (k_minibatch_iterate: a warp per row of M_t, the next M_{t+1} prefetched, s_t in fp64 in a fixed order, the
// two divisions of step 5 in fp64 rounded once to fp32).  The MAVP loops contain no multiply (gram = min1,
// the paper's reading P:266); gram = dot forms x_ij x_ik (reading R14).  The 1/s scaling is one
// fp64 division per entry of M_t.
#include <algorithm>
#include <cstdio>

#include "../../include/mapi.h"
#include "host_common.h"
#include "mapi_common.cuh"
#include "minibatch.h"

using namespace mapi_host;

namespace mapi_mb {

constexpr int kMaxD = 64;       // D <= 64: a row of M_t is at most two terms per lane
constexpr int kChunk = 4096;    // samples per gram CTA
constexpr int kFold = 128;      // fp32 chain length (T1's bound)
constexpr int kGramThreads = 1024;
constexpr int kIterThreads = 1024;

inline size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
inline int64_t nchunks_of(int64_t s) { return (s + kChunk - 1) / kChunk; }

// workspace: [status 256: status, iters_done, bad index flag][part T x nchunks x D^2 f32][M T x D^2 f32]
size_t minibatch_ws_bytes(int64_t D, int64_t s, int64_t T) {
    if (D < 1 || s < 1 || T < 1) return 0;
    return 256 + al256(4 * (size_t)(T * nchunks_of(s) * D * D)) + al256(4 * (size_t)(T * D * D));
}

// One CTA per (chunk c, iteration t): part[t][c][j][k] = sum over the chunk's samples, in batch order, of
// term(x_ij, x_ik).  PP = pairs (j, k) per thread.
template <int OP, int PP>
__global__ void __launch_bounds__(kGramThreads) k_minibatch_gram(const float* __restrict__ X, int64_t N, int D,
                                                                  int64_t ldx, const int32_t* __restrict__ batch,
                                                                  int32_t s, int nchunks, float* __restrict__ part,
                                                                  int32_t* __restrict__ status) {
    extern __shared__ float xs[];  // kFold x D staged sample rows
    const int c = blockIdx.x, t = blockIdx.y, tid = threadIdx.x;
    const int npairs = D * D;
    const int32_t i0 = c * kChunk, i1 = min(s, i0 + kChunk);
    const int32_t* b = batch + (int64_t)t * s;
    int pj[PP], pk[PP];
    double acc[PP];
#pragma unroll
    for (int u = 0; u < PP; ++u) {
        const int p = tid + u * kGramThreads;
        pj[u] = p < npairs ? p / D : 0;
        pk[u] = p < npairs ? p % D : 0;
        acc[u] = 0.0;
    }
    int bad = 0;
    for (int32_t f0 = i0; f0 < i1; f0 += kFold) {
        const int cnt = min(kFold, i1 - f0);
        __syncthreads();  // the previous fold's reads are done
        for (int e = tid; e < cnt * D; e += kGramThreads) {
            const int i = e / D, j = e - i * D;
            const int64_t idx = b[f0 + i];
            const bool ok = idx >= 0 && idx < N;
            bad |= !ok;
            xs[e] = ok ? __ldg(X + idx * ldx + j) : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PP; ++u) {
            float a32 = 0.0f;
            for (int i = 0; i < cnt; ++i) a32 += mapi::mavp_term<OP>(xs[i * D + pj[u]], xs[i * D + pk[u]]);
            acc[u] += (double)a32;
        }
    }
    if (bad) atomicOr(status + 2, 1);
    float* out = part + ((int64_t)t * nchunks + c) * npairs;
#pragma unroll
    for (int u = 0; u < PP; ++u) {
        const int p = tid + u * kGramThreads;
        if (p < npairs) out[p] = (float)acc[u];
    }
}

// M_t[j][k] = fp32((sum of the chunk partials in chunk order, fp64) / s)
__global__ void k_minibatch_reduce(int64_t total, int npairs, int nchunks, int32_t s, const float* __restrict__ part,
                                   float* __restrict__ M) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = e / npairs, p = e - t * npairs;
        double a = 0.0;
        for (int c = 0; c < nchunks; ++c) a += (double)part[(t * nchunks + c) * npairs + p];
        M[e] = (float)(a / (double)s);
    }
}

// The dependent chain: one CTA, warp r owns rows r and r + 32 of M_t (lane l: columns l and l + 32).
__global__ void __launch_bounds__(kIterThreads, 1) k_minibatch_iterate(const float* __restrict__ M, int D, int32_t T,
                                                                        float beta, const float* __restrict__ w0,
                                                                        const float* __restrict__ wprev0,
                                                                        float* __restrict__ wprev_out,
                                                                        float* __restrict__ w_out,
                                                                        float* __restrict__ w_l2_out,
                                                                        float* __restrict__ norms,
                                                                        int32_t* __restrict__ status) {
    __shared__ float w[kMaxD], wp[kMaxD], ya[kMaxD];
    __shared__ double y[kMaxD];
    __shared__ double s_st;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int npairs = D * D;
    if (tid < kMaxD) {
        w[tid] = tid < D ? w0[tid] : 0.0f;
        wp[tid] = (wprev0 && tid < D) ? wprev0[tid] : 0.0f;  // w_{-1} = 0 (R15) unless a run is continued
    }
    // this lane's entries of M_t: rows warp, warp + 32; columns lane, lane + 32
    auto load_m = [&](int32_t t, float (&m)[4]) {
        const float* Mt = M + (int64_t)t * npairs;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int j = warp + 32 * a, k = lane + 32 * b;
                m[2 * a + b] = (t < T && j < D && k < D) ? __ldg(Mt + j * D + k) : 0.0f;
            }
    };
    float m[4], mn[4];
    load_m(0, m);
    __syncthreads();
    int32_t done = 0, st_code = 0;
    for (int32_t t = 0; t < T; ++t) {
        load_m(t + 1, mn);  // M does not depend on w: the next iteration's entries are in flight
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const int j = warp + 32 * a;
            float acc = mapi::mavp_term<0>(m[2 * a], w[lane]) + mapi::mavp_term<0>(m[2 * a + 1], w[lane + 32]);
            acc = mapi::warp_sum(acc);  // (padding entries of m and w are 0)
            if (lane == 0 && j < D) ya[j] = acc;
        }
        __syncthreads();
        if (warp == 0) {  // the momentum term (Alg. 3's one product per output) and s_t, outside the MAVP loop
            double p = 0.0;
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int j = lane + 32 * a;
                if (j < D) {
                    const double yj = (double)ya[j] - (double)beta * (double)wp[j];
                    y[j] = yj;
                    p += fabs(yj);
                }
            }
            p = mapi::warp_sum(p);
            if (lane == 0) s_st = p;
        }
        __syncthreads();
        const double st = s_st;
        if (!(st > 0.0) || isinf(st)) {  // uniform
            st_code = (st == 0.0) ? MAPI_ERR_DEGENERATE : MAPI_ERR_NONFINITE;
            break;
        }
        if (tid < D) {  // step 5, verbatim: both vectors divided by ||w_{t+1}||_1
            const float wt = w[tid];
            wp[tid] = (float)((double)wt / st);
            w[tid] = (float)(y[tid] / st);
        }
        if (tid == 0 && norms) norms[t] = (float)st;
        done = t + 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) m[q] = mn[q];
        __syncthreads();
    }
    if (tid == 0) {
        status[0] = st_code;
        status[1] = done;
    }
    if (tid < D) {
        w_out[tid] = w[tid];
        if (wprev_out) wprev_out[tid] = wp[tid];
    }
    if (w_l2_out) {  // Alg. 3 line 7
        if (warp == 0) {
            const double a = lane < D ? (double)w[lane] : 0.0, b = lane + 32 < D ? (double)w[lane + 32] : 0.0;
            const double q = mapi::warp_sum(a * a + b * b);
            if (lane == 0) s_st = sqrt(q);
        }
        __syncthreads();
        if (tid < D) w_l2_out[tid] = s_st > 0.0 ? (float)((double)w[tid] / s_st) : 0.0f;
    }
}

template <int OP>
mapi_status launch_gram(const float* X, int64_t N, int D, int64_t ldx, const int32_t* batch, int32_t s, int32_t T,
                        int nchunks, float* part, int32_t* status, cudaStream_t st) {
    const size_t smem = sizeof(float) * (size_t)kFold * (size_t)D;
    const dim3 grid((unsigned)nchunks, (unsigned)T);
    const int pp = (D * D + kGramThreads - 1) / kGramThreads;
    if (pp <= 1) k_minibatch_gram<OP, 1><<<grid, kGramThreads, smem, st>>>(X, N, D, ldx, batch, s, nchunks, part, status);
    else if (pp <= 2) k_minibatch_gram<OP, 2><<<grid, kGramThreads, smem, st>>>(X, N, D, ldx, batch, s, nchunks, part, status);
    else k_minibatch_gram<OP, 4><<<grid, kGramThreads, smem, st>>>(X, N, D, ldx, batch, s, nchunks, part, status);
    MAPI_LAUNCHED();
    return MAPI_OK;
}

}  // namespace mapi_mb

using namespace mapi_mb;

extern "C" mapi_status mapi_minibatch(int32_t gram_op, const float* X, int64_t N, int64_t D, int64_t ldx,
                                      const int32_t* batch, int32_t s, int32_t T, float beta, const float* w0,
                                      const float* w_prev0, float* w_out, float* w_l2_out, float* w_prev_out,
                                      float* norms, int32_t* iters_done, void* ws, size_t ws_bytes,
                                      mapi_stream_t stream) {
    if (gram_op != MAPI_OP_MIN1 && gram_op != MAPI_OP_DOT)
        return fail(MAPI_ERR_BAD_PARAM, "gram_op (%d) must be MAPI_OP_MIN1 or MAPI_OP_DOT", gram_op);
    if (!X || !batch || !w0 || !w_out) return fail(MAPI_ERR_NULL, "X / batch / w0 / w_out is NULL");
    if (N < 1 || D < 1 || ldx < D) return fail(MAPI_ERR_SHAPE, "N (%lld), D (%lld), ldx (%lld): need N >= 1, 1 <= D <= ldx",
                                               (long long)N, (long long)D, (long long)ldx);
    if (D > kMaxD) return fail(MAPI_ERR_SHAPE, "D (%lld) > %d: the mini-batch path holds a row of M_t in one warp", (long long)D, kMaxD);
    if (s < 1 || T < 1) return fail(MAPI_ERR_BAD_PARAM, "s (%d) and T (%d) must be >= 1", s, T);
    if (T > 65535) return fail(MAPI_ERR_SHAPE, "T (%d) > 65535 (grid limit); split the run", T);
    if (!(beta == beta) || isinf(beta)) return fail(MAPI_ERR_BAD_PARAM, "beta must be finite");
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    const size_t need = minibatch_ws_bytes(D, s, T);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    mapi_status stt = device_info(d);
    if (stt != MAPI_OK) return stt;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int nchunks = (int)nchunks_of(s), npairs = (int)(D * D);
    char* p = static_cast<char*>(ws);
    int32_t* status = reinterpret_cast<int32_t*>(p);
    float* part = reinterpret_cast<float*>(p + 256);
    float* M = reinterpret_cast<float*>(p + 256 + al256(4 * (size_t)T * (size_t)nchunks * (size_t)npairs));
    MAPI_CUDA(cudaMemsetAsync(status, 0, 256, st));
    Timer timer(st);
    timer.start();
    stt = gram_op == MAPI_OP_DOT ? launch_gram<2>(X, N, (int)D, ldx, batch, s, T, nchunks, part, status, st)
                                 : launch_gram<0>(X, N, (int)D, ldx, batch, s, T, nchunks, part, status, st);
    if (stt != MAPI_OK) return stt;
    const int64_t total = (int64_t)T * npairs;
    k_minibatch_reduce<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4 * d.sms), 256, 0, st>>>(total, npairs, nchunks, s,
                                                                                                  part, M);
    MAPI_LAUNCHED();
    k_minibatch_iterate<<<1, kIterThreads, 0, st>>>(M, (int)D, T, beta, w0, w_prev0, w_prev_out, w_out, w_l2_out, norms,
                                                    status);
    MAPI_LAUNCHED();
    timer.stop();
    int32_t h[3] = {0, 0, 0};
    MAPI_CUDA(cudaMemcpyAsync(h, status, sizeof(h), cudaMemcpyDeviceToHost, st));
    MAPI_CUDA(cudaStreamSynchronize(st));
    timer.harvest();
    if (iters_done) *iters_done = h[1];
    if (h[2]) return fail(MAPI_ERR_BAD_PARAM, "a batch index is outside [0, N)");
    if (h[0] == MAPI_ERR_DEGENERATE) return fail(MAPI_ERR_DEGENERATE, "||w_{t+1}||_1 == 0 at iteration %d", h[1]);
    if (h[0] == MAPI_ERR_NONFINITE) return fail(MAPI_ERR_NONFINITE, "||w_{t+1}||_1 is not finite at iteration %d", h[1]);
    return MAPI_OK;
}
