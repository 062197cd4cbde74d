// single.cuh — K6t: the whole MAPI iteration of a small matrix (n <= 256, BASELINE configs[0]) in ONE CTA,
// with the matrix held in registers + tensor memory.
//
// Alg. 1 at n = 256 is a 65,536-term MAVP per iteration: too little work to spread over a grid or
// even a cluster (K6r, one 8-CTA cluster: ~2 us per iteration, of which the cluster barrier and the DSMEM
// y exchange are half).  One SM holds the whole 256 KB matrix: 128 KB in registers (128 floats per thread,
// 256 threads) and 128 KB in tensor memory (256 of the 512 TMEM columns, `tcgen05.st` once, `tcgen05.ld`
// per iteration — TMEM as plain storage, no MMA: MAVP is not a contraction).  Thread (warp w, lane l) owns
// ROW r = 128 (w / 4) + 32 (w % 4) + l entirely (TMEM lane = r mod 128, the lane quarter its warp may
// access), so a row sum needs no cross-thread reduction: columns [0, 128) come from its registers,
// [128, 256) from its TMEM lane, w_t is read from shared memory as warp-wide broadcasts (every lane reads
// the same float4).  4 fp32 chains of 64 terms (FMNMX.XORSIGN + FADD2), pairwise.  Epilogue per iteration:
// s_t = fp64 per-warp butterflies then the 8 warp partials in warp order (one __syncthreads), each thread
// forms its own w_{t+1,r} = fp32(y_r / s_t) (fp64 division, as K6r) and its |delta| term (second
// __syncthreads).  No grid, cluster or global-memory exchange at all.  Deterministic.
// Requirements: n <= 256 (rows and columns beyond n are zero-padded on chip), 1 CTA (one SM).
#pragma once
#include "dense.cuh"
#include "mapi_common.cuh"
#include "resident.cuh"

namespace mapi {

constexpr int kSingleN = 256;        // max n
constexpr int kSingleThreads = 256;  // one row per thread
constexpr int kSingleRegCols = 128;  // columns held in registers; the rest in TMEM
inline size_t single_smem_bytes() { return sizeof(float) * kSingleN * (kSingleRegCols + 4); }  // staging

template <int OP>
__global__ void __launch_bounds__(kSingleThreads, 1) k_iterate_single(IterArgs p) {
    __shared__ __align__(16) float w_s[kSingleN];
    __shared__ double wsum[kSingleThreads / 32], dsum[kSingleThreads / 32];
    __shared__ uint32_t tslot;
    const int64_t n = p.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q = warp & 3, rh = warp >> 2;
    const int r = 128 * rh + 32 * q + lane;  // this thread's row (= tid)
    const bool live = r < n;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tslot;
    const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(128 * rh);

    // ---- one-time staging, one 128-column half at a time through shared memory: coalesced global reads
    // (a warp reads consecutive columns of one row), then thread r takes row r (stride 132 floats: the
    // quarter-warp phases of LDS.128 hit distinct banks).  Half 0 -> registers, half 1 -> TMEM; zero
    // beyond n.
    extern __shared__ __align__(16) float stage[];  // kSingleN x kStageLd
    constexpr int kStageLd = kSingleRegCols + 4;
    auto stage_half = [&](int h) {
        for (int e = tid; e < kSingleN * kSingleRegCols; e += kSingleThreads) {
            const int row = e / kSingleRegCols, col = kSingleRegCols * h + (e % kSingleRegCols);
            stage[row * kStageLd + (e % kSingleRegCols)] =
                (row < n && col < n) ? __ldg(p.A + (int64_t)row * p.lda + col) : 0.0f;
        }
        __syncthreads();
    };
    const float4* src = reinterpret_cast<const float4*>(stage + r * kStageLd);
    float areg[kSingleRegCols];
    stage_half(0);
#pragma unroll
    for (int m = 0; m < kSingleRegCols / 4; ++m) {
        const float4 x = src[m];
        areg[4 * m] = x.x; areg[4 * m + 1] = x.y; areg[4 * m + 2] = x.z; areg[4 * m + 3] = x.w;
    }
    __syncthreads();
    stage_half(1);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float v[32];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const float4 x = src[8 * c + m];
            v[4 * m] = x.x; v[4 * m + 1] = x.y; v[4 * m + 2] = x.z; v[4 * m + 3] = x.w;
        }
        tmem_st32(ta + (uint32_t)(32 * c), v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // v is rewritten next chunk
    }
    w_s[tid] = tid < n ? p.b0[tid] : 0.0f;
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();

    int32_t done = 0, status = kStOk;
    const float4* w4 = reinterpret_cast<const float4*>(w_s);
    for (int32_t t = 0; t < p.iters; ++t) {
        unsigned long long c0 = 0, c1 = 0;  // (chain 0, 1), (chain 2, 3) packed for FADD2
        float at[32];
        tmem_ld32(ta, at);  // TMEM chunk 0 in flight during the register half
#pragma unroll
        for (int m = 0; m < kSingleRegCols / 4; ++m) {
            const float4 w = w4[m];  // broadcast
            c0 = res_fadd2(c0, res_pack2(mavp_term<OP>(areg[4 * m], w.x), mavp_term<OP>(areg[4 * m + 1], w.y)));
            c1 = res_fadd2(c1, res_pack2(mavp_term<OP>(areg[4 * m + 2], w.z), mavp_term<OP>(areg[4 * m + 3], w.w)));
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            tmem_wait_ld(at);
            float a[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) a[k] = at[k];
            if (c + 1 < 4) tmem_ld32(ta + (uint32_t)(32 * (c + 1)), at);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const float4 w = w4[kSingleRegCols / 4 + 8 * c + m];
                c0 = res_fadd2(c0, res_pack2(mavp_term<OP>(a[4 * m], w.x), mavp_term<OP>(a[4 * m + 1], w.y)));
                c1 = res_fadd2(c1, res_pack2(mavp_term<OP>(a[4 * m + 2], w.z), mavp_term<OP>(a[4 * m + 3], w.w)));
            }
        }
        const float y = (__uint_as_float((uint32_t)c0) + __uint_as_float((uint32_t)(c0 >> 32))) +
                        (__uint_as_float((uint32_t)c1) + __uint_as_float((uint32_t)(c1 >> 32)));
        // s_t (rows beyond n contribute 0)
        double ap = warp_sum(norm_part<OP>(y));
        if (lane == 0) wsum[warp] = ap;
        __syncthreads();  // also: every thread finished reading w_t
        double sd = 0.0;
#pragma unroll
        for (int i = 0; i < kSingleThreads / 32; ++i) sd += wsum[i];
        sd = norm_final<OP>(sd);
        if (!(sd > 0.0) || isinf(sd)) {  // uniform across the CTA
            status = (sd == 0.0) ? kStDegenerate : kStNonfinite;
            break;
        }
        // w_{t+1,r} = fp32(y_r / s_t) (fp64 division, one per thread); delta in fp64
        const float wn = live ? (float)((double)y / sd) : 0.0f;
        const double dp = warp_sum((double)fabsf(wn - w_s[r]));
        if (lane == 0) dsum[warp] = dp;
        w_s[r] = wn;
        __syncthreads();
        double delta = 0.0;
#pragma unroll
        for (int i = 0; i < kSingleThreads / 32; ++i) delta += dsum[i];
        if (tid == 0) {
            if (p.norms) p.norms[t] = (float)sd;
            if (p.deltas) p.deltas[t] = (float)delta;
        }
        done = t + 1;
        if (p.tol > 0.0f && delta < (double)p.tol) break;
    }
    if (live) p.w_out[r] = w_s[r];
    if (p.w_l2) {
        // the final l2 copy in-kernel, bitwise k_l2_copy's result: fp32 squares, warp butterflies, then
        // one butterfly over the warp partials padded with zeros to 32 (k_l2_copy's 1024-thread block_sum
        // sees exactly these values for n <= 256)
        const float wv = live ? w_s[r] : 0.0f;
        float part = 0.0f;
        part += wv * wv;
        part = warp_sum(part);
        __shared__ float l2s[kSingleThreads / 32 + 1];
        __syncthreads();
        if (lane == 0) l2s[warp] = part;
        __syncthreads();
        if (warp == 0) {
            float x = lane < kSingleThreads / 32 ? l2s[lane] : 0.0f;
            x = warp_sum(x);
            if (lane == 0) l2s[kSingleThreads / 32] = x;
        }
        __syncthreads();
        const float l2 = sqrtf(l2s[kSingleThreads / 32]);
        if (live) p.w_l2[r] = l2 > 0.0f ? wv / l2 : 0.0f;
    }
    if (tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

}  // namespace mapi
