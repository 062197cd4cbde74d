// bulk.cuh — K2t: persistent MAPI iteration fed by TMA bulk copies (mid-size n, A L2-resident).
//
// Alg. 1 for matrices that fit in L2 (cfg2's 64 MiB D_i): every iteration re-reads A from
// L2, so the per-row register kernel (K2) is LATENCY-bound — 16 warps x 8 x 16 B loads in flight per
// SM cover only ~64 KB of the 453 KB an SM reads per iteration (ncu: L2 hit 96.6%, L2 throughput 27%,
// issue 22%, long-scoreboard + barrier stalls).  Here every warp streams its own work items through
// SP private 4 KB shared-memory slots with `cp.async.bulk` (the TMA engine: no registers held,
// completion counted as tx bytes on one mbarrier per slot), SP items ahead of its consumption, so
// NC x SP x 4 KB (~190 KB) per SM is in flight.  A does not depend on w, so a warp keeps issuing the
// next iteration's copies before the grid barrier: the memory pipeline never drains.
//
// Work items: (local row r, 1024-float chunk q) of the CTA's contiguous rows [r0, r1), row-major, the
// same every iteration; warp c owns items c, c + NC, ...  A chunk partial is a warp butterfly of 32
// lane partials (4 accumulators x 8 terms, pairwise tree), stored per (r, q); y_row = sum_q partial
// in chunk order.  Deterministic for a given (n, grid).  Requirements: A and lda 16 B-aligned
// (n % 4 == 0, lda % 4 == 0); 1 CTA per SM (cooperative launch).
//
// Slots are private to a warp and reused only after the same warp consumed them (__syncwarp before
// the re-issue), so no "empty" barrier is needed and a full-barrier wait is never more than one
// phase ahead.  On an early stop (tol / degenerate) each warp waits for the copies it issued beyond
// the last iteration before the CTA exits (no async copy outlives the CTA).
#pragma once
#include "dense.cuh"
#include "mapi_common.cuh"

namespace mapi {

constexpr int kBulkNC = 16;                       // warps per CTA (each its own copy issuer)
constexpr int kBulkThreads = kBulkNC * 32;
#ifndef MAPI_BULK_CHUNK
#define MAPI_BULK_CHUNK 1024
#endif
constexpr int kBulkChunk = MAPI_BULK_CHUNK;       // floats per ring slot (4 KB)
constexpr int kBulkMaxSlots = 64;                 // per CTA (kBulkNC x slots per warp)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_test(bar, parity)) {
    }
}
// 1-D bulk copy global -> shared (TMA), completion as tx bytes on `bar`; L2 evict-last hint (A is
// re-read every iteration and is meant to stay resident).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
inline size_t bulk_fixed_smem(int64_t n, int64_t rows_max) {
    const int64_t cpr = (n + kBulkChunk - 1) / kBulkChunk;
    size_t b = sizeof(float) * (size_t)(cpr * kBulkChunk);           // w_t, zero-padded to whole chunks
    b += sizeof(float) * (size_t)((rows_max * cpr + 3) & ~int64_t(3));  // chunk partials
    b += sizeof(double) * 40;                                          // reduction scratch + flags
    b += 2 * sizeof(uint64_t) * kBulkMaxSlots;                         // full / empty mbarriers
    return (b + 127) & ~size_t(127);
}

#ifdef MAPI_BULK_TRACE
__device__ long long g_bulk_trace[6 * 512];  // investigation builds only (scripts/probe_k2t.cu)
#define BULK_STAMP(t, k) \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (t) < 512) g_bulk_trace[(t) * 6 + (k)] = clock64()
#else
#define BULK_STAMP(t, k)
#endif

template <int OP>
__global__ void __launch_bounds__(kBulkThreads, 1) k_iterate_bulk(IterArgs p, int slots) {
    extern __shared__ __align__(16) float ws_[];
    const int64_t n = p.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int SP = slots / kBulkNC;                                    // slots per warp (>= 2)
    const int64_t cpr = (n + kBulkChunk - 1) / kBulkChunk;             // chunks per row
    const int64_t r0 = (int64_t)blockIdx.x * n / gridDim.x, r1 = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
    const int64_t rows = r1 - r0, rows_max = (n + gridDim.x - 1) / gridDim.x;
    const int items = (int)(rows * cpr), cpr_i = (int)cpr;
    const int nj = items > warp ? (items - warp + kBulkNC - 1) / kBulkNC : 0;  // this warp's items / iteration
    // shared layout (bulk_fixed_smem + slots x 4 KB): [ring][w][partials][scratch][mbarriers]
    float* ring = ws_;
    float* w_s = ring + (size_t)slots * kBulkChunk;
    float* part = w_s + cpr * kBulkChunk;
    double* red = reinterpret_cast<double*>(part + ((rows_max * cpr + 3) & ~int64_t(3)));
    uint64_t* full = reinterpret_cast<uint64_t*>(red + 40) + warp * SP;  // this warp's slots
    float* my_ring = ring + (size_t)warp * SP * kBulkChunk;

    for (int64_t k = tid; k < cpr * kBulkChunk; k += blockDim.x) w_s[k] = k < n ? p.b0[k] : 0.0f;
    if (lane == 0)
        for (int j = 0; j < SP; ++j) mbar_init(full + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // load cursor (iteration lt, item j = lj of this warp, slot ls) — lane 0 issues
    uint64_t pol = 0;
    if (lane == 0) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    int lt = 0, lj = 0, ls = 0;
    int64_t issued = 0, consumed = 0;
    auto issue = [&]() {
        if (nj == 0 || lt >= p.iters) return;
        if (lane == 0) {
            const int i = warp + kBulkNC * lj, r = i / cpr_i, q = i - r * cpr_i;
            const uint32_t bytes = (uint32_t)(4 * min((int64_t)kBulkChunk, n - (int64_t)q * kBulkChunk));
            mbar_expect_tx(full + ls, bytes);
            bulk_g2s(my_ring + (size_t)ls * kBulkChunk, p.A + (r0 + r) * p.lda + (int64_t)q * kBulkChunk, bytes,
                     full + ls, pol);
        }
        ++issued;
        if (++ls == SP) ls = 0;
        if (++lj == nj) { lj = 0; ++lt; }
    };
    for (int j = 0; j < SP; ++j) issue();

    int cs = 0;        // consume slot
    uint32_t cph = 0;  // its phase
    int32_t done = 0, status = kStOk;
    const float4* w4 = reinterpret_cast<const float4*>(w_s);
    for (int32_t t = 0; t < p.iters; ++t) {
        float* y = p.y + (t & 1) * n;
        BULK_STAMP(t, 0);
        for (int j = 0; j < nj; ++j) {
            const int i = warp + kBulkNC * j, q = i % cpr_i;
            mbar_wait(full + cs, cph);
            const float4* a4 = reinterpret_cast<const float4*>(my_ring + (size_t)cs * kBulkChunk);
            const int lim4 = (int)(min((int64_t)kBulkChunk, n - (int64_t)q * kBulkChunk) >> 2);  // valid float4s
            float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int jj = 0; jj < kBulkChunk / 128; ++jj) {
                const int e = lane + 32 * jj;
                if (e < lim4) {
                    const float4 a = a4[e], w = w4[q * (kBulkChunk / 4) + e];
                    acc[0] += mavp_term<OP>(a.x, w.x);
                    acc[1] += mavp_term<OP>(a.y, w.y);
                    acc[2] += mavp_term<OP>(a.z, w.z);
                    acc[3] += mavp_term<OP>(a.w, w.w);
                }
            }
            __syncwarp();  // every lane is done with the slot: refill it SP items ahead
            ++consumed;
            if (++cs == SP) { cs = 0; cph ^= 1u; }
            issue();
            const float v = warp_sum(tree_sum(acc));
            if (lane == 0) part[i] = v;
        }
        BULK_STAMP(t, 1);
        __syncthreads();
        BULK_STAMP(t, 2);
        // rows of this CTA: y = sum of chunk partials in chunk order; |y| partial (a1-a3)
        double abs_part = 0.0;
        for (int64_t r = tid; r < rows; r += blockDim.x) {
            float v = 0.0f;
            for (int64_t q = 0; q < cpr; ++q) v += part[r * cpr + q];
            y[r0 + r] = v;
            abs_part += norm_part<OP>(v);
        }
        const double cta_abs = block_sum(abs_part, red);
        double* slots_g = reinterpret_cast<double*>(p.slots);
        if (tid == 0) slots_g[(t & 1) * gridDim.x + blockIdx.x] = cta_abs;
        grid_barrier(p.bar, (unsigned int)(t + 1) * gridDim.x);  // the issued copies keep flowing
        BULK_STAMP(t, 3);
        // the y loads of the normalisation do not depend on s_t: issue them together with the slot
        // loads (one L2 round trip after the barrier instead of two)
        constexpr int YR = 16;  // y values held per thread (n <= 8192 with 512 threads); the rest streams
        float yr[YR];
#pragma unroll
        for (int q = 0; q < YR; ++q) {
            const int64_t k = tid + (int64_t)q * kBulkThreads;
            yr[q] = k < n ? __ldcg(y + k) : 0.0f;
        }
        // s_t in the same fixed fp64 order in every CTA
        double s;
        {
            if (warp == 0) {
                double pt = 0.0;
                for (int c = lane; c < (int)gridDim.x; c += 32) pt += __ldcg(slots_g + (t & 1) * gridDim.x + c);
                pt = warp_sum(pt);
                if (lane == 0) red[32] = pt;
            }
            __syncthreads();
            s = norm_final<OP>(red[32]);
            __syncthreads();
        }
        if (!(s > 0.0) || isinf(s)) {  // uniform across the grid
            status = (s == 0.0) ? kStDegenerate : kStNonfinite;
            break;
        }
        BULK_STAMP(t, 4);
        // w_{t+1} = fp32(y / s_t) (fp64 division), delta_t in fp64
        double dpart = 0.0;
        // y / s_t for n elements per CTA per iteration: one IEEE fp64 reciprocal of s_t, then per element
        // q0 = y r, q = q0 + (y - q0 s) r (the residual-corrected quotient DDIV itself computes, without
        // its special-case paths: y and s are finite fp32-range values here).  Measured ~1,200 of ~25,700
        // cycles per iteration cheaper than the DDIV sequence (scripts/probe_k2t.cu); the fp32 rounding
        // of the result can differ from fp32(y / s) only when y / s lies within an fp64 ulp of an fp32
        // rounding boundary.
        const double rs = 1.0 / s;
#pragma unroll
        for (int q = 0; q < YR; ++q) {
            const int64_t k = tid + (int64_t)q * kBulkThreads;
            if (k < n) {
                const double q0 = (double)yr[q] * rs;
                const float wn = (float)fma(fma(-q0, s, (double)yr[q]), rs, q0);
                dpart += (double)fabsf(wn - w_s[k]);
                w_s[k] = wn;
            }
        }
        for (int64_t k = tid + (int64_t)YR * kBulkThreads; k < n; k += blockDim.x) {
            const double yk = (double)__ldcg(y + k), q0 = yk * rs;
            const float wn = (float)fma(fma(-q0, s, yk), rs, q0);
            dpart += (double)fabsf(wn - w_s[k]);
            w_s[k] = wn;
        }
        const double delta = block_sum(dpart, red);  // also orders the w_s writes before reuse
        BULK_STAMP(t, 5);
        if (blockIdx.x == 0 && tid == 0) {
            if (p.norms) p.norms[t] = (float)s;
            if (p.deltas) p.deltas[t] = (float)delta;
        }
        done = t + 1;
        if (p.tol > 0.0f && delta < (double)p.tol) break;
    }
    // drain the copies issued beyond the last consumed item (early stop)
    for (; consumed < issued; ++consumed) {
        mbar_wait(full + cs, cph);
        if (++cs == SP) { cs = 0; cph ^= 1u; }
    }
    // final iterate out: CTA c writes its row range of its (identical) copy
    for (int64_t k = r0 + tid; k < r1; k += blockDim.x) p.w_out[k] = w_s[k];
    if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
}

}  // namespace mapi
