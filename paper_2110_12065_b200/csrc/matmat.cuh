// matmat.cuh — K8: the MAVP matrix product (matrix extension)
//
//   C[i][j] = (1/d) ( a_i (op) b_j ),   a_i = row i of A (m x K), b_j = row j of B (p x K)
//
// With A = B = V (pixels x N mean-removed samples) and d = N - 1 this is the min-covariance of
// Alg. 2 step 4; d = N gives Eq. (5).
//
// Tile: 64 A-rows x 256 B-rows per CTA, 256 threads; thread (warp w, lane l) owns rows i = w + 8 ii and
// columns j = l + 32 jj (ii, jj < 8): A reads are warp-wide broadcasts, B reads conflict-free LDS.128,
// and the C stores of a warp are 128 B coalesced.  K runs in 32-wide stages through a 3-deep shared
// memory ring (cp.async 16 B when rows are 16 B aligned and K % 4 == 0, 4 B copies otherwise);
// the k loop of the last stage stops at K (rounded up to 4; the staged tail is zero), per term one
// FMNMX.XORSIGN + half an FADD2 (pairs of columns), folded every 128 terms; the epilogue applies the
// scalar factor 1/d of Eq. (5) ("1/N X (+) X^T") as one multiply per element, outside the MAVP
// loop.  Bound: ALU pipe for large K, HBM writes of C for small K (the paper's N = 10 samples).
#pragma once
#include "batched.cuh"

namespace mapi {

constexpr int kMmI = 64, kMmJ = 256, kMmK = 32, kMmThreads = 256, kMmStages = 3, kMmLd = kMmK + 4;

inline size_t matmat_smem_bytes() { return sizeof(float) * kMmStages * (kMmI + kMmJ) * kMmLd; }

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}

// Persistent over output tiles: CTA c owns tiles c, c + G, ... (row-major over (i-tile, j-tile)); the
// (tile, stage) sequence of a CTA is one continuous cp.async pipeline, so the staging of the next tile
// overlaps the compute and the C stores of the current one.  V16: 16 B copies (rows 16 B aligned and
// K % 4 == 0); otherwise 4 B copies of the K columns (e.g. the paper's N = 10 samples).
template <int OP, bool V16>
__global__ void __launch_bounds__(kMmThreads, 1) k_mavp_matmat(const float* __restrict__ A, int64_t m, int64_t K,
                                                               int64_t lda, const float* __restrict__ B, int64_t p,
                                                               int64_t ldb, float d, float* __restrict__ C,
                                                               int64_t ldc) {
    extern __shared__ __align__(16) float smem[];
    float* As = smem;                              // [stage][64][kMmLd]
    float* Bs = smem + kMmStages * kMmI * kMmLd;   // [stage][256][kMmLd]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tj = (p + kMmJ - 1) / kMmJ, ntiles = ((m + kMmI - 1) / kMmI) * tj;
    const int64_t nst = (K + kMmK - 1) / kMmK;  // stages per tile
    const int64_t G = gridDim.x;
    const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - blockIdx.x + G - 1) / G : 0;
    const int64_t units = my_tiles * nst;
    if (units == 0) return;

    // load cursor
    int64_t l_tile = blockIdx.x, l_s = 0;
    auto load_next = [&](int slot) {
        const int64_t i0 = (l_tile / tj) * kMmI, j0 = (l_tile % tj) * kMmJ, k0 = l_s * kMmK;
        float* as = As + slot * kMmI * kMmLd;
        float* bs = Bs + slot * kMmJ * kMmLd;
        if constexpr (V16) {
#pragma unroll
            for (int q = tid; q < kMmI * (kMmK / 4); q += kMmThreads) {
                const int r = q >> 3, kq = (q & 7) * 4;
                const bool in = i0 + r < m && k0 + kq < K;
                cp_async16(as + r * kMmLd + kq, in ? (const void*)(A + (i0 + r) * lda + k0 + kq) : (const void*)A,
                           in ? 16 : 0);
            }
#pragma unroll
            for (int q = tid; q < kMmJ * (kMmK / 4); q += kMmThreads) {
                const int r = q >> 3, kq = (q & 7) * 4;
                const bool in = j0 + r < p && k0 + kq < K;
                cp_async16(bs + r * kMmLd + kq, in ? (const void*)(B + (j0 + r) * ldb + k0 + kq) : (const void*)B,
                           in ? 16 : 0);
            }
        } else {
            // columns [0, kw) of the stage: kw = K - k0 rounded up to 4 (the tail is zero-filled)
            const int kw = (int)min((int64_t)kMmK, (K - k0 + 3) & ~int64_t(3));
            for (int q = tid; q < kMmI * kw; q += kMmThreads) {
                const int r = q / kw, kk = q - r * kw;
                const bool in = i0 + r < m && k0 + kk < K;
                cp_async4(as + r * kMmLd + kk, in ? (const void*)(A + (i0 + r) * lda + k0 + kk) : (const void*)A,
                          in ? 4 : 0);
            }
            for (int q = tid; q < kMmJ * kw; q += kMmThreads) {
                const int r = q / kw, kk = q - r * kw;
                const bool in = j0 + r < p && k0 + kk < K;
                cp_async4(bs + r * kMmLd + kk, in ? (const void*)(B + (j0 + r) * ldb + k0 + kk) : (const void*)B,
                          in ? 4 : 0);
            }
        }
        if (++l_s == nst) {
            l_s = 0;
            l_tile += G;
        }
    };

    unsigned long long acc[8][4], tot[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = tot[i][j] = 0ull;
    const float inv_d = 1.0f / d;

    load_next(0);
    cp_async_commit();
    if (units > 1) load_next(1);
    cp_async_commit();
    int slot = 0, lslot = 2, nfold = 0;
    int64_t c_tile = blockIdx.x, c_s = 0;  // compute cursor
    for (int64_t u = 0; u < units; ++u) {
        cp_async_wait<1>();
        __syncthreads();
        if (u + 2 < units) load_next(lslot);
        cp_async_commit();
        lslot = lslot == kMmStages - 1 ? 0 : lslot + 1;
        const float* as = As + slot * kMmI * kMmLd + warp * kMmLd;
        const float* bs = Bs + slot * kMmJ * kMmLd + lane * kMmLd;
        slot = slot == kMmStages - 1 ? 0 : slot + 1;
        const int kend = (int)min((int64_t)kMmK, (K - c_s * kMmK + 3) & ~int64_t(3));  // zero-filled tail
#pragma unroll 2
        for (int kq = 0; kq < kend; kq += 4) {
            float4 a4[8], b4[8];
#pragma unroll
            for (int ii = 0; ii < 8; ++ii) a4[ii] = *reinterpret_cast<const float4*>(as + ii * 8 * kMmLd + kq);
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) b4[jj] = *reinterpret_cast<const float4*>(bs + jj * 32 * kMmLd + kq);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
#pragma unroll
                for (int ii = 0; ii < 8; ++ii) {
                    const float a = c == 0 ? a4[ii].x : c == 1 ? a4[ii].y : c == 2 ? a4[ii].z : a4[ii].w;
#pragma unroll
                    for (int jp = 0; jp < 4; ++jp) {
                        const float4& x0 = b4[2 * jp];
                        const float4& x1 = b4[2 * jp + 1];
                        const float b0 = c == 0 ? x0.x : c == 1 ? x0.y : c == 2 ? x0.z : x0.w;
                        const float b1 = c == 0 ? x1.x : c == 1 ? x1.y : c == 2 ? x1.z : x1.w;
                        acc[ii][jp] = fadd2(acc[ii][jp], pack2(mavp_term<OP>(a, b0), mavp_term<OP>(a, b1)));
                    }
                }
            }
        }
        const bool tile_end = c_s + 1 == nst;
        if (++nfold == kFoldStages || tile_end) {
#pragma unroll
            for (int ii = 0; ii < 8; ++ii)
#pragma unroll
                for (int jp = 0; jp < 4; ++jp) {
                    tot[ii][jp] = fadd2(tot[ii][jp], acc[ii][jp]);
                    acc[ii][jp] = 0ull;
                }
            nfold = 0;
        }
        if (tile_end) {  // epilogue: C = (1/d) * sum (Eq. 5's scalar factor), coalesced along j
            const int64_t i0 = (c_tile / tj) * kMmI, j0 = (c_tile % tj) * kMmJ;
#pragma unroll
            for (int ii = 0; ii < 8; ++ii) {
                const int64_t i = i0 + warp + 8 * ii;
#pragma unroll
                for (int jp = 0; jp < 4; ++jp) {
                    const int64_t ja = j0 + lane + 64 * jp, jb = ja + 32;
                    if (i < m) {
                        float* crow = C + i * ldc;
                        if (ja < p) crow[ja] = d == 1.0f ? lo_of(tot[ii][jp]) : inv_d * lo_of(tot[ii][jp]);
                        if (jb < p) crow[jb] = d == 1.0f ? hi_of(tot[ii][jp]) : inv_d * hi_of(tot[ii][jp]);
                    }
                    tot[ii][jp] = 0ull;
                }
            }
            c_s = 0;
            c_tile += G;
        } else {
            ++c_s;
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// K8s: small K (K <= 12 — the paper's N = 10 samples; Alg. 2 step 4 on 128^2-pixel images gives a
// 16384^2 C from only 10 terms per element).  There the tiled kernel is bound by its per-element
// staging (4 B cp.async per value) and by 1 CTA/SM of 234-register threads (ncu: issue 49%, warps
// active 12.5%, "wait" stalls), not by the 10 FMNMX per output.  K8s keeps a 256-column j-tile of B in
// REGISTERS (lane owns columns j0 + lane + 32 jj, jj < 8: 8 x KP values) and sweeps 32-row i-tiles of
// A through a double-buffered shared-memory stage (32 x K floats, warp-broadcast reads): per output
// K terms (FMNMX.XORSIGN, FADD2 over column pairs), the 1/d scale and one coalesced store.  Units =
// (j-tile, i-tile) in j-major order split evenly over a persistent grid, so a CTA reloads B only when
// its range crosses a j-tile.  Per element the k order is ascending from 0, as in K8 for K <= 32: the
// two kernels give bitwise-identical C (tested).
constexpr int kMsThreads = 256;
#ifndef MAPI_MS_JJ
#define MAPI_MS_JJ 4
#endif
constexpr int kMsJJ = MAPI_MS_JJ;          // B columns per lane (registers: kMsJJ x KP)
constexpr int kMsII = 32 / kMsJJ;          // A rows per warp  (accumulators: kMsII x kMsJJ)
constexpr int kMsI = 8 * kMsII, kMsJ = 32 * kMsJJ;

template <int OP, int KP>
__global__ void __launch_bounds__(kMsThreads) k_mavp_matmat_smallk(const float* __restrict__ A, int64_t m, int K,
                                                                 int64_t lda, const float* __restrict__ B,
                                                                 int64_t p, int64_t ldb, float d,
                                                                 float* __restrict__ C, int64_t ldc) {
    constexpr int JP = kMsJJ / 2, AR = (kMsI * KP + kMsThreads - 1) / kMsThreads;
    __shared__ float As[2][kMsI][KP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ni = (m + kMsI - 1) / kMsI, nj = (p + kMsJ - 1) / kMsJ, units = ni * nj;
    const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
    if (u0 >= u1) return;
    const float inv_d = 1.0f / d;
    float breg[kMsJJ][KP];
    int64_t cur_jt = -1;
    // A stage of unit u into registers (AR values per thread: kMsI x K floats)
    float ar[AR];
    auto load_a = [&](int64_t u) {
        const int64_t i0 = (u % ni) * kMsI;
#pragma unroll
        for (int h = 0; h < AR; ++h) {
            const int idx = tid + h * kMsThreads;
            const int r = idx / K, k = idx - r * K;
            ar[h] = (idx < kMsI * K && i0 + r < m) ? __ldg(A + (i0 + r) * lda + k) : 0.0f;
        }
    };
    auto store_a = [&](int buf) {
#pragma unroll
        for (int h = 0; h < AR; ++h) {
            const int idx = tid + h * kMsThreads;
            if (idx < kMsI * K) {
                const int r = idx / K, k = idx - r * K;
                As[buf][r][k] = ar[h];
            }
        }
    };
    load_a(u0);
    store_a(0);
    __syncthreads();
    int buf = 0;
    for (int64_t u = u0; u < u1; ++u) {
        const int64_t jt = u / ni, i0 = (u % ni) * kMsI, j0 = jt * kMsJ;
        if (jt != cur_jt) {  // (re)load this j-tile's B columns into registers
#pragma unroll
            for (int jj = 0; jj < kMsJJ; ++jj) {
                const int64_t j = j0 + lane + 32 * jj;
#pragma unroll
                for (int k = 0; k < KP; ++k) breg[jj][k] = (j < p && k < K) ? __ldg(B + j * ldb + k) : 0.0f;
            }
            cur_jt = jt;
        }
        if (u + 1 < u1) load_a(u + 1);  // next stage in flight during this unit's compute
        unsigned long long acc[kMsII][JP];
#pragma unroll
        for (int ii = 0; ii < kMsII; ++ii)
#pragma unroll
            for (int jp = 0; jp < JP; ++jp) acc[ii][jp] = 0ull;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            if (k < K) {
#pragma unroll
                for (int ii = 0; ii < kMsII; ++ii) {
                    const float a = As[buf][warp + 8 * ii][k];
#pragma unroll
                    for (int jp = 0; jp < JP; ++jp)
                        acc[ii][jp] = fadd2(acc[ii][jp], pack2(mavp_term<OP>(a, breg[2 * jp][k]),
                                                               mavp_term<OP>(a, breg[2 * jp + 1][k])));
                }
            }
        }
#pragma unroll
        for (int ii = 0; ii < kMsII; ++ii) {
            const int64_t i = i0 + warp + 8 * ii;
            if (i < m) {
                float* crow = C + i * ldc;
#pragma unroll
                for (int jp = 0; jp < JP; ++jp) {
                    const int64_t ja = j0 + lane + 64 * jp, jb = ja + 32;
                    if (ja < p) crow[ja] = d == 1.0f ? lo_of(acc[ii][jp]) : inv_d * lo_of(acc[ii][jp]);
                    if (jb < p) crow[jb] = d == 1.0f ? hi_of(acc[ii][jp]) : inv_d * hi_of(acc[ii][jp]);
                }
            }
        }
        if (u + 1 < u1) {
            store_a(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
}

}  // namespace mapi
