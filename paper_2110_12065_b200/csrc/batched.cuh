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
#include <cstdlib>
#include <cstring>
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
inline size_t batched_part_bytes(int64_t n, int32_t k);
inline size_t batched_ws_bytes(int64_t n, int32_t k) {
    const int64_t rb = (n + 255) / 256;
    return 256 + bal256(8 * (size_t)k) + bal256(4 * (size_t)k) + 2 * bal256(4 * (size_t)k * n) +
           bal256(batched_part_bytes(n, k)) + bal256(4 * (size_t)k * rb);
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
    p += bal256(batched_part_bytes(n, k));
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

// Y[v][j] = sum_s part[s][v][j] (s ascending); colpart[v][blk] = sum_{j in blk} |Y[v][j]| (l1, MAPI) or
// Y[v][j]^2 (sq: l2, the RPI comparator of Eq. 1).
__global__ void __launch_bounds__(256) k_batched_reduce(int64_t n, int32_t kv, int ks,
                                                        const float* __restrict__ part, float* __restrict__ Y,
                                                        float* __restrict__ colpart, int64_t rb, bool sq) {
    __shared__ float red[33];
    const int v = blockIdx.y;
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    float y = 0.0f;
    if (j < n) {
        for (int s = 0; s < ks; ++s) y += part[((int64_t)s * kv + v) * n + j];
        Y[(int64_t)v * n + j] = y;
    }
    const float a = block_sum(sq ? y * y : fabsf(y), red);
    if (threadIdx.x == 0) colpart[(int64_t)v * rb + blockIdx.x] = a;
}

// Per vector v (one CTA each): s = sum colpart (fixed order; sq: its square root, the l2 norm of RPI),
// W = Y / s, delta, trace, stop.
__global__ void __launch_bounds__(1024) k_batched_normalize(int64_t n, int32_t kv, int32_t t, float tol,
                                                            const float* __restrict__ Y,
                                                            const float* __restrict__ colpart, int64_t rb,
                                                            float* __restrict__ W, float* norms, float* deltas,
                                                            int32_t* status, int32_t* stop, bool sq) {
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
    const float s = sq ? sqrtf(red[32]) : red[32];
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

// ---------------------------------------------------------------------------------------------
// K4 v2 (default when rows are 16 B aligned): stream-K persistent tiles.
//
// Work = (row tile of 256 rows) x (vector tile of 64) x (k stage of 32): U units, split into equal
// contiguous ranges over G = #SMs CTAs (one CTA per SM), so every SM gets the same number of k-stages
// (no wave quantisation).  A CTA accumulates consecutive stages of one tile in registers and writes
// a partial tile when the tile (or its range) ends; k_batched_reduce2 adds the <= kMaxParts partials
// of each tile in CTA order (deterministic).  Stages are staged global -> shared with cp.async
// (16 B, zero-filled out of range) in a 3-deep ring.  Thread (tr, tv) = (lane, warp) owns rows
// tr + 32 i and vectors tv + 8 j (i, j < 8): A reads are conflict-free LDS.128 across the warp, W
// reads are warp-wide broadcasts.  Inner loop per term: FMNMX.XORSIGN + half an FADD2 (pairs of
// vectors); accumulators are folded every kFoldStages stages into a second set (chains <= 128 terms).
constexpr int kB2M = 256, kB2V = 64, kB2K = 32, kB2Threads = 256, kB2Stages = 3, kB2Ld = kB2K + 4;
constexpr int kFoldStages = 4;  // 4 x 32 = 128 terms per fp32 chain before folding
constexpr int kMaxParts = 8;

struct StreamK {
    int64_t row_tiles, vec_tiles, kstages, units;
    int grid;
};

inline StreamK streamk_plan(int64_t n, int32_t k, int sms) {
    StreamK p;
    p.row_tiles = (n + kB2M - 1) / kB2M;
    p.vec_tiles = (k + kB2V - 1) / kB2V;
    p.kstages = (n + kB2K - 1) / kB2K;
    p.units = p.row_tiles * p.vec_tiles * p.kstages;
    p.grid = (int)std::min<int64_t>(sms, std::max<int64_t>(1, p.units));
    return p;
}

// first CTA whose range [c*U/G, (c+1)*U/G) contains unit u
__host__ __device__ inline int64_t streamk_cta_of(int64_t u, int64_t U, int64_t G) {
    int64_t c = (u * G) / U;
    while (c + 1 < G && ((c + 1) * U) / G <= u) ++c;
    while (c > 0 && (c * U) / G > u) --c;
    return c;
}

inline bool streamk_ok(int64_t n, int32_t k, int sms) {
    const StreamK p = streamk_plan(n, k, sms);
    const int64_t max_parts = (p.kstages * p.grid + p.units - 1) / p.units + 1;  // ranges spanning a tile
    return max_parts <= kMaxParts;
}

__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
    return ((unsigned long long)__float_as_uint(hi) << 32) | (unsigned long long)__float_as_uint(lo);
}
__device__ __forceinline__ float lo_of(unsigned long long x) { return __uint_as_float((unsigned)(x & 0xffffffffu)); }
__device__ __forceinline__ float hi_of(unsigned long long x) { return __uint_as_float((unsigned)(x >> 32)); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// TV = vectors per thread (8: 256 threads, fold accumulators in registers; 4: 512 threads = 4 warps per
// scheduler for latency hiding, fold accumulators in shared memory).
template <int TV>
struct SkCfg {
    static constexpr int threads = 32 * (kB2V / TV);
    static constexpr int vstride = kB2V / TV;      // vectors of a thread: warp + vstride * j
    static constexpr bool smem_fold = TV == 4;
};

template <int OP, int TV>
__global__ void __launch_bounds__(SkCfg<TV>::threads, 1) k_batched_streamk(const float* __restrict__ A, int64_t n,
                                                                           int64_t lda, const float* __restrict__ W,
                                                                           int32_t kv, StreamK plan,
                                                                           float* __restrict__ part) {
    constexpr int NT = SkCfg<TV>::threads, VS = SkCfg<TV>::vstride, TP = TV / 2;  // TP: vector pairs
    extern __shared__ __align__(16) float smem[];
    float* As = smem;                                   // [stage][256][kB2Ld]
    float* Ws = smem + kB2Stages * kB2M * kB2Ld;        // [stage][64][kB2Ld]
    unsigned long long* fold = reinterpret_cast<unsigned long long*>(Ws + kB2Stages * kB2V * kB2Ld);  // [8*TP][NT]
    const int tid = threadIdx.x, tr = tid & 31, tv = tid >> 5;
    const int64_t U = plan.units, G = gridDim.x;
    const int64_t u0 = ((int64_t)blockIdx.x * U) / G, u1 = (((int64_t)blockIdx.x + 1) * U) / G;
    if (u0 >= u1) return;

    // load cursor: the (tile, k-stage) of the next stage to stage into shared memory
    int64_t l_tile = u0 / plan.kstages, l_ks = u0 % plan.kstages;
    constexpr int AQ = kB2M * (kB2K / 4) / NT;   // A chunks per thread per stage (8 or 4)
    constexpr int WQ = kB2V * (kB2K / 4) / NT;   // W chunks per thread per stage (2 or 1)
    constexpr int RS = NT / 8;                   // row stride between a thread's chunks
    const float* pA[AQ];
    const float* pW[WQ];
    uint32_t a_ok = 0, w_ok = 0;
    const int tr8 = tid >> 3, kq4 = (tid & 7) * 4;
    auto set_tile = [&](int64_t tile) {
        const int64_t rt = tile / plan.vec_tiles, vt = tile - rt * plan.vec_tiles;
        const int64_t row0 = rt * kB2M, v0 = vt * kB2V;
        a_ok = w_ok = 0;
#pragma unroll
        for (int i = 0; i < AQ; ++i) {
            const int64_t row = row0 + tr8 + RS * i;
            pA[i] = A + (row < n ? row : 0) * lda + kq4;
            a_ok |= (row < n ? 1u : 0u) << i;
        }
#pragma unroll
        for (int i = 0; i < WQ; ++i) {
            const int64_t v = v0 + tr8 + RS * i;
            pW[i] = W + (v < kv ? v : 0) * n + kq4;
            w_ok |= (v < kv ? 1u : 0u) << i;
        }
    };
    set_tile(l_tile);
    auto load_next = [&](int slot) {
        const int64_t k0 = l_ks * kB2K;
        const bool k_in = k0 + kq4 < n;
        float* as = As + slot * kB2M * kB2Ld + tr8 * kB2Ld + kq4;
        float* ws = Ws + slot * kB2V * kB2Ld + tr8 * kB2Ld + kq4;
#pragma unroll
        for (int i = 0; i < AQ; ++i) {
            const bool in = k_in && ((a_ok >> i) & 1u);
            cp_async16(as + RS * i * kB2Ld, in ? (const void*)(pA[i] + k0) : (const void*)A, in ? 16 : 0);
        }
#pragma unroll
        for (int i = 0; i < WQ; ++i) {
            const bool in = k_in && ((w_ok >> i) & 1u);
            cp_async16(ws + RS * i * kB2Ld, in ? (const void*)(pW[i] + k0) : (const void*)W, in ? 16 : 0);
        }
        if (++l_ks == plan.kstages) {
            l_ks = 0;
            set_tile(++l_tile);
        }
    };

    unsigned long long acc[8][TP];
    unsigned long long tot[SkCfg<TV>::smem_fold ? 1 : 8][SkCfg<TV>::smem_fold ? 1 : TP];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < TP; ++j) acc[i][j] = 0ull;
    if constexpr (SkCfg<TV>::smem_fold) {
#pragma unroll
        for (int q = 0; q < 8 * TP; ++q) fold[q * NT + tid] = 0ull;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < TP; ++j) tot[i][j] = 0ull;
    }

    const int64_t nst = u1 - u0;
    load_next(0);
    cp_async_commit();
    if (nst > 1) load_next(1);
    cp_async_commit();
    int nfold = 0, slot = 0, lslot = 2;
    int64_t c_tile = u0 / plan.kstages, c_ks = u0 % plan.kstages;  // compute cursor
    for (int64_t st = 0; st < nst; ++st) {
        cp_async_wait<1>();
        __syncthreads();
        if (st + 2 < nst) load_next(lslot);
        cp_async_commit();
        lslot = lslot == kB2Stages - 1 ? 0 : lslot + 1;
        const float* as = As + slot * kB2M * kB2Ld + tr * kB2Ld;
        const float* ws = Ws + slot * kB2V * kB2Ld + tv * kB2Ld;
        slot = slot == kB2Stages - 1 ? 0 : slot + 1;
#pragma unroll 2
        for (int kq = 0; kq < kB2K; kq += 4) {
            float4 a4[8], w4[TV];
#pragma unroll
            for (int i = 0; i < 8; ++i) a4[i] = *reinterpret_cast<const float4*>(as + i * 32 * kB2Ld + kq);
#pragma unroll
            for (int j = 0; j < TV; ++j) w4[j] = *reinterpret_cast<const float4*>(ws + j * VS * kB2Ld + kq);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float a = c == 0 ? a4[i].x : c == 1 ? a4[i].y : c == 2 ? a4[i].z : a4[i].w;
#pragma unroll
                    for (int jp = 0; jp < TP; ++jp) {
                        const float4& x0 = w4[2 * jp];
                        const float4& x1 = w4[2 * jp + 1];
                        const float w0 = c == 0 ? x0.x : c == 1 ? x0.y : c == 2 ? x0.z : x0.w;
                        const float w1 = c == 0 ? x1.x : c == 1 ? x1.y : c == 2 ? x1.z : x1.w;
                        acc[i][jp] = fadd2(acc[i][jp], pack2(mavp_term<OP>(a, w0), mavp_term<OP>(a, w1)));
                    }
                }
            }
        }
        const bool tile_end = (st + 1 == nst) || (c_ks + 1 == plan.kstages);
        if (++nfold == kFoldStages || tile_end) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < TP; ++j) {
                    if constexpr (SkCfg<TV>::smem_fold) {
                        unsigned long long& f = fold[(i * TP + j) * NT + tid];
                        f = fadd2(f, acc[i][j]);
                    } else {
                        tot[i][j] = fadd2(tot[i][j], acc[i][j]);
                    }
                    acc[i][j] = 0ull;
                }
            nfold = 0;
        }
        if (tile_end) {
            // partial slot of this CTA within the tile: CTA index minus the tile's first CTA
            const int64_t p = (int64_t)blockIdx.x - streamk_cta_of(c_tile * plan.kstages, U, G);
            float* out = part + ((c_tile * kMaxParts + p) * kB2V) * kB2M;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int jp = 0; jp < TP; ++jp) {
                    const int r = tr + 32 * i, v = tv + VS * (2 * jp);
                    unsigned long long x;
                    if constexpr (SkCfg<TV>::smem_fold) {
                        x = fold[(i * TP + jp) * NT + tid];
                        fold[(i * TP + jp) * NT + tid] = 0ull;
                    } else {
                        x = tot[i][jp];
                        tot[i][jp] = 0ull;
                    }
                    out[(int64_t)v * kB2M + r] = lo_of(x);
                    out[(int64_t)(v + VS) * kB2M + r] = hi_of(x);
                }
        }
        if (++c_ks == plan.kstages) {
            c_ks = 0;
            ++c_tile;
        }
    }
    cp_async_wait<0>();
}

// Y[v][j] = sum of the tile's partials in CTA order; colpart[v][blk] = sum |Y[v][j]| (sq: Y^2) over 256 rows.
__global__ void __launch_bounds__(256) k_batched_reduce2(int64_t n, int32_t kv, StreamK plan, int G,
                                                         const float* __restrict__ part, float* __restrict__ Y,
                                                         float* __restrict__ colpart, int64_t rb, bool sq) {
    __shared__ float red[33];
    const int v = blockIdx.y;
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    float y = 0.0f;
    if (j < n) {
        const int64_t rt = j / kB2M, vt = v / kB2V;
        const int64_t tile = rt * plan.vec_tiles + vt;
        const int64_t c0 = streamk_cta_of(tile * plan.kstages, plan.units, G);
        const int64_t c1 = streamk_cta_of(tile * plan.kstages + plan.kstages - 1, plan.units, G);
        for (int64_t p = 0; p <= c1 - c0; ++p)
            y += part[((tile * kMaxParts + p) * kB2V + (v - vt * kB2V)) * kB2M + (j - rt * kB2M)];
        Y[(int64_t)v * n + j] = y;
    }
    const float a = block_sum(sq ? y * y : fabsf(y), red);
    if (threadIdx.x == 0) colpart[(int64_t)v * rb + blockIdx.x] = a;
}

inline size_t streamk_part_bytes(int64_t n, int32_t k) {
    const int64_t tiles = ((n + kB2M - 1) / kB2M) * ((k + kB2V - 1) / kB2V);
    return sizeof(float) * (size_t)tiles * kMaxParts * kB2V * kB2M;
}
template <int TV>
inline size_t streamk_smem_bytes() {
    return sizeof(float) * kB2Stages * (kB2M + kB2V) * kB2Ld +
           (SkCfg<TV>::smem_fold ? sizeof(unsigned long long) * 8 * (TV / 2) * SkCfg<TV>::threads : 0);
}

static thread_local char g_batched_err[256] = "";
inline const char* batched_last_error() { return g_batched_err; }

inline size_t batched_part_bytes(int64_t n, int32_t k) {
    return std::max(sizeof(float) * (size_t)64 * k * n, streamk_part_bytes(n, k));
}

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
    // v2 (stream-K) needs 16 B-aligned rows of A and of W (n % 4 == 0); MAPI_BATCHED_PATH=v1 forces v1
    const char* env = getenv("MAPI_BATCHED_PATH");
    const bool v2 = !(env && strcmp(env, "v1") == 0) && reinterpret_cast<uintptr_t>(A) % 16 == 0 && lda % 4 == 0 &&
                    n % 4 == 0 && streamk_ok(n, k, sms);
    const StreamK plan = streamk_plan(n, k, sms);
    // v2 (256 threads, 8x8 register tiles) is the default; MAPI_BATCHED_PATH=v3 selects the 512-thread
    // 8x4 variant with the fold in shared memory (measured 63.5% vs 64.5% of the FMNMX peak at cfg4)
    const bool v3 = env && strcmp(env, "v3") == 0;
    auto k2 = op == 2 ? k_batched_streamk<2, 8> : (op == 1 ? k_batched_streamk<1, 8> : k_batched_streamk<0, 8>);
    auto k3 = op == 2 ? k_batched_streamk<2, 4> : (op == 1 ? k_batched_streamk<1, 4> : k_batched_streamk<0, 4>);
    const bool sq = op == 2;  // RPI: l2 normalisation (Eq. 1)
    const size_t sm2 = streamk_smem_bytes<8>(), sm3 = streamk_smem_bytes<4>();
    if (v2) {
        if ((e = cudaFuncSetAttribute(v3 ? k3 : k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(v3 ? sm3 : sm2))) !=
            cudaSuccess)
            return batched_cuda_fail(e, "smem attribute");
    }
    if (timing) cudaEventRecord(*ev_a, s);
    for (int32_t t = 0; t < iters; ++t) {
        if (v2) {
            if (v3)
                k3<<<plan.grid, SkCfg<4>::threads, sm3, s>>>(A, n, lda, B.W, k, plan, B.part);
            else
                k2<<<plan.grid, SkCfg<8>::threads, sm2, s>>>(A, n, lda, B.W, k, plan, B.part);
            k_batched_reduce2<<<gr, 256, 0, s>>>(n, k, plan, plan.grid, B.part, B.Y, B.colpart, B.rb, sq);
        } else {
            if (op == 2)
                k_batched_partial<2><<<gp, kBThreads, 0, s>>>(A, n, lda, B.W, k, kslice, B.part);
            else if (op == 1)
                k_batched_partial<1><<<gp, kBThreads, 0, s>>>(A, n, lda, B.W, k, kslice, B.part);
            else
                k_batched_partial<0><<<gp, kBThreads, 0, s>>>(A, n, lda, B.W, k, kslice, B.part);
            k_batched_reduce<<<gr, 256, 0, s>>>(n, k, ks, B.part, B.Y, B.colpart, B.rb, sq);
        }
        k_batched_normalize<<<k, 1024, 0, s>>>(n, k, t, tol, B.Y, B.colpart, B.rb, B.W, norms, deltas, B.status,
                                               B.stop, sq);
        launches.fetch_add(3, std::memory_order_relaxed);
        if ((e = cudaGetLastError()) != cudaSuccess) return batched_cuda_fail(e, "batched launch");
    }
    if (timing) cudaEventRecord(*ev_b, s);
    if ((e = cudaMemcpyAsync(W_out, B.W, 4 * (size_t)k * n, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return batched_cuda_fail(e, "copy W");
    return MAPI_OK;
}

// Sync, read per-vector status / iteration counts; returns the status of the first vector that stopped
// on an error (its index in *bad, its iteration count in *bad_iter), MAPI_OK if none did.
inline mapi_status batched_finish(void* ws, int64_t n, int32_t k, cudaStream_t s, int32_t* iters_done,
                                  int32_t* bad, int32_t* bad_iter) {
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
        if (h[2 * v] != 0 && worst == MAPI_OK) {
            worst = (mapi_status)h[2 * v];
            *bad = v;
            *bad_iter = h[2 * v + 1];
        }
    }
    free(h);
    return worst;
}

}  // namespace mapi
