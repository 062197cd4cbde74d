// resident.cuh — K2r: persistent MAPI iteration with the whole matrix held ON CHIP (TMEM + shared memory).
//
// Alg. 1 for mid-size n (cfg2's 4096 x 4096 D_i = 64 MiB).  Every iteration of K2t
// re-reads A from L2 (~453 KB per SM per iteration, L2-bandwidth/latency bound at ~13 us/iteration).
// But 148 SMs hold 148 x (256 KB TMEM + 227 KB shared memory) = 70 MB on chip, more than D_i.  K2r
// loads its CTA's rows ONCE per call, into tensor memory (`tcgen05.st`, 16 rows of 4096) and shared
// memory (kResSmemRows rows), and every iteration reads them back with `tcgen05.ld` / `LDS.128`: no
// L2 or HBM traffic for A inside the loop.  TMEM is used purely as storage (no MMA: MAVP is not a
// contraction, the tensor cores cannot compute sign(a w) min(|a|,|w|)).
//
// Thread mapping (NW warps, 1 CTA per SM, cooperative launch): quarter q = warp % 4 (the TMEM lane
// quarter a warp may access), group g = warp / 4.  Thread (q, lane) is "column lane" L = 32q + lane
// and owns the 32 columns [32L, 32L + 32) of EVERY row of the CTA (n <= 4096 = 128 x 32), so it keeps
// those 32 entries of w_t in registers for the whole pass.  Local rows 0..15 live in TMEM (row i =
// TMEM columns [32i, 32i + 32) of the 128 lanes), local rows 16.. in shared memory (row-major, 4096
// floats per row); group g computes TMEM rows [g TR, (g+1) TR) and shared rows [g SR, (g+1) SR).
// Within a row slice, the 8 float4 chunks are visited in the lane-rotated order c = (m + lane) % 8
// (conflict-free LDS.128: the 8 lanes of a quarter-warp phase hit 8 distinct 4-bank groups); the
// TMEM copy and the w registers are stored in the same rotated order so the pairing is static.
//
// Per iteration: every thread forms its 32-term partial of each of its rows (4 chains: FMNMX.XORSIGN
// + FADD2, pairwise), the warp reduces its P partials across the 32 lanes with a reduce-scatter
// butterfly (P + log2 steps shuffles instead of 5P), the 4 quarters meet in shared memory
// (y_i = (q0 + q1) + (q2 + q3)), warp 0 writes y and the CTA's fp64 |y| partial, ONE grid barrier,
// then every CTA forms s_t (fixed order), w_{t+1} = fp32(y/s_t) for all n and the fp64 delta_t
// exactly as K2t does (identical bits and stop decision in every CTA).  Deterministic for a given
// (n, grid).  Requirements: n <= 4096, ceil(n / grid) <= 16 + kResSmemRows, 1 CTA per SM.
#pragma once
#include "dense.cuh"
#include "mapi_common.cuh"

namespace mapi {

constexpr int kResLanes = 128;                   // TMEM lanes = column lanes
constexpr int kResCPL = 32;                      // columns per lane
constexpr int kResNPad = kResLanes * kResCPL;    // 4096: padded row length (max n)
constexpr int kResTmemRows = 512 / kResCPL;      // 16 rows in the 512 TMEM columns
constexpr int kResSmemRows = 12;                 // rows in shared memory (192 KB)
constexpr int kResMaxRows = kResTmemRows + kResSmemRows;
constexpr int kResDeflMax = 8;                   // fused deflation: at most 8 previous components

// smem_rows = rows kept in shared memory (kResSmemRows minus the register-resident rows)
inline size_t resident_smem_bytes(int smem_rows = kResSmemRows) {
    return sizeof(float) * ((size_t)smem_rows * kResNPad + kResNPad + 4 * 32) + sizeof(double) * 64 + 16;
}

__device__ __forceinline__ void tmem_ld32(uint32_t ta, float (&v)[32]) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta));
}
// wait for this thread's outstanding tcgen05.ld; the loaded registers are "+r" operands, so no use of
// them can be scheduled above the wait (the load writes them asynchronously)
__device__ __forceinline__ void tmem_wait_ld(float (&v)[32]) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.wait::ld.sync.aligned;"
        : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
          "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]),
          "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
          "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
        :
        : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t ta, const float (&v)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(ta), "r"(__float_as_uint(v[0])),
                 "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3]))
                 : "memory");
}
__device__ __forceinline__ void st_tagged(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_tagged(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_cluster_f64(double* local, uint32_t rank, double v) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
// fixed-shape pairwise tree over NW per-warp partials in shared memory (same order in every CTA)
template <int NW>
__device__ __forceinline__ double res_tree(const double* v) {
    double a[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) a[i] = v[i];
#pragma unroll
    for (int h = NW / 2; h > 0; h >>= 1)
#pragma unroll
        for (int i = 0; i < h; ++i) a[i] = a[2 * i] + a[2 * i + 1];
    return a[0];
}
__device__ __forceinline__ void tmem_st32(uint32_t ta, const float (&v)[32]) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ unsigned long long res_fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long res_pack2(float x, float y) {
    return (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(y) << 32);
}

// 32 terms (one row slice) against the thread's 32 w registers: 4 chains of 8 (two FADD2 pairs),
// pairwise final tree.  Same pairing in every row, TMEM or shared.
template <int OP>
__device__ __forceinline__ float res_row32(const float (&a)[32], const float (&w)[32]) {
    unsigned long long p0 = 0, p1 = 0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        p0 = res_fadd2(p0, res_pack2(mavp_term<OP>(a[4 * m], w[4 * m]), mavp_term<OP>(a[4 * m + 1], w[4 * m + 1])));
        p1 = res_fadd2(p1, res_pack2(mavp_term<OP>(a[4 * m + 2], w[4 * m + 2]), mavp_term<OP>(a[4 * m + 3], w[4 * m + 3])));
    }
    return (__uint_as_float((uint32_t)p0) + __uint_as_float((uint32_t)(p0 >> 32))) +
           (__uint_as_float((uint32_t)p1) + __uint_as_float((uint32_t)(p1 >> 32)));
}

// Reduce PP per-lane partials across the 32 lanes: reduce-scatter butterfly (at offset o the lanes with
// bit o set keep the upper half of the live values, the others the lower half; each adds its partner's
// copy), then plain butterfly steps.  Returns the full 32-lane sum of value index res_row_of<PP>(lane).
template <int PP>
__device__ __forceinline__ float res_lane_reduce(float (&v)[PP], int lane) {
#pragma unroll
    for (int j = 0; (PP >> j) > 1; ++j) {
        const int o = 16 >> j, half = PP >> (j + 1);
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = up ? v[i] : v[i + half];
            const float keep = up ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    float x = v[0];
    constexpr int LOGPP = PP >= 16 ? 4 : (PP >= 8 ? 3 : (PP >= 4 ? 2 : (PP >= 2 ? 1 : 0)));
#pragma unroll
    for (int o = 16 >> LOGPP; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
template <int PP>
__device__ __forceinline__ int res_row_of(int lane) {
    int r = 0;
#pragma unroll
    for (int j = 0; (PP >> j) > 1; ++j) r = 2 * r + ((lane >> (4 - j)) & 1);
    return r;
}

// one-time load of a 32-column row slice in rotated chunk order (zero beyond n / for absent rows)
__device__ __forceinline__ void res_load_slice(const float* A, int64_t lda, int64_t n, int64_t row, bool valid,
                                               int L, int lane, bool vec4, float (&v)[32]) {
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const int c = (m + lane) & 7;
        const int64_t k0 = (int64_t)kResCPL * L + 4 * c;
        const float* src = A + row * lda + k0;
        if (valid && vec4 && k0 + 3 < n) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(src));
            v[4 * m] = x.x; v[4 * m + 1] = x.y; v[4 * m + 2] = x.z; v[4 * m + 3] = x.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) v[4 * m + e] = (valid && k0 + e < n) ? __ldg(src + e) : 0.0f;
        }
    }
}

#ifdef MAPI_RES_TRACE
__device__ long long g_res_trace[8 * 512];  // investigation builds only (scripts/probe_k2r.cu)
__device__ int g_res_polls[148 * 512];  // poll rounds of thread 0 per (CTA, iteration)
#define RES_STAMP(t, k) \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (t) < 512) g_res_trace[(t) * 8 + (k)] = clock64()
#define RES_POLLS(t, c) \
    if (threadIdx.x == 0 && (t) < 512 && blockIdx.x < 148) g_res_polls[blockIdx.x * 512 + (t)] = (c)
#else
#define RES_POLLS(t, c)
#define RES_STAMP(t, k)
#endif

// CL: 1 = every CTA gathers all of y_t and forms all n quotients itself; 2 = CTA pairs (a 2-CTA
// cluster: 148 SMs hold 74 pairs) split the epilogue: each CTA polls HALF of y_t (halving the L2 read
// volume of the exchange, the bound of a poll round) and forms half of w_{t+1}, written into both CTAs'
// shared memory with DSMEM stores; the |y| and delta partials cross the pair the same way, each behind
// one barrier.cluster (release / acquire).
template <int OP, int NW, int CL = 1, int RR = 0>
__global__ void __launch_bounds__(NW * 32, 1) k_iterate_resident(IterArgs p) {
    constexpr int NT = NW * 32, G = NW / 4;                    // threads, warp groups
    constexpr int SMR = kResSmemRows - G * RR;                 // rows in shared memory
    constexpr int TR = kResTmemRows / G, SR = SMR / G, P = TR + RR + SR;
    constexpr int PP = P <= 2 ? 2 : (P <= 4 ? 4 : (P <= 8 ? 8 : 16));
    static_assert(kResTmemRows % G == 0 && SMR % G == 0 && SMR >= 0 && P <= 16, "row split");
    extern __shared__ __align__(16) float ws_[];
    float* a_s = ws_;                                           // SMR x 4096
    float* w_s = a_s + (size_t)SMR * kResNPad;                  // 4096 (w_t, zero-padded)
    float* yq = w_s + kResNPad;                                 // [4][32] quarter partials of y
    double* red = reinterpret_cast<double*>(yq + 4 * 32);       // 64: per-warp partials
    uint32_t* tslot = reinterpret_cast<uint32_t*>(red + 64);
    const int64_t n = p.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q = warp & 3, g = warp >> 2;
    const int L = 32 * q + lane;
    const int64_t r0 = (int64_t)blockIdx.x * n / gridDim.x, r1 = (int64_t)(blockIdx.x + 1) * n / gridDim.x;
    const int R = (int)(r1 - r0);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *tslot;
    const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(kResCPL * TR * g);

    // ---- one-time staging of this CTA's rows (A does not change across iterations)
    const bool vec4 = (n % 4 == 0) && (p.lda % 4 == 0) && ((reinterpret_cast<uintptr_t>(p.A) & 15) == 0);
    float areg[RR > 0 ? RR : 1][32];
    if (NW == 8 && p.dk > 0) {  // (the 16-warp variant has no register room for it: never fused)
        // fused L2 deflation (mapi_pca_topk): stage D_i = fp32(C - sum_{m<dk} p_m r_m^T) straight from C
        // instead of a separate build kernel writing D_i to memory.  Per element the same fp64 sequence as
        // k_build_deflated (v = C; v = fma(-p_m[row], r_m[col], v), m ascending; one rounding): bitwise the
        // same D_i.  Position-major: at position m every lane handles its column chunk (m + lane) % 8 (the
        // rotated layout) of all its rows, with r_m of those 4 columns in registers, the rows' p_m values
        // in shared memory (staged once) and all the rows' C loads of a position in flight together.
        constexpr int NR = TR + SR;  // TMEM + shared rows per thread (register rows: a row-major pass below)
        double* p_s = reinterpret_cast<double*>(w_s);  // [kResMaxRows][kResDeflMax], w_s is free until later
        for (int e = tid; e < kResMaxRows * kResDeflMax; e += NT) {
            const int i = e / kResDeflMax, mm = e % kResDeflMax;
            p_s[e] = (i < R && mm < p.dk) ? -__ldg(p.dP + (int64_t)mm * n + r0 + i) : 0.0;
        }
        __syncthreads();
        auto row_of = [&](int j) {  // local row index of this thread's j-th row (TMEM, then shared)
            return j < TR ? g * TR + j : kResTmemRows + G * RR + g * SR + (j - TR);
        };
        // rows per load batch (register budget: r_m of 4 columns = 64 registers)
        constexpr int NB = NR % 4 == 0 ? 4 : (NR % 2 == 0 ? 2 : 1);
#pragma unroll 1
        for (int m = 0; m < 8; ++m) {
            const int c = (m + lane) & 7;
            const int64_t k0 = (int64_t)kResCPL * L + 4 * c;
            double r4[kResDeflMax][4];
#pragma unroll
            for (int mm = 0; mm < kResDeflMax; ++mm)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    r4[mm][e] = (mm < p.dk && k0 + e < n) ? __ldg(p.dR + (int64_t)mm * n + k0 + e) : 0.0;
#pragma unroll 1
            for (int jb = 0; jb < NR; jb += NB) {
            float x[NB][4];
#pragma unroll
            for (int jj = 0; jj < NB; ++jj) {
                const int j = jb + jj;
                const int i = row_of(j);
                const bool valid = i < R;
                const float* src = p.A + (r0 + (valid ? i : 0)) * p.lda + k0;
                if (valid && vec4 && k0 + 3 < n) {
                    const float4 t = __ldg(reinterpret_cast<const float4*>(src));
                    x[jj][0] = t.x; x[jj][1] = t.y; x[jj][2] = t.z; x[jj][3] = t.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) x[jj][e] = (valid && k0 + e < n) ? __ldg(src + e) : 0.0f;
                }
            }
#pragma unroll
            for (int jj = 0; jj < NB; ++jj) {
                const int j = jb + jj;
                const int i = row_of(j);
                double v[4] = {(double)x[jj][0], (double)x[jj][1], (double)x[jj][2], (double)x[jj][3]};
#pragma unroll
                for (int mm = 0; mm < kResDeflMax; ++mm) {
                    if (mm < p.dk) {
                        const double pm = p_s[i * kResDeflMax + mm];
#pragma unroll
                        for (int e = 0; e < 4; ++e) v[e] = fma(pm, r4[mm][e], v[e]);
                    }
                }
                float o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) o[e] = (i < R && k0 + e < n) ? (float)v[e] : 0.0f;
                if (j < TR) {
                    tmem_st4(ta + (uint32_t)(kResCPL * j + 4 * m), o);
                } else {
                    reinterpret_cast<float4*>(a_s + (size_t)(g * SR + (j - TR)) * kResNPad)[8 * L + c] =
                        make_float4(o[0], o[1], o[2], o[3]);
                }
            }
            }
        }
        // register rows, row-major (static register indices): chunk by chunk with r_m from L2
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
            const int i = kResTmemRows + g * RR + rr;
            float x[32];
            res_load_slice(p.A, p.lda, n, r0 + i, i < R, L, lane, vec4, x);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int c = (m + lane) & 7;
                const int64_t k0 = (int64_t)kResCPL * L + 4 * c;
                double v[4] = {(double)x[4 * m], (double)x[4 * m + 1], (double)x[4 * m + 2], (double)x[4 * m + 3]};
                for (int mm = 0; mm < p.dk; ++mm) {
                    const double pm = p_s[i * kResDeflMax + mm];
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        v[e] = fma(pm, k0 + e < n ? __ldg(p.dR + (int64_t)mm * n + k0 + e) : 0.0, v[e]);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) areg[rr][4 * m + e] = (i < R && k0 + e < n) ? (float)v[e] : 0.0f;
            }
        }
        __syncthreads();  // p_s (in w_s) is overwritten below
    } else {
    // two rows' loads in flight at a time (the staging is latency-bound: one row per trip took ~2x longer)
#pragma unroll 1
    for (int r = 0; r < TR; r += 2) {
        const int i = g * TR + r;
        float v[32], u[32];
        res_load_slice(p.A, p.lda, n, r0 + i, i < R, L, lane, vec4, v);
        if (r + 1 < TR) res_load_slice(p.A, p.lda, n, r0 + i + 1, i + 1 < R, L, lane, vec4, u);
        tmem_st32(ta + (uint32_t)(kResCPL * r), v);
        if (r + 1 < TR) tmem_st32(ta + (uint32_t)(kResCPL * (r + 1)), u);
    }
#pragma unroll
    for (int r = 0; r < RR; ++r) {
        const int i = kResTmemRows + g * RR + r;
        res_load_slice(p.A, p.lda, n, r0 + i, i < R, L, lane, vec4, areg[r]);
    }
#pragma unroll 1
    for (int r = 0; r < SR; r += 2) {
        float v[2][32];
#pragma unroll
        for (int h = 0; h < 2; ++h)
            if (r + h < SR) {
                const int i = kResTmemRows + G * RR + g * SR + r + h;
                res_load_slice(p.A, p.lda, n, r0 + i, i < R, L, lane, vec4, v[h]);
            }
#pragma unroll
        for (int h = 0; h < 2; ++h)
            if (r + h < SR) {
                float4* dst = reinterpret_cast<float4*>(a_s + (size_t)(g * SR + r + h) * kResNPad) + 8 * L;
#pragma unroll
                for (int m = 0; m < 8; ++m)
                    dst[(m + lane) & 7] = make_float4(v[h][4 * m], v[h][4 * m + 1], v[h][4 * m + 2], v[h][4 * m + 3]);
            }
    }
    }
    for (int k = tid; k < kResNPad; k += NT) w_s[k] = k < n ? p.b0[k] : 0.0f;
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();

    float wr[32];  // w_t at this thread's columns, rotated order
    auto load_w = [&]() {
        const float4* src = reinterpret_cast<const float4*>(w_s) + 8 * L;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const float4 x = src[(m + lane) & 7];
            wr[4 * m] = x.x; wr[4 * m + 1] = x.y; wr[4 * m + 2] = x.z; wr[4 * m + 3] = x.w;
        }
    };
    load_w();

    int32_t done = 0, status = kStOk;
    uint64_t* yt = reinterpret_cast<uint64_t*>(p.y);  // [2][n] tagged words: (t + 1) << 32 | bits(y)
    double* wsum = red;                               // [CL * NW] per-warp |y| partials
    double* dsum = red + 32;                          // [CL * NW] per-warp delta partials
    constexpr int YH = kResNPad / NT / CL;            // y values per thread in the normalisation
    const uint32_t half = CL == 2 ? cluster_ctarank() : 0u;
    const int64_t kb = (int64_t)half * (kResNPad / CL);  // first element of this CTA's share
    for (int32_t t = 0; t < p.iters; ++t) {
        uint64_t* yb = yt + (t & 1) * n;
        const uint32_t tag = (uint32_t)t + 1u;
        RES_STAMP(t, 0);
        float part[PP];
#pragma unroll
        for (int r = 0; r < PP; ++r) part[r] = 0.0f;
        // TMEM row i is in flight while shared-memory row i is computed (the two read paths overlap).
        // Row guards are warp-uniform (tcgen05.ld / wait are .sync.aligned).
        float at[32];
        if (g * TR < R) tmem_ld32(ta, at);
#pragma unroll
        for (int i = 0; i < (TR > SR + RR ? TR : SR + RR); ++i) {
            if (i < RR) {  // register row (rows beyond R were staged as zeros: no guard needed)
                part[TR + i] = res_row32<OP>(areg[i], wr);
            } else if (i < RR + SR && kResTmemRows + G * RR + g * SR + (i - RR) < R) {
                const int sr = i - RR;
                const float4* src = reinterpret_cast<const float4*>(a_s + (size_t)(g * SR + sr) * kResNPad) + 8 * L;
                float as[32];
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const float4 x = src[(m + lane) & 7];
                    as[4 * m] = x.x; as[4 * m + 1] = x.y; as[4 * m + 2] = x.z; as[4 * m + 3] = x.w;
                }
                part[TR + RR + sr] = res_row32<OP>(as, wr);
            }
            if (i < TR && g * TR + i < R) {
                tmem_wait_ld(at);
                part[i] = res_row32<OP>(at, wr);
                if (i + 1 < TR && g * TR + i + 1 < R) tmem_ld32(ta + (uint32_t)(kResCPL * (i + 1)), at);
            }
        }
        RES_STAMP(t, 1);
        const float rv = res_lane_reduce<PP>(part, lane);
        {
            const int ri = res_row_of<PP>(lane);
            if ((lane & (32 / PP - 1)) == 0 && ri < P) {
                const int i = ri < TR ? g * TR + ri
                            : (ri < TR + RR ? kResTmemRows + g * RR + (ri - TR)
                                            : kResTmemRows + G * RR + g * SR + (ri - TR - RR));
                yq[q * 32 + i] = rv;
            }
        }
        __syncthreads();
        // publish this CTA's rows: one 8-byte word per row carries the value AND its iteration tag, so
        // the exchange needs no grid barrier, fence or counter (a reader that sees the tag sees the value)
        RES_STAMP(t, 2);
        if (warp == 0 && lane < R) {
            const float v = (yq[lane] + yq[32 + lane]) + (yq[64 + lane] + yq[96 + lane]);
            st_tagged(yb + r0 + lane, ((uint64_t)tag << 32) | __float_as_uint(v));
        }
        RES_STAMP(t, 3);
        // gather y_t (this CTA's share: all of it for CL = 1, half for CL = 2): every thread polls its YH
        // words until they carry this iteration's tag
        float yr[YH];
        int rounds = 0;
        {
            uint32_t pending = 0;
#pragma unroll
            for (int j = 0; j < YH; ++j) {
                yr[j] = 0.0f;
                if (kb + tid + (int64_t)j * NT < n) pending |= 1u << j;
            }
            while (pending) {
                ++rounds;
                uint64_t xv[YH];  // all loads of a round in flight together, then the tag checks
#pragma unroll
                for (int j = 0; j < YH; ++j)
                    xv[j] = (pending & (1u << j)) ? ld_tagged(yb + kb + tid + (int64_t)j * NT) : 0;
#pragma unroll
                for (int j = 0; j < YH; ++j) {
                    if ((pending & (1u << j)) && (uint32_t)(xv[j] >> 32) == tag) {
                        yr[j] = __uint_as_float((uint32_t)xv[j]);
                        pending &= ~(1u << j);
                    }
                }
            }
        }
        RES_POLLS(t, rounds);
        RES_STAMP(t, 4);
        // s_t: per-thread fp64 partials in a fixed order, warp butterflies, then the CL x NW warp partials
        // (half 0's warps, then half 1's) in a fixed tree: the same element -> thread mapping in every CTA
        // and cluster gives identical s_t everywhere
        {
            double ap = 0.0;
#pragma unroll
            for (int j = 0; j < YH; ++j) {
                const double yd = (double)yr[j];
                ap += (OP == 2) ? yd * yd : fabs(yd);
            }
            ap = warp_sum(ap);
            if (lane == 0) {
                wsum[half * NW + warp] = ap;
                if constexpr (CL == 2) st_cluster_f64(&wsum[half * NW + warp], half ^ 1u, ap);
            }
        }
        if constexpr (CL == 2) cluster_sync_all(); else __syncthreads();
        RES_STAMP(t, 5);
        const double s = norm_final<OP>(res_tree<CL * NW>(wsum));
        if (!(s > 0.0) || isinf(s)) {  // uniform across the grid
            status = (s == 0.0) ? kStDegenerate : kStNonfinite;
            break;
        }
        // w_{t+1} = fp32(y / s_t) with s_t in fp64, evaluated in fp32 pairs: 1/s_t = rh + rl (fp64
        // reciprocal split into two floats), q = p + (e + y rl) with p = y rh and e = fma(y, rh, -p) its
        // exact error: |q - y/s_t| ~ 2^-47 |q|, so the fp32 result equals fp32(y / s_t) except when y/s_t
        // lies within ~2^-47 (relative) of an fp32 rounding boundary.  No fp64 conversion per element
        // (F2F is the bottleneck of a per-element fp64 quotient: 4096 per CTA per iteration).  delta_t:
        // fp32 |w_{t+1} - w_t| per element, fp32 within a thread (YH terms), fp64 across threads.
        // Branch-free over the padded 4096: beyond n, y = 0 and w_s = 0, so w stays 0 and adds 0 to delta.
        const double rs = 1.0 / s;
        const float rh = (float)rs, rl = (float)(rs - (double)rh);
        float dv = 0.0f;
#pragma unroll
        for (int j = 0; j < YH; ++j) {
            const int k = (int)kb + tid + j * NT;
            const float pj = yr[j] * rh;
            const float wn = pj + fmaf(yr[j], rl, fmaf(yr[j], rh, -pj));
            dv += fabsf(wn - w_s[k]);
            w_s[k] = wn;
            if constexpr (CL == 2) st_cluster(&w_s[k], half ^ 1u, wn);
        }
        double dpart = (double)dv;
        RES_STAMP(t, 7);
        dpart = warp_sum(dpart);
        if (lane == 0) {
            dsum[half * NW + warp] = dpart;
            if constexpr (CL == 2) st_cluster_f64(&dsum[half * NW + warp], half ^ 1u, dpart);
        }
        // orders the w_s writes (both halves) before load_w
        if constexpr (CL == 2) cluster_sync_all(); else __syncthreads();
        RES_STAMP(t, 6);
        const double delta = res_tree<CL * NW>(dsum);
        if (blockIdx.x == 0 && tid == 0) {
            if (p.norms) p.norms[t] = (float)s;
            if (p.deltas) p.deltas[t] = (float)delta;
        }
        done = t + 1;
        if (p.tol > 0.0f && delta < (double)p.tol) break;
        load_w();
    }
    if constexpr (CL == 2) cluster_sync_all();  // no DSMEM access may target an exited CTA
    for (int64_t k = r0 + tid; k < r1; k += NT) p.w_out[k] = w_s[k];
    if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

}  // namespace mapi
