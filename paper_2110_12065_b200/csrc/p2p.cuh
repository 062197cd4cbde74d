// p2p.cuh — multi-GPU MAPI with the exchange fused into the persistent iteration kernels (SURVEY §8(e),
// NEXT-4): K2p (row-sharded full rows) and K2sp (the symmetric kernel K2s with its
// upper-triangle task list split over the ranks).  One cooperative launch per rank runs all iterations.
//
// Every rank owns an EXCHANGE buffer in its HBM (mapi_p2p_alloc, mapped into every peer with CUDA IPC):
//     [flag u64 @0][y: 2 parities x world x n f32 @256][rank totals: 2 parities x world f64]
// The arrival protocol (both kernels), global iteration e, parity e & 1:
//   1. the CTAs store their share of the exchanged data into every rank's buffer (NVLink P2P stores,
//      coalesced: consecutive threads on consecutive elements) and fence at system scope;
//   2. a LOCAL grid barrier (gpu scope): every store of this rank is ordered before it;
//   3. CTA 0 release-adds 1 to every rank's flag (system scope): ONE arrival per rank per iteration;
//   4. every CTA waits (acquire, system scope) until its own flag reaches base + (e + 1 - epoch0) x world.
// A rank can be at most one iteration ahead of the slowest (it needs everyone's arrival to leave one), and
// its next writes go to the other parity, which the slow rank has finished reading.  The flag counts
// monotonically across calls (the host carries epoch and flag base: + published and + published x world),
// so no reset or host barrier is needed between calls.  A 10 s %globaltimer bound on the wait turns a
// missing peer into an error instead of a hang.  The CTA count G must be the same on every rank (it sets
// the row ownership and the fixed summation orders): the host agrees on it (min over the ranks) and passes
// it in.  On one GPU (world = 1, peer 0 = own buffer) the same code runs with local stores — that is what
// the GPU tests exercise; the cross-GPU ordering is the argument above (system-scope fence + release /
// acquire, causally chained through the local barrier).
#pragma once
#include "dense.cuh"
#include "mapi_common.cuh"
#include "sym.cuh"

namespace mapi {

constexpr int kP2pMaxGrid = 1024;
constexpr int kP2pMaxWorld = 64;
constexpr unsigned long long kP2pTimeoutNs = 10ull * 1000 * 1000 * 1000;  // 10 s without all arrivals
constexpr int kStP2pTimeout = 8;                                            // reported as MAPI_ERR_CUDA

__host__ __device__ inline size_t p2p_al(size_t b) { return (b + 255) & ~size_t(255); }
inline size_t p2p_exchange_bytes(int64_t n, int world) {
    return 256 + p2p_al(sizeof(float) * 2 * (size_t)world * (size_t)n) + p2p_al(sizeof(double) * 2 * (size_t)world);
}
__device__ __forceinline__ float* p2p_y(unsigned long long base) { return reinterpret_cast<float*>(base + 256); }
__device__ __forceinline__ double* p2p_rtot(unsigned long long base, int64_t n, int world) {
    return reinterpret_cast<double*>(base + 256 + p2p_al(sizeof(float) * 2 * (size_t)world * (size_t)n));
}

// steps 2-4 of the protocol (the caller has stored and fenced).  Returns false on a timed-out wait.
__device__ __forceinline__ bool p2p_arrive_wait(const unsigned long long* s_peer, int P, unsigned int* bar,
                                                unsigned int bar_target, unsigned long long* my_flag,
                                                unsigned long long flag_target, int* s_abort) {
    grid_barrier(bar, bar_target);
    if (blockIdx.x == 0 && threadIdx.x < P) {
        unsigned long long* f = reinterpret_cast<unsigned long long*>(s_peer[threadIdx.x]);
        asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(f) : "memory");
    }
    if (threadIdx.x == 0) {
        unsigned long long v, t0, now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        *s_abort = 0;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory");
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            if (v < flag_target && now - t0 > kP2pTimeoutNs) {  // a peer never arrived: fail, do not hang
                *s_abort = 1;
                break;
            }
        } while (v < flag_target);
    }
    __syncthreads();
    return *s_abort == 0;
}

// =============================================================================== K2p (row-sharded)
// Rank r holds rows [row0, row0 + m) of A.  Iteration t (global e), CTA c (rows c, c + G, ... of the local
// block, CTA-cooperative as K2c): y rows -> the OWN buffer's y[e & 1][row0 + row] and a per-CTA fp64 |y|
// partial -> local grid barrier -> CTA c copies the contiguous slice [c m / G, (c + 1) m / G) of the rank's
// rows to every peer; CTA 0 forms the rank total of |y| (the K2c order) and stores it into every rank's
// rank-total slot -> the arrival protocol -> s_t = the rank totals in rank order (on one rank: exactly
// K2c's s_t), w_{t+1} = fp32(y / s_t) from the full y, delta_t: identical bits and stop decision on every
// rank, no all-reduce.  The first load of iteration t+1 is issued before the exchange (A does not depend on w).
struct P2PArgs {
    const float* A;      // local rows (m x n, lda)
    int64_t m, n, lda, row0;
    const float* b0;     // full start vector (n)
    int32_t iters;
    float tol;
    int32_t rank, world;
    const unsigned long long* peers;  // device array: exchange base of every rank (peers[rank] = own)
    unsigned long long epoch0;        // global iteration index of this call's t = 0
    unsigned long long flag_base;     // own flag value before this call (epoch0 * world)
    float* w_out;                     // full w (n)
    float *norms, *deltas;
    int32_t* status;
    unsigned int* bar;                // local grid barrier counter (zeroed per call)
    double* cslots;                   // [2][G] per-CTA |y| partials (local workspace)
};

template <int OP, int POL, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_iterate_p2p(P2PArgs p) {
    constexpr int STEP = 256;
    extern __shared__ __align__(16) float ws_[];
    const int64_t n = p.n, m = p.m;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, P = p.world;
    const int64_t rows_cta = m > blockIdx.x ? (m - blockIdx.x + G - 1) / G : 0;  // local rows c, c+G, ...
    float* w_s = ws_;
    float* part = ws_ + ((n + 7) & ~int64_t(7));
    double* red = reinterpret_cast<double*>(part + ((rows_cta * NW + 1) & ~int64_t(1)));
    __shared__ unsigned long long s_peer[kP2pMaxWorld];
    __shared__ int s_abort;
    const int64_t cfull = n / STEP;
    const int c0 = (int)(warp * cfull / NW), c1 = (int)((warp + 1) * cfull / NW);
    const int spr = c1 - c0;
    const int nsteps = (int)rows_cta * spr;
    const int64_t tail0 = cfull * STEP;
    const bool has_tail = tail0 < n && warp == NW - 1;
    const int64_t rstride = (int64_t)G * p.lda;
    const float* abase = p.A + (int64_t)blockIdx.x * p.lda + (int64_t)c0 * STEP + lane * 8;
    const unsigned long long own = p.peers[p.rank];
    unsigned long long* my_flag = reinterpret_cast<unsigned long long*>(own);
    const float* y_own = p2p_y(own);
    const double* rtot_own = p2p_rtot(own, n, P);
    unsigned int epoch = 0;
    // this CTA's slice of the rank's rows for the copy-out
    const int64_t sl0 = m * blockIdx.x / G, sl1 = m * (blockIdx.x + 1) / G;

    for (int64_t k = tid; k < n; k += blockDim.x) w_s[k] = p.b0[k];
    for (int q = tid; q < P; q += blockDim.x) s_peer[q] = p.peers[q];

    float buf[2][8], acc[8];
    int lr = 0, lq = 0;
    auto load = [&](float (&b)[8]) {
        ld_stream<8, POL>(abase + lr * rstride + (int64_t)lq * STEP, b);
        if (++lq == spr) { lq = 0; ++lr; }
    };
    if (nsteps > 0) load(buf[0]);
    __syncthreads();
    int32_t done = 0, status = kStOk;

    for (int32_t t = 0; t < p.iters; ++t) {
        const unsigned long long e = p.epoch0 + (unsigned long long)t;
        const int par = (int)(e & 1);
        float* ypar_own = const_cast<float*>(y_own) + (int64_t)par * P * n;
        int cr = 0, cq = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
        auto finish_row = [&]() {
            float v = tree_sum(acc);
            if (has_tail) {
                const float* a = p.A + ((int64_t)blockIdx.x + (int64_t)cr * G) * p.lda;
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
        {  // rows: explicit register double buffer (as K2c)
            int s = 0;
            for (; s + 1 < nsteps; s += 2) {
                load(buf[1]);
                consume(buf[0]);
                if (s + 2 < nsteps) load(buf[0]);
                consume(buf[1]);
            }
            if (s < nsteps) consume(buf[0]);
        }
        if (spr == 0)
            for (cr = 0; cr < (int)rows_cta; ++cr) finish_row();
        lr = 0;
        lq = 0;
        if (t + 1 < p.iters && nsteps > 0) load(buf[0]);  // next iteration's first chunk, across the exchange
        __syncthreads();
        // ---- the rank's y rows into the own buffer, the CTA's fp64 |y| partial
        double abs_part = 0.0;
        for (int64_t r = tid; r < rows_cta; r += blockDim.x) {
            float v = 0.0f;
#pragma unroll 8
            for (int q = 0; q < NW; ++q) v += part[r * NW + q];
            __stcg(ypar_own + p.row0 + blockIdx.x + r * G, v);
            abs_part += norm_part<OP>(v);
        }
        const double cta_abs = block_sum(abs_part, red);
        if (tid == 0) p.cslots[par * kP2pMaxGrid + blockIdx.x] = cta_abs;
        grid_barrier(p.bar, ++epoch * G);
        // ---- copy-out: this CTA's contiguous slice of the rank's rows to every peer (coalesced), CTA 0 the
        // rank total of |y| (lane-strided over the CTA partials, butterfly: K2c's order)
        for (int q = 0; q < P; ++q) {
            if (q == p.rank) continue;
            float* yq = p2p_y(s_peer[q]) + (int64_t)par * P * n + p.row0;
            for (int64_t i = sl0 + tid; i < sl1; i += blockDim.x) yq[i] = __ldcg(ypar_own + p.row0 + i);
        }
        if (blockIdx.x == 0 && warp == 0) {
            double pp = 0.0;
            for (int c = lane; c < G; c += 32) pp += __ldcg(p.cslots + par * kP2pMaxGrid + c);
            pp = warp_sum(pp);
            for (int q = lane; q < P; q += 32) p2p_rtot(s_peer[q], n, P)[par * P + p.rank] = pp;
        }
        __threadfence_system();
        if (!p2p_arrive_wait(s_peer, P, p.bar, ++epoch * G, my_flag, p.flag_base + (unsigned long long)(t + 1) * P,
                             &s_abort)) {
            status = kStP2pTimeout;
            break;
        }
        // ---- s_t from the rank totals in rank order: identical on every rank
        double sd;
        {
            if (tid == 0) {
                double pp = 0.0;
                for (int q = 0; q < P; ++q) pp += __ldcg(rtot_own + par * P + q);
                red[32] = pp;
            }
            __syncthreads();
            sd = norm_final<OP>(red[32]);
            __syncthreads();
        }
        if (!(sd > 0.0) || isinf(sd)) {
            status = (sd == 0.0) ? kStDegenerate : kStNonfinite;
            break;
        }
        double dpart = 0.0;
        for (int64_t k = tid; k < n; k += blockDim.x) {
            const float wn = (float)((double)__ldcg(ypar_own + k) / sd);
            dpart += (double)fabsf(wn - w_s[k]);
            w_s[k] = wn;
        }
        const double delta = block_sum(dpart, red);
        if (blockIdx.x == 0 && tid == 0) {
            if (p.norms) p.norms[t] = (float)sd;
            if (p.deltas) p.deltas[t] = (float)delta;
        }
        done = t + 1;
        if (p.tol > 0.0f && delta < (double)p.tol) break;
    }
    const int64_t per = (n + G - 1) / G;
    const int64_t k0 = (int64_t)blockIdx.x * per, k1 = min(n, k0 + per);
    for (int64_t k = k0 + tid; k < k1; k += blockDim.x) p.w_out[k] = w_s[k];
    if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
}

inline size_t p2p_smem_bytes(int64_t m, int64_t n, int grid, int nw) {
    const int64_t rows_cta = (m + grid - 1) / grid;
    return sizeof(float) * (size_t)(((n + 7) & ~int64_t(7)) + ((rows_cta * nw + 1) & ~int64_t(1))) +
           sizeof(double) * 33;
}

// =============================================================================== K2sp (sharded K2s)
// Rank r of P runs the tasks [tlo, thi) = [r T / P, (r + 1) T / P) of K2s's upper-triangle task list and
// holds only the rows of their strips, [row0, row1) (sym_shard_rows).  Iteration t (global e):
//   tasks (local counter) -> local barrier -> lagged stop test on delta_{t-1} -> every CTA reduces, for its
//   owned rows (the K2s ownership over all n rows), the partials of this rank's tasks only (sym_reduce
//   <SHARDED>) and stores them as y_r[j] (fp32) into every rank's buffer y[e & 1][r][j] (owned rows are
//   contiguous: coalesced) -> the arrival protocol -> y_j = fp32(sum_q y_q[j] in rank order, fp64) for
//   the owned rows, |y| partial -> local barrier -> s_t -> w_{t+1} tagged words (local) + delta partial.
// Every rank forms the same y, s, w and stop decision.  On one rank y_j = fp32(fp64(fp32(tot))) = the K2s
// value: K2sp is bitwise K2s there (tested).  Per iteration and rank: 1/P of the triangle's HBM bytes,
// world x n x 4 bytes out and in over NVLink, one flag round trip.
struct SymShardArgs {
    SymArgs sa;                        // it.A = the held rows [row0, row1), lda
    int64_t row0, tlo, thi;
    int32_t rank, world;
    const unsigned long long* peers;
    unsigned long long epoch0, flag_base;
};

template <int OP>
__global__ void __launch_bounds__(kSymThreads, 1) k_iterate_sym_sharded(SymShardArgs x) {
    extern __shared__ __align__(16) float sm_[];
    const SymArgs& sa = x.sa;
    float* wj_s = sm_ + (threadIdx.x >> 5) * kSymRB;
    double* red = reinterpret_cast<double*>(reinterpret_cast<char*>(sm_) + kSymSmemRegion);
    __shared__ unsigned long long s_peer[kP2pMaxWorld];
    __shared__ int s_abort;
    const IterArgs& p = sa.it;
    const int64_t n = p.n;
    const int tid = threadIdx.x;
    const int G = gridDim.x, P = x.world;
    const int64_t o0 = sym_own_start(blockIdx.x, G, n), o1 = sym_own_start(blockIdx.x + 1, G, n);
    unsigned long long* wtag = sa.wtag;
    float* yg = sa.yg;
    double* slotA = reinterpret_cast<double*>(p.slots);
    double* slotD = slotA + 2 * G;
    const unsigned long long own = x.peers[x.rank];
    unsigned long long* my_flag = reinterpret_cast<unsigned long long*>(own);
    const float* y_own = p2p_y(own);
    unsigned int epoch = 0;
    const uint64_t keep = sym_keep_policy();
    for (int q = tid; q < P; q += blockDim.x) s_peer[q] = x.peers[q];
    for (int64_t j = o0 + tid; j < o1; j += blockDim.x) sym_st_tag(wtag + j, sym_tagged(1u, p.b0[j]));
    grid_barrier(p.bar, ++epoch * G);

    int32_t done = 0, status = kStOk;
    bool stopped = false;
    int32_t t = 0;
    for (; t < p.iters; ++t) {
        const unsigned long long e = x.epoch0 + (unsigned long long)t;
        const int par = (int)(e & 1);
        const unsigned long long* wcur = wtag + (t & 1) * n;
        unsigned long long* wnext = wtag + ((t + 1) & 1) * n;
        const uint32_t tag = (uint32_t)t + 1u;
        sym_tasks<OP>(sa, p.A, x.row0, x.tlo, x.thi, p.bar + 32 + (t & 1), wcur, tag, wj_s, keep);
        grid_barrier(p.bar, ++epoch * G);
        if (blockIdx.x == 0 && tid == 0) p.bar[32 + ((t + 1) & 1)] = 0u;
        if (t > 0) {
            const double delta = sym_slots_sum(slotD + ((t - 1) & 1) * G, red, 33);
            if (blockIdx.x == 0 && tid == 0 && p.deltas) p.deltas[t - 1] = (float)delta;
            done = t;
            if (p.tol > 0.0f && delta < (double)p.tol) {
                stopped = true;
                break;
            }
        }
        // ---- this rank's partial y of the owned rows into every rank's buffer
        sym_reduce<true>(sa, o0, o1, x.tlo, x.thi, reinterpret_cast<double*>(sm_), [&](int64_t j, float v) {
            for (int q = 0; q < P; ++q) p2p_y(s_peer[q])[((int64_t)par * P + x.rank) * n + j] = v;
        });
        __threadfence_system();
        if (!p2p_arrive_wait(s_peer, P, p.bar, ++epoch * G, my_flag, x.flag_base + (unsigned long long)(t + 1) * P,
                             &s_abort)) {
            status = kStP2pTimeout;
            done = t;
            stopped = true;
            break;
        }
        // ---- y of the owned rows: the ranks' partials in rank order
        double abs_part = 0.0;
        for (int64_t j = o0 + tid; j < o1; j += blockDim.x) {
            double acc = 0.0;
            for (int q = 0; q < P; ++q) acc += (double)__ldcg(y_own + ((int64_t)par * P + q) * n + j);
            const float v = (float)acc;
            yg[j] = v;
            abs_part += norm_part<OP>(v);
        }
        const double cta_abs = block_sum(abs_part, red);
        if (tid == 0) slotA[(t & 1) * G + blockIdx.x] = cta_abs;
        grid_barrier(p.bar, ++epoch * G);
        const double sd = norm_final<OP>(sym_slots_sum(slotA + (t & 1) * G, red, 32));
        if (!(sd > 0.0) || isinf(sd)) {
            status = (sd == 0.0) ? kStDegenerate : kStNonfinite;
            done = t;
            stopped = true;
            break;
        }
        if (blockIdx.x == 0 && tid == 0 && p.norms) p.norms[t] = (float)sd;
        double dpart = 0.0;
        for (int64_t j = o0 + tid; j < o1; j += blockDim.x) {
            const float wn = (float)((double)__ldcg(yg + j) / sd);
            const float wo = __uint_as_float((uint32_t)sym_ld_tag(wcur + j));
            dpart += (double)fabsf(wn - wo);
            sym_st_tag(wnext + j, sym_tagged(tag + 1u, wn));
        }
        const double cta_d = block_sum(dpart, red);
        if (tid == 0) slotD[(t & 1) * G + blockIdx.x] = cta_d;
    }
    if (!stopped) {
        grid_barrier(p.bar, ++epoch * G);
        const double delta = sym_slots_sum(slotD + ((t - 1) & 1) * G, red, 33);
        if (blockIdx.x == 0 && tid == 0 && p.deltas) p.deltas[t - 1] = (float)delta;
        done = t;
    }
    const unsigned long long* wfin = wtag + (done & 1) * n;
    for (int64_t j = o0 + tid; j < o1; j += blockDim.x) p.w_out[j] = __uint_as_float((uint32_t)sym_ld_tag(wfin + j));
    if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
}

}  // namespace mapi
