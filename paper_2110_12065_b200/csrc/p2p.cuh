// p2p.cuh — K2p: row-sharded MAPI with the y exchange fused into the persistent iteration kernel
// (DESIGN.md §8).  One cooperative launch per rank runs all iterations.
//
// Rank r of P holds rows [row0, row0 + m) of A (m = n / P).  Every rank owns an EXCHANGE buffer in its
// own HBM (allocated by mapi_p2p_alloc, mapped into every peer with CUDA IPC over NVLink):
//     [flag u64 @0][y 2 x n f32 @256][slots 2 x P x kP2pMaxGrid f64]
// Iteration t on rank r, CTA c (rows c, c + G, ... of the local block, CTA-cooperative as in K2c):
//   1. y_j = (A_local (+) w_t)_j for its rows; fp64 partial of ||y||.
//   2. stores y_j into y[t & 1][row0 + j] of EVERY rank's exchange buffer and its partial into
//      slots[t & 1][r * G + c] of every rank (P2P stores through NVLink; the local rank is peer r).
//   3. fence.sys, then one system-scope release-add of 1 on every rank's flag.
//   4. waits (acquire.sys) until its own flag reaches base + (e + 1) * P * G (e = the global
//      iteration index): every CTA of every rank has published iteration t.  This also replaces the
//      local grid barrier.
//   5. s_t = sum of the P * G partials in (rank, CTA) order -> identical on every rank; w_{t+1} =
//      fp32(y / s_t) from the local y copy (L2, bypassing L1), delta_t in fp64 fixed order -> the
//      same stop decision on every rank, no all-reduce.
// Buffers alternate by the GLOBAL iteration parity e & 1, and e and the flag base continue across
// calls (the host passes both; they are the same on every rank because every rank stops at the same
// iteration), so no reset / host barrier is needed between calls: a rank can be at most one iteration
// ahead of the slowest (it needs everyone's signal to leave an iteration), and its writes then go to
// the other parity, which the slow rank has finished reading.
// On one GPU (P = 1, peer 0 = own buffer) the same code runs with local stores — that is what the
// tests exercise; the P > 1 ordering argument is above (NVLink P2P stores + sys-scope release/acquire).
#pragma once
#include "dense.cuh"
#include "mapi_common.cuh"

namespace mapi {

constexpr int kP2pMaxGrid = 1024;  // slots per rank per parity
constexpr int kP2pMaxWorld = 64;
constexpr unsigned long long kP2pTimeoutNs = 10ull * 1000 * 1000 * 1000;  // 10 s without all arrivals
constexpr int kStP2pTimeout = 8;                                            // reported as MAPI_ERR_CUDA

inline size_t p2p_exchange_bytes(int64_t n, int world) {
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    return 256 + al(sizeof(float) * 2 * (size_t)n) + al(sizeof(double) * 2 * (size_t)world * kP2pMaxGrid);
}

struct P2PArgs {
    const float* A;      // local rows (m x n, lda)
    int64_t m, n, lda, row0;
    const float* b0;     // full start vector (n)
    int32_t iters;
    float tol;
    int32_t rank, world;
    const unsigned long long* peers;  // device array: exchange base of every rank (peers[rank] = own)
    unsigned long long epoch0;        // global iteration index of this call's t = 0
    unsigned long long flag_base;     // own flag value before this call (epoch0 * world * G)
    float* w_out;                     // full w (n)
    float *norms, *deltas;
    int32_t* status;
};

__device__ __forceinline__ float* p2p_y(unsigned long long base) { return reinterpret_cast<float*>(base + 256); }
__device__ __forceinline__ double* p2p_slots(unsigned long long base, int64_t n) {
    return reinterpret_cast<double*>(base + 256 + ((sizeof(float) * 2 * (size_t)n + 255) & ~size_t(255)));
}

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
    const double* slots_own = p2p_slots(own, n);

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
        // ---- publish: y rows into every rank's y[par], the fp64 partial into every rank's slots
        double abs_part = 0.0;
        for (int64_t r = tid; r < rows_cta; r += blockDim.x) {
            float v = 0.0f;
#pragma unroll 8
            for (int q = 0; q < NW; ++q) v += part[r * NW + q];
            const int64_t row = p.row0 + blockIdx.x + r * G;
            for (int q = 0; q < P; ++q) p2p_y(s_peer[q])[(int64_t)par * n + row] = v;
            abs_part += norm_part<OP>(v);
        }
        const double cta_abs = block_sum(abs_part, red);
        if (tid < P)
            p2p_slots(s_peer[tid], n)[((int64_t)par * P + p.rank) * kP2pMaxGrid + blockIdx.x] = cta_abs;
        __threadfence_system();  // this thread's P2P stores before the CTA's release below
        __syncthreads();
        if (tid < P) {  // one system-scope release-add per destination rank
            unsigned long long* f = reinterpret_cast<unsigned long long*>(s_peer[tid]);
            asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(f) : "memory");
        }
        if (tid == 0) {
            const unsigned long long target = p.flag_base + (unsigned long long)(t + 1) * P * G;
            unsigned long long v, t0, now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            s_abort = 0;
            do {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flag) : "memory");
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (v < target && now - t0 > kP2pTimeoutNs) {  // a peer never arrived: fail, do not hang
                    s_abort = 1;
                    break;
                }
            } while (v < target);
        }
        __syncthreads();
        if (s_abort) {
            status = kStP2pTimeout;
            break;
        }
        // ---- s_t over the P x G partials in (rank, CTA) order: identical on every rank
        double sd;
        {
            if (warp == 0) {
                double pp = 0.0;
                for (int q = 0; q < P; ++q) {
                    double pq = 0.0;
                    for (int c = lane; c < G; c += 32) pq += __ldcg(slots_own + ((int64_t)par * P + q) * kP2pMaxGrid + c);
                    pp += warp_sum(pq);
                }
                if (lane == 0) red[32] = pp;
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
            const float wn = (float)((double)__ldcg(y_own + (int64_t)par * n + k) / sd);
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

}  // namespace mapi
