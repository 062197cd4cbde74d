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
#include <cstdlib>
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
// by rounding noise; the paper computes in double (MATLAB).  The fp64 iterate is never stored: w_t is
// a pure function of (S_{t-1}, s_{t-1}, e_{t-1}), so the next launch recomputes it bit-exactly from
// the previous gather output (e is double-buffered) and two fp64 scalars — 20 B/node of traffic
// per normalise instead of 32 B/node with an fp64 w array.
//
// workspace: [hdr 256: status[2] @0, stop @8, counter u32 @12, s f64 @16, hist (S, s) x 2 f64 @32]
//            [e0 n f32][e1 n f32][v n f32]
//            [slotS 2*G f64][slotY G f64][slotD G f64]
//            [merge-path partition: (i,k) x (T+1) i32][carry_row T i32][carry_val T f32][gsum T x 8 f64]
// T = number of merge-path tiles = ceil((n + nnz) / kMpTile).
#ifndef MAPI_MP_THREADS
#define MAPI_MP_THREADS 128
#endif
constexpr int kMpThreads = MAPI_MP_THREADS;
#ifndef MAPI_MP_IPT
#define MAPI_MP_IPT 12
#endif
constexpr int kMpIpt = MAPI_MP_IPT;                          // merge items (rows + nonzeros) per thread
constexpr int kMpTile = kMpThreads * kMpIpt;        // 1536 items per CTA (sweep: r01_summary.md)
constexpr int kMpWarps = kMpThreads / 32;           // per-warp fp64 partials of sum e

struct CsrWs {
    int32_t* status;
    int32_t* stop;
    uint32_t* counter;
    double* s;
    double* hist;  // [2][2]: (S_t, s_t) of the last normalised iteration t, slot (t + 1) & 1
    float *e[2], *v;
    double *slotS, *slotY, *slotD;
    int32_t *part_i, *part_k, *carry_row;
    float* carry_val;
    double* gsum;
    int64_t tiles;
};

inline int64_t mp_tiles(int64_t n, int64_t nnz) { return (n + nnz + kMpTile - 1) / kMpTile; }

// n: nodes (the e / v arrays); m: rows this workspace gathers (m = n on one GPU, the owned block when sharded)
inline size_t csr_rank_ws_bytes(int64_t n, int64_t nnz, int64_t m = -1) {
    const int64_t T = mp_tiles(m < 0 ? n : m, nnz);
    return 256 + 3 * cal256(4 * (size_t)n) + 4 * cal256(8 * (size_t)kCsrMaxGrid) +
           2 * cal256(4 * (size_t)(T + 1)) + 2 * cal256(4 * (size_t)T) + cal256(8 * (size_t)T * kMpWarps);
}

inline CsrWs carve_csr(void* ws, int64_t n, int64_t nnz, int64_t m = -1) {
    char* p = static_cast<char*>(ws);
    CsrWs c;
    c.tiles = mp_tiles(m < 0 ? n : m, nnz);
    c.status = reinterpret_cast<int32_t*>(p);
    c.stop = reinterpret_cast<int32_t*>(p + 8);
    c.counter = reinterpret_cast<uint32_t*>(p + 12);
    c.s = reinterpret_cast<double*>(p + 16);
    c.hist = reinterpret_cast<double*>(p + 32);
    p += 256;
    for (int b = 0; b < 2; ++b) {
        c.e[b] = reinterpret_cast<float*>(p);
        p += cal256(4 * (size_t)n);
    }
    c.v = reinterpret_cast<float*>(p);
    p += cal256(4 * (size_t)n);
    c.slotS = reinterpret_cast<double*>(p);
    p += 2 * cal256(8 * (size_t)kCsrMaxGrid);
    c.slotY = reinterpret_cast<double*>(p);
    p += cal256(8 * (size_t)kCsrMaxGrid);
    c.slotD = reinterpret_cast<double*>(p);
    p += cal256(8 * (size_t)kCsrMaxGrid);
    c.part_i = reinterpret_cast<int32_t*>(p);
    p += cal256(4 * (size_t)(c.tiles + 1));
    c.part_k = reinterpret_cast<int32_t*>(p);
    p += cal256(4 * (size_t)(c.tiles + 1));
    c.carry_row = reinterpret_cast<int32_t*>(p);
    p += cal256(4 * (size_t)c.tiles);
    c.carry_val = reinterpret_cast<float*>(p);
    p += cal256(4 * (size_t)c.tiles);
    c.gsum = reinterpret_cast<double*>(p);
    return c;
}

// x / d for the n node quotients of an iteration, given rd = 1/d (one IEEE fp64 division per CTA):
// q0 = x rd, q = q0 + (x - q0 d) rd — the residual-corrected quotient DDIV itself computes, without its
// special-case paths (x, d are finite and normal here); used by every kernel that forms w so that a
// recomputed w_t is bit-identical to the one formed the iteration before.
__device__ __forceinline__ double qdiv(double x, double d, double rd) {
    const double q0 = x * rd;
    return fma(fma(-q0, d, x), rd, q0);
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

// same, reading the slots through L2 (written by other CTAs of the running launch)
__device__ __forceinline__ double slots_sum_cg(const double* slots, int count, double* red) {
    if (threadIdx.x < 32) {
        double part = 0.0;
        for (int c = threadIdx.x; c < count; c += 32) part += __ldcg(slots + c);
        part = warp_sum(part);
        if (threadIdx.x == 0) red[32] = part;
    }
    __syncthreads();
    const double r = red[32];
    __syncthreads();
    return r;
}

// K3a at t = 0: w_0 = b0 (checked >= 0), v_j, S partials (slot parity 0).
__global__ void __launch_bounds__(kCsrThreads) k_rank_init(int64_t n, const float* __restrict__ b0,
                                                           const float* __restrict__ bg, const float* __restrict__ cap,
                                                           float* __restrict__ v, double* __restrict__ slotS,
                                                           int32_t* status, int32_t* stop) {
    __shared__ double red[33];
    double sp = 0.0;
    bool neg = false;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double wj = (double)b0[j];
        neg |= wj < 0.0;
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

// ---- K3b: merge-path gather-sum  e_i = sum_{e in row i} v[col_idx[e]]  (fp32)
// The (n row ends) + (nnz nonzeros) merge list is cut into equal tiles of kMpTile items, so hub
// rows (97k edges) and empty rows (52% at cfg5) cost the same per item (Merrill & Garland's
// merge-based SpMV decomposition, re-derived for a value-free gather-sum).  Every row end is
// emitted exactly once; a row that spans threads collects the preceding threads' carries in thread
// order, and a row that spans CTAs gets the CTA carry-outs added by k_rank_fixup in CTA order, so
// the summation order is fixed for a given graph.

// L2 policy knobs for the gather (K3b): the col_idx / row_ptr streams are read once per
// iteration (evict-first, no L1 allocation) so that they do not push the 16 MB gathered vector v out
// of L2 / L1; the gathers themselves ask L2 to keep v (evict-last).
#ifndef MAPI_CSR_HINT
#define MAPI_CSR_HINT 1
#endif
#ifndef MAPI_CSR_SHARE
#define MAPI_CSR_SHARE 1
#endif
__device__ __forceinline__ uint64_t l2_policy_stream() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_keep() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p, uint64_t pol) {
#if MAPI_CSR_HINT
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ float ld_keep_f32(const float* p, uint64_t pol) {
#if MAPI_CSR_HINT
    float r;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
    return r;
#else
    return __ldg(p);
#endif
}

// merge-path search on diagonal d: the number of row ends consumed before d
__device__ __forceinline__ int64_t mp_search(int64_t d, const int32_t* __restrict__ row_end, int64_t n,
                                             int64_t nnz) {
    int64_t lo = max((int64_t)0, d - nnz), hi = min(d, n);
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)row_end[mid] <= d - 1 - mid) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// once per call: tile start coordinates (i, k) for every tile boundary
__global__ void k_mp_partition(int64_t n, int64_t nnz, const int32_t* __restrict__ row_ptr, int64_t tiles,
                               int32_t* __restrict__ part_i, int32_t* __restrict__ part_k) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > tiles) return;
    const int64_t d = min(c * kMpTile, n + nnz);
    const int64_t i = mp_search(d, row_ptr + 1, n, nnz);
    part_i[c] = (int32_t)i;
    part_k[c] = (int32_t)(d - i);
}

// Per-tile shared memory of the merge-path gather (one 128-thread group's worth).
struct MpSmem {
    int32_t* buf;   // kMpTileBuf words: row ends, then gathered values
    float* fp;      // kMpThreads
    int32_t* wl_row;
    int32_t* wf_row;
    float* wl_val;  // kMpWarps each
};
constexpr int kMpTileBuf = kMpTile + 2 + (kMpTile + 2) / 32 + 1;

// One merge-path tile (kMpThreads threads: tid = thread within the group, sync = its barrier).  HUB > 0:
// v[0 .. HUB) is read from `hub` (a shared-memory copy, bitwise the same values) instead of L2.
template <int HUB, typename Sync>
__device__ __forceinline__ void mp_tile(int64_t tile, int tid, const Sync& sync, const MpSmem& sm, const float* hub,
                                        int64_t n, int64_t nnz, const int32_t* __restrict__ row_ptr,
                                        const int32_t* __restrict__ col_idx, const float* __restrict__ v,
                                        const int32_t* __restrict__ part_i, const int32_t* __restrict__ part_k,
                                        float* __restrict__ e, int32_t* __restrict__ carry_row,
                                        float* __restrict__ carry_val, double* __restrict__ gsum, uint64_t pol_s,
                                        uint64_t pol_k) {
    // shared arrays indexed through pad(): one spare word per 8 so that the lane-strided reads of the
    // consume loop (thread t walks ~8 consecutive items) hit 32 distinct banks instead of 4
    // the stop flag (written by the previous launch) is read together with the partition, not
    // ahead of it: one global round trip before the streams start instead of two
    const int lane = tid & 31, warp = tid >> 5;
    const int32_t i0 = part_i[tile], i1 = part_i[tile + 1];
    const int32_t k0 = part_k[tile], k1 = part_k[tile + 1];
    const int nrows = i1 - i0, nk = k1 - k0;  // nrows + nk == items of this tile
    // one spare word per 32: the staging writes (32 consecutive items per warp) are conflict-free and
    // the consume loop's ~8-apart lane reads land on distinct banks
    auto pad = [](int x) { return x + (x >> 5); };
    // one buffer: nrows + 1 row ends, then nk values (nrows + nk <= kMpTile); half the shared memory
    // of two full-size arrays, which leaves more of the unified L1 to cache the gathered v
    int32_t* s_end = sm.buf;
    float* s_val = reinterpret_cast<float*>(sm.buf) + pad(nrows + 1) + 1;
    float* s_fp = sm.fp;  // segmented prefix of the threads' carries
    int32_t* wl_row = sm.wl_row;
    int32_t* wf_row = sm.wf_row;
    float* wl_val = sm.wl_val;
    // stage row ends (rows i0 .. i1, the last possibly partial) and gathered values
    for (int r = tid; r <= nrows; r += kMpThreads)
        s_end[pad(r)] = (i0 + r < n) ? ld_stream_i32(row_ptr + i0 + r + 1, pol_s) : (int32_t)nnz;
    // nk <= kMpTile = kMpIpt * kMpThreads: all kMpIpt column ids first, then all gathers in flight
    int32_t cj[kMpIpt];
#pragma unroll
    for (int u = 0; u < kMpIpt; ++u) {
        const int j = tid + u * kMpThreads;
        cj[u] = j < nk ? ld_stream_i32(col_idx + k0 + j, pol_s) : -1;
    }
    float xv[kMpIpt];
#pragma unroll
    for (int u = 0; u < kMpIpt; ++u) {
        if constexpr (HUB > 0) {
            // branch-free, so the 12 global gathers still issue back to back: hub lanes load v[0] (one
            // shared sector) and take the shared-memory copy instead
            const bool inhub = (unsigned)cj[u] < (unsigned)HUB;
            const float g = ld_keep_f32(v + (inhub || cj[u] < 0 ? 0 : cj[u]), pol_k);
            const float h = hub[inhub ? cj[u] : 0];
            xv[u] = cj[u] < 0 ? 0.0f : (inhub ? h : g);
        } else {
            xv[u] = cj[u] >= 0 ? ld_keep_f32(v + cj[u], pol_k) : 0.0f;
        }
    }
    double gpart = 0.0;
#pragma unroll
    for (int u = 0; u < kMpIpt; ++u) {
        const int j = tid + u * kMpThreads;
        if (j < nk) s_val[pad(j)] = xv[u];
        gpart += (double)xv[u];
    }
    sync();
    // this thread's diagonal within the tile (merge-path search in shared memory)
    const int items = nrows + nk;
    const int dt = min(tid * kMpIpt, items);
    int lo = max(0, dt - nk), hi = min(dt, nrows);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_end[pad(mid)] - k0 <= dt - 1 - mid) lo = mid + 1;
        else hi = mid;
    }
    int ri = lo, kj = dt - lo;
    float acc = 0.0f, own_first = 0.0f;
    int first_row = -1;  // first row this thread emits (local index); earlier threads may feed it
    const int dend = min(dt + kMpIpt, items);
    int32_t cur_end = ri < nrows ? s_end[pad(ri)] - k0 : 0x7fffffff;  // end of row ri, tile-relative
    for (int d = dt; d < dend; ++d) {
        if (kj >= cur_end) {  // the end of row ri (ri < nrows)
            if (first_row < 0) {
                first_row = ri;
                own_first = acc;
            } else {
                e[i0 + ri] = acc;  // started inside this thread: complete
            }
            acc = 0.0f;
            ++ri;
            cur_end = ri < nrows ? s_end[pad(ri)] - k0 : 0x7fffffff;
        } else {
            acc += s_val[pad(kj)];
            ++kj;
        }
    }
    // Carries: thread t leaves row ri open with partial acc.  Rows are non-decreasing in t, so the
    // threads open on one row form a contiguous run; a segmented inclusive scan (keyed by row) gives
    // each thread the sum of its run so far.  Warp level: Hillis-Steele shuffles; block level: the
    // trailing runs of the preceding warps, nearest first.  Fixed order -> deterministic.
    float pv = acc;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const float ov = __shfl_up_sync(0xffffffffu, pv, off);
        const int orow = __shfl_up_sync(0xffffffffu, ri, off);
        if (lane >= off && orow == ri) pv += ov;
    }
    if (lane == 31) {
        wl_row[warp] = ri;
        wl_val[warp] = pv;
    }
    if (lane == 0) wf_row[warp] = ri;
    sync();
    if (ri == wf_row[warp]) {  // my run reaches the start of my warp: add preceding warps' tails
        float extra = 0.0f;
        for (int q = warp - 1; q >= 0; --q) {
            if (wl_row[q] != ri) break;
            extra += wl_val[q];
            if (wf_row[q] != ri) break;
        }
        pv += extra;
    }
    s_fp[tid] = pv;
    sync();
    // the first row this thread emits was left open by thread tid-1 (its carry row is this thread's
    // start row), so its preceding partials are exactly s_fp[tid-1]
    if (first_row >= 0) e[i0 + first_row] = (tid > 0 ? s_fp[tid - 1] : 0.0f) + own_first;
    if (tid == kMpThreads - 1) {  // CTA carry-out: the run still open on the tile's last row
        carry_row[tile] = (ri < nrows || (ri == nrows && i1 < n)) ? i0 + ri : -1;
        carry_val[tile] = pv;
    }
    // fp64 sum of this tile's gathered values, per warp (k_rank_fixup adds the warps in order)
    gpart = warp_sum(gpart);
    if (lane == 0) gsum[tile * kMpWarps + warp] = gpart;
}

__global__ void __launch_bounds__(kMpThreads) k_rank_rows_mp(int64_t n, int64_t nnz, const int32_t* __restrict__ row_ptr,
                                                             const int32_t* __restrict__ col_idx,
                                                             const float* __restrict__ v,
                                                             const int32_t* __restrict__ part_i,
                                                             const int32_t* __restrict__ part_k, float* __restrict__ e,
                                                             int32_t* __restrict__ carry_row,
                                                             float* __restrict__ carry_val, double* __restrict__ gsum,
                                                             const int32_t* stop) {
    // the stop flag (written by the previous launch) is read together with the partition, not ahead of
    // it: one global round trip before the streams start instead of two
    const int32_t halt = *stop;
    __shared__ int32_t s_buf[kMpTileBuf];
    __shared__ float s_fp[kMpThreads];
    __shared__ int32_t wl_row[kMpWarps], wf_row[kMpWarps];
    __shared__ float wl_val[kMpWarps];
    if (halt) return;
    const MpSmem sm{s_buf, s_fp, wl_row, wf_row, wl_val};
    mp_tile<0>((int64_t)blockIdx.x, threadIdx.x, [] { __syncthreads(); }, sm, nullptr, n, nnz, row_ptr, col_idx, v,
               part_i, part_k, e, carry_row, carry_val, gsum, l2_policy_stream(), l2_policy_keep());
}

// K3h (opt-in, MAPI_CSR_HUB=1; measured slower, see csr_rank_run): the same tiles, persistent (kHubCtas
// CTAs per SM, kHubGroups independent 128-thread groups each with its own named barrier), with the first
// HUB entries of v copied once per launch into shared memory.  After mapi_csr_reorder (ids by descending
// out-degree) those are the highest out-degree sources (cfg5: the first 12,288 ids carry ~37% of the
// edges), whose gathers then cost shared-memory wavefronts instead of one L1 wavefront per lane.  The
// gather-only probe gained 30% this way (profiles/r01_probe_hub.log), but the persistent tile loop itself
// runs at half K3's rate.  Bitwise the same e as k_rank_rows_mp.
constexpr int kHubGroups = 8;
#ifndef MAPI_CSR_HUBN
#define MAPI_CSR_HUBN 12288
#endif
#ifndef MAPI_CSR_HUB_CTAS
#define MAPI_CSR_HUB_CTAS 2
#endif
constexpr int kHub = MAPI_CSR_HUBN;           // v entries in shared memory per CTA
constexpr int kHubCtas = MAPI_CSR_HUB_CTAS;   // CTAs per SM (each with its own hub copy)
inline size_t hub_smem_bytes() {
    return sizeof(float) * kHub + kHubGroups * (sizeof(int32_t) * kMpTileBuf + sizeof(float) * kMpThreads +
                                                  sizeof(int32_t) * 2 * kMpWarps + sizeof(float) * kMpWarps);
}
template <int HUB>
__global__ void __launch_bounds__(kMpThreads * kHubGroups, kHubCtas) k_rank_rows_mp_hub(
    int64_t n, int64_t nnz, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
    const float* __restrict__ v, const int32_t* __restrict__ part_i, const int32_t* __restrict__ part_k,
    float* __restrict__ e, int32_t* __restrict__ carry_row, float* __restrict__ carry_val, double* __restrict__ gsum,
    const int32_t* stop, int64_t tiles) {
    if (*(volatile const int32_t*)stop) return;
    extern __shared__ __align__(16) float hsm_[];
    float* hub = hsm_;
    for (int i = threadIdx.x; i < HUB; i += kMpThreads * kHubGroups) hub[i] = i < n ? __ldg(v + i) : 0.0f;
    const int g = threadIdx.x / kMpThreads, gtid = threadIdx.x % kMpThreads;
    char* gp = reinterpret_cast<char*>(hsm_ + HUB) +
               (size_t)g * (sizeof(int32_t) * kMpTileBuf + sizeof(float) * kMpThreads + sizeof(int32_t) * 2 * kMpWarps +
                            sizeof(float) * kMpWarps);
    MpSmem sm;
    sm.buf = reinterpret_cast<int32_t*>(gp);
    sm.fp = reinterpret_cast<float*>(sm.buf + kMpTileBuf);
    sm.wl_row = reinterpret_cast<int32_t*>(sm.fp + kMpThreads);
    sm.wf_row = sm.wl_row + kMpWarps;
    sm.wl_val = reinterpret_cast<float*>(sm.wf_row + kMpWarps);
    __syncthreads();
    const uint64_t pol_s = l2_policy_stream(), pol_k = l2_policy_keep();
    auto sync = [g] { asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kMpThreads) : "memory"); };
    for (int64_t tile = (int64_t)blockIdx.x * kHubGroups + g; tile < tiles; tile += (int64_t)gridDim.x * kHubGroups)
        mp_tile<HUB>(tile, gtid, sync, sm, hub, n, nnz, row_ptr, col_idx, v, part_i, part_k, e, carry_row, carry_val,
                     gsum, pol_s, pol_k);
}

// CTA carry-outs into the rows they belong to (tile order), and the fp64 partials of sum_i e_i.
__global__ void __launch_bounds__(256) k_rank_fixup(int64_t tiles, const int32_t* __restrict__ carry_row,
                                                    const float* __restrict__ carry_val,
                                                    const double* __restrict__ gsum, float* __restrict__ e,
                                                    double* __restrict__ slotY, const int32_t* stop) {
    __shared__ double red[33];
    if (*(volatile const int32_t*)stop) return;
    double g = 0.0;  // grid-stride over tiles: any graph size with a bounded grid
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < tiles; c += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int q = 0; q < kMpWarps; ++q) g += gsum[c * kMpWarps + q];
        const int32_t r = carry_row[c];
        if (r >= 0 && (c == 0 || carry_row[c - 1] != r)) {
            float sum = 0.0f;
            for (int64_t q = c; q < tiles && carry_row[q] == r; ++q) sum += carry_val[q];
            e[r] += sum;  // the emitting tile (after this run) already wrote its part
        }
    }
    const double G = block_sum(g, red);
    if (threadIdx.x == 0) slotY[blockIdx.x] = G;
}

// K3c+d: s = ||y||_1 = n S + sum_i e_i (fp64), w_new = (S + e_j) / s (fp64), w_old recomputed from the
// previous gather (bit-identical to last launch's w_new), delta partials, next v_j and S partials; the
// last CTA to finish (counter) sums the delta partials in slot order and writes delta_t, the trace,
// iters_done and the stop flag.  (One fp64 product n*S per iteration: the l1 norm of the background.)
template <bool V4>
__global__ void __launch_bounds__(kCsrThreads, 4) k_rank_normalize(
    int64_t n, const float* __restrict__ e, const float* __restrict__ e_prev, const float* __restrict__ b0,
    double* __restrict__ hist, const double* __restrict__ slotS_cur, double* __restrict__ slotS_next, int nS,
    const double* __restrict__ slotY, int nY, const float* __restrict__ bg, const float* __restrict__ cap,
    float* __restrict__ v, double* __restrict__ slotD, double* s_out, uint32_t* counter, int32_t t, float tol,
    float* deltas, int32_t* status, int32_t* stop) {
    __shared__ double red[33];
    __shared__ int s_last;
    if (*(volatile const int32_t*)stop) return;
    const double S = slots_sum(slotS_cur, nS, red);
    const double s = (double)n * S + slots_sum(slotY, nY, red);
    if (!(s > 0.0) || isinf(s)) {  // uniform across CTAs: CTA 0 reports, nothing is updated
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            *s_out = s;
            status[0] = (s == 0.0) ? 4 : 6;
            *stop = 1;
        }
        return;
    }
    // w_old = w_t: b0 at t = 0, else (S_{t-1} + e_{t-1}) / s_{t-1} exactly as the last launch formed it
    const bool first = e_prev == nullptr;
    const double Sp = first ? 0.0 : hist[(t & 1) * 2], sp_ = first ? 1.0 : hist[(t & 1) * 2 + 1];
    const double rs = 1.0 / s, rsp = 1.0 / sp_;
    auto w_old = [&](int64_t j, float ep) -> double { return first ? (double)b0[j] : qdiv(Sp + (double)ep, sp_, rsp); };
    double dp = 0.0, sn = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t j0 = 0;
    if constexpr (V4) {
        // groups of 4 consecutive nodes, two groups per trip: 16 B vector loads, 8 nodes in flight
        const int64_t groups = n / 4;
        for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += 2 * stride) {
            float4 ev[2], pv[2], bv[2], cv[2];
            const bool two = g + stride < groups;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q == 1 && !two) break;
                const int64_t gg = g + q * stride;
                ev[q] = reinterpret_cast<const float4*>(e)[gg];
                pv[q] = reinterpret_cast<const float4*>(first ? b0 : e_prev)[gg];
                bv[q] = __ldg(reinterpret_cast<const float4*>(bg) + gg);
                cv[q] = __ldg(reinterpret_cast<const float4*>(cap) + gg);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q == 1 && !two) break;
                const int64_t gg = g + q * stride;
                const float ee[4] = {ev[q].x, ev[q].y, ev[q].z, ev[q].w};
                const float pp[4] = {pv[q].x, pv[q].y, pv[q].z, pv[q].w};
                const float bb[4] = {bv[q].x, bv[q].y, bv[q].z, bv[q].w};
                const float cc[4] = {cv[q].x, cv[q].y, cv[q].z, cv[q].w};
                float vn[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double wn = qdiv(S + (double)ee[i], s, rs);
                    const double wo = first ? (double)pp[i] : qdiv(Sp + (double)pp[i], sp_, rsp);
                    dp += fabs(wn - wo);
                    vn[i] = csr_v(wn, bb[i], cc[i]);
                    sn += fmin((double)bb[i], wn);
                }
                reinterpret_cast<float4*>(v)[gg] = make_float4(vn[0], vn[1], vn[2], vn[3]);
            }
        }
        j0 = groups * 4;
    }
    for (int64_t j = j0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const double wn = qdiv(S + (double)e[j], s, rs);
        dp += fabs(wn - w_old(j, first ? 0.0f : e_prev[j]));
        const float b = bg[j];
        v[j] = csr_v(wn, b, cap[j]);
        sn += fmin((double)b, wn);
    }
    const double D = block_sum(dp, red);
    const double Sn = block_sum(sn, red);
    if (threadIdx.x == 0) {
        slotD[blockIdx.x] = D;
        slotS_next[blockIdx.x] = Sn;
        __threadfence();
        s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    // K3d (last CTA): delta_t in slot order, trace, iters_done, (S_t, s_t) for the next launch, stop
    __threadfence();
    const double d = slots_sum_cg(slotD, gridDim.x, red);
    if (threadIdx.x == 0) {
        *counter = 0u;
        *s_out = s;
        hist[((t + 1) & 1) * 2] = S;
        hist[((t + 1) & 1) * 2 + 1] = s;
        if (deltas) deltas[t] = (float)d;
        status[1] = t + 1;
        if (tol > 0.0f && d < (double)tol) *stop = 1;
    }
}

// Final outputs: w = (S + e) / s of the last normalised iteration (b0 if none), recomputed in fp64
// exactly as the loop formed it; w_out = fp32(w) and the per-CTA sums of w^2 (pass 1), then the
// optional l2 copy (pass 2).
struct RankLast {
    const float* e;
    double S, s;
    bool none;
};
__device__ __forceinline__ RankLast rank_last(const float* e0, const float* e1, const double* hist,
                                              const int32_t* status) {
    const int32_t done = status[1];
    RankLast r;
    r.none = done == 0;
    const int32_t last = done - 1;
    r.e = (last & 1) ? e1 : e0;
    r.S = r.none ? 0.0 : hist[((last + 1) & 1) * 2];
    r.s = r.none ? 1.0 : hist[((last + 1) & 1) * 2 + 1];
    return r;
}
__global__ void __launch_bounds__(kCsrThreads) k_rank_output(int64_t n, const float* __restrict__ e0,
                                                            const float* __restrict__ e1, const double* hist,
                                                            const int32_t* status, const float* __restrict__ b0,
                                                            float* __restrict__ w_out, double* __restrict__ slotQ) {
    __shared__ double red[33];
    const RankLast L = rank_last(e0, e1, hist, status);
    const double rls = 1.0 / L.s;
    double part = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double x = L.none ? (double)b0[j] : qdiv(L.S + (double)L.e[j], L.s, rls);
        w_out[j] = (float)x;
        part = fma(x, x, part);
    }
    const double q = block_sum(part, red);
    if (threadIdx.x == 0) slotQ[blockIdx.x] = q;
}
__global__ void __launch_bounds__(kCsrThreads) k_rank_output_l2(int64_t n, const float* __restrict__ e0,
                                                               const float* __restrict__ e1, const double* hist,
                                                               const int32_t* status, const float* __restrict__ b0,
                                                               const double* __restrict__ slotQ, int nq,
                                                               float* __restrict__ w_l2) {
    __shared__ double red[33];
    const RankLast L = rank_last(e0, e1, hist, status);
    const double rls = 1.0 / L.s;
    const double l2 = sqrt(slots_sum(slotQ, nq, red));
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double x = L.none ? (double)b0[j] : qdiv(L.S + (double)L.e[j], L.s, rls);
        w_l2[j] = l2 > 0.0 ? (float)(x / l2) : 0.0f;
    }
}

inline mapi_status csr_rank_run(int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* col_idx,
                                const float* cap, const float* bg, const float* b0, int32_t max_iters, float tol,
                                float* w_out, float* w_l2_out, float* deltas, void* ws, int sms, cudaStream_t s,
                                cudaEvent_t* ev_a, cudaEvent_t* ev_b, std::atomic<uint64_t>& launches) {
    CsrWs W = carve_csr(ws, n, nnz);
    cudaError_t err = cudaMemsetAsync(ws, 0, 256, s);
    if (err != cudaSuccess) return csr_cuda_fail(err, "memset");
    const int gcol = (int)std::min<int64_t>({(n + kCsrThreads - 1) / kCsrThreads, (int64_t)4 * sms, (int64_t)kCsrMaxGrid});
    const int64_t T = W.tiles;
    // 16 B vector path for the node arrays when the caller's b0 / bg / cap are 16 B aligned
    const bool v4 = (reinterpret_cast<uintptr_t>(bg) % 16 == 0) && (reinterpret_cast<uintptr_t>(cap) % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(b0) % 16 == 0);
    const int gfix = (int)std::min<int64_t>((T + 255) / 256, kCsrMaxGrid);
    // K3h (persistent, shared-memory hub copy of v) only when MAPI_CSR_HUB=1 (=2: persistent without the
    // hub copy); bitwise the same gather as K3.  Measured SLOWER on cfg5 (K3 3.68k it/s; K3h 2.3k on the
    // relabelled graph; the 104 KB carve-out alone 1.67k: it displaces the L1 cache, whose 13% hit rate on
    // the hottest v lines K3 relies on): the default stays the one-tile-per-CTA K3.
    const char* he = getenv("MAPI_CSR_HUB");
    const bool hub = he && (he[0] == '1' || he[0] == '2');
    const bool persist_only = he && he[0] == '2';
    const unsigned hub_grid =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * kHubCtas, (T + kHubGroups - 1) / kHubGroups));
    if (hub) {
        err = cudaFuncSetAttribute(k_rank_rows_mp_hub<kHub>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)hub_smem_bytes());
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_rank_rows_mp_hub<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)hub_smem_bytes());
        if (err != cudaSuccess) return csr_cuda_fail(err, "hub kernel smem");
    }
    // (investigation) MAPI_CSR_CARVEOUT=<percent>: shared-memory carve-out preference of K3, i.e. how much
    // of the unified L1 stays cache for the gathered v
    if (const char* co = getenv("MAPI_CSR_CARVEOUT")) {
        err = cudaFuncSetAttribute(k_rank_rows_mp, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(co));
        if (err != cudaSuccess) return csr_cuda_fail(err, "carveout");
    }
    k_mp_partition<<<(unsigned)((T + 1 + 255) / 256), 256, 0, s>>>(n, nnz, row_ptr, T, W.part_i, W.part_k);
    launches.fetch_add(1, std::memory_order_relaxed);
    if (ev_a) cudaEventRecord(*ev_a, s);
    k_rank_init<<<gcol, kCsrThreads, 0, s>>>(n, b0, bg, cap, W.v, W.slotS, W.status, W.stop);
    launches.fetch_add(1, std::memory_order_relaxed);
    for (int32_t t = 0; t < max_iters; ++t) {
        double* S_cur = W.slotS + (t & 1) * kCsrMaxGrid;
        double* S_next = W.slotS + ((t + 1) & 1) * kCsrMaxGrid;
        float* e_cur = W.e[t & 1];
        const float* e_prev = t == 0 ? nullptr : W.e[(t + 1) & 1];
        if (hub && persist_only)
            k_rank_rows_mp_hub<0><<<hub_grid, kMpThreads * kHubGroups, hub_smem_bytes(), s>>>(
                n, nnz, row_ptr, col_idx, W.v, W.part_i, W.part_k, e_cur, W.carry_row, W.carry_val, W.gsum, W.stop, T);
        else if (hub)
            k_rank_rows_mp_hub<kHub><<<hub_grid, kMpThreads * kHubGroups, hub_smem_bytes(), s>>>(
                n, nnz, row_ptr, col_idx, W.v, W.part_i, W.part_k, e_cur, W.carry_row, W.carry_val, W.gsum, W.stop, T);
        else
            k_rank_rows_mp<<<(unsigned)T, kMpThreads, 0, s>>>(n, nnz, row_ptr, col_idx, W.v, W.part_i, W.part_k,
                                                              e_cur, W.carry_row, W.carry_val, W.gsum, W.stop);
        k_rank_fixup<<<gfix, 256, 0, s>>>(T, W.carry_row, W.carry_val, W.gsum, e_cur, W.slotY, W.stop);
        if (v4)
            k_rank_normalize<true><<<gcol, kCsrThreads, 0, s>>>(n, e_cur, e_prev, b0, W.hist, S_cur, S_next, gcol,
                                                                W.slotY, gfix, bg, cap, W.v, W.slotD, W.s, W.counter,
                                                                t, tol, deltas, W.status, W.stop);
        else
            k_rank_normalize<false><<<gcol, kCsrThreads, 0, s>>>(n, e_cur, e_prev, b0, W.hist, S_cur, S_next, gcol,
                                                                 W.slotY, gfix, bg, cap, W.v, W.slotD, W.s, W.counter,
                                                                 t, tol, deltas, W.status, W.stop);
        launches.fetch_add(3, std::memory_order_relaxed);
        if ((err = cudaGetLastError()) != cudaSuccess) return csr_cuda_fail(err, "rank launch");
    }
    if (ev_b) cudaEventRecord(*ev_b, s);
    k_rank_output<<<gcol, kCsrThreads, 0, s>>>(n, W.e[0], W.e[1], W.hist, W.status, b0, w_out, W.slotD);
    launches.fetch_add(1, std::memory_order_relaxed);
    if (w_l2_out) {
        k_rank_output_l2<<<gcol, kCsrThreads, 0, s>>>(n, W.e[0], W.e[1], W.hist, W.status, b0, W.slotD, gcol,
                                                      w_l2_out);
        launches.fetch_add(1, std::memory_order_relaxed);
    }
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

// ------------------------------------------------------------------ K3n: the ranking over ranks
// SURVEY 8(e) / DESIGN.md 8: rank r owns the destination rows [row0, row0 + m) of the graph (its sub-CSR:
// row_ptr rebased to 0, GLOBAL source ids in col_idx); every rank keeps the full n-node state (e, v and
// the fp64 scalars) and runs the SAME node kernels on it, so w, s_t, delta_t and the stop decision are
// bitwise identical on every rank.  Per iteration t:
//   rows:       e_t[row0 .. row0 + m) = gather-sum of v_t over the rank's edges  (K3b on the sub-CSR)
//   exchange:   all-gather of the e_t blocks (the caller's collective: NCCL; n * 4 bytes in total)
//   normalize:  sum_i e_i over all n in a fixed order -> s_t, then K3c+d unchanged (w, v_{t+1}, S, delta)
// The per-iteration launches are enqueued by the caller (one call per step), so the collective sits
// between them on the same stream; after a tol stop the remaining launches exit at once.
inline int csr_node_grid(int64_t n, int sms) {
    return (int)std::min<int64_t>({(n + kCsrThreads - 1) / kCsrThreads, (int64_t)4 * sms, (int64_t)kCsrMaxGrid});
}

// sum_i e_i over all n nodes: per-CTA fp64 partials in a fixed (grid-stride, then block tree) order
__global__ void __launch_bounds__(kCsrThreads) k_rank_esum(int64_t n, const float* __restrict__ e,
                                                           double* __restrict__ slotY, const int32_t* stop) {
    __shared__ double red[33];
    if (*(volatile const int32_t*)stop) return;
    double g = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        g += (double)e[j];
    const double G = block_sum(g, red);
    if (threadIdx.x == 0) slotY[blockIdx.x] = G;
}

inline mapi_status csr_shard_begin(int64_t n, int64_t m, int64_t nnz, const int32_t* row_ptr, const float* cap,
                                   const float* bg, const float* b0, void* ws, int sms, cudaStream_t s,
                                   std::atomic<uint64_t>& launches) {
    CsrWs W = carve_csr(ws, n, nnz, m);
    cudaError_t err = cudaMemsetAsync(ws, 0, 256, s);
    if (err != cudaSuccess) return csr_cuda_fail(err, "memset");
    if (m > 0) {
        k_mp_partition<<<(unsigned)((W.tiles + 1 + 255) / 256), 256, 0, s>>>(m, nnz, row_ptr, W.tiles, W.part_i,
                                                                              W.part_k);
        launches.fetch_add(1, std::memory_order_relaxed);
    }
    k_rank_init<<<csr_node_grid(n, sms), kCsrThreads, 0, s>>>(n, b0, bg, cap, W.v, W.slotS, W.status, W.stop);
    launches.fetch_add(1, std::memory_order_relaxed);
    if ((err = cudaGetLastError()) != cudaSuccess) return csr_cuda_fail(err, "shard begin launch");
    return MAPI_OK;
}

// iteration t's gather over the owned rows; *e_out = the n-float device array e_t whose block
// [row0, row0 + m) is now valid and whose other blocks the exchange fills
inline mapi_status csr_shard_rows(int64_t n, int64_t m, int64_t row0, int64_t nnz, const int32_t* row_ptr,
                                  const int32_t* col_idx, int32_t t, float** e_out, void* ws, cudaStream_t s,
                                  std::atomic<uint64_t>& launches) {
    CsrWs W = carve_csr(ws, n, nnz, m);
    float* e_cur = W.e[t & 1];
    if (e_out) *e_out = e_cur;
    if (m == 0) return MAPI_OK;
    const int64_t T = W.tiles;
    const int gfix = (int)std::min<int64_t>((T + 255) / 256, kCsrMaxGrid);
    k_rank_rows_mp<<<(unsigned)T, kMpThreads, 0, s>>>(m, nnz, row_ptr, col_idx, W.v, W.part_i, W.part_k,
                                                      e_cur + row0, W.carry_row, W.carry_val, W.gsum, W.stop);
    // the carries of rows spanning tiles; its slotY output (the LOCAL sum of e) is overwritten by
    // csr_shard_normalize's sum over all n
    k_rank_fixup<<<gfix, 256, 0, s>>>(T, W.carry_row, W.carry_val, W.gsum, e_cur + row0, W.slotY, W.stop);
    launches.fetch_add(2, std::memory_order_relaxed);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return csr_cuda_fail(err, "shard rows launch");
    return MAPI_OK;
}

// after the exchange: s_t, w_{t+1}, v_{t+1}, S_{t+1}, delta_t, trace and stop flag, on the full state
inline mapi_status csr_shard_normalize(int64_t n, int64_t m, int64_t nnz, const float* cap, const float* bg,
                                       const float* b0, int32_t t, float tol, float* deltas, void* ws, int sms,
                                       cudaStream_t s, std::atomic<uint64_t>& launches) {
    CsrWs W = carve_csr(ws, n, nnz, m);
    const int gcol = csr_node_grid(n, sms);
    const bool v4 = (reinterpret_cast<uintptr_t>(bg) % 16 == 0) && (reinterpret_cast<uintptr_t>(cap) % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(b0) % 16 == 0);
    double* S_cur = W.slotS + (t & 1) * kCsrMaxGrid;
    double* S_next = W.slotS + ((t + 1) & 1) * kCsrMaxGrid;
    float* e_cur = W.e[t & 1];
    const float* e_prev = t == 0 ? nullptr : W.e[(t + 1) & 1];
    k_rank_esum<<<gcol, kCsrThreads, 0, s>>>(n, e_cur, W.slotY, W.stop);
    if (v4)
        k_rank_normalize<true><<<gcol, kCsrThreads, 0, s>>>(n, e_cur, e_prev, b0, W.hist, S_cur, S_next, gcol, W.slotY,
                                                            gcol, bg, cap, W.v, W.slotD, W.s, W.counter, t, tol, deltas,
                                                            W.status, W.stop);
    else
        k_rank_normalize<false><<<gcol, kCsrThreads, 0, s>>>(n, e_cur, e_prev, b0, W.hist, S_cur, S_next, gcol,
                                                             W.slotY, gcol, bg, cap, W.v, W.slotD, W.s, W.counter, t,
                                                             tol, deltas, W.status, W.stop);
    launches.fetch_add(2, std::memory_order_relaxed);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return csr_cuda_fail(err, "shard normalize launch");
    return MAPI_OK;
}

inline mapi_status csr_shard_output(int64_t n, int64_t m, int64_t nnz, const float* b0, float* w_out, float* w_l2_out,
                                    void* ws, int sms, cudaStream_t s, std::atomic<uint64_t>& launches) {
    CsrWs W = carve_csr(ws, n, nnz, m);
    const int gcol = csr_node_grid(n, sms);
    k_rank_output<<<gcol, kCsrThreads, 0, s>>>(n, W.e[0], W.e[1], W.hist, W.status, b0, w_out, W.slotD);
    launches.fetch_add(1, std::memory_order_relaxed);
    if (w_l2_out) {
        k_rank_output_l2<<<gcol, kCsrThreads, 0, s>>>(n, W.e[0], W.e[1], W.hist, W.status, b0, W.slotD, gcol, w_l2_out);
        launches.fetch_add(1, std::memory_order_relaxed);
    }
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return csr_cuda_fail(err, "shard output launch");
    return MAPI_OK;
}

}  // namespace mapi
