// sym.cuh — K2s: persistent MAPI iteration for SYMMETRIC matrices reading only the upper triangle.
//
// MAPI's dense inputs are covariance matrices (Eq. 2 / Eq. 5: C = X X^T / N), symmetric by
// construction, and at n = 32768 (BASELINE configs[2]) an iteration is bound by the 4 GiB read of A.  A
// stored element a_jk (k > j) appears in two MAVP terms of y = A (+) w (Eq. 3, matrix extension
// P:69-70): term(a_jk, w_k) in y_j and term(a_kj, w_j) = term(a_jk, w_j) in y_k.  K2s reads each
// upper-triangle element once (half the HBM bytes) and forms BOTH terms — still one FMNMX.XORSIGN per term
// and no multiply, n^2 terms per iteration, exactly the same sum as the full read:
//     y_j = sum_{k >= j} term(a_jk, w_k)  [row terms]  +  sum_{k < j} term(a_kj, w_k)  [column terms].
//
// Tasks: (row block b of kSymRB = 128 rows, column chunk c of kSymCC = 256 columns = 1 KB per row) with
// chunk end > block start, i.e. chunks c >= b / 2; warps take tasks from a per-iteration atomic counter
// (~7 per warp at n = 32768; dynamic because SMs stream at different rates).  A warp streams its task row by row (lane l holds columns
// c0 + 8l .. +8 of the row: one 256-bit evict-first load; two 4-row batches in flight): the row term of the
// lane's 8 elements against w_k (registers, loaded once per task) is summed in a tree, and the 8 row
// partials of an 8-row group cross the warp in one reduce-scatter butterfly (9 shuffles) -> P_row[c][j]; the column terms against w_j (a shared-memory broadcast) accumulate per
// lane in 8 registers over the task's 64 rows (64-term chains) -> P_col[b][k].  On the diagonal tasks
// the row term keeps k >= j and the column term k > j; everything below the diagonal is skipped (never
// read into a result: the tests fill it with NaN).  w_t lives in global memory (L2) as tagged words: a task
// reads its 256 w_k (8 words per lane) and its 128 w_j (staged per warp in shared memory).
//
// Per iteration, two grid barriers: tasks -> | -> the stop test on delta_{t-1} (lagged, below) -> each CTA sums
// the partials of the rows it OWNS (a range balanced by partial count, fp64, fixed combine order):
// y_j = sum_{c >= c(j)} P_row[c][j] + sum_{b <= b(j)} P_col[b][j] (fp32 chains <= 256 terms inside the
// partials, fp64 across them: within T1), fp64 |y| partial per CTA -> | -> s_t (fixed order, every
// CTA), the owner forms w_{t+1,j} = fp32(y_j / s_t) (fp64 division, as K2c), its delta partial, and PUBLISHES
// w_{t+1,j} as one tagged 8-byte word ((t + 2) << 32 | bits) — no third barrier: the next iteration's tasks
// poll the words of their rows / columns until the tag is current (a reader that sees the tag sees the
// value: single-copy atomic 64-bit words, no fence).  delta_t is summed after the next iteration's first
// barrier, so a tol stop at t (delta_t < tol) is decided one task phase late and that phase's partials are
// discarded: the outputs are exactly those of stopping at t.  Nothing is replicated per CTA (K2c forms all n
// quotients in every CTA).  Deterministic for a given (n, grid).  Requirements: n % 8 == 0, lda % 8 == 0,
// 32 B-aligned A (the caller falls back to the full-matrix kernels otherwise); wtag 2n words zeroed per call,
// yg n floats, slots >= 4 x grid doubles.
#pragma once
#include "dense.cuh"
#include "mapi_common.cuh"
#include "resident.cuh"  // res_lane_reduce (reduce-scatter butterfly)

namespace mapi {

constexpr int kSymRB = 128;        // rows per task (column-partial chain length: T1's 128-term limit)
constexpr int kSymCC = 256;        // columns per task (one 1 KB row chunk per warp row)
constexpr int kSymPrefetchRows = 16;  // default of SymArgs::prefetch_rows (sweep: profiles/r02_probe_k2s_prefetch.log)
constexpr int kSymNW = 16;         // warps per CTA
constexpr int kSymThreads = kSymNW * 32;
constexpr int kSymCR = kSymCC / kSymRB;  // chunks per row block (2): tasks of block b start at chunk b / 2

struct SymArgs {
    IterArgs it;
    float* prow;  // [nc][n] row partials
    float* pcol;  // [nb][n] column partials
    unsigned long long* wtag;  // [2][n] tagged w words ((t + 1) << 32 | bits(w_t)), zeroed per call
    float* yg;                 // [n] y of the owned rows
    int32_t prefetch_rows;     // K2s: rows per first-wave task prefetched into L2 across the epilogue (0: off)
};

__host__ __device__ inline int64_t sym_nb(int64_t n) { return (n + kSymRB - 1) / kSymRB; }
__host__ __device__ inline int64_t sym_nc(int64_t n) { return (n + kSymCC - 1) / kSymCC; }
// sum_{x < j} floor(x / m)
__host__ __device__ inline int64_t sym_floor_sum(int64_t j, int64_t m) {
    const int64_t q = j / m, r = j % m;
    return m * q * (q - 1) / 2 + r * q;
}
// first task of row block b: sum_{b' < b} (nc - b' / kSymCR)
__host__ __device__ inline int64_t sym_task_start(int64_t b, int64_t nc) { return b * nc - sym_floor_sum(b, kSymCR); }
// partials summed for row j: row partials of chunks [j / CC, nc) + column partials of blocks [0, j / RB]
__host__ __device__ inline int64_t sym_partials_before(int64_t j, int64_t nc) {  // sum over rows < j
    return j * (nc + 1) - sym_floor_sum(j, kSymCC) + sym_floor_sum(j, kSymRB);
}
// phase-2 row ownership: CTA c owns rows [own(c), own(c+1)), balanced by the number of partials to sum
// (rows near n sum ~3x more partials than rows near 0)
__host__ __device__ inline int64_t sym_own_start(int64_t c, int64_t grid, int64_t n) {
    const int64_t nc = sym_nc(n), total = sym_partials_before(n, nc);
    int64_t lo = 0, hi = n;  // smallest j with F(j) * grid >= c * total
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((double)sym_partials_before(mid, nc) * (double)grid >= (double)c * (double)total) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}
// row-tiled partial layout: element (j, q) of an array with m entries per row at sym_tile(j, m) + 32 q
__host__ __device__ inline int64_t sym_tile(int64_t j, int64_t m) { return (j >> 5) * 32 * m + (j & 31); }
inline size_t sym_partials_bytes(int64_t n) {
    const int64_t np = (n + 31) & ~int64_t(31);  // whole 32-row tiles
    return sizeof(float) * (size_t)np * (size_t)(sym_nb(n) + sym_nc(n));
}
// per-warp w_j staging (phase 1) / one fp64 sub-sum per thread (phase 2), then the reduction scratch
constexpr int kSymSmemRegion = (kSymNW * kSymRB * 4 > kSymThreads * 8) ? kSymNW * kSymRB * 4 : kSymThreads * 8;  // bytes
inline size_t sym_smem_bytes(int64_t /*n*/) { return kSymSmemRegion + sizeof(double) * 40; }

// partial stores ask L2 to keep the lines (evict_last): the next phase re-reads them, while A streams
// through L2 evict-first
__device__ __forceinline__ uint64_t sym_keep_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void sym_st_keep(float* p, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void sym_st4_keep(float* p, float a, float b, float c, float d, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c),
                 "f"(d), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ unsigned long long sym_ld_tag(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void sym_st_tag(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long sym_tagged(uint32_t tag, float w) {
    return ((unsigned long long)tag << 32) | (unsigned long long)__float_as_uint(w);
}
// N tagged words of w_t (tag t + 1) from wt[idx[i]]: all loads in flight, then re-polled until current
template <int N>
__device__ __forceinline__ void sym_wait_words(const unsigned long long* wt, const int64_t (&idx)[N], uint32_t tag,
                                               float (&out)[N]) {
    unsigned long long v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = idx[i] >= 0 ? sym_ld_tag(wt + idx[i]) : sym_tagged(tag, 0.0f);
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int i = 0; i < N; ++i) ok &= (uint32_t)(v[i] >> 32) == tag;
        if (ok) break;
#pragma unroll
        for (int i = 0; i < N; ++i)
            if ((uint32_t)(v[i] >> 32) != tag) v[i] = sym_ld_tag(wt + idx[i]);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = __uint_as_float((uint32_t)v[i]);
}

template <int OP>
__device__ __forceinline__ float sym_tree8(const float (&a)[8], const float (&w)[8]) {
    float t[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) t[e] = mavp_term<OP>(a[e], w[e]);
    return tree_sum(t);
}

#ifdef MAPI_SYM_TRACE
__device__ long long g_sym_trace[6 * 512];  // investigation builds only (scripts/probe_k2s.cu)
__device__ long long g_sym_cta[2 * 256 * 32];  // per-CTA task-phase start / end (globaltimer), iteration < 32
#define SYM_STAMP(t, k) \
    if (blockIdx.x == 0 && threadIdx.x == 0 && (t) < 512) g_sym_trace[(t) * 6 + (k)] = clock64(); \
    if (threadIdx.x == 0 && (k) <= 1 && (t) < 32 && blockIdx.x < 256) { \
        long long gt; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt)); g_sym_cta[((t) * 256 + blockIdx.x) * 2 + (k)] = gt; }
#else
#define SYM_STAMP(t, k)
#endif

// task index of (row block b, chunk c) (c >= b / kSymCR)
__host__ __device__ inline int64_t sym_task_index(int64_t b, int64_t c, int64_t nc) {
    return sym_task_start(b, nc) + c - b / kSymCR;
}
// Sharded K2s: rank r of P takes the contiguous task range [tlo, thi) = [r T / P, (r + 1) T / P).  For row j
// its valid partials on rank r: row partials of chunks [c_lo, c_hi) (tasks of strip b(j) in the range, from
// c(j) on) and column partials of row blocks [b_lo, b_hi) (tasks (b, c(j)), b <= b(j), in the range; their
// index grows with b).  On one rank both are the full lists.
struct SymValid {
    int64_t c_lo, c_hi, b_lo, b_hi;
};
__host__ __device__ inline SymValid sym_valid(int64_t j, int64_t n, int64_t tlo, int64_t thi) {
    const int64_t nc = sym_nc(n), B = j / kSymRB, C = j / kSymCC;
    SymValid v;
    const int64_t s0 = sym_task_start(B, nc), half = B / kSymCR;  // strip B: chunks half .. nc-1
    v.c_lo = tlo - s0 + half;
    v.c_hi = thi - s0 + half;
    v.c_lo = v.c_lo < C ? C : v.c_lo;
    v.c_hi = v.c_hi > nc ? nc : v.c_hi;
    if (v.c_hi < v.c_lo) v.c_hi = v.c_lo;
    // column partials: the b in [0, B] with tlo <= index(b, C) < thi
    int64_t lo = 0, hi = B + 1;  // first b with index >= tlo
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sym_task_index(mid, C, nc) >= tlo) hi = mid;
        else lo = mid + 1;
    }
    v.b_lo = lo;
    hi = B + 1;  // first b with index >= thi
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sym_task_index(mid, C, nc) >= thi) hi = mid;
        else lo = mid + 1;
    }
    v.b_hi = lo;
    return v;
}
// the rows rank r's tasks read: strips b(tlo) .. b(thi - 1)
__host__ __device__ inline void sym_shard_rows(int64_t n, int64_t tlo, int64_t thi, int64_t& r0, int64_t& r1) {
    const int64_t nb = sym_nb(n), nc = sym_nc(n);
    auto strip = [&](int64_t task) {
        int64_t lo = 0, hi = nb - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (sym_task_start(mid, nc) <= task) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    if (thi <= tlo) {
        r0 = r1 = 0;
        return;
    }
    r0 = strip(tlo) * kSymRB;
    r1 = (strip(thi - 1) + 1) * kSymRB;
    if (r1 > n) r1 = n;
}

// ---- phase 1 of K2s: the upper-triangle tasks [tlo, thi) of w_t (tagged words wcur, tag), taken from a
// counter (`ctr`, zeroed, counts from 0).  A rows are addressed relative to row r0 (the sharded ranks hold
// only the rows of their strips).
template <int OP>
__device__ __forceinline__ void sym_tasks(const SymArgs& sa, const float* A, int64_t r0, int64_t tlo, int64_t thi,
                                          unsigned int* ctr, const unsigned long long* wcur, uint32_t tag,
                                          float* wj_s, uint64_t keep) {
    const IterArgs& p = sa.it;
    const int64_t n = p.n;
    const int lane = threadIdx.x & 31;
    const int64_t nb = sym_nb(n), nc = sym_nc(n);
    auto fetch = [&]() -> unsigned int {
        unsigned int v = 0;
        if (lane == 0) v = atomicAdd(ctr, 1u);
        return v;
    };
    unsigned int nxt = fetch();
    for (int64_t task = tlo + __shfl_sync(0xffffffffu, nxt, 0); task < thi;) {
        nxt = fetch();
        int64_t lo = 0, hi = nb - 1;  // row block: last b with start(b) <= task
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (sym_task_start(mid, nc) <= task) lo = mid;
            else hi = mid - 1;
        }
        const int64_t b = lo, c = b / kSymCR + (task - sym_task_start(b, nc));
        const int64_t j0 = b * kSymRB, j1 = min(n, j0 + kSymRB), c0 = c * kSymCC;
        const int64_t kl = c0 + 8 * lane;  // this lane's first column
        const bool live = kl < n;          // n % 8 == 0: a lane is all in or all out
        const bool diag = c0 < j1;         // some element with k <= j: masked path
        const int rows = (int)(j1 - j0);
        float* prow = sa.prow + c * 32;  // + sym_tile(j) for row j
        const float* base = A + (j0 - r0) * p.lda + kl;
        float a[2][4][8];
        auto load = [&](float (&buf)[4][8], int rb) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                // (on diagonal tasks a lane whose 8 columns all lie below the row's diagonal loads nothing:
                // every one of its terms is masked)
                if (live && rb + r < rows && kl + 7 >= j0 + rb + r)
                    ld_stream<8, 0>(base + (int64_t)(rb + r) * p.lda, buf[r]);
                else
#pragma unroll
                    for (int e = 0; e < 8; ++e) buf[r][e] = 0.0f;
            }
        };
        load(a[0], 0);  // A does not depend on w: in flight while the w words are polled
        float wk[8], col[8];
        {
            int64_t idx[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) idx[e] = live ? kl + e : -1;
            sym_wait_words<8>(wcur, idx, tag, wk);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) col[e] = 0.0f;
        __syncwarp();  // the previous task's reads of wj_s are done
        {
            int64_t idx[kSymRB / 32];
            float v[kSymRB / 32];
#pragma unroll
            for (int i = 0; i < kSymRB / 32; ++i) idx[i] = (32 * i + lane < rows) ? j0 + 32 * i + lane : -1;
            sym_wait_words<kSymRB / 32>(wcur, idx, tag, v);
#pragma unroll
            for (int i = 0; i < kSymRB / 32; ++i) wj_s[32 * i + lane] = v[i];
        }
        __syncwarp();
        // partial layouts are row-tiled ([j / 32][chunk or block][j % 32]): phase 2 reads all partials of
        // 32 consecutive rows as one contiguous run
        float pr[8];  // per-lane row partials of the current 8-row group
        // rows rb .. rb+3 of the group -> pr[h*4 .. h*4+3] (rows beyond the task add zeros and are
        // never stored)
        auto consume = [&](const float (&buf)[4][8], int rb, int h) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t j = j0 + rb + r;
                const float wj = wj_s[rb + r];
                if (!diag) {
                    pr[4 * h + r] = sym_tree8<OP>(buf[r], wk);
#pragma unroll
                    for (int e = 0; e < 8; ++e) col[e] += mavp_term<OP>(buf[r][e], wj);
                } else {
                    float tr[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int64_t k = kl + e;
                        tr[e] = k >= j ? mavp_term<OP>(buf[r][e], wk[e]) : 0.0f;
                        if (k > j) col[e] += mavp_term<OP>(buf[r][e], wj);
                    }
                    pr[4 * h + r] = tree_sum(tr);
                }
            }
        };
        // the 8 row partials of a group across the warp: reduce-scatter butterfly (9 shuffles for 8
        // rows); lanes with (lane & 3) == 0 hold row res_row_of<8>(lane) and store it
        auto finish_group = [&](int rb) {
            const float v = res_lane_reduce<8>(pr, lane);
            const int ri = res_row_of<8>(lane);
            if ((lane & 3) == 0 && rb + ri < rows) sym_st_keep(prow + sym_tile(j0 + rb + ri, nc), v, keep);
        };
        for (int rb = 0; rb < rows; rb += 8) {
            load(a[1], rb + 4);
            consume(a[0], rb, 0);
            if (rb + 8 < rows) load(a[0], rb + 8);
            consume(a[1], rb + 4, 1);
            finish_group(rb);
        }
        if (live) {  // columns kl .. kl+7 lie in one 32-column tile
            float* pc = sa.pcol + b * 32 + sym_tile(kl, nb);
            sym_st4_keep(pc, col[0], col[1], col[2], col[3], keep);
            sym_st4_keep(pc + 4, col[4], col[5], col[6], col[7], keep);
        }
        task = tlo + __shfl_sync(0xffffffffu, nxt, 0);
    }
}

// ---- phase 2 of K2s: y_j of the owned rows [o0, o1) from the partials (SHARDED: only the partials of the
// task range [tlo, thi); the others are skipped as zeros, which leaves the sums unchanged).  `subs`
// threads per row (the most that fit the owned rows in one pass), consecutive threads on consecutive rows
// (coalesced partial reads); sub k takes partials q = k, k + subs, ... in ascending order, 48 loads in
// flight, each batch summed by a fixed fp32 pairwise tree and accumulated in fp64; the subs meet in shared
// memory and are added in sub order.  out(j, v) receives fp32(y_j) (for the owner) .
template <bool SHARDED, typename Out>
__device__ __forceinline__ void sym_reduce(const SymArgs& sa, int64_t o0, int64_t o1, int64_t tlo, int64_t thi,
                                           double* redp, Out out) {
    const int64_t n = sa.it.n, nb = sym_nb(n), nc = sym_nc(n);
    const int tid = threadIdx.x;
    const int64_t rown = o1 - o0;
    const int subs = rown * 8 <= kSymThreads ? 8 : (rown * 4 <= kSymThreads ? 4 : (rown * 2 <= kSymThreads ? 2 : 1));
    const int rpp = kSymThreads / subs;  // rows per pass
    const int rl = tid % rpp, sub = tid / rpp;
    for (int64_t pbase = o0; pbase < o1; pbase += rpp) {
        const int64_t j = pbase + rl;
        double acc = 0.0;
        if (j < o1) {
            const int64_t cj = j / kSymCC, bj = j / kSymRB;
            const int64_t nrow = nc - cj, ntot = nrow + bj + 1;
            const float* prow_j = sa.prow + sym_tile(j, nc) + cj * 32;  // + q * 32
            const float* pcol_j = sa.pcol + sym_tile(j, nb);            // + b * 32
            SymValid vr{cj, nc, 0, bj + 1};
            if constexpr (SHARDED) vr = sym_valid(j, n, tlo, thi);
            for (int64_t q0 = sub; q0 < ntot; q0 += 48 * subs) {
                float v[48];
#pragma unroll
                for (int u = 0; u < 48; ++u) {
                    const int64_t q = q0 + (int64_t)u * subs;
                    if constexpr (SHARDED) {
                        const bool isrow = q < nrow;
                        const int64_t x = isrow ? cj + q : q - nrow;
                        const bool ok = q < ntot && (isrow ? (x >= vr.c_lo && x < vr.c_hi) : (x >= vr.b_lo && x < vr.b_hi));
                        v[u] = ok ? (isrow ? __ldcg(prow_j + q * 32) : __ldcg(pcol_j + (q - nrow) * 32)) : 0.0f;
                    } else {
                        v[u] = q < ntot ? (q < nrow ? __ldcg(prow_j + q * 32) : __ldcg(pcol_j + (q - nrow) * 32))
                                        : 0.0f;
                    }
                }
                // pairwise fp32 tree over the batch (6 levels), one fp64 add per batch: a per-element
                // fp64 conversion (F2F, a slow pipe) made this phase F2F-bound
#pragma unroll
                for (int h = 24; h >= 3; h >>= 1)
#pragma unroll
                    for (int u = 0; u < h; ++u) v[u] = v[2 * u] + v[2 * u + 1];
                acc += (double)((v[0] + v[1]) + v[2]);
            }
        }
        redp[tid] = acc;
        __syncthreads();
        if (tid < rpp && pbase + tid < o1) {
            double tot = 0.0;
            for (int k = 0; k < subs; ++k) tot += redp[k * rpp + tid];
            out(pbase + tid, (float)tot);
        }
        __syncthreads();
    }
}

// sum of the G fp64 slots of a parity in a fixed order (warp 0 lane-strided, butterfly), broadcast
__device__ __forceinline__ double sym_slots_sum(const double* slots, double* red, int k) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) {
        double pp = 0.0;
        for (int cc = lane; cc < (int)gridDim.x; cc += 32) pp += __ldcg(slots + cc);
        pp = warp_sum(pp);
        if (lane == 0) red[k] = pp;
    }
    __syncthreads();
    const double v = red[k];
    __syncthreads();
    return v;
}

template <int OP>
__global__ void __launch_bounds__(kSymThreads, 1) k_iterate_sym(SymArgs sa) {
    extern __shared__ __align__(16) float sm_[];
    float* wj_s = sm_ + (threadIdx.x >> 5) * kSymRB;             // per warp: w_j of its task's rows
    double* red = reinterpret_cast<double*>(reinterpret_cast<char*>(sm_) + kSymSmemRegion);
    const IterArgs& p = sa.it;
    const int64_t n = p.n;
    const int tid = threadIdx.x;
    const int64_t ntasks = sym_task_start(sym_nb(n), sym_nc(n));
    const int64_t o0 = sym_own_start(blockIdx.x, gridDim.x, n), o1 = sym_own_start(blockIdx.x + 1, gridDim.x, n);
    unsigned long long* wtag = sa.wtag;  // [2][n] by iteration parity
    float* yg = sa.yg;
    double* slotA = reinterpret_cast<double*>(p.slots);  // [2][grid] |y| partials
    double* slotD = slotA + 2 * gridDim.x;              // [2][grid] delta partials
    unsigned int epoch = 0;
    const uint64_t keep = sym_keep_policy();
    for (int64_t j = o0 + tid; j < o1; j += blockDim.x) sym_st_tag(wtag + j, sym_tagged(1u, p.b0[j]));
    grid_barrier(p.bar, ++epoch * gridDim.x);

    int32_t done = 0, status = kStOk;
    bool stopped = false;
    int32_t t = 0;
    for (; t < p.iters; ++t) {
        const unsigned long long* wcur = wtag + (t & 1) * n;  // w_t, tag t + 1
        unsigned long long* wnext = wtag + ((t + 1) & 1) * n;
        const uint32_t tag = (uint32_t)t + 1u;
        SYM_STAMP(t, 0);
        // ---- phase 1: upper-triangle tasks from a per-iteration counter (SMs stream at different rates: a
        // static deal left the fastest CTAs idle ~40 us per iteration); a task's partials do not depend on
        // which warp computes them, so the results stay bitwise reproducible
        sym_tasks<OP>(sa, p.A, 0, 0, ntasks, p.bar + 32 + (t & 1), wcur, tag, wj_s, keep);
        SYM_STAMP(t, 1);
        grid_barrier(p.bar, ++epoch * gridDim.x);
        SYM_STAMP(t, 2);
        // every warp is past its last fetch of iteration t - 1's counter: re-arm it for iteration t + 1
        if (blockIdx.x == 0 && tid == 0) p.bar[32 + ((t + 1) & 1)] = 0u;
        // ---- the lagged stop test: delta_{t-1} (partials written before this barrier) decides whether w_t
        // is the result; this iteration's task partials are then discarded
        if (t > 0) {
            const double delta = sym_slots_sum(slotD + ((t - 1) & 1) * gridDim.x, red, 33);
            if (blockIdx.x == 0 && tid == 0 && p.deltas) p.deltas[t - 1] = (float)delta;
            done = t;
            if (p.tol > 0.0f && delta < (double)p.tol) {
                stopped = true;
                break;
            }
        }
        // ---- phase 2: y_j of the owned rows, |y| partial
        double abs_part = 0.0;
        sym_reduce<false>(sa, o0, o1, 0, ntasks, reinterpret_cast<double*>(sm_), [&](int64_t j, float v) {
            yg[j] = v;
            abs_part += norm_part<OP>(v);
        });
        const double cta_abs = block_sum(abs_part, red);  // its barriers also publish yg to this CTA
        if (tid == 0) slotA[(t & 1) * gridDim.x + blockIdx.x] = cta_abs;
        // HBM is idle from here until the next tasks start (barrier, s_t, the w publish: ~16 us): pull the
        // first rows of the next iteration's first wave of tasks (counter values 0 .. G kSymNW - 1) into L2
        // (bulk prefetches: no registers, nothing to wait for; A does not depend on w)
        if (sa.prefetch_rows > 0 && t + 1 < p.iters) {
            const int64_t task = (int64_t)blockIdx.x * kSymNW + (tid >> 5);
            if (task < ntasks) {
                const int64_t nbk = sym_nb(n), nck = sym_nc(n);
                int64_t lo = 0, hi = nbk - 1;  // row block: last b with start(b) <= task
                while (lo < hi) {
                    const int64_t mid = (lo + hi + 1) >> 1;
                    if (sym_task_start(mid, nck) <= task) lo = mid;
                    else hi = mid - 1;
                }
                const int64_t c0 = (lo / kSymCR + (task - sym_task_start(lo, nck))) * kSymCC, j0 = lo * kSymRB;
                const uint32_t bytes = (uint32_t)min((int64_t)kSymCC, n - c0) * 4u;
                for (int r = tid & 31; r < sa.prefetch_rows && r < kSymRB && j0 + r < n; r += 32) {
                    const float* src = p.A + (j0 + r) * p.lda + c0;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
                }
            }
        }
        SYM_STAMP(t, 3);
        grid_barrier(p.bar, ++epoch * gridDim.x);
        SYM_STAMP(t, 4);
        // ---- s_t: the same fixed-order fp64 sum in every CTA
        const double sd = norm_final<OP>(sym_slots_sum(slotA + (t & 1) * gridDim.x, red, 32));
        if (!(sd > 0.0) || isinf(sd)) {  // uniform across the grid
            status = (sd == 0.0) ? kStDegenerate : kStNonfinite;
            done = t;
            stopped = true;
            break;
        }
        if (blockIdx.x == 0 && tid == 0 && p.norms) p.norms[t] = (float)sd;
        // ---- w_{t+1} = fp32(y / s_t) (fp64 division, as K2c) for the owned rows: published as tagged words
        // (tag t + 2) for the next tasks; the delta partial (summed after the next barrier)
        double dpart = 0.0;
        for (int64_t j = o0 + tid; j < o1; j += blockDim.x) {
            const float wn = (float)((double)__ldcg(yg + j) / sd);
            const float wo = __uint_as_float((uint32_t)sym_ld_tag(wcur + j));
            dpart += (double)fabsf(wn - wo);
            sym_st_tag(wnext + j, sym_tagged(tag + 1u, wn));
        }
        const double cta_d = block_sum(dpart, red);
        if (tid == 0) slotD[(t & 1) * gridDim.x + blockIdx.x] = cta_d;
    }
    if (!stopped) {  // ran all iterations: delta of the last one
        grid_barrier(p.bar, ++epoch * gridDim.x);
        const double delta = sym_slots_sum(slotD + ((t - 1) & 1) * gridDim.x, red, 33);
        if (blockIdx.x == 0 && tid == 0 && p.deltas) p.deltas[t - 1] = (float)delta;
        done = t;
    }
    // w_done (on a degenerate stop: the last good iterate), from the owned tagged words
    const unsigned long long* wfin = wtag + (done & 1) * n;
    for (int64_t j = o0 + tid; j < o1; j += blockDim.x) p.w_out[j] = __uint_as_float((uint32_t)sym_ld_tag(wfin + j));
    if (blockIdx.x == 0 && tid == 0) {
        p.status[0] = status;
        p.status[1] = done;
    }
}

}  // namespace mapi
