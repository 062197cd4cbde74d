// csr_plan.cu — K3s: the segmented MAPI ranking step (Eq. 13) for sm_100a.
//
// The ranking step is (K3; reading Q10)
//     y_i = S + sum_{j -> i} v_j,   S = sum_j min(bg_j, w_j),   v_j = min(max(w_j - bg_j, 0), cap_j)
// i.e. a gather-sum of v over each row's sources.  On the CSR layout (K3, csr.cuh) every one of the E'
// gathers is a scattered 4-byte L2 read that costs one L1TEX wavefront: ~245 us per iteration at cfg5
// against ~60 us of HBM traffic.  K3s changes the LAYOUT, not the arithmetic:
//   * sources with out-degree >= 1 get compact ids by DESCENDING out-degree (ties by id); compact id p
//     lives in segment p / 32767 at local offset p % 32767 (offset 32767 is a zero slot);
//   * the edges are stored segment-major, then by destination row, then in CSR order, as 16-bit words
//     `local offset | end-of-piece << 15`, where a piece is a run of <= kPieceMax edges of one row inside
//     one segment (hub rows are split so every piece is short);
//   * per iteration each CTA copies the v values of one segment (128 KB) into SHARED memory and streams
//     its contiguous, piece-aligned share of the words: every gather is a shared-memory load, every piece
//     sum a plain fp32 partial written in piece order (no atomics);
//   * the node pass sums row i's pieces in (segment, piece) order through a static slot list (pieces
//     sorted by row), forms y_i = S + e_i and the fp64 node state exactly as K3 does.
// Everything runs in ONE persistent cooperative launch: init, then per iteration phase A (pieces) ->
// grid barrier -> phase B (nodes) -> grid barrier -> identical stop decision in every CTA.  A tol stop
// ends the launch on the device.  Deterministic: every sum has a fixed order for a given plan.
//
// Numerics are K3's (csr.cuh): fp32 gather sums, fp64 per-node state (R9), w_t never stored but
// recomputed bit-exactly from (S_{t-1}, s_{t-1}, e_{t-1}); the l1 norm s = n S + sum e with sum e taken in
// fp64 over the gathered values.  Operator DOT (RPI, reading R13): v_j = cap_j w_j, S = sum bg_j w_j.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/mapi.h"
#include "csr_plan.h"
#include "host_common.h"
#include "mapi_common.cuh"

using namespace mapi_host;

namespace mapi_plan {

constexpr int kSegShift = 15;
constexpr int kSegStride = 1 << kSegShift;  // floats of v per segment in the compact vector (128 KB)
constexpr int kSegSrc = kSegStride - 1;      // sources per segment; local offset kSegSrc = the zero slot
constexpr uint16_t kDummy = (uint16_t)kSegSrc;  // padding word: the zero slot, no end flag
constexpr int kPieceMax = 256;               // edges per piece
constexpr int kSegAlign = 16;                // segment starts in the word array: one thread's 16 words
constexpr int kThreads = 1024;               // planned kernel: one CTA of 32 warps per SM
constexpr int kWpt = 16;                     // words per thread per tile (two 16 B loads)
constexpr int kTile = kThreads * kWpt;       // 16384 words per CTA tile
constexpr int kMaxGrid = 1024;
constexpr int kPieceWeight = 2;              // CTA balance: an edge weighs 1, a piece 2 more (its store)
constexpr int kWarps = kThreads / 32;
constexpr uint64_t kMagic = 0x4d415049504c414eull;  // "MAPIPLAN"

inline size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
inline int64_t max_segments(int64_t n) { return (n + kSegSrc - 1) / kSegSrc; }

// ------------------------------------------------------------------------------- plan layout
// [hdr 256: magic, n, nnz, nsrc, npieces, nwords, nseg, grid]
// [q n i32: compact v index seg*32768 + off, -1 if dangling]   [segb nseg+1 i32: padded word start]
// [ctab grid+1 i32: CTA word ranges]  [ctap grid+1 i32: CTA first piece]
// [rsp n+1 i32: row i's slots]  [pos npieces i32: slot -> piece]  [words nwords u16]
struct PlanView {
    int32_t *q, *segb, *ctab, *ctap, *rsp, *pos;
    uint16_t* words;
};
inline PlanView plan_view(void* plan, int64_t n, int64_t nseg, int grid, int64_t npieces) {
    char* p = static_cast<char*>(plan) + 256;
    PlanView v;
    v.q = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)n);
    v.segb = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)(nseg + 1));
    v.ctab = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)(grid + 1));
    v.ctap = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)(grid + 1));
    v.rsp = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)(n + 1));
    v.pos = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)std::max<int64_t>(npieces, 1));
    v.words = reinterpret_cast<uint16_t*>(p);
    return v;
}
inline size_t plan_bytes_exact(int64_t n, int64_t nseg, int grid, int64_t npieces, int64_t nwords) {
    return 256 + al256(4 * (size_t)n) + al256(4 * (size_t)(nseg + 1)) + 2 * al256(4 * (size_t)(grid + 1)) +
           al256(4 * (size_t)(n + 1)) + al256(4 * (size_t)std::max<int64_t>(npieces, 1)) + al256(2 * (size_t)nwords);
}
inline int64_t nwords_bound(int64_t nnz, int64_t nseg) { return nnz + (int64_t)kSegAlign * (nseg + 1); }

size_t plan_bytes_bound(int64_t n, int64_t nnz) {
    if (n < 1 || nnz < 0) return 0;
    const int64_t nseg = max_segments(n);
    // npieces <= nnz (every piece holds >= 1 edge)
    return plan_bytes_exact(n, nseg, kMaxGrid, nnz, nwords_bound(nnz, nseg));
}

// ------------------------------------------------------------------------------- build workspace
struct BuildWs {
    uint32_t *outdeg, *skey, *skey2;
    int32_t *sval, *sval2;
    int32_t* erow;
    uint32_t *ekey, *ekey2;
    int32_t *eval, *eval2;
    int32_t* srow;
    uint16_t* soff;
    int32_t *runb, *runb2;
    uint32_t *pe, *pid;
    int32_t *prow, *pend, *piota, *prow2;
    int32_t *segstart, *rcnt;
    uint32_t* counter;  // [0] nsrc
    void* cub;
    size_t cub_bytes;
};

struct MaxOp {
    __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

inline size_t cub_bytes_needed(int64_t n, int64_t nnz) {
    const int nn = (int)std::max<int64_t>(n, 1), ne = (int)std::max<int64_t>(nnz, 1);
    size_t a = 0, b = 0, c = 0, d = 0, e = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, std::max(nn, ne), 0, 32);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, ne);
    cub::DeviceScan::InclusiveScan(nullptr, c, (const int32_t*)nullptr, (int32_t*)nullptr, MaxOp{}, ne);
    cub::DeviceScan::ExclusiveSum(nullptr, d, (const int32_t*)nullptr, (int32_t*)nullptr, nn + 1);
    e = std::max(std::max(a, b), std::max(c, d));
    return e + 1024;
}

size_t plan_build_ws_bytes(int64_t n, int64_t nnz) {
    if (n < 1 || nnz < 0) return 0;
    const size_t N = 4 * (size_t)(n + 1), E = 4 * (size_t)std::max<int64_t>(nnz, 1);
    return 256 + 5 * al256(N) + 10 * al256(E) + al256(2 * (size_t)std::max<int64_t>(nnz, 1)) + 5 * al256(E) +
           al256(4 * (size_t)(max_segments(n) + 1)) + al256(N) + al256(cub_bytes_needed(n, nnz));
}

inline BuildWs carve_build(void* ws, int64_t n, int64_t nnz) {
    char* p = static_cast<char*>(ws);
    BuildWs b;
    b.counter = reinterpret_cast<uint32_t*>(p);
    p += 256;
    const size_t N = al256(4 * (size_t)(n + 1)), E = al256(4 * (size_t)std::max<int64_t>(nnz, 1));
    auto takeN = [&]() { char* r = p; p += N; return r; };
    auto takeE = [&]() { char* r = p; p += E; return r; };
    b.outdeg = reinterpret_cast<uint32_t*>(takeN());
    b.skey = reinterpret_cast<uint32_t*>(takeN());
    b.skey2 = reinterpret_cast<uint32_t*>(takeN());
    b.sval = reinterpret_cast<int32_t*>(takeN());
    b.sval2 = reinterpret_cast<int32_t*>(takeN());
    b.erow = reinterpret_cast<int32_t*>(takeE());
    b.ekey = reinterpret_cast<uint32_t*>(takeE());
    b.ekey2 = reinterpret_cast<uint32_t*>(takeE());
    b.eval = reinterpret_cast<int32_t*>(takeE());
    b.eval2 = reinterpret_cast<int32_t*>(takeE());
    b.srow = reinterpret_cast<int32_t*>(takeE());
    b.runb = reinterpret_cast<int32_t*>(takeE());
    b.runb2 = reinterpret_cast<int32_t*>(takeE());
    b.pe = reinterpret_cast<uint32_t*>(takeE());
    b.pid = reinterpret_cast<uint32_t*>(takeE());
    b.soff = reinterpret_cast<uint16_t*>(p);
    p += al256(2 * (size_t)std::max<int64_t>(nnz, 1));
    b.prow = reinterpret_cast<int32_t*>(takeE());
    b.pend = reinterpret_cast<int32_t*>(takeE());
    b.piota = reinterpret_cast<int32_t*>(takeE());
    b.prow2 = reinterpret_cast<int32_t*>(takeE());
    takeE();  // spare
    b.segstart = reinterpret_cast<int32_t*>(p);
    p += al256(4 * (size_t)(max_segments(n) + 1));
    b.rcnt = reinterpret_cast<int32_t*>(takeN());
    b.cub = p;
    b.cub_bytes = cub_bytes_needed(n, nnz);
    return b;
}

// ------------------------------------------------------------------------------- build kernels
__global__ void kp_outdeg(int64_t nnz, const int32_t* __restrict__ col_idx, uint32_t* __restrict__ outdeg) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(outdeg + col_idx[e], 1u);  // integer histogram: order-independent
}

// sort key: descending out-degree (dangling last), value = id (stable sort keeps ties by ascending id)
__global__ void kp_src_keys(int64_t n, const uint32_t* __restrict__ outdeg, uint32_t* __restrict__ key,
                            int32_t* __restrict__ val, uint32_t* nsrc) {
    uint32_t cnt = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t d = outdeg[j];
        key[j] = 0xffffffffu - d;
        val[j] = (int32_t)j;
        cnt += d > 0;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nsrc, cnt);
}

__global__ void kp_q(int64_t nsrc, const int32_t* __restrict__ order, int32_t* __restrict__ q) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nsrc; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t seg = p / kSegSrc, off = p - seg * kSegSrc;
        q[order[p]] = (int32_t)(seg * kSegStride + off);
    }
}

// per edge: its row (binary search in row_ptr), segment key, edge id
__global__ void kp_edges(int64_t n, int64_t nnz, const int32_t* __restrict__ row_ptr,
                         const int32_t* __restrict__ col_idx, const int32_t* __restrict__ q,
                         int32_t* __restrict__ erow, uint32_t* __restrict__ ekey, int32_t* __restrict__ eval) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n - 1;  // the row i with row_ptr[i] <= e < row_ptr[i+1]
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if ((int64_t)row_ptr[mid] <= e) lo = mid;
            else hi = mid - 1;
        }
        erow[e] = (int32_t)lo;
        ekey[e] = (uint32_t)(q[col_idx[e]] >> kSegShift);
        eval[e] = (int32_t)e;
    }
}

// sorted position k: row, local offset, run-start marker (max-scanned into the run begin), segment starts
__global__ void kp_sorted(int64_t nnz, const uint32_t* __restrict__ eks, const int32_t* __restrict__ evs,
                          const int32_t* __restrict__ erow, const int32_t* __restrict__ col_idx,
                          const int32_t* __restrict__ q, int32_t* __restrict__ srow, uint16_t* __restrict__ soff,
                          int32_t* __restrict__ runmark, int32_t* __restrict__ segstart) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t e = evs[k];
        const int32_t row = erow[e];
        const uint32_t seg = eks[k];
        srow[k] = row;
        soff[k] = (uint16_t)(q[col_idx[e]] & (kSegStride - 1));
        bool start = k == 0;
        if (!start) {
            const uint32_t sp = eks[k - 1];
            start = sp != seg || erow[evs[k - 1]] != row;
            if (sp != seg) segstart[seg] = (int32_t)k;
        } else {
            segstart[seg] = 0;
        }
        runmark[k] = start ? (int32_t)k : 0;
    }
}

// end-of-piece flags: the run ends, or the piece reached kPieceMax edges
__global__ void kp_piece_end(int64_t nnz, const int32_t* __restrict__ runb, const int32_t* __restrict__ runmark,
                             uint32_t* __restrict__ pe) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        // runmark[k+1] != 0 <=> a run starts at k+1 (k+1 > 0)
        const bool next_run = (k + 1 == nnz) || runmark[k + 1] != 0;
        const bool full = ((k - runb[k] + 1) % kPieceMax) == 0;
        pe[k] = (next_run || full) ? 1u : 0u;
    }
}

// per piece (at its last edge k): its row and its (unpadded) end; per-row piece counts
__global__ void kp_pieces(int64_t nnz, const uint32_t* __restrict__ pe, const uint32_t* __restrict__ pid,
                          const int32_t* __restrict__ srow, int32_t* __restrict__ prow, int32_t* __restrict__ pend,
                          int32_t* __restrict__ piota, int32_t* __restrict__ rcnt) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        if (!pe[k]) continue;
        const uint32_t p = pid[k];
        prow[p] = srow[k];
        pend[p] = (int32_t)(k + 1);
        piota[p] = (int32_t)p;
        atomicAdd(rcnt + srow[k], 1);
    }
}

// padded segment starts (one thread: nseg is small)
__global__ void kp_segb(int32_t nseg, int64_t nnz, int32_t* __restrict__ segstart, int32_t* __restrict__ segb) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    segstart[nseg] = (int32_t)nnz;
    int64_t acc = 0;
    for (int32_t s = 0; s < nseg; ++s) {
        segb[s] = (int32_t)acc;
        const int64_t cnt = (int64_t)segstart[s + 1] - segstart[s];
        acc += (cnt + kSegAlign - 1) / kSegAlign * kSegAlign;
    }
    segb[nseg] = (int32_t)acc;
}

__global__ void kp_fill_words(int64_t nwords, uint16_t* __restrict__ words) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nwords; k += (int64_t)gridDim.x * blockDim.x)
        words[k] = kDummy;
}

__global__ void kp_words(int64_t nnz, const uint32_t* __restrict__ eks, const uint16_t* __restrict__ soff,
                         const uint32_t* __restrict__ pe, const int32_t* __restrict__ segstart,
                         const int32_t* __restrict__ segb, uint16_t* __restrict__ words) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t s = eks[k];
        words[k + segb[s] - segstart[s]] = (uint16_t)(soff[k] | (pe[k] << 15));
    }
}

// CTA c's first piece: the pieces whose cumulative weight (edges + kPieceWeight per piece) is <= c W / G;
// its word range starts at that piece's first (padded) word.  Piece-aligned boundaries: no carries
// between CTAs.
__global__ void kp_cta(int grid, int64_t nnz, int64_t npieces, int64_t nwords, const int32_t* __restrict__ pend,
                       const uint32_t* __restrict__ eks, const int32_t* __restrict__ segstart,
                       const int32_t* __restrict__ segb, int32_t* __restrict__ ctab, int32_t* __restrict__ ctap) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > grid) return;
    if (c == 0 || c == grid) {
        ctab[c] = c == 0 ? 0 : (int32_t)nwords;
        ctap[c] = c == 0 ? 0 : (int32_t)npieces;
        return;
    }
    const double W = (double)nnz + (double)kPieceWeight * (double)npieces;
    const double target = W * (double)c / (double)grid;
    int64_t lo = 0, hi = npieces;  // count of pieces p with Wend(p) <= target
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const double wend = (double)pend[mid] + (double)kPieceWeight * (double)(mid + 1);
        if (wend <= target) lo = mid + 1;
        else hi = mid;
    }
    const int64_t P = lo;
    ctap[c] = (int32_t)P;
    if (P >= npieces) {
        ctab[c] = (int32_t)nwords;
    } else {
        const int64_t k = P == 0 ? 0 : pend[P - 1];  // first edge of piece P
        const uint32_t s = eks[k];
        ctab[c] = (int32_t)(k + segb[s] - segstart[s]);
    }
}

}  // namespace mapi_plan

// ================================================================================ run
namespace mapi_plan {

// workspace: [hdr 256: status[2] @0, stop @8, bar u32 @12, hist (S, s) x 2 f64 @32, flags @96]
//            [e0 n f32][e1 n f32][vc nseg*32768 f32][part npieces f32]
//            [slotS 2*G f64][slotY G f64][slotD G f64][slotQ G f64]
struct RunWs {
    int32_t* status;
    int32_t* stop;
    unsigned* bar;
    double* hist;
    float *e0, *e1, *vc, *part;
    double *slotS, *slotY, *slotD, *slotQ;
};
inline size_t run_ws_exact(int64_t n, int64_t nseg, int64_t npieces) {
    return 256 + 2 * al256(4 * (size_t)n) + al256(4 * (size_t)kSegStride * (size_t)std::max<int64_t>(nseg, 1)) +
           al256(4 * (size_t)std::max<int64_t>(npieces, 1)) + 5 * al256(8 * (size_t)kMaxGrid);
}
size_t rank_plan_ws_bytes(int64_t n, int64_t nnz) {
    if (n < 1 || nnz < 0) return 0;
    return run_ws_exact(n, max_segments(n), std::max<int64_t>(nnz, 1));
}
inline RunWs carve_run(void* ws, int64_t n, int64_t nseg, int64_t npieces) {
    char* p = static_cast<char*>(ws);
    RunWs r;
    r.status = reinterpret_cast<int32_t*>(p);
    r.stop = reinterpret_cast<int32_t*>(p + 8);
    r.bar = reinterpret_cast<unsigned*>(p + 12);
    r.hist = reinterpret_cast<double*>(p + 32);
    p += 256;
    r.e0 = reinterpret_cast<float*>(p); p += al256(4 * (size_t)n);
    r.e1 = reinterpret_cast<float*>(p); p += al256(4 * (size_t)n);
    r.vc = reinterpret_cast<float*>(p); p += al256(4 * (size_t)kSegStride * (size_t)std::max<int64_t>(nseg, 1));
    r.part = reinterpret_cast<float*>(p); p += al256(4 * (size_t)std::max<int64_t>(npieces, 1));
    r.slotS = reinterpret_cast<double*>(p); p += 2 * al256(8 * (size_t)kMaxGrid);
    r.slotY = reinterpret_cast<double*>(p); p += al256(8 * (size_t)kMaxGrid);
    r.slotD = reinterpret_cast<double*>(p); p += al256(8 * (size_t)kMaxGrid);
    r.slotQ = reinterpret_cast<double*>(p);
    return r;
}

struct RunArgs {
    int64_t n;
    int32_t nseg, iters;
    float tol;
    const int32_t *q, *segb, *ctab, *ctap, *rsp, *pos;
    const uint16_t* words;
    const float *cap, *bg, *b0;
    float* deltas;
    RunWs w;
};

// x / d for the node quotients given rd = 1/d: the residual-corrected quotient (as csr.cuh's qdiv), so a
// recomputed w_t is bit-identical to the one formed the iteration before
__device__ __forceinline__ double qdiv(double x, double d, double rd) {
    const double q0 = x * rd;
    return fma(fma(-q0, d, x), rd, q0);
}
// per-node terms: v_j and the background part of S.  min-type (Eq. 13 via F7): v = min(max(w - bg, 0), cap),
// S += min(bg, w).  DOT (RPI on G, reading R13): v = cap w, S += bg w.
template <int OP>
__device__ __forceinline__ float node_v(double w, float bg, float cap) {
    if constexpr (OP == 2) return (float)((double)cap * w);
    else return (float)fmin(fmax(w - (double)bg, 0.0), (double)cap);
}
template <int OP>
__device__ __forceinline__ double node_s(double w, float bg) {
    if constexpr (OP == 2) return (double)bg * w;
    else return fmin((double)bg, w);
}

// sum of G fp64 slots in a fixed order (warp 0 lane-strided, butterfly), broadcast; slots written by
// other CTAs of this launch are read through L2
__device__ __forceinline__ double slots_sum(const double* slots, int count, double* red) {
    __syncthreads();
    if (threadIdx.x < 32) {
        double part = 0.0;
        for (int c = threadIdx.x; c < count; c += 32) part += __ldcg(slots + c);
        part = mapi::warp_sum(part);
        if (threadIdx.x == 0) red[32] = part;
    }
    __syncthreads();
    return red[32];
}

// segmented-scan element: piece count, carried fp32 sum, "a piece ended here" flag
struct ScanEl {
    int c;
    float v;
    int f;
};
__device__ __forceinline__ ScanEl scan_op(const ScanEl& a, const ScanEl& b) {  // a before b
    return ScanEl{a.c + b.c, b.f ? b.v : a.v + b.v, a.f | b.f};
}

struct PlanSmem {
    ScanEl wtot[kWarps];   // warp inclusive totals
    ScanEl wpre[kWarps];   // exclusive warp prefixes (incl. the tile carry)
    ScanEl total;          // tile carry-out
    double red[33];
};

template <int OP>
__global__ void __launch_bounds__(kThreads, 1) k_rank_plan(RunArgs a) {
    extern __shared__ __align__(16) float vseg[];  // kSegStride floats
    __shared__ PlanSmem sm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t n = a.n;
    RunWs& W = a.w;
    unsigned epoch = 0;
    // node range of this CTA (phase B / init): contiguous, multiple of 4
    const int64_t chunk = ((n + G - 1) / G + 3) & ~int64_t(3);
    const int64_t j0 = std::min<int64_t>(n, (int64_t)c * chunk), j1 = std::min<int64_t>(n, j0 + chunk);

    // ---- init: w_0 = b0 (>= 0), v, S_0 partials (parity 0)
    {
        double sp = 0.0;
        int neg = 0;
        for (int64_t j = j0 + tid; j < j1; j += kThreads) {
            const double wj = (double)a.b0[j];
            neg |= wj < 0.0;
            const float b = a.bg[j];
            const int32_t qj = a.q[j];
            if (qj >= 0) W.vc[qj] = node_v<OP>(wj, b, a.cap[j]);
            sp += node_s<OP>(wj, b);
        }
        if (__syncthreads_or(neg) && tid == 0) {
            W.status[0] = MAPI_ERR_NEGATIVE;
            W.stop[0] = 1;
        }
        const double S = mapi::block_sum(sp, sm.red);
        if (tid == 0) W.slotS[c] = S;
        mapi::grid_barrier(W.bar, ++epoch * G);
        if (*(volatile int32_t*)W.stop) return;
    }

    // CTA word range and first piece; the segment holding its first word
    const int32_t cb = a.ctab[c], ce = a.ctab[c + 1];
    const int32_t p0 = a.ctap[c];
    int s0 = 0;
    {
        int lo = 0, hi = a.nseg - 1;  // largest s with segb[s] <= cb
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (a.segb[mid] <= cb) lo = mid;
            else hi = mid - 1;
        }
        s0 = lo;
    }
    const float4* vc4 = reinterpret_cast<const float4*>(W.vc);
    const uint4* words4 = reinterpret_cast<const uint4*>(a.words);

    for (int32_t t = 0; t < a.iters; ++t) {
        // ================= phase A: piece partials of e_i = sum_{j -> i} v_j (fp32), fp64 sum of the gathers
        double gp = 0.0;
        int32_t piece = p0;
        float carry = 0.0f;
        int32_t pb = cb;
        for (int s = s0; pb < ce; ++s) {
            const int32_t run_end = min(ce, a.segb[s + 1]);
            if (run_end <= pb) continue;
            __syncthreads();  // the previous run's gathers are done
            for (int i = tid; i < kSegStride / 4; i += kThreads) reinterpret_cast<float4*>(vseg)[i] = __ldcg(vc4 + (int64_t)s * (kSegStride / 4) + i);
            __syncthreads();
            for (int32_t base = pb & ~(kWpt - 1); base < run_end; base += kTile) {
                const int32_t idx = base + tid * kWpt;
                uint32_t wd[8];
                if (idx < run_end && idx + kWpt > pb) {
                    const uint4 A = __ldcs(words4 + idx / 8), B = __ldcs(words4 + idx / 8 + 1);
                    wd[0] = A.x; wd[1] = A.y; wd[2] = A.z; wd[3] = A.w;
                    wd[4] = B.x; wd[5] = B.y; wd[6] = B.z; wd[7] = B.w;
                    if (idx < pb || idx + kWpt > run_end) {  // the CTA's first / last 16 words: mask others'
#pragma unroll
                        for (int h = 0; h < 8; ++h) {
                            const int32_t x0 = idx + 2 * h;
                            uint32_t lo16 = wd[h] & 0xffffu, hi16 = wd[h] >> 16;
                            if (x0 < pb || x0 >= run_end) lo16 = kDummy;
                            if (x0 + 1 < pb || x0 + 1 >= run_end) hi16 = kDummy;
                            wd[h] = lo16 | (hi16 << 16);
                        }
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < 8; ++h) wd[h] = (uint32_t)kDummy | ((uint32_t)kDummy << 16);
                }
                float x[kWpt];
                uint32_t fl = 0;
#pragma unroll
                for (int h = 0; h < 8; ++h) {
                    const uint32_t lo16 = wd[h] & 0xffffu, hi16 = wd[h] >> 16;
                    x[2 * h] = vseg[lo16 & 0x7fffu];
                    x[2 * h + 1] = vseg[hi16 & 0x7fffu];
                    fl |= (lo16 >> 15) << (2 * h);
                    fl |= (hi16 >> 15) << (2 * h + 1);
                }
                const int cnt = __popc(fl);
                const int last = fl ? 31 - __clz(fl) : -1;
                float tail = 0.0f;
#pragma unroll
                for (int i = 0; i < kWpt; ++i) {
                    gp += (double)x[i];
                    if (i > last) tail += x[i];
                }
                // block-wide segmented scan of (cnt, tail, cnt > 0): warp level
                ScanEl el{cnt, tail, cnt > 0};
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    ScanEl o;
                    o.c = __shfl_up_sync(0xffffffffu, el.c, off);
                    o.v = __shfl_up_sync(0xffffffffu, el.v, off);
                    o.f = __shfl_up_sync(0xffffffffu, el.f, off);
                    if (lane >= off) el = scan_op(o, el);
                }
                ScanEl ex;  // warp-exclusive
                ex.c = __shfl_up_sync(0xffffffffu, el.c, 1);
                ex.v = __shfl_up_sync(0xffffffffu, el.v, 1);
                ex.f = __shfl_up_sync(0xffffffffu, el.f, 1);
                if (lane == 0) ex = ScanEl{0, 0.0f, 0};
                if (lane == 31) sm.wtot[warp] = el;
                __syncthreads();
                if (warp == 0) {  // warp prefixes, the tile carry first
                    ScanEl x0 = sm.wtot[lane];
                    ScanEl inc = x0;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        ScanEl o;
                        o.c = __shfl_up_sync(0xffffffffu, inc.c, off);
                        o.v = __shfl_up_sync(0xffffffffu, inc.v, off);
                        o.f = __shfl_up_sync(0xffffffffu, inc.f, off);
                        if (lane >= off) inc = scan_op(o, inc);
                    }
                    const ScanEl init{0, carry, 0};
                    ScanEl exw;
                    exw.c = __shfl_up_sync(0xffffffffu, inc.c, 1);
                    exw.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
                    exw.f = __shfl_up_sync(0xffffffffu, inc.f, 1);
                    sm.wpre[lane] = lane == 0 ? init : scan_op(init, exw);
                    if (lane == 31) sm.total = scan_op(init, inc);
                }
                __syncthreads();
                const ScanEl pre = scan_op(sm.wpre[warp], ex);  // everything before this thread
                const ScanEl tot = sm.total;
                // walk: complete this thread's pieces, first one carrying the preceding threads' sums
                float acc = pre.v;
                int k = 0;
                float* out = W.part + piece + pre.c;
#pragma unroll
                for (int i = 0; i < kWpt; ++i) {
                    acc += x[i];
                    if ((fl >> i) & 1u) {
                        __stcg(out + k, acc);
                        acc = 0.0f;
                        ++k;
                    }
                }
                carry = tot.v;
                piece += tot.c;
            }
            pb = run_end;
        }
        const double Gs = mapi::block_sum(gp, sm.red);
        if (tid == 0) W.slotY[c] = Gs;
        mapi::grid_barrier(W.bar, ++epoch * G);

        // ================= phase B: s = n S + sum e, w_{t+1} = (S + e) / s (fp64), delta, next v and S
        const double S = slots_sum(W.slotS + (t & 1) * kMaxGrid, G, sm.red);
        const double s = (double)n * S + slots_sum(W.slotY, G, sm.red);
        if (!(s > 0.0) || isinf(s)) {  // uniform: every CTA sees the same s
            if (c == 0 && tid == 0) {
                W.status[0] = (s == 0.0) ? MAPI_ERR_DEGENERATE : MAPI_ERR_NONFINITE;
                W.stop[0] = 1;
            }
            return;
        }
        const bool first = t == 0;
        // (S_{t-1}, s_{t-1}) written by CTA 0 last iteration: read through L2 (L1 is not coherent)
        const double Sp = first ? 0.0 : __ldcg(W.hist + (t & 1) * 2);
        const double sp_ = first ? 1.0 : __ldcg(W.hist + (t & 1) * 2 + 1);
        const double rs = 1.0 / s, rsp = 1.0 / sp_;
        float* e_cur = (t & 1) ? W.e1 : W.e0;
        const float* e_prev = (t & 1) ? W.e0 : W.e1;
        double dp = 0.0, sn = 0.0;
        for (int64_t j = j0 + tid; j < j1; j += kThreads) {
            const int32_t r0 = __ldg(a.rsp + j), r1 = __ldg(a.rsp + j + 1);
            float e = 0.0f;
            for (int32_t r = r0; r < r1; ++r) e += __ldcg(W.part + __ldg(a.pos + r));
            const double wn = qdiv(S + (double)e, s, rs);
            const double wo = first ? (double)a.b0[j] : qdiv(Sp + (double)__ldcg(e_prev + j), sp_, rsp);
            dp += fabs(wn - wo);
            const float b = a.bg[j];
            const int32_t qj = a.q[j];
            if (qj >= 0) W.vc[qj] = node_v<OP>(wn, b, a.cap[j]);
            sn += node_s<OP>(wn, b);
            e_cur[j] = e;
        }
        const double D = mapi::block_sum(dp, sm.red);
        const double Sn = mapi::block_sum(sn, sm.red);
        if (tid == 0) {
            W.slotD[c] = D;
            W.slotS[((t + 1) & 1) * kMaxGrid + c] = Sn;
        }
        mapi::grid_barrier(W.bar, ++epoch * G);
        const double d = slots_sum(W.slotD, G, sm.red);
        if (c == 0 && tid == 0) {
            W.hist[((t + 1) & 1) * 2] = S;
            W.hist[((t + 1) & 1) * 2 + 1] = s;
            if (a.deltas) a.deltas[t] = (float)d;
            W.status[1] = t + 1;
        }
        if (a.tol > 0.0f && d < (double)a.tol) break;  // uniform decision
    }
}

// Outputs: w = (S + e)/s of the last iteration (b0 if none) in fp64 as the loop formed it; w_out = fp32(w),
// per-CTA sums of w^2, then the optional l2 copy.
struct Last {
    const float* e;
    double S, s;
    bool none;
};
__device__ __forceinline__ Last last_iter(const RunWs& W) {
    const int32_t done = W.status[1];
    Last r;
    r.none = done == 0;
    const int32_t last = done - 1;
    r.e = (last & 1) ? W.e1 : W.e0;
    r.S = r.none ? 0.0 : W.hist[((last + 1) & 1) * 2];
    r.s = r.none ? 1.0 : W.hist[((last + 1) & 1) * 2 + 1];
    return r;
}
__global__ void __launch_bounds__(256) k_plan_output(int64_t n, RunWs W, const float* __restrict__ b0,
                                                     float* __restrict__ w_out) {
    __shared__ double red[33];
    const Last L = last_iter(W);
    const double rls = 1.0 / L.s;
    double part = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double x = L.none ? (double)b0[j] : qdiv(L.S + (double)L.e[j], L.s, rls);
        w_out[j] = (float)x;
        part = fma(x, x, part);
    }
    const double qs = mapi::block_sum(part, red);
    if (threadIdx.x == 0) W.slotQ[blockIdx.x] = qs;
}
__global__ void __launch_bounds__(256) k_plan_output_l2(int64_t n, RunWs W, const float* __restrict__ b0, int nq,
                                                        float* __restrict__ w_l2) {
    __shared__ double red[33];
    const Last L = last_iter(W);
    const double rls = 1.0 / L.s;
    if (threadIdx.x < 32) {
        double p = 0.0;
        for (int c = threadIdx.x; c < nq; c += 32) p += W.slotQ[c];
        p = mapi::warp_sum(p);
        if (threadIdx.x == 0) red[32] = p;
    }
    __syncthreads();
    const double l2 = sqrt(red[32]);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double x = L.none ? (double)b0[j] : qdiv(L.S + (double)L.e[j], L.s, rls);
        w_l2[j] = l2 > 0.0 ? (float)(x / l2) : 0.0f;
    }
}

}  // namespace mapi_plan

// ================================================================================ C ABI
using namespace mapi_plan;

extern "C" {

mapi_status mapi_csr_plan(int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* col_idx, void* plan,
                          size_t plan_bytes, mapi_csr_plan_info* info, void* ws, size_t ws_bytes,
                          mapi_stream_t stream) {
    if (n < 1) return fail(MAPI_ERR_SHAPE, "n (%lld) must be >= 1", (long long)n);
    if (n >= (int64_t)INT32_MAX - kSegStride)
        return fail(MAPI_ERR_SHAPE, "n (%lld) out of the int32 index range", (long long)n);
    if (nnz < 0 || nnz >= (int64_t)INT32_MAX - kSegAlign * (max_segments(n) + 2))
        return fail(MAPI_ERR_SHAPE, "nnz (%lld) out of the int32 index range", (long long)nnz);
    if (!row_ptr || !plan || !info || (nnz > 0 && !col_idx))
        return fail(MAPI_ERR_NULL, "row_ptr / col_idx / plan / info is NULL");
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    if (ws_bytes < plan_build_ws_bytes(n, nnz))
        return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, plan_build_ws_bytes(n, nnz));
    if (plan_bytes < plan_bytes_bound(n, nnz))
        return fail(MAPI_ERR_WORKSPACE, "plan_bytes (%zu) < required (%zu)", plan_bytes, plan_bytes_bound(n, nnz));
    Device d;
    mapi_status st = device_info(d);
    if (st != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int occ = 0;
    MAPI_CUDA(cudaFuncSetAttribute(k_rank_plan<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kSegStride));
    MAPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rank_plan<0>, kThreads, 4 * kSegStride));
    if (occ < 1) return fail(MAPI_ERR_CUDA, "planned ranking kernel does not fit on an SM");
    const int grid = std::min(d.sms, kMaxGrid);
    BuildWs B = carve_build(ws, n, nnz);
    const unsigned g1 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * (int64_t)d.sms));
    const unsigned ge = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nnz + 255) / 256, 16 * (int64_t)d.sms));
    MAPI_CUDA(cudaMemsetAsync(B.counter, 0, 256, s));
    MAPI_CUDA(cudaMemsetAsync(B.outdeg, 0, 4 * (size_t)n, s));
    MAPI_CUDA(cudaMemsetAsync(B.rcnt, 0, 4 * (size_t)(n + 1), s));
    if (nnz > 0) {
        kp_outdeg<<<ge, 256, 0, s>>>(nnz, col_idx, B.outdeg);
        MAPI_LAUNCHED();
    }
    kp_src_keys<<<g1, 256, 0, s>>>(n, B.outdeg, B.skey, B.sval, B.counter);
    MAPI_LAUNCHED();
    size_t tb = B.cub_bytes;
    MAPI_CUDA(cub::DeviceRadixSort::SortPairs(B.cub, tb, B.skey, B.skey2, B.sval, B.sval2, (int)n, 0, 32, s));
    uint32_t nsrc_h = 0;
    MAPI_CUDA(cudaMemcpyAsync(&nsrc_h, B.counter, 4, cudaMemcpyDeviceToHost, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    const int64_t nsrc = nsrc_h;
    const int32_t nseg = (int32_t)std::max<int64_t>(1, (nsrc + kSegSrc - 1) / kSegSrc);
    PlanView P = plan_view(plan, n, nseg, grid, std::max<int64_t>(nnz, 1));  // pos sized by the bound for now
    MAPI_CUDA(cudaMemsetAsync(P.q, 0xff, 4 * (size_t)n, s));
    if (nsrc > 0) {
        kp_q<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nsrc + 255) / 256, 8 * (int64_t)d.sms)), 256, 0, s>>>(
            nsrc, B.sval2, P.q);
        MAPI_LAUNCHED();
    }
    int64_t npieces = 0, nwords = 0;
    if (nnz > 0) {
        kp_edges<<<ge, 256, 0, s>>>(n, nnz, row_ptr, col_idx, P.q, B.erow, B.ekey, B.eval);
        MAPI_LAUNCHED();
        int bits = 1;
        while ((1ll << bits) < (int64_t)nseg) ++bits;
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceRadixSort::SortPairs(B.cub, tb, B.ekey, B.ekey2, B.eval, B.eval2, (int)nnz, 0, bits, s));
        kp_sorted<<<ge, 256, 0, s>>>(nnz, B.ekey2, B.eval2, B.erow, col_idx, P.q, B.srow, B.soff, B.runb, B.segstart);
        MAPI_LAUNCHED();
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceScan::InclusiveScan(B.cub, tb, B.runb, B.runb2, MaxOp{}, (int)nnz, s));
        kp_piece_end<<<ge, 256, 0, s>>>(nnz, B.runb2, B.runb, B.pe);
        MAPI_LAUNCHED();
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceScan::ExclusiveSum(B.cub, tb, B.pe, B.pid, (int)nnz, s));
        uint32_t last[2] = {0, 0};
        MAPI_CUDA(cudaMemcpyAsync(&last[0], B.pid + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
        MAPI_CUDA(cudaMemcpyAsync(&last[1], B.pe + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
        MAPI_CUDA(cudaStreamSynchronize(s));
        npieces = (int64_t)last[0] + last[1];
        kp_pieces<<<ge, 256, 0, s>>>(nnz, B.pe, B.pid, B.srow, B.prow, B.pend, B.piota, B.rcnt);
        MAPI_LAUNCHED();
        kp_segb<<<1, 32, 0, s>>>(nseg, nnz, B.segstart, P.segb);
        MAPI_LAUNCHED();
        int32_t nw = 0;
        MAPI_CUDA(cudaMemcpyAsync(&nw, P.segb + nseg, 4, cudaMemcpyDeviceToHost, s));
        MAPI_CUDA(cudaStreamSynchronize(s));
        nwords = nw;
    } else {
        MAPI_CUDA(cudaMemsetAsync(P.segb, 0, 4 * (size_t)(nseg + 1), s));
    }
    // final layout with the exact piece count (pos shrinks; words follow it)
    P = plan_view(plan, n, nseg, grid, npieces);
    if (nwords > 0) {
        kp_fill_words<<<(unsigned)std::min<int64_t>((nwords + 255) / 256, 16 * (int64_t)d.sms), 256, 0, s>>>(nwords, P.words);
        MAPI_LAUNCHED();
        kp_words<<<ge, 256, 0, s>>>(nnz, B.ekey2, B.soff, B.pe, B.segstart, P.segb, P.words);
        MAPI_LAUNCHED();
        // slots: pieces stably sorted by row (the (segment, piece) order within a row is kept)
        int rbits = 1;
        while ((1ll << rbits) < n) ++rbits;
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceRadixSort::SortPairs(B.cub, tb, B.prow, B.prow2, B.piota, P.pos, (int)npieces, 0, rbits, s));
    }
    tb = B.cub_bytes;
    MAPI_CUDA(cub::DeviceScan::ExclusiveSum(B.cub, tb, B.rcnt, P.rsp, (int)(n + 1), s));
    kp_cta<<<(unsigned)((grid + 1 + 127) / 128), 128, 0, s>>>(grid, nnz, npieces, nwords, B.pend, B.ekey2, B.segstart,
                                                               P.segb, P.ctab, P.ctap);
    MAPI_LAUNCHED();
    struct {
        uint64_t magic;
        int64_t n, nnz, nsrc, npieces, nwords;
        int32_t nseg, grid;
    } hdr = {kMagic, n, nnz, nsrc, npieces, nwords, nseg, grid};
    MAPI_CUDA(cudaMemcpyAsync(plan, &hdr, sizeof(hdr), cudaMemcpyHostToDevice, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    info->n = n;
    info->nnz = nnz;
    info->nsrc = nsrc;
    info->npieces = npieces;
    info->nwords = nwords;
    info->nseg = nseg;
    info->grid = grid;
    return MAPI_OK;
}

mapi_status mapi_rank_csr_plan(int32_t op, const void* plan, const mapi_csr_plan_info* info, const float* cap,
                               const float* bg, const float* b0, int32_t max_iters, float tol, float* w_out,
                               float* w_l2_out, float* deltas, int32_t* iters_done, void* ws, size_t ws_bytes,
                               mapi_stream_t stream) {
    if (op != MAPI_OP_MIN1 && op != MAPI_OP_MIN2 && op != MAPI_OP_DOT)
        return fail(MAPI_ERR_BAD_PARAM, "op (%d) must be MAPI_OP_MIN1, MAPI_OP_MIN2 or MAPI_OP_DOT", op);
    if (!plan || !info || !cap || !bg || !b0 || !w_out) return fail(MAPI_ERR_NULL, "a required pointer is NULL");
    const int64_t n = info->n;
    if (n < 1 || info->nnz < 0 || info->grid < 1 || info->grid > kMaxGrid || info->nseg < 1 ||
        info->npieces < 0 || info->npieces > std::max<int64_t>(info->nnz, 0) || info->nwords < 0)
        return fail(MAPI_ERR_SHAPE, "plan info is inconsistent (n %lld, nnz %lld, grid %d, nseg %d)", (long long)n,
                    (long long)info->nnz, info->grid, info->nseg);
    if (max_iters < 1) return fail(MAPI_ERR_BAD_PARAM, "max_iters (%d) must be >= 1", max_iters);
    if (!(tol >= 0.0f)) return fail(MAPI_ERR_BAD_PARAM, "tol must be >= 0");
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    const size_t need = run_ws_exact(n, info->nseg, info->npieces);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    mapi_status st = device_info(d);
    if (st != MAPI_OK) return st;
    if (info->grid > d.sms)
        return fail(MAPI_ERR_SHAPE, "plan built for %d CTAs; this device has %d SMs", info->grid, d.sms);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const PlanView P = plan_view(const_cast<void*>(plan), n, info->nseg, info->grid, info->npieces);
    RunArgs a;
    a.n = n;
    a.nseg = info->nseg;
    a.iters = max_iters;
    a.tol = tol;
    a.q = P.q; a.segb = P.segb; a.ctab = P.ctab; a.ctap = P.ctap; a.rsp = P.rsp; a.pos = P.pos; a.words = P.words;
    a.cap = cap; a.bg = bg; a.b0 = b0; a.deltas = deltas;
    a.w = carve_run(ws, n, info->nseg, info->npieces);
    MAPI_CUDA(cudaMemsetAsync(ws, 0, 256, s));
    // the compact vector's zero slots (offset 32767 of each segment) and unused tail stay 0
    MAPI_CUDA(cudaMemsetAsync(a.w.vc, 0, 4 * (size_t)kSegStride * (size_t)info->nseg, s));
    auto kern = op == MAPI_OP_DOT ? k_rank_plan<2> : k_rank_plan<0>;
    MAPI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kSegStride));
    Timer timer(s);
    void* args[] = {&a};
    timer.start();
    MAPI_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(info->grid), dim3(kThreads), args,
                                          (size_t)4 * kSegStride, s));
    timer.stop();
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const int gout = (int)std::min<int64_t>((n + 255) / 256, std::min(4 * d.sms, kMaxGrid));
    k_plan_output<<<gout, 256, 0, s>>>(n, a.w, b0, w_out);
    MAPI_LAUNCHED();
    if (w_l2_out) {
        k_plan_output_l2<<<gout, 256, 0, s>>>(n, a.w, b0, gout, w_l2_out);
        MAPI_LAUNCHED();
    }
    int32_t h[2] = {0, 0};
    MAPI_CUDA(cudaMemcpyAsync(h, a.w.status, sizeof(h), cudaMemcpyDeviceToHost, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    timer.harvest();
    if (iters_done) *iters_done = h[1];
    if (h[0] == MAPI_ERR_NEGATIVE) return fail(MAPI_ERR_NEGATIVE, "b0 has a negative entry");
    if (h[0] == MAPI_ERR_DEGENERATE) return fail(MAPI_ERR_DEGENERATE, "||G (+) w_t||_1 == 0 at iteration %d", h[1]);
    if (h[0] == MAPI_ERR_NONFINITE)
        return fail(MAPI_ERR_NONFINITE, "||G (+) w_t||_1 is not finite at iteration %d", h[1]);
    return MAPI_OK;
}

}  // extern "C"
