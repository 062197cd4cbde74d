// csr_plan.cu — K3s: the segmented MAPI ranking step (Eq. 13) for sm_100a.
//
// The ranking step is (K3; reading Q10)
//     y_i = S + e_i,   e_i = sum_{j -> i} v_j,   S = sum_j min(bg_j, w_j),   v_j = min(max(w_j - bg_j, 0), cap_j)
// i.e. a gather-sum of v over each row's sources.  On the CSR layout (K3, csr.cuh) every one of the E'
// gathers is a scattered 4-byte L2 read that costs one L1TEX wavefront: ~245 us per iteration at cfg5
// against ~60 us of HBM traffic.  K3s changes the LAYOUT, not the arithmetic:
//   * "plan order": sources (out-degree >= 1) by DESCENDING out-degree, then dangling nodes that have
//     in-edges, then ISOLATED nodes (no in- and no out-edges); ties by id.  Every per-node array of the run
//     (bg, cap, e, the v vector) is kept in plan order, so the node pass streams it contiguously;
//   * source p lives in segment p / 32767 at local offset p % 32767 of the compact v vector (offset 32767 of
//     every segment is a zero slot);
//   * the edges are stored segment-major, then by the PLAN position of their destination row, then in CSR
//     order, as 16-bit words `local offset | end-of-fragment << 15`.  Segment starts are aligned to the
//     512-word warp tile; a "fragment" is a maximal run of one row inside one segment and one tile;
//   * phase A: each CTA copies the v values of one segment (128 KB) into SHARED memory and its warps stream
//     512-word tiles: every gather is a shared-memory load; a warp-level segmented scan (no block
//     synchronisation) closes the fragments, which are written in fragment order (coalesced) at the tile's
//     precomputed fragment base;
//   * phase B: the live nodes are cut into batches (<= 4096 rows, <= 48K slots); a batch's fragment sums are
//     gathered in (segment, fragment) order — contiguous runs of `part`, coalesced — through the static list
//     bfrag into shared memory at their slot (row-sorted) positions brel, and every row sums its slots in
//     (segment, position) order in fp64;
//   * isolated nodes all have y_i = S and the same bg (checked at run time), so from iteration 1 on they are
//     one class: count x (their delta and S terms) instead of ~43% of cfg5's node traffic.
// Everything runs in ONE persistent cooperative launch: init, then per iteration phase A -> grid barrier ->
// phase B -> grid barrier -> identical stop decision in every CTA.  A tol stop ends the launch on the device.
// Deterministic: every sum has a fixed order for a given plan.
//
// Numerics: fp32 sums inside a fragment (<= 512 terms, ~6.5 on average at cfg5), the fragments of a row
// summed in fp64; the per-node state is fp64 (R9): e_i is stored in fp64, so w_t = (S_{t-1} + e_{t-1}) /
// s_{t-1} is recomputed bit-exactly from it; the l1 norm s = n S + sum e with sum e taken in fp64 over the
// fragment sums.  Operator DOT (RPI, reading R13): v_j = cap_j w_j, S = sum bg_j w_j.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
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
constexpr int kLaneW = 16;                   // words per lane per tile (two 16 B loads)
constexpr int kTileW = 32 * kLaneW;          // 512 words per warp tile; segment starts are tile-aligned
constexpr int kThreads = 1024;               // planned kernel: one CTA of 32 warps per SM
constexpr int kWarps = kThreads / 32;
constexpr int kMaxGrid = 1024;
constexpr int kStageF = kWarps * kTileW;     // phase A per-warp fragment stages (floats after the segment)
constexpr int kSmemF = kSegStride + kStageF; // dynamic shared floats; phase B stages a batch's slots in all of it
constexpr size_t kPlanSmem = sizeof(float) * (size_t)kSmemF;
constexpr int kNodeK = 4;                    // rows per thread per batch
constexpr int kBatchRows = kNodeK * kThreads;
constexpr int kSlotBlock = 16384;            // a batch never spans two slot blocks (plus its last row): the bound's block
constexpr int kSlotBlockRun = 32768;         // the block the plan is cut with (>= kSlotBlock): 893 instead of 1,201
                                             // batches at cfg5, phase B 75 -> 67 us (profiles/r02_probe_k3s_slotblock.log)
constexpr int kUnitBig = 256;                // phase A work units (tiles), taken dynamically: big ones first,
constexpr int kUnitSmall = kWarps;           // then one tile per warp for the last 1/8 of the tiles
constexpr uint64_t kMagic = 0x4d41504950334c4eull;

inline size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
inline int64_t max_segments(int64_t n) { return std::max<int64_t>(1, (n + kSegSrc - 1) / kSegSrc); }
inline int64_t nwords_bound(int64_t nnz, int64_t nseg) {
    return (nnz + kTileW - 1) / kTileW * kTileW + (int64_t)kTileW * nseg;
}
inline int64_t nbatch_bound(int64_t n, int64_t nnz) { return n / kBatchRows + nnz / kSlotBlock + 2; }
inline int64_t nunits_bound(int64_t ntiles, int64_t nseg) { return ntiles / kUnitSmall + nseg + 2; }

// ------------------------------------------------------------------------------- plan layout
// [hdr 256][perm n i32: plan position -> node id][segb nseg+1 i32: padded word start of each segment]
// [units 3 nunits i32: phase A work units (first tile, end tile, segment) in scheduling order]
// [fbase ntiles+1 i32: first fragment of each tile][rsp n+1 i32: plan position -> its first slot]
// [words nwords u16: source offsets][wflags nwords/16 u32: per lane chunk of 16 words, the end-of-fragment flags
//  (low 16 bits) and the number of fragments that end in the tile's preceding chunks (high 16 bits)]
// [bfrag nfrag i32: fragments in (batch, fragment) order][brel nfrag u16: their slot within the batch]
// [bstart nbatch+1 i32: batch rows]
struct PlanView {
    int32_t *perm, *segb, *units, *fbase, *rsp;
    uint16_t* words;
    uint32_t* wflags;
    int32_t* bfrag;
    uint16_t* brel;
    int32_t* bstart;
};
inline PlanView plan_view(void* plan, int64_t n, int64_t nseg, int64_t nunits, int64_t nwords, int64_t nfrag) {
    const int64_t ntiles = nwords / kTileW;
    char* p = static_cast<char*>(plan) + 256;
    PlanView v;
    v.perm = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)n);
    v.segb = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)(nseg + 1));
    v.units = reinterpret_cast<int32_t*>(p); p += al256(12 * (size_t)std::max<int64_t>(nunits, 1));
    v.fbase = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)(ntiles + 1));
    v.rsp = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)(n + 1));
    v.words = reinterpret_cast<uint16_t*>(p); p += al256(2 * (size_t)std::max<int64_t>(nwords, 1));
    v.wflags = reinterpret_cast<uint32_t*>(p); p += al256(4 * (size_t)std::max<int64_t>(nwords / kLaneW, 1));
    v.bfrag = reinterpret_cast<int32_t*>(p); p += al256(4 * (size_t)std::max<int64_t>(nfrag, 1));
    v.brel = reinterpret_cast<uint16_t*>(p); p += al256(2 * (size_t)std::max<int64_t>(nfrag, 1));
    v.bstart = reinterpret_cast<int32_t*>(p);
    return v;
}
inline size_t plan_bytes_exact(int64_t n, int64_t nseg, int64_t nunits, int64_t nwords, int64_t nfrag, int64_t nbatch) {
    const int64_t ntiles = nwords / kTileW;
    return 256 + al256(4 * (size_t)n) + al256(4 * (size_t)(nseg + 1)) + al256(12 * (size_t)std::max<int64_t>(nunits, 1)) +
           al256(4 * (size_t)(ntiles + 1)) + al256(4 * (size_t)(n + 1)) + al256(2 * (size_t)std::max<int64_t>(nwords, 1)) +
           al256(4 * (size_t)std::max<int64_t>(nwords / kLaneW, 1)) +
           al256(4 * (size_t)std::max<int64_t>(nfrag, 1)) + al256(2 * (size_t)std::max<int64_t>(nfrag, 1)) +
           al256(4 * (size_t)(nbatch + 1));
}

size_t plan_bytes_bound(int64_t n, int64_t nnz) {
    if (n < 1 || nnz < 0) return 0;
    const int64_t nseg = max_segments(n);
    // nfrag <= nnz (every fragment holds >= 1 edge)
    const int64_t nw = nwords_bound(nnz, nseg);
    return plan_bytes_exact(n, nseg, nunits_bound(nw / kTileW, nseg), nw, nnz, nbatch_bound(n, nnz));
}

// ------------------------------------------------------------------------------- build workspace
struct BuildWs {
    uint32_t* counter;  // [0] nsrc, [1] isolated nodes, [2] max slots of a batch
    uint32_t *outdeg, *skey, *skey2;
    int32_t *sval, *inv, *rcnt, *segb, *bflag, *bincl;
    int32_t *segcnt, *segstart, *tcnt;
    uint64_t *ekey, *ekey2;
    uint32_t *eoff, *eoff2, *fstart, *fid;
    int32_t *frow, *frow2, *fidx, *pos, *fslot, *fbat, *fbat2;
    void* cub;
    size_t cub_bytes;
};

inline size_t cub_bytes_needed(int64_t n, int64_t nnz, int64_t ntiles) {
    const int nn = (int)std::max<int64_t>(n + 1, 1), ne = (int)std::max<int64_t>(nnz, 1);
    size_t a = 0, b = 0, c = 0, d = 0, f = 0, g = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, nn, 0, 32);
    cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, ne, 0, 64);
    cub::DeviceRadixSort::SortPairs(nullptr, c, (const int32_t*)nullptr, (int32_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, ne, 0, 32);
    cub::DeviceScan::ExclusiveSum(nullptr, d, (const uint32_t*)nullptr, (uint32_t*)nullptr, ne);
    cub::DeviceScan::ExclusiveSum(nullptr, f, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)std::max<int64_t>(std::max<int64_t>(n, ntiles) + 1, 1));
    cub::DeviceScan::InclusiveSum(nullptr, g, (const int32_t*)nullptr, (int32_t*)nullptr, nn);
    return std::max({a, b, c, d, f, g}) + 1024;
}

size_t plan_build_ws_bytes(int64_t n, int64_t nnz) {
    if (n < 1 || nnz < 0) return 0;
    const int64_t nseg = max_segments(n), ntiles = nwords_bound(nnz, nseg) / kTileW;
    const size_t N = al256(4 * (size_t)(n + 1)), E = al256(4 * (size_t)std::max<int64_t>(nnz, 1));
    return 256 + 10 * N + 2 * al256(4 * (size_t)(nseg + 1)) + al256(4 * (size_t)(ntiles + 1)) + 4 * E /*ekey x2*/ +
           11 * E + al256(cub_bytes_needed(n, nnz, ntiles));
}

inline BuildWs carve_build(void* ws, int64_t n, int64_t nnz) {
    const int64_t nseg = max_segments(n), ntiles = nwords_bound(nnz, nseg) / kTileW;
    char* p = static_cast<char*>(ws);
    BuildWs b;
    b.counter = reinterpret_cast<uint32_t*>(p);
    p += 256;
    const size_t N = al256(4 * (size_t)(n + 1)), E = al256(4 * (size_t)std::max<int64_t>(nnz, 1));
    auto take = [&](size_t bytes) { char* r = p; p += bytes; return r; };
    b.outdeg = reinterpret_cast<uint32_t*>(take(N));
    b.skey = reinterpret_cast<uint32_t*>(take(N));
    b.skey2 = reinterpret_cast<uint32_t*>(take(N));
    b.sval = reinterpret_cast<int32_t*>(take(N));
    b.inv = reinterpret_cast<int32_t*>(take(N));
    b.rcnt = reinterpret_cast<int32_t*>(take(N));
    b.segb = reinterpret_cast<int32_t*>(take(N));  // nseg + 1 <= n + 1
    b.bflag = reinterpret_cast<int32_t*>(take(N));
    b.bincl = reinterpret_cast<int32_t*>(take(N));
    take(N);  // spare
    b.segcnt = reinterpret_cast<int32_t*>(take(al256(4 * (size_t)(nseg + 1))));
    b.segstart = reinterpret_cast<int32_t*>(take(al256(4 * (size_t)(nseg + 1))));
    b.tcnt = reinterpret_cast<int32_t*>(take(al256(4 * (size_t)(ntiles + 1))));
    b.ekey = reinterpret_cast<uint64_t*>(take(2 * E));
    b.ekey2 = reinterpret_cast<uint64_t*>(take(2 * E));
    b.eoff = reinterpret_cast<uint32_t*>(take(E));
    b.eoff2 = reinterpret_cast<uint32_t*>(take(E));
    b.fstart = reinterpret_cast<uint32_t*>(take(E));
    b.fid = reinterpret_cast<uint32_t*>(take(E));
    b.frow = reinterpret_cast<int32_t*>(take(E));
    b.frow2 = reinterpret_cast<int32_t*>(take(E));
    b.fidx = reinterpret_cast<int32_t*>(take(E));
    b.pos = reinterpret_cast<int32_t*>(take(E));
    b.fslot = reinterpret_cast<int32_t*>(take(E));
    b.fbat = reinterpret_cast<int32_t*>(take(E));
    b.fbat2 = reinterpret_cast<int32_t*>(take(E));
    b.cub = p;
    b.cub_bytes = cub_bytes_needed(n, nnz, ntiles);
    return b;
}

// ------------------------------------------------------------------------------- build kernels
#define GRID_STRIDE(i, count) \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (count); i += (int64_t)gridDim.x * blockDim.x)

__global__ void kp_outdeg(int64_t nnz, const int32_t* __restrict__ col_idx, uint32_t* __restrict__ outdeg) {
    GRID_STRIDE(e, nnz) atomicAdd(outdeg + col_idx[e], 1u);  // integer histogram: order-independent
}

// plan-order key: sources by descending out-degree, then dangling nodes with in-edges, then isolated nodes;
// value = id (the stable sort keeps ties by ascending id)
__global__ void kp_src_keys(int64_t n, const uint32_t* __restrict__ outdeg, const int32_t* __restrict__ row_ptr,
                            uint32_t* __restrict__ key, int32_t* __restrict__ val, uint32_t* counter) {
    uint32_t ns = 0, ni = 0;
    GRID_STRIDE(j, n) {
        const uint32_t d = outdeg[j];
        const bool has_in = row_ptr[j + 1] > row_ptr[j];
        key[j] = d > 0 ? 0xfffffffdu - d : (has_in ? 0xfffffffeu : 0xffffffffu);
        val[j] = (int32_t)j;
        ns += d > 0;
        ni += (d == 0 && !has_in);
    }
    ns = __reduce_add_sync(0xffffffffu, ns);
    ni = __reduce_add_sync(0xffffffffu, ni);
    if ((threadIdx.x & 31) == 0) {
        if (ns) atomicAdd(counter + 0, ns);
        if (ni) atomicAdd(counter + 1, ni);
    }
}

__global__ void kp_inv(int64_t n, const int32_t* __restrict__ perm, int32_t* __restrict__ inv) {
    GRID_STRIDE(p, n) inv[perm[p]] = (int32_t)p;
}

// per edge: key = (segment of its source, plan position of its row), value = the source's local offset
__global__ void kp_edges(int64_t n, int64_t nnz, const int32_t* __restrict__ row_ptr,
                         const int32_t* __restrict__ col_idx, const int32_t* __restrict__ inv,
                         uint64_t* __restrict__ ekey, uint32_t* __restrict__ eoff) {
    GRID_STRIDE(e, nnz) {
        int64_t lo = 0, hi = n - 1;  // the row i with row_ptr[i] <= e < row_ptr[i+1]
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if ((int64_t)row_ptr[mid] <= e) lo = mid;
            else hi = mid - 1;
        }
        const int32_t ps = inv[col_idx[e]];
        const uint32_t seg = (uint32_t)(ps / kSegSrc), off = (uint32_t)(ps - (int32_t)seg * kSegSrc);
        ekey[e] = ((uint64_t)seg << 32) | (uint32_t)inv[lo];
        eoff[e] = off;
    }
}

// segment of each sorted edge: counts and first positions
// The edges are sorted by segment: only the run boundaries write (segstart = first edge of the segment's run,
// segcnt = one past its last edge until kp_segb turns it into the count; both zeroed before, so a segment
// without edges keeps 0 / 0).  (A per-edge atomicAdd on the ~60 counters took 41 of the plan build's 50 ms.)
__global__ void kp_segcount(int64_t nnz, const uint64_t* __restrict__ ek, int32_t* __restrict__ segcnt,
                            int32_t* __restrict__ segstart) {
    GRID_STRIDE(k, nnz) {
        const uint32_t seg = (uint32_t)(ek[k] >> 32);
        if (k == 0) {
            segstart[seg] = 0;
        } else {
            const uint32_t prev = (uint32_t)(ek[k - 1] >> 32);
            if (prev != seg) {
                segstart[seg] = (int32_t)k;
                segcnt[prev] = (int32_t)k;
            }
        }
        if (k == nnz - 1) segcnt[seg] = (int32_t)nnz;
    }
}

// run ends -> counts, and the padded segment starts, tile-aligned (one thread: nseg is small)
__global__ void kp_segb(int32_t nseg, int32_t* __restrict__ segcnt, const int32_t* __restrict__ segstart,
                        int32_t* __restrict__ segb) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    int64_t acc = 0;
    for (int32_t s = 0; s < nseg; ++s) {
        const int32_t cnt = segcnt[s] > 0 ? segcnt[s] - segstart[s] : 0;
        segcnt[s] = cnt;
        segb[s] = (int32_t)acc;
        acc += ((int64_t)cnt + kTileW - 1) / kTileW * kTileW;
    }
    segb[nseg] = (int32_t)acc;
}

__device__ __forceinline__ int64_t padded_pos(int64_t k, uint32_t seg, const int32_t* segstart, const int32_t* segb) {
    return k - segstart[seg] + segb[seg];
}

// a fragment starts where the (segment, row) run starts or a tile starts
__global__ void kp_fstart(int64_t nnz, const uint64_t* __restrict__ ek, const int32_t* __restrict__ segstart,
                          const int32_t* __restrict__ segb, uint32_t* __restrict__ fstart) {
    GRID_STRIDE(k, nnz) {
        const uint64_t key = ek[k];
        const int64_t pw = padded_pos(k, (uint32_t)(key >> 32), segstart, segb);
        fstart[k] = (k == 0 || ek[k - 1] != key || pw % kTileW == 0) ? 1u : 0u;
    }
}

// fragment rows / ids, per-row and per-tile fragment counts, and the words
__global__ void kp_frag(int64_t nnz, const uint64_t* __restrict__ ek, const uint32_t* __restrict__ eoff,
                        const uint32_t* __restrict__ fstart, const uint32_t* __restrict__ fid,
                        const int32_t* __restrict__ segstart, const int32_t* __restrict__ segb,
                        int32_t* __restrict__ frow, int32_t* __restrict__ fidx, int32_t* __restrict__ rcnt,
                        int32_t* __restrict__ tcnt, uint16_t* __restrict__ words) {
    GRID_STRIDE(k, nnz) {
        const uint64_t key = ek[k];
        const int64_t pw = padded_pos(k, (uint32_t)(key >> 32), segstart, segb);
        const bool end = (k + 1 == nnz) || fstart[k + 1];
        words[pw] = (uint16_t)(eoff[k] | (end ? 0x8000u : 0u));
        if (fstart[k]) {
            const uint32_t f = fid[k];
            const int32_t row = (int32_t)(uint32_t)key;
            frow[f] = row;
            fidx[f] = (int32_t)f;
            atomicAdd(rcnt + row, 1);
            atomicAdd(tcnt + pw / kTileW, 1);
        }
    }
}

__global__ void kp_fill_words(int64_t nwords, uint16_t* __restrict__ words) {
    GRID_STRIDE(k, nwords) words[k] = kDummy;
}
// per lane chunk of 16 words: the end flags as a 16-bit mask and, in the high half, the number of fragments
// ending in the tile's preceding chunks (the lane's first position in the warp's fragment stage: static, so
// the run kernel needs no warp scan of the counts); the words keep only the source offset.  A warp of this
// kernel covers exactly one tile (32 consecutive chunks: the block size and nchunks are multiples of 32).
__global__ void kp_wflags(int64_t nchunks, uint16_t* __restrict__ words, uint32_t* __restrict__ wflags) {
    GRID_STRIDE(ch, nchunks) {
        uint32_t m = 0;
        for (int i = 0; i < kLaneW; ++i) {
            const uint16_t w = words[ch * kLaneW + i];
            m |= (uint32_t)(w >> 15) << i;
            words[ch * kLaneW + i] = (uint16_t)(w & 0x7fffu);
        }
        const int lane = threadIdx.x & 31;
        int c = __popc(m);
        const int cnt = c;
        for (int off = 1; off < 32; off <<= 1) {
            const int co = __shfl_up_sync(0xffffffffu, c, off);
            if (lane >= off) c += co;
        }
        wflags[ch] = m | ((uint32_t)(c - cnt) << 16);
    }
}

// Bank-conflict-aware word order (plan time; after kp_wflags: the words are 15-bit source offsets, the end flags
// sit in wflags).  Phase A's gather step i reads, warp-wide, word 16 l + i of every lane l from the shared
// segment: a random 32-address gather costs ~3.9 extra shared-memory wavefronts (ncu: 44% of K3s's shared
// wavefronts were conflict replays, profiles/r02_cfg5_k3s_raw.csv).  The words of one lane that belong to the
// same fragment may be summed in any fixed order, so within each (lane chunk, fragment) group the offsets are
// re-assigned to the group's steps greedily, lanes in order, each word to the free step where its bank is
// used by the fewest other lanes; kDeconflictRounds passes, a lane's own words taken out of the counts before
// it is re-assigned.  One warp per tile; only the order of the fp32 additions inside a fragment changes (fixed
// by the plan: deterministic).
constexpr int kDeconflictRounds = 2;  // sweep: profiles/r02_probe_k3s_deconflict.log (1: 6,279, 2: 6,300, 3: 6,309, 8: 6,315 it/s)
__global__ void __launch_bounds__(256) kp_deconflict(int64_t ntiles, uint16_t* __restrict__ words,
                                                     const uint32_t* __restrict__ wflags, int rounds) {
    __shared__ uint8_t cnt[8][kLaneW][32];  // per warp: lanes using (step, bank)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t tile = (int64_t)blockIdx.x * 8 + warp; tile < ntiles; tile += (int64_t)gridDim.x * 8) {
        for (int i = lane; i < kLaneW * 32; i += 32) (&cnt[warp][0][0])[i] = 0;
        __syncwarp();
        uint16_t* w = words + tile * kTileW + kLaneW * lane;
        const uint32_t fl = wflags[tile * 32 + lane] & 0xffffu;
        uint16_t x[kLaneW], out[kLaneW];
#pragma unroll
        for (int i = 0; i < kLaneW; ++i) out[i] = w[i];
        for (int round = 0; round < rounds; ++round) {
            for (int l = 0; l < 32; ++l) {
                if (lane == l) {
                    for (int i = 0; i < kLaneW; ++i) {
                        x[i] = out[i];
                        if (round > 0) --cnt[warp][i][x[i] & 31];
                    }
                    int g0 = 0;
                    while (g0 < kLaneW) {
                        int g1 = g0;  // the group ends at the first end flag at or after g0 (or with the chunk)
                        while (g1 < kLaneW - 1 && !((fl >> g1) & 1u)) ++g1;
                        uint32_t free_steps = ((2u << g1) - 1u) & ~((1u << g0) - 1u);
                        for (int k = g0; k <= g1; ++k) {
                            const uint16_t a = x[k];
                            const int bank = a & 31;
                            int best = g0, bestc = 1 << 30;
                            for (int st = g0; st <= g1; ++st) {
                                if (!((free_steps >> st) & 1u)) continue;
                                const int c = cnt[warp][st][bank];
                                if (c < bestc) {
                                    bestc = c;
                                    best = st;
                                }
                            }
                            out[best] = a;
                            free_steps &= ~(1u << best);
                            ++cnt[warp][best][bank];
                        }
                        g0 = g1 + 1;
                    }
                }
                __syncwarp();
            }
        }
#pragma unroll
        for (int i = 0; i < kLaneW; ++i) w[i] = out[i];
        __syncwarp();
    }
}

__global__ void kp_fslot(int64_t nfrag, const int32_t* __restrict__ pos, int32_t* __restrict__ fslot) {
    GRID_STRIDE(r, nfrag) fslot[pos[r]] = (int32_t)r;
}

// batch starts over the live rows: every kBatchRows rows and wherever the slot position enters a new slot
// block, so a batch holds <= kBatchRows rows and < kSlotBlock + (its last row's slots) slots
__global__ void kp_bflag(int64_t nlive, const int32_t* __restrict__ rsp, int32_t* __restrict__ flag, int32_t slot_block) {
    GRID_STRIDE(r, nlive) flag[r] = (r == 0 || r % kBatchRows == 0 || rsp[r] / slot_block != rsp[r - 1] / slot_block);
}
__global__ void kp_bstart(int64_t nlive, const int32_t* __restrict__ flag, const int32_t* __restrict__ incl,
                          int32_t* __restrict__ bstart) {
    GRID_STRIDE(r, nlive) if (flag[r]) bstart[incl[r] - 1] = (int32_t)r;
    if (blockIdx.x == 0 && threadIdx.x == 0) bstart[incl[nlive - 1]] = (int32_t)nlive;
}
__global__ void kp_fbat(int64_t nfrag, const int32_t* __restrict__ frow, const int32_t* __restrict__ incl,
                        int32_t* __restrict__ fbat, int32_t* __restrict__ fidx) {
    GRID_STRIDE(f, nfrag) {
        fbat[f] = incl[frow[f]] - 1;
        fidx[f] = (int32_t)f;
    }
}
// slot of each listed fragment relative to its batch's first slot; the largest batch (shared capacity)
__global__ void kp_brel(int64_t nfrag, const int32_t* __restrict__ bfrag, const int32_t* __restrict__ fbat,
                        const int32_t* __restrict__ fslot, const int32_t* __restrict__ bstart,
                        const int32_t* __restrict__ rsp, uint16_t* __restrict__ brel, uint32_t* maxslots) {
    GRID_STRIDE(k, nfrag) {
        const int32_t f = bfrag[k], b = fbat[f];
        const int32_t R0 = rsp[bstart[b]], R1 = rsp[bstart[b + 1]];
        const int32_t rel = fslot[f] - R0;
        brel[k] = (uint16_t)min(rel, 65535);
        if (k == (int64_t)R0) atomicMax(maxslots, (uint32_t)(R1 - R0));
    }
}

}  // namespace mapi_plan

// ================================================================================ run
namespace mapi_plan {

// workspace: [hdr 256: status[2] @0, stop @8, bar u32 @12, non-uniform isolated bg @16, unit counters u32 x 4
//            @20, hist (S, s) x 2 f64 @48]
//            [e0 n f64][e1 n f64][bgp n f32][capp n f32][vc nseg*32768 f32][part nfrag f32]
//            [slotY nunits f64: phase A unit sums][slotD nbatch f64][slotS 2 x nbatch f64: batch partials]
//            [slotDi G f64][slotSi 2 x G f64: isolated-node partials per CTA][slotQ G f64]
struct RunWs {
    int32_t* status;
    int32_t* stop;
    unsigned* bar;
    int32_t* iso_mixed;
    unsigned* ctr;  // [0..1] phase A unit counters, [2..3] phase B batch counters (by iteration parity)
    double* hist;
    double *e0, *e1;
    float *bgp, *capp, *vc, *part;
    double *slotY, *slotD, *slotS, *slotDi, *slotSi, *slotQ;
    int64_t nbatch;
};
inline size_t run_ws_exact(int64_t n, int64_t nseg, int64_t nfrag, int64_t nunits, int64_t nbatch) {
    return 256 + 2 * al256(8 * (size_t)n) + 2 * al256(4 * (size_t)n) +
           al256(4 * (size_t)kSegStride * (size_t)std::max<int64_t>(nseg, 1)) +
           al256(4 * (size_t)std::max<int64_t>(nfrag, 1)) + al256(8 * (size_t)std::max<int64_t>(nunits, 1)) +
           3 * al256(8 * (size_t)std::max<int64_t>(nbatch, 1)) + 4 * al256(8 * (size_t)kMaxGrid);
}
size_t rank_plan_ws_bytes(int64_t n, int64_t nnz) {
    if (n < 1 || nnz < 0) return 0;
    const int64_t nseg = max_segments(n), nw = nwords_bound(nnz, nseg);
    return run_ws_exact(n, nseg, std::max<int64_t>(nnz, 1), nunits_bound(nw / kTileW, nseg), nbatch_bound(n, nnz));
}
inline RunWs carve_run(void* ws, int64_t n, int64_t nseg, int64_t nfrag, int64_t nunits, int64_t nbatch) {
    char* p = static_cast<char*>(ws);
    RunWs r;
    r.status = reinterpret_cast<int32_t*>(p);
    r.stop = reinterpret_cast<int32_t*>(p + 8);
    r.bar = reinterpret_cast<unsigned*>(p + 12);
    r.iso_mixed = reinterpret_cast<int32_t*>(p + 16);
    r.ctr = reinterpret_cast<unsigned*>(p + 20);
    r.hist = reinterpret_cast<double*>(p + 48);
    p += 256;
    r.e0 = reinterpret_cast<double*>(p); p += al256(8 * (size_t)n);
    r.e1 = reinterpret_cast<double*>(p); p += al256(8 * (size_t)n);
    r.bgp = reinterpret_cast<float*>(p); p += al256(4 * (size_t)n);
    r.capp = reinterpret_cast<float*>(p); p += al256(4 * (size_t)n);
    r.vc = reinterpret_cast<float*>(p); p += al256(4 * (size_t)kSegStride * (size_t)std::max<int64_t>(nseg, 1));
    r.part = reinterpret_cast<float*>(p); p += al256(4 * (size_t)std::max<int64_t>(nfrag, 1));
    r.slotY = reinterpret_cast<double*>(p); p += al256(8 * (size_t)std::max<int64_t>(nunits, 1));
    const size_t B = al256(8 * (size_t)std::max<int64_t>(nbatch, 1));
    r.slotD = reinterpret_cast<double*>(p); p += B;
    r.slotS = reinterpret_cast<double*>(p); p += 2 * B;  // parity q at slotS + q * (B / 8)
    r.slotDi = reinterpret_cast<double*>(p); p += al256(8 * (size_t)kMaxGrid);
    r.slotSi = reinterpret_cast<double*>(p); p += 2 * al256(8 * (size_t)kMaxGrid);
    r.slotQ = reinterpret_cast<double*>(p);
    r.nbatch = (int64_t)(B / 8);  // parity stride of slotS
    return r;
}

struct RunArgs {
    int64_t n, nlive, nsrc;
    int32_t nseg, iters, nunits, nbatch;
    float tol;
    const int32_t *perm, *segb, *units, *fbase, *rsp, *bstart, *bfrag;
    const uint16_t *brel, *words;
    const uint32_t* wflags;
    const float *cap, *bg, *b0;
    float* deltas;
    unsigned long long* trace;  // optional: phase stamps (globaltimer), see PLAN_STAMP
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
    // rounding to fp32 is monotone and 0 / cap are fp32 values, so clamping after the rounding gives exactly
    // fp32(min(max(w - bg, 0), cap)) with one conversion less (F2F.F64.F32 + DADD issue at 16 lanes/clk/SM,
    // profiles/r02_probe_fp64.log)
    else return fminf(fmaxf((float)(w - (double)bg), 0.0f), cap);
}
template <int OP>
__device__ __forceinline__ double node_s(double w, float bg) {
    if constexpr (OP == 2) return (double)bg * w;
    else return fmin((double)bg, w);
}
// compact v index of plan position p < nsrc
__device__ __forceinline__ int64_t vc_index(int64_t p) {
    const int64_t seg = p / kSegSrc;
    return seg * kSegStride + (p - seg * kSegSrc);
}

// two block sums at once (one set of barriers), results broadcast
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    a = mapi::warp_sum(a);
    b = mapi::warp_sum(b);
    __syncthreads();
    if (lane == 0) {
        red[warp] = a;
        red[40 + warp] = b;
    }
    __syncthreads();
    if (warp == 0) {
        double x = red[lane], y = red[40 + lane];
        x = mapi::warp_sum(x);
        y = mapi::warp_sum(y);
        if (lane == 0) {
            red[32] = x;
            red[72] = y;
        }
    }
    __syncthreads();
    a = red[32];
    b = red[72];
}

// one 512-word tile: 16 words per lane (lane l: words 16 l .. 16 l + 15, end flags fl), gathers from the shared
// segment (shared address sb).  The lane's fragments are closed in word order into the warp's stage at their
// fragment positions (static: the plan stores each lane's first position beside its flags), the run carried in
// from the preceding lanes (a segmented warp scan of the lanes' open tails) is added to the lane's first fragment, and
// the warp writes the stage to part[fb ..) with coalesced stores.  Returns the fp64 sum of the fragment sums
// (lane partials of the fragment sums it stores, in fp32, one conversion per lane).
__device__ __forceinline__ double plan_tile(const uint4 (&wd)[2], uint32_t fl, uint32_t sb, int32_t fb,
                                            float* __restrict__ stage, float* __restrict__ part, int lane) {
    const uint32_t u[8] = {wd[0].x, wd[0].y, wd[0].z, wd[0].w, wd[1].x, wd[1].y, wd[1].z, wd[1].w};
    float x[kLaneW];
#pragma unroll
    for (int h = 0; h < 8; ++h) {
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[2 * h]) : "r"(sb + ((u[h] & 0xffffu) << 2)));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x[2 * h + 1]) : "r"(sb + ((u[h] >> 16) << 2)));
    }
    // fl: the lane's end-of-fragment flags (low half) and its first stage position (high half, from the plan)
    const int cnt = __popc(fl & 0xffffu);
    const int before = (int)(fl >> 16);
    const int total = __shfl_sync(0xffffffffu, before + cnt, 31);
    // close the lane's fragments (the first one without the carried run); acc ends as the open tail
    float acc = 0.0f;
    float* st = stage + before;
#pragma unroll
    for (int i = 0; i < kLaneW; ++i) {
        acc += x[i];
        if ((fl >> i) & 1u) {
            *st++ = acc;
            acc = 0.0f;
        }
    }
    // inclusive segmented scan over lanes of (has flag, open tail): the run carried into the next lane.  A
    // lane is final once a flag has been seen within its reach (f) or its reach covers lane 0; with ~2.5
    // fragment ends per lane that is the case for every lane after one or two of the five steps, and the
    // remaining steps would change nothing: leave early (same values, bit for bit)
    int f = cnt > 0;
    float v = acc;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int fo = __shfl_up_sync(0xffffffffu, f, off);
        const float vo = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) {
            if (!f) v = vo + v;
            f |= fo;
        }
        if (__all_sync(0xffffffffu, f || lane < 2 * off)) break;
    }
    const float carry = __shfl_up_sync(0xffffffffu, v, 1);
    if (lane > 0 && cnt > 0) stage[before] += carry;
    __syncwarp();
    float ls = 0.0f;
    for (int i = lane; i < total; i += 32) {
        const float y = stage[i];
        __stcg(part + fb + i, y);
        ls += y;
    }
    __syncwarp();  // the stage is reused by the warp's next tile
    return (double)ls;
}

// A tile's loads in a FIXED order (asm volatile: not reordered against each other): the two 16-byte word
// loads first, then the tile's fragment base and the lane's flags.  Phase A's time moved between 78 and 88 us
// with edits elsewhere in the kernel; ncu's source view of a slow build showed the first word load 15% of the
// phase on the long scoreboard after the compiler had hoisted the flags / base loads above it
// (profiles/r02_exp_k3s_tma_phaseb.log).
__device__ __forceinline__ void tile_loads(const uint4* words4, const uint32_t* wflags, const int32_t* fbase,
                                           int32_t tile, int lane, uint4 (&w)[2], uint32_t& fl, int32_t& fb) {
    const uint4* p = words4 + (int64_t)tile * (kTileW / 8) + 2 * lane;
    asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0].x), "=r"(w[0].y), "=r"(w[0].z), "=r"(w[0].w) : "l"(p));
    asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[1].x), "=r"(w[1].y), "=r"(w[1].z), "=r"(w[1].w) : "l"(p + 1));
    asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(fb) : "l"(fbase + tile));
    asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(fl) : "l"(wflags + (int64_t)tile * 32 + lane));
}

// trace layout: [64 iterations][4] CTA 0 stamps, then per CTA [4] sums over iterations 3..63 of the stamps'
// differences (phase A, barrier 1, phase B, barrier 2 + stop test), ns
#define PLAN_STAMP(k)                                                                                    \
    if (a.trace && tid == 0 && t < 64) {                                                                 \
        unsigned long long gt_;                                                                          \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                                          \
        if (c == 0) a.trace[t * 4 + (k)] = gt_;                                                          \
        if (t >= 3 && (k) > 0) a.trace[256 + c * 4 + (k) - 1] += gt_ - tprev_;                           \
        if (t >= 3 && (k) == 0) a.trace[256 + c * 4 + 3] += gt_ - tprev_;                               \
        tprev_ = gt_;                                                                                    \
    }

template <int OP>
__global__ void __launch_bounds__(kThreads, 1) k_rank_plan(RunArgs a) {
    extern __shared__ __align__(16) float vseg[];  // phase A: segment (kSegStride) + warp stages; phase B: slots
    __shared__ double red[80];
    __shared__ int32_t s_next[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t n = a.n, nlive = a.nlive, niso = n - nlive;
    const int32_t nb = a.nbatch;
    RunWs& W = a.w;
    const int64_t SB = W.nbatch;  // parity stride of slotS
    unsigned epoch = 0;
    const int64_t i0 = nlive + niso * c / G, i1 = nlive + niso * (c + 1) / G;  // isolated-node slice
    const float bg_iso = niso > 0 ? a.bg[a.perm[nlive]] : 0.0f;

    // ---- init: plan-order copies of bg / cap, w_0 = b0 (>= 0), v, S_0 partials per batch (parity 0)
    {
        int neg = 0, mixed = 0;
        for (int32_t b = (int32_t)((int64_t)nb * c / G); b < (int32_t)((int64_t)nb * (c + 1) / G); ++b) {
            double sp = 0.0;
            for (int64_t p = a.bstart[b] + tid; p < a.bstart[b + 1]; p += kThreads) {
                const int32_t id = a.perm[p];
                const double wj = (double)a.b0[id];
                neg |= wj < 0.0;
                const float bgj = a.bg[id], cp = a.cap[id];
                W.bgp[p] = bgj;
                W.capp[p] = cp;
                if (p < a.nsrc) W.vc[vc_index(p)] = node_v<OP>(wj, bgj, cp);
                sp += node_s<OP>(wj, bgj);
            }
            const double S = mapi::block_sum(sp, red);
            if (tid == 0) W.slotS[b] = S;
        }
        double sp = 0.0;
        for (int64_t p = i0 + tid; p < i1; p += kThreads) {
            const int32_t id = a.perm[p];
            const double wj = (double)a.b0[id];
            neg |= wj < 0.0;
            const float bgj = a.bg[id];
            W.bgp[p] = bgj;
            mixed |= __float_as_uint(bgj) != __float_as_uint(bg_iso);
            sp += node_s<OP>(wj, bgj);
        }
        if (__syncthreads_or(neg) && tid == 0) {
            W.status[0] = MAPI_ERR_NEGATIVE;
            W.stop[0] = 1;
        }
        if (__syncthreads_or(mixed) && tid == 0) atomicOr(W.iso_mixed, 1);
        const double S = mapi::block_sum(sp, red);
        if (tid == 0) W.slotSi[c] = S;
        mapi::grid_barrier(W.bar, ++epoch * G);
        if (*(volatile int32_t*)W.stop) return;
    }
    const bool iso_class = *(volatile int32_t*)W.iso_mixed == 0;

    const float4* vc4 = reinterpret_cast<const float4*>(W.vc);
    const uint4* words4 = reinterpret_cast<const uint4*>(a.words);
    float* wstage = vseg + kSegStride + warp * kTileW;
    const uint32_t sb_seg = (uint32_t)__cvta_generic_to_shared(vseg);
    unsigned long long tprev_ = 0;
    double Sprev = 0.0, sprev = 1.0;  // (S, s) of the previous iteration
    int cur_seg = -1;  // the segment held in shared memory (phase B overwrites it)

    for (int32_t t = 0; t < a.iters; ++t) {
        PLAN_STAMP(0);
        // ================= phase A: fragment sums of e_i (fp32) over units taken from a counter; per unit the
        // fp64 sum of its fragment sums (slotY[unit]: a fixed order whichever CTA ran it)
        {
            unsigned* ctr = W.ctr + (t & 1);
            if (tid == 0) s_next[0] = (int32_t)atomicAdd(ctr, 1u);
            __syncthreads();
            int q = 0;
            for (int32_t u = s_next[0]; u < a.nunits; u = s_next[q]) {
                const int32_t ta = __ldg(a.units + 3 * u), tb = __ldg(a.units + 3 * u + 1), seg = __ldg(a.units + 3 * u + 2);
                if (tid == 0) s_next[q ^ 1] = (int32_t)atomicAdd(ctr, 1u);  // the next unit, fetched early
                if (seg != cur_seg) {  // uniform across the block
                    __syncthreads();  // the previous unit's gathers are done
                    const float4* src = vc4 + (int64_t)seg * (kSegStride / 4);
                    float4 r[kSegStride / 4 / kThreads];
#pragma unroll
                    for (int i = 0; i < kSegStride / 4 / kThreads; ++i) r[i] = __ldcg(src + tid + i * kThreads);
#pragma unroll
                    for (int i = 0; i < kSegStride / 4 / kThreads; ++i)
                        reinterpret_cast<float4*>(vseg)[tid + i * kThreads] = r[i];
                    __syncthreads();
                    cur_seg = seg;
                }
                double gp = 0.0;
                int32_t tile = ta + warp;
                uint4 cur[2], nxt[2];
                int32_t fb = 0, fbn = 0;
                uint32_t fl = 0, fln = 0;
                if (tile < tb) tile_loads(words4, a.wflags, a.fbase, tile, lane, cur, fl, fb);
                for (; tile < tb; tile += kWarps) {
                    const int32_t tn = tile + kWarps;
                    // the warp's next tile, in flight while this one is gathered
                    if (tn < tb) tile_loads(words4, a.wflags, a.fbase, tn, lane, nxt, fln, fbn);
                    if (lane == 0 && tn + kWarps < tb) {  // two tiles ahead: into L2 (no registers held)
                        const uint16_t* pf = a.words + (int64_t)(tn + kWarps) * kTileW;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(kTileW * 2) : "memory");
                    }
                    gp += plan_tile(cur, fl, sb_seg, fb, wstage, W.part, lane);
                    cur[0] = nxt[0];
                    cur[1] = nxt[1];
                    fl = fln;
                    fb = fbn;
                }
                const double ug = mapi::block_sum(gp, red);  // its barriers also publish s_next[q ^ 1]
                if (tid == 0) W.slotY[u] = ug;
                q ^= 1;
            }
        }
        PLAN_STAMP(1);
        mapi::grid_barrier(W.bar, ++epoch * G);
        PLAN_STAMP(2);
        // every CTA is past iteration t - 1's counters: re-arm them for iteration t + 1
        if (c == 0 && tid == 0) {
            W.ctr[(t + 1) & 1] = 0u;
            W.ctr[2 + ((t + 1) & 1)] = 0u;
        }

        // ================= phase B: s = n S + sum e, w_{t+1} = (S + e) / s (fp64), delta, next v and S
        // S = the batches' and the isolated slices' partials, sum e = the units' partials: all loads in flight
        // at once, one pair of block sums (fixed order: thread-strided partials, then the block tree)
        double S = 0.0, ye = 0.0;
        {
            const double* ps = W.slotS + (t & 1) * SB;
            const double* pi = W.slotSi + (t & 1) * kMaxGrid;
            for (int64_t k = tid; k < nb; k += kThreads) S += __ldcg(ps + k);
            for (int64_t k = tid; k < G; k += kThreads) S += __ldcg(pi + k);
            for (int64_t k = tid; k < a.nunits; k += kThreads) ye += __ldcg(W.slotY + k);
            block_sum2(S, ye, red);
        }
        const double s = (double)n * S + ye;
        if (!(s > 0.0) || isinf(s)) {  // uniform: every CTA sees the same s
            if (c == 0 && tid == 0) {
                W.status[0] = (s == 0.0) ? MAPI_ERR_DEGENERATE : MAPI_ERR_NONFINITE;
                W.stop[0] = 1;
            }
            return;
        }
        const bool first = t == 0;
        // (S_{t-1}, s_{t-1}): every CTA formed the same values last iteration
        const double Sp = Sprev, sp_ = sprev;
        const double rs = 1.0 / s, rsp = 1.0 / sp_;
        double* e_cur = (t & 1) ? W.e1 : W.e0;
        const double* e_prev = (t & 1) ? W.e0 : W.e1;
        double* slotSn = W.slotS + ((t + 1) & 1) * SB;
        cur_seg = -1;  // the batches overwrite the shared segment
        {
            unsigned* ctr = W.ctr + 2 + (t & 1);
            if (tid == 0) s_next[0] = (int32_t)atomicAdd(ctr, 1u);
            __syncthreads();
            int q = 0;
            for (int32_t b = s_next[0]; b < nb; b = s_next[q]) {
                if (tid == 0) s_next[q ^ 1] = (int32_t)atomicAdd(ctr, 1u);
                const int64_t bs = a.bstart[b], be = a.bstart[b + 1];
                int32_t r0[kNodeK], r1[kNodeK];
                double eo[kNodeK], e[kNodeK];
                float bgv[kNodeK], cpv[kNodeK];
#pragma unroll
                for (int k = 0; k < kNodeK; ++k) {
                    const int64_t p = bs + tid + (int64_t)k * kThreads;
                    const bool in = p < be;
                    r0[k] = in ? __ldg(a.rsp + p) : 0;
                    r1[k] = in ? __ldg(a.rsp + p + 1) : 0;
                    eo[k] = in ? (first ? (double)a.b0[a.perm[p]] : __ldcg(e_prev + p)) : 0.0;
                    bgv[k] = in ? W.bgp[p] : 0.0f;
                    cpv[k] = in ? W.capp[p] : 0.0f;
                    e[k] = 0.0;
                }
                const int32_t R0 = __ldg(a.rsp + bs), R1 = __ldg(a.rsp + be);
                __syncthreads();  // the previous batch's (or phase A's) shared reads are done
                {
                    constexpr int kU = 4;
                    for (int32_t kb = R0 + tid; kb < R1; kb += kU * kThreads) {
                        int32_t f[kU], rl[kU];
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            const int32_t k = kb + u * kThreads;
                            f[u] = k < R1 ? __ldg(a.bfrag + k) : -1;
                            rl[u] = k < R1 ? (int32_t)__ldg(a.brel + k) : 0;
                        }
                        float v[kU];
#pragma unroll
                        for (int u = 0; u < kU; ++u) v[u] = f[u] >= 0 ? __ldcg(W.part + f[u]) : 0.0f;
#pragma unroll
                        for (int u = 0; u < kU; ++u)
                            if (f[u] >= 0) vseg[rl[u]] = v[u];
                    }
                }
                __syncthreads();
#pragma unroll
                for (int k = 0; k < kNodeK; ++k)
                    for (int32_t r = r0[k]; r < r1[k]; ++r) e[k] += (double)vseg[r - R0];
                double dp = 0.0, sn = 0.0;
#pragma unroll
                for (int k = 0; k < kNodeK; ++k) {
                    const int64_t p = bs + tid + (int64_t)k * kThreads;
                    if (p >= be) continue;
                    const double wn = qdiv(S + e[k], s, rs);
                    const double wo = first ? eo[k] : qdiv(Sp + eo[k], sp_, rsp);
                    dp += fabs(wn - wo);
                    if (p < a.nsrc) W.vc[vc_index(p)] = node_v<OP>(wn, bgv[k], cpv[k]);
                    sn += node_s<OP>(wn, bgv[k]);
                    e_cur[p] = e[k];
                }
                block_sum2(dp, sn, red);  // its barriers also publish s_next[q ^ 1]
                if (tid == 0) {
                    W.slotD[b] = dp;
                    slotSn[b] = sn;
                }
                q ^= 1;
            }
        }
        // isolated nodes: y = S for all; per node on the first iteration (w_0 = b0 differs) or when their bg
        // differ, else one class term
        {
            double dp = 0.0, sn = 0.0;
            const double wn = qdiv(S, s, rs);
            if (first || !iso_class) {
                const double wc = first ? 0.0 : qdiv(Sp, sp_, rsp);
                for (int64_t p = i0 + tid; p < i1; p += kThreads) {
                    const double wo = first ? (double)a.b0[a.perm[p]] : wc;
                    dp += fabs(wn - wo);
                    sn += node_s<OP>(wn, W.bgp[p]);
                }
            } else if (c == 0 && tid == 0 && niso > 0) {
                dp += (double)niso * fabs(wn - qdiv(Sp, sp_, rsp));
                sn += (double)niso * node_s<OP>(wn, bg_iso);
            }
            block_sum2(dp, sn, red);
            if (tid == 0) {
                W.slotDi[c] = dp;
                W.slotSi[((t + 1) & 1) * kMaxGrid + c] = sn;
            }
        }
        PLAN_STAMP(3);
        mapi::grid_barrier(W.bar, ++epoch * G);
        double dpart = 0.0;
        for (int64_t k = tid; k < nb; k += kThreads) dpart += __ldcg(W.slotD + k);
        for (int64_t k = tid; k < G; k += kThreads) dpart += __ldcg(W.slotDi + k);
        const double d = mapi::block_sum(dpart, red);
        Sprev = S;
        sprev = s;
        if (c == 0 && tid == 0) {
            W.hist[((t + 1) & 1) * 2] = S;
            W.hist[((t + 1) & 1) * 2 + 1] = s;
            if (a.deltas) a.deltas[t] = (float)d;
            W.status[1] = t + 1;
        }
        if (a.tol > 0.0f && d < (double)a.tol) break;  // uniform decision
    }
}

// Outputs: w = (S + e)/s of the last iteration (b0 if none) in fp64 as the loop formed it (e = 0 for the
// isolated nodes); w_out = fp32(w) in node-id order, per-CTA sums of w^2, then the optional l2 copy.
struct Last {
    const double* e;
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
__global__ void __launch_bounds__(256) k_plan_output(int64_t n, int64_t nlive, RunWs W, const int32_t* __restrict__ perm,
                                                     const float* __restrict__ b0, float* __restrict__ w_out) {
    __shared__ double red[33];
    const Last L = last_iter(W);
    const double rls = 1.0 / L.s;
    double part = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t id = perm[p];
        const double x = L.none ? (double)b0[id] : qdiv(L.S + (p < nlive ? L.e[p] : 0.0), L.s, rls);
        w_out[id] = (float)x;
        part = fma(x, x, part);
    }
    const double qs = mapi::block_sum(part, red);
    if (threadIdx.x == 0) W.slotQ[blockIdx.x] = qs;
}
__global__ void __launch_bounds__(256) k_plan_output_l2(int64_t n, int64_t nlive, RunWs W,
                                                        const int32_t* __restrict__ perm,
                                                        const float* __restrict__ b0, int nq,
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
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t id = perm[p];
        const double x = L.none ? (double)b0[id] : qdiv(L.S + (p < nlive ? L.e[p] : 0.0), L.s, rls);
        w_l2[id] = l2 > 0.0 ? (float)(x / l2) : 0.0f;
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
    if (nnz < 0 || nwords_bound(nnz, max_segments(n)) >= (int64_t)INT32_MAX)
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
    MAPI_CUDA(cudaFuncSetAttribute(k_rank_plan<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPlanSmem));
    MAPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rank_plan<0>, kThreads, kPlanSmem));
    if (occ < 1) return fail(MAPI_ERR_CUDA, "planned ranking kernel does not fit on an SM");
    const int grid = std::min(d.sms, kMaxGrid);
    BuildWs B = carve_build(ws, n, nnz);
    auto blocks = [&](int64_t items, int per_sm) {
        return (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)per_sm * d.sms));
    };
    const unsigned gn = blocks(n, 8), ge = blocks(nnz, 16);
    const int64_t nseg_max = max_segments(n), ntiles_max = nwords_bound(nnz, nseg_max) / kTileW;
    MAPI_CUDA(cudaMemsetAsync(B.counter, 0, 256, s));
    MAPI_CUDA(cudaMemsetAsync(B.outdeg, 0, 4 * (size_t)n, s));
    MAPI_CUDA(cudaMemsetAsync(B.rcnt, 0, 4 * (size_t)(n + 1), s));
    MAPI_CUDA(cudaMemsetAsync(B.segcnt, 0, 4 * (size_t)(nseg_max + 1), s));
    MAPI_CUDA(cudaMemsetAsync(B.segstart, 0, 4 * (size_t)(nseg_max + 1), s));
    MAPI_CUDA(cudaMemsetAsync(B.tcnt, 0, 4 * (size_t)(ntiles_max + 1), s));
    if (nnz > 0) {
        kp_outdeg<<<ge, 256, 0, s>>>(nnz, col_idx, B.outdeg);
        MAPI_LAUNCHED();
    }
    kp_src_keys<<<gn, 256, 0, s>>>(n, B.outdeg, row_ptr, B.skey, B.sval, B.counter);
    MAPI_LAUNCHED();
    // plan order into the plan's first array (its offset does not depend on the later sizes)
    int32_t* perm = plan_view(plan, n, 1, 0, 0, 0).perm;
    size_t tb = B.cub_bytes;
    MAPI_CUDA(cub::DeviceRadixSort::SortPairs(B.cub, tb, B.skey, B.skey2, B.sval, perm, (int)n, 0, 32, s));
    kp_inv<<<gn, 256, 0, s>>>(n, perm, B.inv);
    MAPI_LAUNCHED();
    uint32_t cnt_h[2] = {0, 0};
    MAPI_CUDA(cudaMemcpyAsync(cnt_h, B.counter, 8, cudaMemcpyDeviceToHost, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    const int64_t nsrc = cnt_h[0], nlive = n - (int64_t)cnt_h[1];
    const int32_t nseg = (int32_t)std::max<int64_t>(1, (nsrc + kSegSrc - 1) / kSegSrc);
    if (nnz > 0) {
        kp_edges<<<ge, 256, 0, s>>>(n, nnz, row_ptr, col_idx, B.inv, B.ekey, B.eoff);
        MAPI_LAUNCHED();
        int bits = 0;
        while ((1ll << bits) < (int64_t)nseg) ++bits;
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceRadixSort::SortPairs(B.cub, tb, B.ekey, B.ekey2, B.eoff, B.eoff2, (int)nnz, 0, 32 + bits,
                                                  s));
        kp_segcount<<<ge, 256, 0, s>>>(nnz, B.ekey2, B.segcnt, B.segstart);
        MAPI_LAUNCHED();
    }
    // tile-aligned segment starts: they size the word array
    kp_segb<<<1, 32, 0, s>>>(nseg, B.segcnt, B.segstart, B.segb);
    MAPI_LAUNCHED();
    int64_t nfrag = 0, nwords = 0;
    std::vector<int32_t> segb_h(nseg + 1);
    MAPI_CUDA(cudaMemcpyAsync(segb_h.data(), B.segb, 4 * (size_t)(nseg + 1), cudaMemcpyDeviceToHost, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    nwords = segb_h[nseg];
    const int64_t ntiles = nwords / kTileW;
    // phase A work units in scheduling order: segments from the last to the first, kUnitBig tiles per unit
    // until only 1/8 of all tiles remain, then kUnitSmall (one tile per warp): the dynamically scheduled
    // tail is fine-grained, and consecutive units mostly share a segment
    std::vector<int32_t> units_h;
    {
        int64_t done = 0;
        for (int32_t sg = nseg - 1; sg >= 0; --sg) {
            int64_t ta = segb_h[sg] / kTileW;
            const int64_t te = segb_h[sg + 1] / kTileW;
            while (ta < te) {
                const int64_t size = std::min<int64_t>(te - ta, (ntiles - done) > ntiles / 8 ? kUnitBig : kUnitSmall);
                units_h.push_back((int32_t)ta);
                units_h.push_back((int32_t)(ta + size));
                units_h.push_back(sg);
                ta += size;
                done += size;
            }
        }
    }
    const int64_t nunits = (int64_t)units_h.size() / 3;
    if (nunits > nunits_bound(ntiles, nseg)) return fail(MAPI_ERR_CUDA, "internal: %lld units", (long long)nunits);
    if (nnz > 0) {
        kp_fstart<<<ge, 256, 0, s>>>(nnz, B.ekey2, B.segstart, B.segb, B.fstart);
        MAPI_LAUNCHED();
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceScan::ExclusiveSum(B.cub, tb, B.fstart, B.fid, (int)nnz, s));
        uint32_t last[2] = {0, 0};
        MAPI_CUDA(cudaMemcpyAsync(&last[0], B.fid + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
        MAPI_CUDA(cudaMemcpyAsync(&last[1], B.fstart + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
        MAPI_CUDA(cudaStreamSynchronize(s));
        nfrag = (int64_t)last[0] + last[1];
    }
    PlanView P = plan_view(plan, n, nseg, nunits, nwords, nfrag);
    MAPI_CUDA(cudaMemcpyAsync(P.segb, B.segb, 4 * (size_t)(nseg + 1), cudaMemcpyDeviceToDevice, s));
    if (nunits > 0)
        MAPI_CUDA(cudaMemcpyAsync(P.units, units_h.data(), 4 * units_h.size(), cudaMemcpyHostToDevice, s));
    if (nnz > 0) {
        kp_fill_words<<<blocks(nwords, 16), 256, 0, s>>>(nwords, P.words);
        MAPI_LAUNCHED();
        kp_frag<<<ge, 256, 0, s>>>(nnz, B.ekey2, B.eoff2, B.fstart, B.fid, B.segstart, P.segb, B.frow, B.fidx, B.rcnt,
                                   B.tcnt, P.words);
        MAPI_LAUNCHED();
        kp_wflags<<<blocks(nwords / kLaneW, 8), 256, 0, s>>>(nwords / kLaneW, P.words, P.wflags);
        MAPI_LAUNCHED();
        {  // investigation switch: MAPI_PLAN_DECONFLICT=<passes> (0: keep the words in destination order)
            const char* dc = getenv("MAPI_PLAN_DECONFLICT");
            const int rounds = dc ? std::max(0, std::min(atoi(dc), 16)) : kDeconflictRounds;
            if (rounds > 0) {
                kp_deconflict<<<blocks(ntiles * 32, 8), 256, 0, s>>>(ntiles, P.words, P.wflags, rounds);
                MAPI_LAUNCHED();
            }
        }
        // row-sorted slots (stable: the (segment, position) order within a row is kept) and their inverse
        int rbits = 1;
        while ((1ll << rbits) < n) ++rbits;
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceRadixSort::SortPairs(B.cub, tb, B.frow, B.frow2, B.fidx, B.pos, (int)nfrag, 0, rbits, s));
        kp_fslot<<<ge, 256, 0, s>>>(nfrag, B.pos, B.fslot);
        MAPI_LAUNCHED();
    }
    tb = B.cub_bytes;
    MAPI_CUDA(cub::DeviceScan::ExclusiveSum(B.cub, tb, B.tcnt, P.fbase, (int)(ntiles + 1), s));
    tb = B.cub_bytes;
    MAPI_CUDA(cub::DeviceScan::ExclusiveSum(B.cub, tb, B.rcnt, P.rsp, (int)(n + 1), s));
    // node-pass batches over the live rows, and the fragments in (batch, fragment) order
    int64_t nbatch = 0;
    if (nlive > 0) {
        // investigation switch: MAPI_PLAN_SLOT_BLOCK=<slots> in [kSlotBlock, 2 kSlotBlock] (fewer, larger batches;
        // nbatch_bound stays valid: it assumes the smallest block)
        const char* sbe = getenv("MAPI_PLAN_SLOT_BLOCK");
        const int32_t slot_block = sbe ? std::max(kSlotBlock, std::min(atoi(sbe), 2 * kSlotBlock)) : kSlotBlockRun;
        kp_bflag<<<blocks(nlive, 8), 256, 0, s>>>(nlive, P.rsp, B.bflag, slot_block);
        MAPI_LAUNCHED();
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceScan::InclusiveSum(B.cub, tb, B.bflag, B.bincl, (int)nlive, s));
        int32_t nb = 0;
        MAPI_CUDA(cudaMemcpyAsync(&nb, B.bincl + nlive - 1, 4, cudaMemcpyDeviceToHost, s));
        MAPI_CUDA(cudaStreamSynchronize(s));
        nbatch = nb;
        if (nbatch > nbatch_bound(n, nnz)) return fail(MAPI_ERR_CUDA, "internal: %lld batches", (long long)nbatch);
        kp_bstart<<<blocks(nlive, 8), 256, 0, s>>>(nlive, B.bflag, B.bincl, P.bstart);
        MAPI_LAUNCHED();
    } else {
        MAPI_CUDA(cudaMemsetAsync(P.bstart, 0, 4, s));
    }
    if (nfrag > 0) {
        kp_fbat<<<ge, 256, 0, s>>>(nfrag, B.frow, B.bincl, B.fbat, B.fidx);
        MAPI_LAUNCHED();
        int bbits = 1;
        while ((1ll << bbits) < nbatch + 1) ++bbits;
        tb = B.cub_bytes;
        MAPI_CUDA(cub::DeviceRadixSort::SortPairs(B.cub, tb, B.fbat, B.fbat2, B.fidx, P.bfrag, (int)nfrag, 0, bbits, s));
        kp_brel<<<ge, 256, 0, s>>>(nfrag, P.bfrag, B.fbat, B.fslot, P.bstart, P.rsp, P.brel, B.counter + 2);
        MAPI_LAUNCHED();
    }
    uint32_t maxslots = 0;
    MAPI_CUDA(cudaMemcpyAsync(&maxslots, B.counter + 2, 4, cudaMemcpyDeviceToHost, s));
    struct {
        uint64_t magic;
        int64_t n, nnz, nsrc, nfrag, nwords, nlive, nbatch, nunits;
        int32_t nseg, grid;
    } hdr = {kMagic, n, nnz, nsrc, nfrag, nwords, nlive, nbatch, nunits, nseg, grid};
    MAPI_CUDA(cudaMemcpyAsync(plan, &hdr, sizeof(hdr), cudaMemcpyHostToDevice, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    if (maxslots > (uint32_t)kSmemF)
        return fail(MAPI_ERR_SHAPE, "a node batch gathers %u fragment sums (> %d): a row with this many fragments "
                    "needs the plan-free path (mapi_rank_csr)", maxslots, kSmemF);
    info->n = n;
    info->nnz = nnz;
    info->nsrc = nsrc;
    info->npieces = nfrag;
    info->nwords = nwords;
    info->nseg = nseg;
    info->grid = grid;
    info->nlive = nlive;
    info->nbatch = nbatch;
    info->nunits = nunits;
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
        info->npieces < 0 || info->npieces > std::max<int64_t>(info->nnz, 0) || info->nwords < 0 ||
        info->nwords % kTileW != 0 || info->nsrc < 0 || info->nsrc > n || info->nlive < info->nsrc ||
        info->nlive > n || info->nbatch < 0 || info->nbatch > nbatch_bound(n, info->nnz) || info->nunits < 0 ||
        info->nunits > nunits_bound(info->nwords / kTileW, info->nseg) || info->nbatch > INT32_MAX ||
        (info->nlive > 0) != (info->nbatch > 0))
        return fail(MAPI_ERR_SHAPE, "plan info is inconsistent (n %lld, nnz %lld, grid %d, nseg %d)", (long long)n,
                    (long long)info->nnz, info->grid, info->nseg);
    if (max_iters < 1) return fail(MAPI_ERR_BAD_PARAM, "max_iters (%d) must be >= 1", max_iters);
    if (!(tol >= 0.0f)) return fail(MAPI_ERR_BAD_PARAM, "tol must be >= 0");
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    const size_t need = run_ws_exact(n, info->nseg, info->npieces, info->nunits, info->nbatch);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    mapi_status st = device_info(d);
    if (st != MAPI_OK) return st;
    if (info->grid > d.sms)
        return fail(MAPI_ERR_SHAPE, "plan built for %d CTAs; this device has %d SMs", info->grid, d.sms);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const PlanView P = plan_view(const_cast<void*>(plan), n, info->nseg, info->nunits, info->nwords, info->npieces);
    RunArgs a;
    a.n = n;
    a.nlive = info->nlive;
    a.nsrc = info->nsrc;
    a.nseg = info->nseg;
    a.nunits = (int32_t)info->nunits;
    a.nbatch = (int32_t)info->nbatch;
    a.iters = max_iters;
    a.tol = tol;
    a.perm = P.perm; a.segb = P.segb; a.units = P.units; a.fbase = P.fbase; a.rsp = P.rsp;
    a.bstart = P.bstart; a.bfrag = P.bfrag; a.brel = P.brel; a.words = P.words; a.wflags = P.wflags;
    a.cap = cap; a.bg = bg; a.b0 = b0; a.deltas = deltas;
    // investigation: MAPI_PLAN_TRACE=1 prints CTA 0's per-phase times (us) of iterations 3..min(iters, 64);
    // MAPI_PLAN_TRACE_FILE=<path> also writes every CTA's phase times
    static const bool trace_on = getenv("MAPI_PLAN_TRACE") && atoi(getenv("MAPI_PLAN_TRACE")) > 0;
    unsigned long long* trace_d = nullptr;
    if (trace_on) {
        MAPI_CUDA(cudaMalloc(&trace_d, 8 * (4 * 64 + 4 * kMaxGrid)));
        MAPI_CUDA(cudaMemsetAsync(trace_d, 0, 8 * (4 * 64 + 4 * kMaxGrid), s));
    }
    a.trace = trace_d;
    a.w = carve_run(ws, n, info->nseg, info->npieces, info->nunits, info->nbatch);
    MAPI_CUDA(cudaMemsetAsync(ws, 0, 256, s));
    // the compact vector's zero slots (offset 32767 of each segment) and unused tail stay 0
    MAPI_CUDA(cudaMemsetAsync(a.w.vc, 0, 4 * (size_t)kSegStride * (size_t)info->nseg, s));
    auto kern = op == MAPI_OP_DOT ? k_rank_plan<2> : k_rank_plan<0>;
    MAPI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPlanSmem));
    Timer timer(s);
    void* args[] = {&a};
    timer.start();
    MAPI_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(info->grid), dim3(kThreads), args, kPlanSmem, s));
    timer.stop();
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const int gout = (int)std::min<int64_t>((n + 255) / 256, std::min(4 * d.sms, kMaxGrid));
    k_plan_output<<<gout, 256, 0, s>>>(n, info->nlive, a.w, P.perm, b0, w_out);
    MAPI_LAUNCHED();
    if (w_l2_out) {
        k_plan_output_l2<<<gout, 256, 0, s>>>(n, info->nlive, a.w, P.perm, b0, gout, w_l2_out);
        MAPI_LAUNCHED();
    }
    int32_t h[2] = {0, 0};
    MAPI_CUDA(cudaMemcpyAsync(h, a.w.status, sizeof(h), cudaMemcpyDeviceToHost, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    timer.harvest();
    if (trace_d) {
        std::vector<unsigned long long> tr(4 * 64 + 4 * kMaxGrid);
        cudaMemcpy(tr.data(), trace_d, 8 * tr.size(), cudaMemcpyDeviceToHost);
        cudaFree(trace_d);
        const int it = std::min(h[1], 64) - 3;
        const char* path = getenv("MAPI_PLAN_TRACE_FILE");
        if (path && it > 0) {  // per-CTA phase times (dynamic scheduling: the barrier waits show the balance)
            FILE* f = fopen(path, "w");
            if (f) {
                fprintf(f, "cta,phaseA_us,bar1_us,phaseB_us,bar2_us\n");
                for (int cc = 0; cc < info->grid; ++cc) {
                    fprintf(f, "%d", cc);
                    for (int k = 0; k < 4; ++k) fprintf(f, ",%.2f", tr[256 + cc * 4 + k] / 1e3 / it);
                    fprintf(f, "\n");
                }
                fclose(f);
            }
        }
        if (it > 0) {
            double ph[4] = {0, 0, 0, 0};
            for (int t = 3; t < 3 + it; ++t) {
                ph[0] += (tr[t * 4 + 1] - tr[t * 4 + 0]) / 1e3;
                ph[1] += (tr[t * 4 + 2] - tr[t * 4 + 1]) / 1e3;
                ph[2] += (tr[t * 4 + 3] - tr[t * 4 + 2]) / 1e3;
                ph[3] += (t + 1 < 64 ? (tr[(t + 1) * 4 + 0] - tr[t * 4 + 3]) / 1e3 : 0.0);
            }
            fprintf(stderr, "[mapi plan trace] us/iteration (CTA 0, %d iterations): phaseA %.1f bar1 %.1f phaseB %.1f bar2 %.1f"
                    " (nbatch %lld, nunits %lld, nfrag %lld, nlive %lld)\n",
                    it, ph[0] / it, ph[1] / it, ph[2] / it, ph[3] / it, (long long)info->nbatch,
                    (long long)info->nunits, (long long)info->npieces, (long long)info->nlive);
        }
    }
    if (iters_done) *iters_done = h[1];
    if (h[0] == MAPI_ERR_NEGATIVE) return fail(MAPI_ERR_NEGATIVE, "b0 has a negative entry");
    if (h[0] == MAPI_ERR_DEGENERATE) return fail(MAPI_ERR_DEGENERATE, "||G (+) w_t||_1 == 0 at iteration %d", h[1]);
    if (h[0] == MAPI_ERR_NONFINITE)
        return fail(MAPI_ERR_NONFINITE, "||G (+) w_t||_1 is not finite at iteration %d", h[1]);
    return MAPI_OK;
}

}  // extern "C"
