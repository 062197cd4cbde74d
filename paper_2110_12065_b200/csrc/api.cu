// api.cu — the C ABI of libmapi.so (declared and documented in include/mapi.h).
//
// Host side only: argument validation, workspace carving, launch-shape selection, kernel
// launches, status read-back.  Every step of the hot path runs in the kernels of
// dense.cuh / deflate.cuh / csr.cuh / batched.cuh; there is no CPU fallback.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>
#include <memory>
#include <thread>

#include "../../include/mapi.h"
#include "host_common.h"
#include "csr_plan.h"
#include "minibatch.h"
#include "batched.cuh"
#include "bulk.cuh"
#include "resident.cuh"
#include "packed.cuh"
#include "single.cuh"
#include "sym.cuh"
#include "reorder.cuh"
#include "csr.cuh"
#include "deflate.cuh"
#include "dense.cuh"
#include "matmat.cuh"
#include "outer.cuh"
#include "p2p.cuh"

using namespace mapi;

using namespace mapi_host;

namespace {

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

template <int V>
using IC = std::integral_constant<int, V>;

template <typename F>
auto with_op(int op, F&& f) {
    return op == 2 ? f(IC<2>{}) : (op == 1 ? f(IC<1>{}) : f(IC<0>{}));
}
template <typename F>
auto with_vec(int vec, F&& f) {
    return vec == 8 ? f(IC<8>{}) : (vec == 4 ? f(IC<4>{}) : f(IC<1>{}));
}
template <typename F>
auto with_pol(int pol, F&& f) {
    return pol == 1 ? f(IC<1>{}) : f(IC<0>{});
}

constexpr int unroll_for(int vec) { return vec == 8 ? 4 : (vec == 4 ? 8 : 16); }

// widest vector the row starts support: 32 B (v8) needs a 32 B-aligned base and lda % 8 == 0
int vec_width(const void* base, int64_t lda) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(base);
    if (a % 32 == 0 && lda % 8 == 0) return 8;
    if (a % 16 == 0 && lda % 4 == 0) return 4;
    return 1;
}

// cache policy: stream with L2 evict-first when the matrix cannot stay L2-resident
int load_policy(const Device& d, int64_t rows, int64_t lda) {
    const double bytes = (double)rows * (double)lda * 4.0;
    return bytes > 0.5 * (double)d.l2_bytes ? 0 : 1;
}

mapi_status check_op(int32_t op, bool dot_ok = false) {
    if (op == MAPI_OP_DOT && dot_ok) return MAPI_OK;
    if (op != MAPI_OP_MIN1 && op != MAPI_OP_MIN2)
        return fail(MAPI_ERR_BAD_PARAM, dot_ok ? "op (%d) must be MAPI_OP_MIN1 (0), MAPI_OP_MIN2 (1) or MAPI_OP_DOT (2)"
                                               : "op (%d) must be MAPI_OP_MIN1 (0) or MAPI_OP_MIN2 (1)",
                    op);
    return MAPI_OK;
}

// ---------------------------------------------------------------------------------------------
// dense iterate workspace: [header 256 B: bar @0, status[2] @64, stop @72]
//                          [slots 2 x 1024 floats][y 2n floats][w n floats]
constexpr int kMaxGrid = 1024;
constexpr int kIterThreads = 512;

// K2p workspace: [status[2] @0, grid-barrier counter @64 | 256][CTA |y| partials 2 x kP2pMaxGrid f64]
size_t sharded_ws_bytes() { return 256 + sizeof(double) * 2 * kP2pMaxGrid; }

size_t iterate_ws_bytes(int64_t n) {
    return 256 + align256(sizeof(double) * 2 * kMaxGrid) + align256(sizeof(double) * 2 * (size_t)n) +
           align256(sizeof(float) * (size_t)n);
}

struct IterWs {
    unsigned int* bar;
    int32_t* status;
    int32_t* stop;
    float* slots;
    float* y;
    float* w;
};

IterWs carve_iterate(void* ws, int64_t n) {
    char* p = static_cast<char*>(ws);
    IterWs w;
    w.bar = reinterpret_cast<unsigned int*>(p);
    w.status = reinterpret_cast<int32_t*>(p + 64);
    w.stop = reinterpret_cast<int32_t*>(p + 72);
    p += 256;
    w.slots = reinterpret_cast<float*>(p);  // holds 2 x kMaxGrid doubles
    p += align256(sizeof(double) * 2 * kMaxGrid);
    w.y = reinterpret_cast<float*>(p);  // 2n floats, or 2n tagged 8-byte words (K2r)
    p += align256(sizeof(double) * 2 * (size_t)n);
    w.w = reinterpret_cast<float*>(p);
    return w;
}

size_t persistent_smem_bytes(int64_t n) { return sizeof(float) * (size_t)((n + 3) & ~int64_t(3)) + sizeof(double) * 33; }

// Dense path selection (K2): "coop" (CTA-cooperative rows, default when A rows are
// 32 B-aligned and n >= 16 chunks of 256), "rows" (one warp per row; any alignment, small n),
// "multi" (two launches per iteration, any n).  MAPI_DENSE_PATH=coop|rows|multi forces one
// (investigation / tests); a forced path that cannot run falls back in the order above.
const char* dense_path_env() {
    const char* e = getenv("MAPI_DENSE_PATH");
    return e ? e : "";
}

bool use_persistent(const Device& d, int64_t n) {
    if (strcmp(dense_path_env(), "multi") == 0) return false;
    return persistent_smem_bytes(n) <= (size_t)d.smem_optin;
}

int coop_warps(int64_t n) { return (n / 256) >= 64 ? 32 : 16; }

// K6 (one 8-CTA cluster, A in distributed shared memory) for small n; MAPI_DENSE_PATH=cluster forces
bool use_cluster(const Device& d, int64_t n) {
    const char* e = dense_path_env();
    if (strcmp(e, "rows") == 0 || strcmp(e, "multi") == 0 || strcmp(e, "coop") == 0 || strcmp(e, "bulk") == 0 ||
        strcmp(e, "resident") == 0)
        return false;
    if (n <= 512) return true;  // K6r (registers) fits any n <= 512
    if (cluster_smem_bytes(n) > (size_t)d.smem_optin) return false;
    return strcmp(e, "cluster") == 0 || strcmp(e, "cluster_smem") == 0;
}

// K2t (TMA bulk-copy ring, bulk.cuh) for mid-size n where A stays L2-resident and the per-row kernel
// is latency-bound; needs 16 B-aligned rows.  MAPI_DENSE_PATH=bulk forces it (any n it can hold).
int bulk_slots(const Device& d, int64_t n) {
    const int64_t grid = std::min<int64_t>(d.sms, n);
    const size_t fixed = bulk_fixed_smem(n, (n + grid - 1) / grid);
    if (fixed >= (size_t)d.smem_optin) return 0;
    const int64_t sl = std::min<int64_t>(kBulkMaxSlots, ((size_t)d.smem_optin - fixed) / (sizeof(float) * kBulkChunk));
    return (int)(sl / kBulkNC * kBulkNC);  // whole slots per warp
}

bool use_bulk(const Device& d, const float* A, int64_t n, int64_t lda) {
    const char* e = dense_path_env();
    if (strcmp(e, "rows") == 0 || strcmp(e, "multi") == 0 || strcmp(e, "coop") == 0) return false;
    if (n % 4 != 0 || lda % 4 != 0 || (reinterpret_cast<uintptr_t>(A) & 15) != 0) return false;
    if (bulk_slots(d, n) < 2 * kBulkNC) return false;
    if (strcmp(e, "bulk") == 0) return true;
    // default: L2-resident A at n >= 3072 (measured vs K2 per-row, profiles/r01_probe_bulk.log:
    // n = 4096 13.4 vs 14.7 us/iteration; at n <= 2048 and for HBM-resident A the others win or tie)
    return n >= 3072 && n < 8192 && (double)n * (double)lda * 4.0 <= 0.6 * (double)d.l2_bytes;
}

bool use_coop(const Device& d, const float* A, int64_t n, int64_t lda) {
    const char* e = dense_path_env();
    if (strcmp(e, "rows") == 0 || strcmp(e, "multi") == 0) return false;
    if (strcmp(e, "bulk") == 0 && use_bulk(d, A, n, lda)) return false;
    if (vec_width(A, lda) != 8) return false;
    if (strcmp(e, "coop") != 0 && n / 256 < 32) return false;  // n < 8192: the per-row kernel is faster
    const int64_t grid = std::min<int64_t>(d.sms, n);
    return coop_smem_bytes(n, (int)grid, coop_warps(n)) <= (size_t)d.smem_optin;
}

// K6t (single.cuh): one CTA, matrix in registers + TMEM, for n <= 256.  MAPI_DENSE_PATH=single forces it.
bool use_single(const Device& d, int64_t n) {
    (void)d;
    const char* e = dense_path_env();
    if (n > kSingleN) return false;
    return strcmp(e, "single") == 0 || e[0] == 0;
}

// K2r (resident.cuh): the whole matrix on chip (TMEM + shared memory) for n <= 4096 when every CTA's
// rows fit (ceil(n / grid) <= 28).  MAPI_DENSE_PATH=resident forces it; default range set by measurement.
bool use_resident(const Device& d, int64_t n) {
    const char* e = dense_path_env();
    if (strcmp(e, "rows") == 0 || strcmp(e, "multi") == 0 || strcmp(e, "coop") == 0 || strcmp(e, "bulk") == 0)
        return false;
    const int64_t grid = std::min<int64_t>(d.sms, n);
    if (n > kResNPad || (n + grid - 1) / grid > kResMaxRows) return false;
    if (resident_smem_bytes() > (size_t)d.smem_optin) return false;
    if (strcmp(e, "resident") == 0) return true;
    // measured (profiles/r01_probe_resident_range.log, us / iteration incl. launch): n = 1536 5.5 vs 6.2
    // (per-row K2), n = 4096 4.7 vs 12.8 (K2t); at n <= 1024 all grid-wide kernels tie at ~5 us (exchange-bound)
    return n > 1024;
}

int resident_warps() {
    const char* e = getenv("MAPI_RES_NW");
    return (e && atoi(e) == 16) ? 16 : 8;  // 8 measured faster at n = 4096 (scripts/probe_k2r.cu)
}

// Runs MAPI on device buffers; no stream sync, no status read-back (caller does both).
// dP / dR / dk: fused L2 deflation of A (only when use_resident(d, n); the caller checks)
mapi_status iterate_launch(const Device& d, int32_t op, const float* A, int64_t n, int64_t lda,
                           const float* b0, int32_t iters, float tol, float* w_out, float* norms,
                           float* deltas, const IterWs& W, cudaStream_t s, Timer* timer,
                           const double* dP = nullptr, const double* dR = nullptr, int32_t dk = 0,
                           float* w_l2 = nullptr, bool* l2_done = nullptr) {
    const int vec = vec_width(A, lda);
    const int pol = load_policy(d, n, lda);
    if (l2_done) *l2_done = false;
    if (dk > 0 && !use_resident(d, n)) return fail(MAPI_ERR_BAD_PARAM, "fused deflation needs the resident path");
    if (use_single(d, n)) {  // (one CTA: no grid barrier counter to reset)
        using KernT = void (*)(IterArgs);
        KernT kern = op == 2 ? k_iterate_single<2> : (op == 1 ? k_iterate_single<1> : k_iterate_single<0>);
        const size_t smem = single_smem_bytes();
        static thread_local KernT attr_done[3] = {nullptr, nullptr, nullptr};  // attribute set once per kernel
        if (attr_done[op] != kern) {
            MAPI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr_done[op] = kern;
        }
        IterArgs a;
        a.A = A; a.n = n; a.lda = lda; a.b0 = b0; a.iters = iters; a.tol = tol;
        a.w_out = w_out; a.norms = norms; a.deltas = deltas; a.y = W.y; a.slots = W.slots;
        a.bar = W.bar; a.status = W.status;
        a.w_l2 = l2_done ? w_l2 : nullptr;
        if (timer) timer->start();
        kern<<<1, kSingleThreads, smem, s>>>(a);
        if (timer) timer->stop();
        g_launches.fetch_add(1, std::memory_order_relaxed);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(MAPI_ERR_CUDA, "single-CTA launch: %s", cudaGetErrorString(e));
        if (l2_done && w_l2) *l2_done = true;
        return MAPI_OK;
    }
    MAPI_CUDA(cudaMemsetAsync(W.bar, 0, 256, s));
    if (use_cluster(d, n)) {
        // K6r (A in registers) for n <= 512 unless MAPI_DENSE_PATH=cluster_smem; K6 (A in shared memory) above
        const bool reg = n <= 512 && strcmp(dense_path_env(), "cluster_smem") != 0;
        using KernT = void (*)(IterArgs);
        KernT kern;
        if (reg) {
            kern = n <= 256 ? (op == 2 ? k_iterate_cluster_reg<2, 1> : (op == 1 ? k_iterate_cluster_reg<1, 1> : k_iterate_cluster_reg<0, 1>))
                            : (op == 2 ? k_iterate_cluster_reg<2, 2> : (op == 1 ? k_iterate_cluster_reg<1, 2> : k_iterate_cluster_reg<0, 2>));
        } else {
            kern = op == 2 ? k_iterate_cluster<2> : (op == 1 ? k_iterate_cluster<1> : k_iterate_cluster<0>);
        }
        const size_t smem = reg ? 0 : cluster_smem_bytes(n);
        if (!reg) MAPI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        IterArgs a;
        a.A = A; a.n = n; a.lda = lda; a.b0 = b0; a.iters = iters; a.tol = tol;
        a.w_out = w_out; a.norms = norms; a.deltas = deltas; a.y = W.y; a.slots = W.slots;
        a.bar = W.bar; a.status = W.status;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kClusterCtas);
        cfg.blockDim = dim3(kClusterThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kClusterCtas;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (timer) timer->start();
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
        if (timer) timer->stop();
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (e != cudaSuccess) return fail(MAPI_ERR_CUDA, "cluster launch (smem %zu): %s", smem, cudaGetErrorString(e));
        return MAPI_OK;
    }
    if (use_coop(d, A, n, lda)) {
        mapi_status st = MAPI_OK;
        auto launch = [&](auto kern, int nw) {
            const int threads = nw * 32;
            // 1 CTA per SM (shared memory holds w); grid <= n so every CTA owns >= 1 row
            const int grid = (int)std::min<int64_t>({(int64_t)d.sms, n, (int64_t)kMaxGrid});
            const size_t smem = coop_smem_bytes(n, grid, nw);
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int occ = 0;
            if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
            if (e != cudaSuccess || occ < 1) {
                st = fail(MAPI_ERR_CUDA, "coop kernel occupancy query failed: %s", cudaGetErrorString(e));
                return 0;
            }
            IterArgs a;
            a.A = A; a.n = n; a.lda = lda; a.b0 = b0; a.iters = iters; a.tol = tol;
            a.w_out = w_out; a.norms = norms; a.deltas = deltas; a.y = W.y; a.slots = W.slots;
            a.bar = W.bar; a.status = W.status;
            void* args[] = {&a};
            if (timer) timer->start();
            e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(threads), args, smem, s);
            if (timer) timer->stop();
            g_launches.fetch_add(1, std::memory_order_relaxed);
            if (e != cudaSuccess)
                st = fail(MAPI_ERR_CUDA, "cooperative launch (grid %d, smem %zu): %s", grid, smem,
                          cudaGetErrorString(e));
            return 0;
        };
        const int nw = coop_warps(n);
        with_op(op, [&](auto OPc) {
            return with_pol(pol, [&](auto POLc) {
                constexpr int OP = decltype(OPc)::value, POL = decltype(POLc)::value;
                return nw == 32 ? launch(k_iterate_coop<OP, POL, 32>, 32) : launch(k_iterate_coop<OP, POL, 16>, 16);
            });
        });
        return st;
    }
    if (use_resident(d, n)) {
        const int grid = (int)std::min<int64_t>(d.sms, n);
        // tagged y words: a tag never matches zeroed memory (tags are t + 1), so each call starts clean
        MAPI_CUDA(cudaMemsetAsync(W.y, 0, sizeof(uint64_t) * 2 * (size_t)n, s));
        // 8 warps with 2 register-resident rows per warp group (4 of the CTA's <= 28 rows in registers, 16 in
        // TMEM, 8 in shared memory); 16 warps (MAPI_RES_NW=16) have no register room for rows
        const int nw = resident_warps();
        const size_t smem = resident_smem_bytes(nw == 8 ? kResSmemRows - 2 * 2 : kResSmemRows);
        using KernT = void (*)(IterArgs);
        KernT kern = nw == 8 ? (op == 2 ? k_iterate_resident<2, 8, 1, 2>
                                        : (op == 1 ? k_iterate_resident<1, 8, 1, 2> : k_iterate_resident<0, 8, 1, 2>))
                             : (op == 2 ? k_iterate_resident<2, 16, 1, 0>
                                        : (op == 1 ? k_iterate_resident<1, 16, 1, 0> : k_iterate_resident<0, 16, 1, 0>));
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(MAPI_ERR_CUDA, "resident kernel smem (%zu): %s", smem, cudaGetErrorString(e));
        IterArgs a;
        a.A = A; a.n = n; a.lda = lda; a.b0 = b0; a.iters = iters; a.tol = tol;
        a.w_out = w_out; a.norms = norms; a.deltas = deltas; a.y = W.y; a.slots = W.slots;
        a.bar = W.bar; a.status = W.status;
        a.dP = dP; a.dR = dR; a.dk = dk;
        void* args[] = {&a};
        if (timer) timer->start();
        e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(nw * 32), args, smem, s);
        if (timer) timer->stop();
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (e != cudaSuccess)
            return fail(MAPI_ERR_CUDA, "resident cooperative launch (grid %d, smem %zu): %s", grid, smem,
                        cudaGetErrorString(e));
        return MAPI_OK;
    }
    if (use_bulk(d, A, n, lda)) {
        const int slots = bulk_slots(d, n);
        const int grid = (int)std::min<int64_t>(d.sms, n);
        const size_t smem = bulk_fixed_smem(n, (n + grid - 1) / grid) + sizeof(float) * kBulkChunk * (size_t)slots;
        auto kern = op == 2 ? k_iterate_bulk<2> : (op == 1 ? k_iterate_bulk<1> : k_iterate_bulk<0>);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(MAPI_ERR_CUDA, "bulk kernel smem (%zu): %s", smem, cudaGetErrorString(e));
        IterArgs a;
        a.A = A; a.n = n; a.lda = lda; a.b0 = b0; a.iters = iters; a.tol = tol;
        a.w_out = w_out; a.norms = norms; a.deltas = deltas; a.y = W.y; a.slots = W.slots;
        a.bar = W.bar; a.status = W.status;
        int sl = slots;
        void* args[] = {&a, &sl};
        if (timer) timer->start();
        e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kBulkThreads), args, smem, s);
        if (timer) timer->stop();
        g_launches.fetch_add(1, std::memory_order_relaxed);
        if (e != cudaSuccess)
            return fail(MAPI_ERR_CUDA, "bulk cooperative launch (grid %d, smem %zu): %s", grid, smem,
                        cudaGetErrorString(e));
        return MAPI_OK;
    }
    if (use_persistent(d, n)) {
        mapi_status st = MAPI_OK;
        with_op(op, [&](auto OPc) {
            return with_vec(vec, [&](auto VECc) {
                return with_pol(pol, [&](auto POLc) {
                    constexpr int OP = decltype(OPc)::value, VEC = decltype(VECc)::value,
                                  POL = decltype(POLc)::value;
                    // mid-size n (< 8192; the matrix is L2-resident and the loop latency-bound): 16 B loads,
                    // 8 in flight per lane (measured 11.3 vs 13.0 us/iteration at n = 4096 for the
                    // default; profiles/r01_probe_dense_mid.log)
                    const bool mid = VEC >= 4 && n < 8192;
                    auto kern = mid ? k_iterate_persistent<OP, (VEC >= 4 ? 4 : VEC), POL, 8, 0, 0, 1>
                                    : k_iterate_persistent<OP, VEC, POL, unroll_for(VEC)>;
                    const size_t smem = persistent_smem_bytes(n);
                    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)smem);
                    int occ = 0;
                    if (e == cudaSuccess)
                        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kIterThreads, smem);
                    if (e != cudaSuccess || occ < 1) {
                        st = fail(MAPI_ERR_CUDA, "persistent kernel occupancy query failed: %s",
                                  cudaGetErrorString(e));
                        return 0;
                    }
                    int64_t want = (n + (kIterThreads / 32) - 1) / (kIterThreads / 32);
                    int grid = (int)std::min<int64_t>({(int64_t)occ * d.sms, want, (int64_t)kMaxGrid});
                    grid = std::max(grid, 1);
                    IterArgs a;
                    a.A = A; a.n = n; a.lda = lda; a.b0 = b0; a.iters = iters; a.tol = tol;
                    a.w_out = w_out; a.norms = norms; a.deltas = deltas; a.y = W.y; a.slots = W.slots;
                    a.bar = W.bar; a.status = W.status;
                    void* args[] = {&a};
                    if (timer) timer->start();
                    e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kIterThreads), args,
                                                    smem, s);
                    if (timer) timer->stop();
                    g_launches.fetch_add(1, std::memory_order_relaxed);
                    if (e != cudaSuccess)
                        st = fail(MAPI_ERR_CUDA, "cooperative launch (grid %d, smem %zu): %s", grid, smem,
                                  cudaGetErrorString(e));
                    return 0;
                });
            });
        });
        return st;
    }
    // multi-launch path
    MAPI_CUDA(cudaMemcpyAsync(W.w, b0, sizeof(float) * (size_t)n, cudaMemcpyDeviceToDevice, s));
    mapi_status st = MAPI_OK;
    if (timer) timer->start();
    with_op(op, [&](auto OPc) {
        return with_vec(vec_width(A, lda) == 8 ? 8 : (vec_width(A, lda) == 4 ? 4 : 1), [&](auto VECc) {
            return with_pol(pol, [&](auto POLc) {
                constexpr int OP = decltype(OPc)::value, VEC = decltype(VECc)::value,
                              POL = decltype(POLc)::value;
                auto kern = k_rows_partial<OP, VEC, POL, unroll_for(VEC)>;
                int occ = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kIterThreads, 0);
                int64_t want = (n + 15) / 16;
                int grid = (int)std::min<int64_t>({(int64_t)std::max(occ, 1) * d.sms, want, (int64_t)kMaxGrid});
                grid = std::max(grid, 1);
                for (int32_t t = 0; t < iters && st == MAPI_OK; ++t) {
                    kern<<<grid, kIterThreads, 0, s>>>(A, n, lda, W.w, W.y, W.slots, W.stop);
                    g_launches.fetch_add(1, std::memory_order_relaxed);
                    k_normalize<<<1, 1024, 0, s>>>(n, W.y, W.slots, grid, W.w, t, tol, norms, deltas,
                                                   W.status, W.stop, OP == 2 ? 1 : 0);
                    g_launches.fetch_add(1, std::memory_order_relaxed);
                    cudaError_t e = cudaGetLastError();
                    if (e != cudaSuccess) st = fail(MAPI_ERR_CUDA, "launch: %s", cudaGetErrorString(e));
                }
                return 0;
            });
        });
    });
    if (timer) timer->stop();
    if (st != MAPI_OK) return st;
    MAPI_CUDA(cudaMemcpyAsync(w_out, W.w, sizeof(float) * (size_t)n, cudaMemcpyDeviceToDevice, s));
    return MAPI_OK;
}

// the two status words come back through a per-thread PINNED buffer (a DMA straight into host memory;
// a pageable destination goes through a staging copy and costs several microseconds more per call)
mapi_status read_status(const IterWs& W, cudaStream_t s, int32_t* iters_done) {
    static thread_local int32_t* pinned = nullptr;
    if (!pinned && cudaHostAlloc(reinterpret_cast<void**>(&pinned), 2 * sizeof(int32_t), cudaHostAllocDefault) != cudaSuccess) {
        pinned = nullptr;
        cudaGetLastError();
    }
    int32_t local[2] = {0, 0};
    int32_t* h = pinned ? pinned : local;
    MAPI_CUDA(cudaMemcpyAsync(h, W.status, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    if (iters_done) *iters_done = h[1];
    if (h[0] == MAPI_ERR_DEGENERATE)
        return fail(MAPI_ERR_DEGENERATE, "||A (+) w_t||_1 == 0 at iteration %d", h[1]);
    if (h[0] == MAPI_ERR_NONFINITE)
        return fail(MAPI_ERR_NONFINITE, "||A (+) w_t||_1 is not finite at iteration %d", h[1]);
    return MAPI_OK;
}

mapi_status validate_dense(int32_t op, const float* A, int64_t n, int64_t lda, const float* b0,
                           int32_t iters, float tol, const float* w_out, void* ws, bool dot_ok = true) {
    mapi_status st = check_op(op, dot_ok);
    if (st != MAPI_OK) return st;
    if (!A) return fail(MAPI_ERR_NULL, "A is NULL");
    if (!b0) return fail(MAPI_ERR_NULL, "b0 is NULL");
    if (!w_out) return fail(MAPI_ERR_NULL, "w_out is NULL");
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    if (n < 1) return fail(MAPI_ERR_SHAPE, "n (%lld) must be >= 1", (long long)n);
    if (lda < n) return fail(MAPI_ERR_SHAPE, "lda (%lld) < n (%lld)", (long long)lda, (long long)n);
    if (iters < 1) return fail(MAPI_ERR_BAD_PARAM, "iters (%d) must be >= 1", iters);
    if (!(tol >= 0.0f)) return fail(MAPI_ERR_BAD_PARAM, "tol (%g) must be >= 0", (double)tol);
    return MAPI_OK;
}

// ---------------------------------------------------------------------------------------------
// K9 outer-product operator: workspace [idx r*M i32][a r*M f32][s r*M f32][part r*NB*q*4 f64][Xc M*N f32]
size_t outer_ws_bytes(int64_t M, int64_t q, int64_t r, int64_t N) {
    return 3 * align256(sizeof(int32_t) * (size_t)(r * M)) +
           align256(sizeof(double) * 4 * (size_t)r * (size_t)outer_blocks(M) * (size_t)q) +
           align256(sizeof(float) * (size_t)M * (size_t)N);
}

// Y = [X -] (W (op) W^T) X [+ bias], r components in sequence (each pass in its own sorted row order)
mapi_status outer_run(int32_t op, const float* W, int64_t M, int64_t r, int64_t ldw, const float* X, int64_t q,
                      int64_t ldx, bool subtract, const float* bias, float* Y, int64_t ldy, char* ws, cudaStream_t s) {
    int32_t* idx = reinterpret_cast<int32_t*>(ws);
    ws += align256(sizeof(int32_t) * (size_t)(r * M));
    float* as = reinterpret_cast<float*>(ws);
    ws += align256(sizeof(float) * (size_t)(r * M));
    float* ss = reinterpret_cast<float*>(ws);
    ws += align256(sizeof(float) * (size_t)(r * M));
    double* part = reinterpret_cast<double*>(ws);
    int P = 1;
    while (P < M) P <<= 1;
    const size_t sort_smem = sizeof(unsigned long long) * (size_t)P;
    MAPI_CUDA(cudaFuncSetAttribute(k_outer_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sort_smem));
    k_outer_sort<<<(unsigned)r, 1024, sort_smem, s>>>(W, M, ldw, idx, as, ss);
    MAPI_LAUNCHED();
    const dim3 grid((unsigned)((q + kOuterThreads - 1) / kOuterThreads), (unsigned)outer_blocks(M));
    for (int c = 0; c < (int)r; ++c) {
        const int acc = c > 0, sub = (c == 0 && subtract) ? 1 : 0;
        const float* bb = (c == (int)r - 1) ? bias : nullptr;
        if (op == 1) {
            k_outer_blocksum<1><<<grid, kOuterThreads, 0, s>>>(X, M, q, ldx, idx, as, ss, c, part);
            k_outer_apply<1><<<grid, kOuterThreads, 0, s>>>(X, M, q, ldx, idx, as, ss, c, part, Y, ldy, acc, sub, bb);
        } else if (op == 2) {
            k_outer_blocksum<2><<<grid, kOuterThreads, 0, s>>>(X, M, q, ldx, idx, as, ss, c, part);
            k_outer_apply<2><<<grid, kOuterThreads, 0, s>>>(X, M, q, ldx, idx, as, ss, c, part, Y, ldy, acc, sub, bb);
        } else {
            k_outer_blocksum<0><<<grid, kOuterThreads, 0, s>>>(X, M, q, ldx, idx, as, ss, c, part);
            k_outer_apply<0><<<grid, kOuterThreads, 0, s>>>(X, M, q, ldx, idx, as, ss, c, part, Y, ldy, acc, sub, bb);
        }
        g_launches.fetch_add(1, std::memory_order_relaxed);
        MAPI_LAUNCHED();
    }
    return MAPI_OK;
}

}  // namespace

// =============================================================================================
extern "C" {

const char* mapi_status_string(mapi_status s) {
    switch (s) {
    case MAPI_OK: return "MAPI_OK";
    case MAPI_ERR_NULL: return "MAPI_ERR_NULL";
    case MAPI_ERR_SHAPE: return "MAPI_ERR_SHAPE";
    case MAPI_ERR_BAD_PARAM: return "MAPI_ERR_BAD_PARAM";
    case MAPI_ERR_DEGENERATE: return "MAPI_ERR_DEGENERATE";
    case MAPI_ERR_NEGATIVE: return "MAPI_ERR_NEGATIVE";
    case MAPI_ERR_NONFINITE: return "MAPI_ERR_NONFINITE";
    case MAPI_ERR_WORKSPACE: return "MAPI_ERR_WORKSPACE";
    case MAPI_ERR_CUDA: return "MAPI_ERR_CUDA";
    }
    return "MAPI_ERR_UNKNOWN";
}

const char* mapi_last_error_message(void) { return g_err; }
uint64_t mapi_launch_count(void) { return g_launches.load(); }
void mapi_set_profiling(int32_t enable) { g_profiling.store(enable ? 1 : 0); }
float mapi_last_kernel_ms(void) { return g_last_kernel_ms; }

// count independent host problems, pipelined: problem i+1's A / b0 host->device copies (a second, copy
// stream) overlap problem i's iterations (the compute stream); two device slots alternate.
// packed: each slot also holds the packed upper triangle (n(n+1)/2 floats) the host sends
// sym: symmetric problems (packed or upper-triangle copies) may run K2s, which needs its partial buffers
size_t iterate_host_many_ws_bytes(int64_t n, int64_t lda, int32_t iters, int32_t count, bool packed = false,
                                  bool sym = false) {
    const size_t slot = align256(sizeof(float) * (size_t)n * (size_t)lda) + 2 * align256(sizeof(float) * (size_t)n) +
                        2 * align256(sizeof(float) * (size_t)std::max(iters, 1)) +
                        (packed ? align256(sizeof(float) * (size_t)packed_floats(n)) : 0);
    return iterate_ws_bytes(n) + 2 * slot + sizeof(int32_t) * 2 * (size_t)std::max(count, 2) +
           ((packed || sym) ? 256 + align256(sym_partials_bytes(n)) : 0);  // (+256: alignment of the partials)
}
// device leading dimension of the unpacked matrix: 32 B-aligned rows (the 256-bit load path)
inline int64_t packed_lda(int64_t n) { return (n + 7) & ~int64_t(7); }

size_t mapi_workspace_size(int32_t op, int64_t n, int64_t nnz, int32_t k) {
    if (n < 0) n = 0;
    if (nnz < 0) nnz = 0;
    if (k < 0) k = 0;
    switch (op) {
    case MAPI_WS_MATVEC: return 0;
    case MAPI_WS_ITERATE: return iterate_ws_bytes(n);
    case MAPI_WS_ITERATE_HOST:  // nnz = lda, k = iters
        return iterate_ws_bytes(n) + align256(sizeof(float) * (size_t)n * (size_t)nnz) +
               4 * align256(sizeof(float) * (size_t)n) + 2 * align256(sizeof(float) * (size_t)k);
    case MAPI_WS_PCA_TOPK:
        return iterate_ws_bytes(n) + align256(sizeof(float) * (size_t)n * (size_t)n) +
               2 * align256(sizeof(double) * (size_t)k * (size_t)n) +
               align256(sizeof(double) * 64 * (size_t)n) + align256(sizeof(float) * (size_t)n) +
               align256(sizeof(int32_t) * 2 * (size_t)k);
    case MAPI_WS_ITERATE_BATCHED: return batched_ws_bytes(n, k);
    case MAPI_WS_MAVP_DEFLATE: return outer_ws_bytes(n, n, 1, 0);
    case MAPI_WS_RECONSTRUCT: return outer_ws_bytes(n, nnz, k, nnz);
    case MAPI_WS_CSR_PREPARE: return csr_prepare_ws_bytes(n, nnz);
    case MAPI_WS_RANK_CSR: return csr_rank_ws_bytes(n, nnz);
    case MAPI_WS_ITERATE_SHARDED: return sharded_ws_bytes();
    case MAPI_WS_ITERATE_HOST_MANY: return iterate_host_many_ws_bytes(n, nnz, k, 2);
    case MAPI_WS_ITERATE_HOST_MANY_PACKED: return iterate_host_many_ws_bytes(n, packed_lda(n), k, 2, true);
    case MAPI_WS_ITERATE_HOST_MANY_SYM: return iterate_host_many_ws_bytes(n, packed_lda(n), k, 2, false, true);
    case MAPI_WS_ITERATE_SYM: return iterate_ws_bytes(n) + align256(sym_partials_bytes(n));
    case MAPI_WS_CSR_REORDER: return reorder_ws_bytes(n);
    case MAPI_WS_CSR_PLAN: return mapi_plan::plan_bytes_bound(n, nnz);
    case MAPI_WS_CSR_PLAN_BUILD: return mapi_plan::plan_build_ws_bytes(n, nnz);
    case MAPI_WS_RANK_CSR_PLAN: return mapi_plan::rank_plan_ws_bytes(n, nnz);
    case MAPI_WS_MINIBATCH: return mapi_mb::minibatch_ws_bytes(n, nnz, k);  // n = D, nnz = s, k = T
    case MAPI_WS_RANK_CSR_SHARD: return csr_rank_ws_bytes(n, nnz, k);  // n nodes, nnz = local edges, k = m
    }
    return 0;
}

mapi_status mapi_mavp_matvec(int32_t op, const float* A, int64_t n_rows, int64_t n_cols, int64_t lda,
                             const float* x, float* y, mapi_stream_t stream) {
    mapi_status st = check_op(op, true);
    if (st != MAPI_OK) return st;
    if (n_rows < 0 || n_cols < 0)
        return fail(MAPI_ERR_SHAPE, "negative size: n_rows %lld, n_cols %lld", (long long)n_rows,
                    (long long)n_cols);
    if (lda < n_cols) return fail(MAPI_ERR_SHAPE, "lda (%lld) < n_cols (%lld)", (long long)lda, (long long)n_cols);
    if (n_rows == 0) return MAPI_OK;
    if (!y) return fail(MAPI_ERR_NULL, "y is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n_cols == 0) {
        MAPI_CUDA(cudaMemsetAsync(y, 0, sizeof(float) * (size_t)n_rows, s));
        return MAPI_OK;
    }
    if (!A) return fail(MAPI_ERR_NULL, "A is NULL");
    if (!x) return fail(MAPI_ERR_NULL, "x is NULL");
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    const size_t smem_x = sizeof(float) * (size_t)n_cols;
    const bool x_in_smem = smem_x <= 200 * 1024;
    int vec = vec_width(A, lda);
    if (!x_in_smem) vec = std::min(vec, vec_width(x, 0));
    const int pol = load_policy(d, n_rows, lda);
    with_op(op, [&](auto OPc) {
        return with_vec(vec, [&](auto VECc) {
            return with_pol(pol, [&](auto POLc) {
                constexpr int OP = decltype(OPc)::value, VEC = decltype(VECc)::value,
                              POL = decltype(POLc)::value;
                auto run = [&](auto kern, size_t smem) {
                    cudaError_t e = cudaSuccess;
                    if (smem > 48 * 1024)
                        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    int occ = 1;
                    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, smem);
                    if (e != cudaSuccess) {
                        st = fail(MAPI_ERR_CUDA, "matvec setup: %s", cudaGetErrorString(e));
                        return 0;
                    }
                    int64_t want = (n_rows + 15) / 16;
                    int grid = (int)std::min<int64_t>((int64_t)std::max(occ, 1) * d.sms, want);
                    kern<<<std::max(grid, 1), 512, smem, s>>>(A, n_rows, n_cols, lda, x, y);
                    g_launches.fetch_add(1, std::memory_order_relaxed);
                    e = cudaGetLastError();
                    if (e != cudaSuccess) st = fail(MAPI_ERR_CUDA, "matvec launch: %s", cudaGetErrorString(e));
                    return 0;
                };
                if (x_in_smem)
                    return run(k_matvec<OP, VEC, POL, false, unroll_for(VEC)>, smem_x);
                return run(k_matvec<OP, VEC, POL, true, unroll_for(VEC)>, (size_t)0);
            });
        });
    });
    return st;
}

mapi_status mapi_mavp_matmat(int32_t op, const float* A, int64_t m, int64_t K, int64_t lda, const float* B,
                             int64_t p, int64_t ldb, float divisor, float* C, int64_t ldc, mapi_stream_t stream) {
    mapi_status st = check_op(op);
    if (st != MAPI_OK) return st;
    if (m < 0 || K < 0 || p < 0)
        return fail(MAPI_ERR_SHAPE, "negative size: m %lld, K %lld, p %lld", (long long)m, (long long)K, (long long)p);
    if (lda < K) return fail(MAPI_ERR_SHAPE, "lda (%lld) < K (%lld)", (long long)lda, (long long)K);
    if (ldb < K) return fail(MAPI_ERR_SHAPE, "ldb (%lld) < K (%lld)", (long long)ldb, (long long)K);
    if (ldc < p) return fail(MAPI_ERR_SHAPE, "ldc (%lld) < p (%lld)", (long long)ldc, (long long)p);
    if (!(divisor > 0.0f) || isinf(divisor))
        return fail(MAPI_ERR_BAD_PARAM, "divisor (%g) must be finite and > 0", (double)divisor);
    if (m == 0 || p == 0) return MAPI_OK;
    if (!C) return fail(MAPI_ERR_NULL, "C is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (K == 0) {
        MAPI_CUDA(cudaMemset2DAsync(C, sizeof(float) * (size_t)ldc, 0, sizeof(float) * (size_t)p, (size_t)m, s));
        return MAPI_OK;
    }
    if (!A || !B) return fail(MAPI_ERR_NULL, "A or B is NULL");
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    const char* mp = getenv("MAPI_MATMAT_PATH");  // "tiled" forces K8 for small K (tests / comparison)
    if (K <= 12 && !(mp && strcmp(mp, "tiled") == 0)) {
        using KernT = void (*)(const float*, int64_t, int, int64_t, const float*, int64_t, int64_t, float, float*,
                               int64_t);
        KernT kern = K <= 4 ? (op == 1 ? k_mavp_matmat_smallk<1, 4> : k_mavp_matmat_smallk<0, 4>)
                   : K <= 8 ? (op == 1 ? k_mavp_matmat_smallk<1, 8> : k_mavp_matmat_smallk<0, 8>)
                            : (op == 1 ? k_mavp_matmat_smallk<1, 12> : k_mavp_matmat_smallk<0, 12>);
        int occ = 1;
        MAPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kMsThreads, 0));
        const int64_t units = ((m + kMsI - 1) / kMsI) * ((p + kMsJ - 1) / kMsJ);
        const unsigned grid = (unsigned)std::min<int64_t>(units, (int64_t)std::max(occ, 1) * d.sms);
        Timer timer(s);
        timer.start();
        kern<<<grid, kMsThreads, 0, s>>>(A, m, (int)K, lda, B, p, ldb, divisor, C, ldc);
        timer.stop();
        MAPI_LAUNCHED();
        if (timer.on) {
            MAPI_CUDA(cudaStreamSynchronize(s));
            timer.harvest();
        }
        return MAPI_OK;
    }
    const bool async = reinterpret_cast<uintptr_t>(A) % 16 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0 &&
                       lda % 4 == 0 && ldb % 4 == 0 && K % 4 == 0;  // 16 B chunks never cross K
    const int64_t ntiles = ((p + kMmJ - 1) / kMmJ) * ((m + kMmI - 1) / kMmI);
    const size_t smem = matmat_smem_bytes();
    auto kern = op == 1 ? (async ? k_mavp_matmat<1, true> : k_mavp_matmat<1, false>)
                        : (async ? k_mavp_matmat<0, true> : k_mavp_matmat<0, false>);
    MAPI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 1;
    MAPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kMmThreads, smem));
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)std::max(occ, 1) * d.sms);
    Timer timer(s);
    timer.start();
    kern<<<grid, kMmThreads, smem, s>>>(A, m, K, lda, B, p, ldb, divisor, C, ldc);
    timer.stop();
    MAPI_LAUNCHED();
    if (timer.on) {
        MAPI_CUDA(cudaStreamSynchronize(s));
        timer.harvest();
    }
    return MAPI_OK;
}

mapi_status mapi_iterate(int32_t op, const float* A, int64_t n, int64_t lda, const float* b0, int32_t iters,
                         float tol, float* w_out, float* w_l2_out, float* norms, float* deltas,
                         int32_t* iters_done, void* ws, size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = validate_dense(op, A, n, lda, b0, iters, tol, w_out, ws);
    if (st != MAPI_OK) return st;
    if (ws_bytes < iterate_ws_bytes(n))
        return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, iterate_ws_bytes(n));
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    IterWs W = carve_iterate(ws, n);
    Timer timer(s);
    bool l2_done = false;
    st = iterate_launch(d, op, A, n, lda, b0, iters, tol, w_out, norms, deltas, W, s, &timer, nullptr, nullptr, 0,
                        w_l2_out, &l2_done);
    if (st != MAPI_OK) return st;
    if (w_l2_out && !l2_done) {
        k_l2_copy<<<1, 1024, 0, s>>>(n, w_out, w_l2_out);
        MAPI_LAUNCHED();
    }
    st = read_status(W, s, iters_done);
    timer.harvest();
    return st;
}

// K2s for symmetric A (sym.cuh): only the upper triangle is read.  Used when the HBM read dominates
// (n >= 8192) and rows are 32 B-aligned; otherwise the full-matrix kernels run (same result up to the
// fp32 summation order).  MAPI_SYM_PATH=full forces the fallback (tests).
bool use_sym(const Device& d, const float* A, int64_t n, int64_t lda) {
    const char* e = getenv("MAPI_SYM_PATH");
    if (e && strcmp(e, "full") == 0) return false;
    if (n % 8 != 0 || lda % 8 != 0 || (reinterpret_cast<uintptr_t>(A) & 31) != 0) return false;
    if (sym_smem_bytes(n) > (size_t)d.smem_optin) return false;
    return n >= 8192 || (e && strcmp(e, "sym") == 0);
}

mapi_status sym_launch(const Device& d, int32_t op, const float* A, int64_t n, int64_t lda, const float* b0,
                       int32_t iters, float tol, float* w_out, float* norms, float* deltas, const IterWs& W,
                       float* partials, cudaStream_t s, Timer* timer) {
    MAPI_CUDA(cudaMemsetAsync(W.bar, 0, 256, s));
    using KernT = void (*)(SymArgs);
    KernT kern = op == 2 ? k_iterate_sym<2> : (op == 1 ? k_iterate_sym<1> : k_iterate_sym<0>);
    const size_t smem = sym_smem_bytes(n);
    MAPI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    MAPI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kSymThreads, smem));
    if (occ < 1) return fail(MAPI_ERR_CUDA, "symmetric kernel does not fit an SM (smem %zu)", smem);
    const int grid = (int)std::min<int64_t>({(int64_t)d.sms, n, (int64_t)kMaxGrid});
    SymArgs a;
    a.it.A = A; a.it.n = n; a.it.lda = lda; a.it.b0 = b0; a.it.iters = iters; a.it.tol = tol;
    a.it.w_out = w_out; a.it.norms = norms; a.it.deltas = deltas; a.it.y = W.y; a.it.slots = W.slots;
    a.it.bar = W.bar; a.it.status = W.status;
    a.prow = partials;
    a.pcol = partials + (size_t)sym_nc(n) * (size_t)((n + 31) & ~int64_t(31));  // row-tiled, whole tiles
    // the y region (2n doubles) holds the tagged w words of both parities, zeroed so no stale tag matches;
    // the w region holds y of the owned rows
    a.wtag = reinterpret_cast<unsigned long long*>(W.y);
    a.yg = W.w;
    {  // investigation switch; the default was chosen from the sweep in profiles/r02_probe_k2s_prefetch.log
        static const int pf = getenv("MAPI_SYM_PREFETCH") ? atoi(getenv("MAPI_SYM_PREFETCH")) : kSymPrefetchRows;
        a.prefetch_rows = std::max(0, std::min(pf, kSymRB));
    }
    MAPI_CUDA(cudaMemsetAsync(W.y, 0, sizeof(unsigned long long) * 2 * (size_t)n, s));
    void* args[] = {&a};
    if (timer) timer->start();
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kSymThreads), args, smem, s);
    if (timer) timer->stop();
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e != cudaSuccess)
        return fail(MAPI_ERR_CUDA, "symmetric cooperative launch (grid %d, smem %zu): %s", grid, smem, cudaGetErrorString(e));
    return MAPI_OK;
}

mapi_status mapi_iterate_sym(int32_t op, const float* A, int64_t n, int64_t lda, const float* b0, int32_t iters,
                             float tol, float* w_out, float* w_l2_out, float* norms, float* deltas,
                             int32_t* iters_done, void* ws, size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = validate_dense(op, A, n, lda, b0, iters, tol, w_out, ws);
    if (st != MAPI_OK) return st;
    const size_t need = mapi_workspace_size(MAPI_WS_ITERATE_SYM, n, 0, 0);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    IterWs W = carve_iterate(ws, n);
    float* partials = reinterpret_cast<float*>(static_cast<char*>(ws) + iterate_ws_bytes(n));
    Timer timer(s);
    st = use_sym(d, A, n, lda) ? sym_launch(d, op, A, n, lda, b0, iters, tol, w_out, norms, deltas, W, partials, s, &timer)
                               : iterate_launch(d, op, A, n, lda, b0, iters, tol, w_out, norms, deltas, W, s, &timer);
    if (st != MAPI_OK) return st;
    if (w_l2_out) {
        k_l2_copy<<<1, 1024, 0, s>>>(n, w_out, w_l2_out);
        MAPI_LAUNCHED();
    }
    st = read_status(W, s, iters_done);
    timer.harvest();
    return st;
}

mapi_status mapi_iterate_host(int32_t op, const float* A_host, int64_t n, int64_t lda, const float* b0_host,
                              int32_t iters, float tol, float* w_out_host, float* w_l2_out_host,
                              float* norms_host, float* deltas_host, int32_t* iters_done, void* ws,
                              size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = validate_dense(op, A_host, n, lda, b0_host, iters, tol, w_out_host, ws);
    if (st != MAPI_OK) return st;
    const size_t need = mapi_workspace_size(MAPI_WS_ITERATE_HOST, n, lda, iters);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* p = static_cast<char*>(ws);
    IterWs W = carve_iterate(p, n);
    p += iterate_ws_bytes(n);
    float* A = reinterpret_cast<float*>(p);
    p += align256(sizeof(float) * (size_t)n * (size_t)lda);
    float* b0 = reinterpret_cast<float*>(p);
    p += align256(sizeof(float) * (size_t)n);
    float* w = reinterpret_cast<float*>(p);
    p += align256(sizeof(float) * (size_t)n);
    float* wl2 = reinterpret_cast<float*>(p);
    p += 2 * align256(sizeof(float) * (size_t)n);
    float* nrm = reinterpret_cast<float*>(p);
    p += align256(sizeof(float) * (size_t)iters);
    float* dlt = reinterpret_cast<float*>(p);
    MAPI_CUDA(cudaMemcpyAsync(A, A_host, sizeof(float) * (size_t)n * (size_t)lda, cudaMemcpyHostToDevice, s));
    MAPI_CUDA(cudaMemcpyAsync(b0, b0_host, sizeof(float) * (size_t)n, cudaMemcpyHostToDevice, s));
    Timer timer(s);
    st = iterate_launch(d, op, A, n, lda, b0, iters, tol, w, nrm, dlt, W, s, &timer);
    if (st != MAPI_OK) return st;
    if (w_l2_out_host) {
        k_l2_copy<<<1, 1024, 0, s>>>(n, w, wl2);
        MAPI_LAUNCHED();
        MAPI_CUDA(cudaMemcpyAsync(w_l2_out_host, wl2, sizeof(float) * (size_t)n, cudaMemcpyDeviceToHost, s));
    }
    MAPI_CUDA(cudaMemcpyAsync(w_out_host, w, sizeof(float) * (size_t)n, cudaMemcpyDeviceToHost, s));
    if (norms_host)
        MAPI_CUDA(cudaMemcpyAsync(norms_host, nrm, sizeof(float) * (size_t)iters, cudaMemcpyDeviceToHost, s));
    if (deltas_host)
        MAPI_CUDA(cudaMemcpyAsync(deltas_host, dlt, sizeof(float) * (size_t)iters, cudaMemcpyDeviceToHost, s));
    st = read_status(W, s, iters_done);
    timer.harvest();
    return st;
}

// mode kFull: A_hosts[i] are full n x lda matrices, copied whole.  kPacked: packed upper triangles
// (n(n+1)/2 floats), unpacked on the device into an n x packed_lda(n) matrix.  kSymUpper: full symmetric
// n x lda host matrices of which only the upper-triangle block rows are copied (one 2-D copy per 128-row
// block: columns [128 b, n) of rows [128 b, 128 b + 128)) into an n x packed_lda(n) device matrix — what
// K2s reads, half the PCIe bytes, no host-side packing.
enum HostMode { kFull = 0, kPacked = 1, kSymUpper = 2 };
static mapi_status host_many_impl(int32_t op, int32_t count, const float* const* A_hosts, int64_t n, int64_t lda,
                                  const float* const* b0_hosts, int32_t iters, float tol, float* const* w_out_hosts,
                                  float* const* norms_hosts, float* const* deltas_hosts, int32_t* iters_done,
                                  void* ws, size_t ws_bytes, mapi_stream_t stream, HostMode mode) {
    if (count < 1) return fail(MAPI_ERR_BAD_PARAM, "count (%d) must be >= 1", count);
    if (!A_hosts || !b0_hosts || !w_out_hosts) return fail(MAPI_ERR_NULL, "A_hosts / b0_hosts / w_out_hosts is NULL");
    const bool packed = mode == kPacked;
    const int64_t lda_host = lda;
    if (mode != kFull) lda = packed_lda(n);
    for (int32_t i = 0; i < count; ++i) {
        mapi_status st = validate_dense(op, A_hosts[i], n, lda, b0_hosts[i], iters, tol, w_out_hosts[i], ws);
        if (st != MAPI_OK) return fail(st, "problem %d: %s", i, g_err);
    }
    if (mode == kSymUpper && lda_host < n)
        return fail(MAPI_ERR_SHAPE, "lda (%lld) < n (%lld)", (long long)lda_host, (long long)n);
    const size_t need = iterate_host_many_ws_bytes(n, lda, iters, count, mode == kPacked, mode == kSymUpper);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    mapi_status st = device_info(d);
    if (st != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* p = static_cast<char*>(ws);
    IterWs W = carve_iterate(p, n);
    p += iterate_ws_bytes(n);
    struct Slot {
        float *A, *b0, *w, *nrm, *dlt, *pk;
    } sl[2];
    for (auto& x : sl) {
        x.A = reinterpret_cast<float*>(p);
        p += align256(sizeof(float) * (size_t)n * (size_t)lda);
        x.pk = nullptr;
        if (packed) {
            x.pk = reinterpret_cast<float*>(p);
            p += align256(sizeof(float) * (size_t)packed_floats(n));
        }
        x.b0 = reinterpret_cast<float*>(p);
        p += align256(sizeof(float) * (size_t)n);
        x.w = reinterpret_cast<float*>(p);
        p += align256(sizeof(float) * (size_t)n);
        x.nrm = reinterpret_cast<float*>(p);
        p += align256(sizeof(float) * (size_t)std::max(iters, 1));
        x.dlt = reinterpret_cast<float*>(p);
        p += align256(sizeof(float) * (size_t)std::max(iters, 1));
    }
    int32_t* st_all = reinterpret_cast<int32_t*>(p);
    p += sizeof(int32_t) * 2 * (size_t)std::max(count, 2);
    // symmetric problems run K2s where it applies (both slots are 256 B-aligned: the same answer for each)
    const bool sym_k = mode != kFull && use_sym(d, sl[0].A, n, lda);
    // K2s partials (the packed input is symmetric), 256 B-aligned (float4 stores)
    float* sym_part = mode != kFull ? reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255)) : nullptr;
    cudaStream_t cs = nullptr;
    cudaEvent_t loaded[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
    auto cleanup = [&]() {
        for (int j = 0; j < 2; ++j) {
            if (loaded[j]) cudaEventDestroy(loaded[j]);
            if (freed[j]) cudaEventDestroy(freed[j]);
        }
        // an error may leave a queued H2D copy into ws on cs: drain it before the caller can reuse ws
        if (cs) {
            cudaStreamSynchronize(cs);
            cudaStreamDestroy(cs);
        }
    };
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    for (int j = 0; j < 2 && e == cudaSuccess; ++j) {
        e = cudaEventCreateWithFlags(&loaded[j], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&freed[j], cudaEventDisableTiming);
    }
    // the copy stream starts after everything already queued on the caller's stream
    if (e == cudaSuccess) e = cudaEventRecord(freed[1], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, freed[1], 0);
    if (e != cudaSuccess) {
        cleanup();
        return fail(MAPI_ERR_CUDA, "stream / event setup: %s", cudaGetErrorString(e));
    }
    Timer timer(s);
    timer.start();
    // copy of problem i into slot i & 1 on the copy stream, after problem i-2 released that slot
    auto issue_copy = [&](int32_t i) {
        Slot& x = sl[i & 1];
        cudaError_t r = cudaSuccess;
        if (i >= 2) r = cudaStreamWaitEvent(cs, freed[i & 1], 0);
        if (r == cudaSuccess) {
            if (mode == kPacked)
                r = cudaMemcpyAsync(x.pk, A_hosts[i], sizeof(float) * (size_t)packed_floats(n), cudaMemcpyHostToDevice,
                                    cs);
            else if (mode == kFull)
                r = cudaMemcpyAsync(x.A, A_hosts[i], sizeof(float) * (size_t)n * (size_t)lda, cudaMemcpyHostToDevice, cs);
            else if (!sym_k)  // the full-matrix kernels will run: the whole matrix
                r = cudaMemcpy2DAsync(x.A, sizeof(float) * (size_t)lda, A_hosts[i], sizeof(float) * (size_t)lda_host,
                                      sizeof(float) * (size_t)n, (size_t)n, cudaMemcpyHostToDevice, cs);
            else
                for (int64_t j0 = 0; j0 < n && r == cudaSuccess; j0 += kSymRB) {
                    const int64_t rows = std::min<int64_t>(kSymRB, n - j0);
                    r = cudaMemcpy2DAsync(x.A + j0 * lda + j0, sizeof(float) * (size_t)lda, A_hosts[i] + j0 * lda_host + j0,
                                          sizeof(float) * (size_t)lda_host, sizeof(float) * (size_t)(n - j0),
                                          (size_t)rows, cudaMemcpyHostToDevice, cs);
                }
        }
        if (r == cudaSuccess) r = cudaMemcpyAsync(x.b0, b0_hosts[i], sizeof(float) * (size_t)n, cudaMemcpyHostToDevice, cs);
        if (r == cudaSuccess) r = cudaEventRecord(loaded[i & 1], cs);
        return r;
    };
    e = issue_copy(0);
    for (int32_t i = 0; i < count && st == MAPI_OK && e == cudaSuccess; ++i) {
        Slot& x = sl[i & 1];
        e = cudaStreamWaitEvent(s, loaded[i & 1], 0);
        if (e != cudaSuccess) break;
        if (packed) {
            const int64_t nb = (n + kPackTile - 1) / kPackTile;
            const int64_t tiles = nb * (nb + 1) / 2;
            k_unpack_sym<<<(unsigned)std::min<int64_t>(tiles, (int64_t)d.sms * 8), 256, 0, s>>>(x.pk, n, x.A, lda);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            if ((e = cudaGetLastError()) != cudaSuccess) break;
        }
        st = sym_k
                 ? sym_launch(d, op, x.A, n, lda, x.b0, iters, tol, x.w, x.nrm, x.dlt, W, sym_part, s, nullptr)
                 : iterate_launch(d, op, x.A, n, lda, x.b0, iters, tol, x.w, x.nrm, x.dlt, W, s, nullptr);
        if (st != MAPI_OK) break;
        // queue the next problem's copy before this one's read-back (a pageable read-back may block the host)
        if (i + 1 < count && (e = issue_copy(i + 1)) != cudaSuccess) break;
        e = cudaMemcpyAsync(st_all + 2 * i, W.status, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(w_out_hosts[i], x.w, sizeof(float) * (size_t)n, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && norms_hosts && norms_hosts[i])
            e = cudaMemcpyAsync(norms_hosts[i], x.nrm, sizeof(float) * (size_t)iters, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && deltas_hosts && deltas_hosts[i])
            e = cudaMemcpyAsync(deltas_hosts[i], x.dlt, sizeof(float) * (size_t)iters, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(freed[i & 1], s);
    }
    timer.stop();
    if (e != cudaSuccess && st == MAPI_OK) st = fail(MAPI_ERR_CUDA, "pipelined host iterate: %s", cudaGetErrorString(e));
    std::vector<int32_t> h(2 * (size_t)count, 0);
    cudaError_t e2 = cudaMemcpyAsync(h.data(), st_all, sizeof(int32_t) * 2 * (size_t)count, cudaMemcpyDeviceToHost, s);
    if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(s);
    cleanup();
    if (st != MAPI_OK) return st;
    if (e2 != cudaSuccess) return fail(MAPI_ERR_CUDA, "status read-back: %s", cudaGetErrorString(e2));
    timer.harvest();
    for (int32_t i = 0; i < count; ++i) {
        if (iters_done) iters_done[i] = h[2 * i + 1];
        if (h[2 * i] != 0)
            return fail((mapi_status)h[2 * i], "problem %d: %s at iteration %d", i,
                        h[2 * i] == MAPI_ERR_DEGENERATE ? "||A (op) w||_1 == 0" : "non-finite norm", h[2 * i + 1]);
    }
    return MAPI_OK;
}

mapi_status mapi_iterate_host_many(int32_t op, int32_t count, const float* const* A_hosts, int64_t n, int64_t lda,
                                   const float* const* b0_hosts, int32_t iters, float tol, float* const* w_out_hosts,
                                   float* const* norms_hosts, float* const* deltas_hosts, int32_t* iters_done,
                                   void* ws, size_t ws_bytes, mapi_stream_t stream) {
    return host_many_impl(op, count, A_hosts, n, lda, b0_hosts, iters, tol, w_out_hosts, norms_hosts, deltas_hosts,
                          iters_done, ws, ws_bytes, stream, kFull);
}

mapi_status mapi_iterate_host_many_sym(int32_t op, int32_t count, const float* const* A_hosts, int64_t n, int64_t lda,
                                       const float* const* b0_hosts, int32_t iters, float tol,
                                       float* const* w_out_hosts, float* const* norms_hosts,
                                       float* const* deltas_hosts, int32_t* iters_done, void* ws, size_t ws_bytes,
                                       mapi_stream_t stream) {
    return host_many_impl(op, count, A_hosts, n, lda, b0_hosts, iters, tol, w_out_hosts, norms_hosts, deltas_hosts,
                          iters_done, ws, ws_bytes, stream, kSymUpper);
}

// LAPACK-style packed upper triangle of a host matrix (row j = A[j, j:]), `threads` host threads (0 = all
// hardware threads): pure data movement for mapi_iterate_host_many_packed callers
mapi_status mapi_pack_upper_host(const float* A, int64_t n, int64_t lda, float* out, int32_t threads) {
    if (!A || !out) return fail(MAPI_ERR_NULL, "A / out is NULL");
    if (n < 1 || lda < n) return fail(MAPI_ERR_SHAPE, "n (%lld) / lda (%lld)", (long long)n, (long long)lda);
    int T = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    T = (int)std::min<int64_t>(T, n);
    std::vector<std::thread> pool;
    // thread k takes rows with balanced element counts: cumulative count of rows < j is j n - j (j - 1) / 2
    auto start = [&](int k) {
        const double total = (double)n * (double)(n + 1) / 2.0, target = total * k / T;
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((double)mid * (double)n - (double)mid * (double)(mid - 1) / 2.0 >= target) hi = mid;
            else lo = mid + 1;
        }
        return lo;
    };
    for (int k = 0; k < T; ++k) {
        const int64_t j0 = start(k), j1 = start(k + 1);
        pool.emplace_back([=]() {
            for (int64_t j = j0; j < j1; ++j)
                memcpy(out + (j * n - j * (j - 1) / 2), A + j * lda + j, sizeof(float) * (size_t)(n - j));
        });
    }
    for (auto& th : pool) th.join();
    return MAPI_OK;
}

mapi_status mapi_iterate_host_many_packed(int32_t op, int32_t count, const float* const* Ap_hosts, int64_t n,
                                          const float* const* b0_hosts, int32_t iters, float tol,
                                          float* const* w_out_hosts, float* const* norms_hosts,
                                          float* const* deltas_hosts, int32_t* iters_done, void* ws, size_t ws_bytes,
                                          mapi_stream_t stream) {
    return host_many_impl(op, count, Ap_hosts, n, 0, b0_hosts, iters, tol, w_out_hosts, norms_hosts, deltas_hosts,
                          iters_done, ws, ws_bytes, stream, kPacked);
}

mapi_status mapi_pca_topk(int32_t op, const float* C, int64_t n, int64_t ldc, int32_t k, int32_t iters,
                          const float* b0, float* P_out, float* norms, float* deltas, void* ws,
                          size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = validate_dense(op, C, n, ldc, b0, iters, 0.0f, P_out, ws);
    if (st != MAPI_OK) return st;
    if (k < 1 || k > n) return fail(MAPI_ERR_BAD_PARAM, "k (%d) must be in [1, n = %lld]", k, (long long)n);
    const size_t need = mapi_workspace_size(MAPI_WS_PCA_TOPK, n, 0, k);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* p = static_cast<char*>(ws);
    IterWs W = carve_iterate(p, n);
    p += iterate_ws_bytes(n);
    float* D = reinterpret_cast<float*>(p);
    p += align256(sizeof(float) * (size_t)n * (size_t)n);
    double* P64 = reinterpret_cast<double*>(p);
    p += align256(sizeof(double) * (size_t)k * (size_t)n);
    double* R = reinterpret_cast<double*>(p);
    p += align256(sizeof(double) * (size_t)k * (size_t)n);
    double* part = reinterpret_cast<double*>(p);
    p += align256(sizeof(double) * 64 * (size_t)n);
    float* wtmp = reinterpret_cast<float*>(p);
    p += align256(sizeof(float) * (size_t)n);
    int32_t* st_all = reinterpret_cast<int32_t*>(p);  // per-vector (status, iters_done), read back once
    const int S = (int)std::min<int64_t>(64, n);
    const int64_t rows_per = (n + S - 1) / S;
    std::vector<std::unique_ptr<Timer>> timers;
    for (int32_t i = 0; i < k; ++i) {
        const float* Ai = C;
        int64_t ld = ldc;
        // MAPI_PCA_FUSE=1: K2r stages D_i itself from C, P and R (bitwise the k_build_deflated result), no
        // D_i round trip through memory.  Measured slower at cfg2 (190k vs 193k it/s: the staging runs at 8
        // warps per SM inside the persistent kernel, the separate build at full occupancy), so the separate
        // build stays the default; tests compare the two bitwise.
        const char* fe = getenv("MAPI_PCA_FUSE");
        const bool fuse = i > 0 && i <= kResDeflMax && use_resident(d, n) && resident_warps() == 8 && fe &&
                          fe[0] == '1';
        if (i > 0 && !fuse) {
            const int gx = (int)std::min<int64_t>((n + 255) / 256, 65535);
            const int gy = (int)std::min<int64_t>(n, 65535);
            const bool v4 = i <= 8 && n % 4 == 0 && ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
            if (v4) {
                const dim3 g((unsigned)((n / 4 + 255) / 256), (unsigned)((n + kDeflRows - 1) / kDeflRows));
                switch (i) {
                    case 1: k_build_deflated_v4<1><<<g, 256, 0, s>>>(C, n, ldc, P64, R, D); break;
                    case 2: k_build_deflated_v4<2><<<g, 256, 0, s>>>(C, n, ldc, P64, R, D); break;
                    case 3: k_build_deflated_v4<3><<<g, 256, 0, s>>>(C, n, ldc, P64, R, D); break;
                    case 4: k_build_deflated_v4<4><<<g, 256, 0, s>>>(C, n, ldc, P64, R, D); break;
                    case 5: k_build_deflated_v4<5><<<g, 256, 0, s>>>(C, n, ldc, P64, R, D); break;
                    case 6: k_build_deflated_v4<6><<<g, 256, 0, s>>>(C, n, ldc, P64, R, D); break;
                    case 7: k_build_deflated_v4<7><<<g, 256, 0, s>>>(C, n, ldc, P64, R, D); break;
                    default: k_build_deflated_v4<8><<<g, 256, 0, s>>>(C, n, ldc, P64, R, D); break;
                }
            } else {
                k_build_deflated<<<dim3(gx, gy), 256, 0, s>>>(C, n, ldc, P64, R, i, D);
            }
            MAPI_LAUNCHED();
            Ai = D;
            ld = n;
        }
        // no host round trip per vector: each vector's status words are copied aside on the stream and
        // read back once after the last vector (a degenerate vector still reports its index)
        timers.emplace_back(new Timer(s));
        st = iterate_launch(d, op, Ai, n, ld, b0, iters, 0.0f, wtmp, norms ? norms + (int64_t)i * iters : nullptr,
                            deltas ? deltas + (int64_t)i * iters : nullptr, W, s, timers.back().get(),
                            fuse ? P64 : nullptr, fuse ? R : nullptr, fuse ? i : 0);
        if (st != MAPI_OK) return st;
        MAPI_CUDA(cudaMemcpyAsync(st_all + 2 * i, W.status, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        k_l2_to_p<<<1, 1024, 0, s>>>(n, wtmp, P64 + (int64_t)i * n, P_out + (int64_t)i * n);
        MAPI_LAUNCHED();
        if (i + 1 < k) {
            k_colsum_partial<<<dim3((unsigned)((n + 255) / 256), S), 256, 0, s>>>(C, n, ldc, P64 + (int64_t)i * n,
                                                                               part, rows_per);
            MAPI_LAUNCHED();
            k_colsum_final<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, S, part, R + (int64_t)i * n);
            MAPI_LAUNCHED();
        }
    }
    std::vector<int32_t> h(2 * (size_t)k, 0);
    MAPI_CUDA(cudaMemcpyAsync(h.data(), st_all, sizeof(int32_t) * 2 * (size_t)k, cudaMemcpyDeviceToHost, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    float total_ms = 0.0f;
    for (auto& t : timers) {
        t->harvest();
        total_ms += g_last_kernel_ms;
    }
    if (g_profiling.load()) g_last_kernel_ms = total_ms;
    for (int32_t i = 0; i < k; ++i) {
        if (h[2 * i] == MAPI_ERR_DEGENERATE)
            return fail(MAPI_ERR_DEGENERATE, "vector %d: ||A (+) w_t||_1 == 0 at iteration %d", i, h[2 * i + 1]);
        if (h[2 * i] == MAPI_ERR_NONFINITE)
            return fail(MAPI_ERR_NONFINITE, "vector %d: ||A (+) w_t||_1 is not finite at iteration %d", i, h[2 * i + 1]);
    }
    return MAPI_OK;
}

mapi_status mapi_iterate_batched(int32_t op, const float* A, int64_t n, int64_t lda, const float* B0, int32_t k,
                                 int32_t iters, float tol, float* W_out, float* norms, float* deltas,
                                 int32_t* iters_done, void* ws, size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = validate_dense(op, A, n, lda, B0, iters, tol, W_out, ws);
    if (st != MAPI_OK) return st;
    if (k < 1) return fail(MAPI_ERR_BAD_PARAM, "k (%d) must be >= 1", k);
    const size_t need = batched_ws_bytes(n, k);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Timer timer(s);
    st = batched_run(op, A, n, lda, B0, k, iters, tol, W_out, norms, deltas, ws, d.sms, s, &timer.a, &timer.b,
                     timer.on, g_launches);
    if (st != MAPI_OK) return fail(st, "%s", batched_last_error());
    int32_t bad = -1, bad_iter = 0;
    st = batched_finish(ws, n, k, s, iters_done, &bad, &bad_iter);
    timer.harvest();
    if (st == MAPI_ERR_CUDA) return fail(st, "%s", batched_last_error());
    if (st != MAPI_OK)
        return fail(st, "vector %d (the first of the k that stopped on an error): %s at iteration %d", bad,
                    st == MAPI_ERR_DEGENERATE ? "||A (+) w_t||_1 == 0" : "||A (+) w_t||_1 is not finite", bad_iter);
    return MAPI_OK;
}

mapi_status mapi_csr_prepare(int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* col_idx, float alpha,
                             float* cap_out, float* bg_out, void* ws, size_t ws_bytes, mapi_stream_t stream) {
    if (n < 1) return fail(MAPI_ERR_SHAPE, "n (%lld) must be >= 1", (long long)n);
    if (nnz < 0 || nnz >= (int64_t)INT32_MAX)
        return fail(MAPI_ERR_SHAPE, "nnz (%lld) must be in [0, 2^31)", (long long)nnz);
    if (n >= (int64_t)INT32_MAX) return fail(MAPI_ERR_SHAPE, "n (%lld) must be < 2^31", (long long)n);
    if (!row_ptr || (nnz > 0 && !col_idx)) return fail(MAPI_ERR_NULL, "row_ptr/col_idx is NULL");
    if (!cap_out || !bg_out) return fail(MAPI_ERR_NULL, "cap_out/bg_out is NULL");
    if (!(alpha > 0.0f && alpha < 1.0f)) return fail(MAPI_ERR_BAD_PARAM, "alpha (%g) must be in (0, 1)", (double)alpha);
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    if (ws_bytes < csr_prepare_ws_bytes(n, nnz))
        return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, csr_prepare_ws_bytes(n, nnz));
    Device d;
    mapi_status st;
    if ((st = device_info(d)) != MAPI_OK) return st;
    st = csr_prepare_run(n, nnz, row_ptr, col_idx, alpha, cap_out, bg_out, ws, d.sms,
                         static_cast<cudaStream_t>(stream), g_launches);
    if (st != MAPI_OK) return fail(st, "%s", csr_last_error());
    return MAPI_OK;
}

mapi_status mapi_rank_csr(int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* col_idx, const float* cap,
                          const float* bg, const float* b0, int32_t max_iters, float tol, float* w_out,
                          float* w_l2_out, float* deltas, int32_t* iters_done, void* ws, size_t ws_bytes,
                          mapi_stream_t stream) {
    if (n < 1) return fail(MAPI_ERR_SHAPE, "n (%lld) must be >= 1", (long long)n);
    if (nnz < 0 || nnz >= (int64_t)INT32_MAX)
        return fail(MAPI_ERR_SHAPE, "nnz (%lld) must be in [0, 2^31)", (long long)nnz);
    if (n >= (int64_t)INT32_MAX) return fail(MAPI_ERR_SHAPE, "n (%lld) must be < 2^31", (long long)n);
    if (!row_ptr || (nnz > 0 && !col_idx) || !cap || !bg || !b0 || !w_out)
        return fail(MAPI_ERR_NULL, "a required pointer (row_ptr/col_idx/cap/bg/b0/w_out) is NULL");
    if (max_iters < 1) return fail(MAPI_ERR_BAD_PARAM, "max_iters (%d) must be >= 1", max_iters);
    if (!(tol >= 0.0f)) return fail(MAPI_ERR_BAD_PARAM, "tol (%g) must be >= 0", (double)tol);
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    if (ws_bytes < csr_rank_ws_bytes(n, nnz))
        return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, csr_rank_ws_bytes(n, nnz));
    Device d;
    mapi_status st;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Timer timer(s);
    st = csr_rank_run(n, nnz, row_ptr, col_idx, cap, bg, b0, max_iters, tol, w_out, w_l2_out, deltas, ws, d.sms, s,
                      timer.on ? &timer.a : nullptr, timer.on ? &timer.b : nullptr, g_launches);
    if (st != MAPI_OK) return fail(st, "%s", csr_last_error());
    st = csr_rank_finish(ws, n, nnz, s, iters_done);
    timer.harvest();
    if (st == MAPI_ERR_CUDA) return fail(st, "%s", csr_last_error());
    if (st == MAPI_ERR_NEGATIVE) return fail(st, "b0 has a negative entry");
    if (st == MAPI_ERR_DEGENERATE) return fail(st, "||G (+) w_t||_1 == 0");
    if (st == MAPI_ERR_NONFINITE) return fail(st, "||G (+) w_t||_1 is not finite");
    return st;
}

// ---- K3n: MAPI ranking with the destination rows partitioned over ranks (csr.cuh)
static mapi_status shard_check(int64_t n, int64_t m, int64_t row0, int64_t nnz, const void* ws, size_t ws_bytes) {
    if (n < 1 || n >= (int64_t)INT32_MAX) return fail(MAPI_ERR_SHAPE, "n (%lld) must be in [1, 2^31)", (long long)n);
    if (nnz < 0 || nnz >= (int64_t)INT32_MAX)
        return fail(MAPI_ERR_SHAPE, "nnz_local (%lld) must be in [0, 2^31)", (long long)nnz);
    if (m < 0 || row0 < 0 || row0 + m > n)
        return fail(MAPI_ERR_SHAPE, "rows [%lld, %lld) are not inside [0, %lld)", (long long)row0,
                    (long long)(row0 + m), (long long)n);
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    if (ws_bytes < csr_rank_ws_bytes(n, nnz, m))
        return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, csr_rank_ws_bytes(n, nnz, m));
    return MAPI_OK;
}

mapi_status mapi_rank_csr_shard_begin(int64_t n, int64_t m, int64_t nnz_local, const int32_t* row_ptr_local,
                                      const float* cap, const float* bg, const float* b0, void* ws, size_t ws_bytes,
                                      mapi_stream_t stream) {
    mapi_status st = shard_check(n, m, 0, nnz_local, ws, ws_bytes);
    if (st != MAPI_OK) return st;
    if ((m > 0 && !row_ptr_local) || !cap || !bg || !b0)
        return fail(MAPI_ERR_NULL, "a required pointer (row_ptr_local/cap/bg/b0) is NULL");
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    st = csr_shard_begin(n, m, nnz_local, row_ptr_local, cap, bg, b0, ws, d.sms, static_cast<cudaStream_t>(stream),
                         g_launches);
    if (st != MAPI_OK) return fail(st, "%s", csr_last_error());
    return MAPI_OK;
}

mapi_status mapi_rank_csr_shard_rows(int64_t n, int64_t m, int64_t row0, int64_t nnz_local,
                                     const int32_t* row_ptr_local, const int32_t* col_idx_local, int32_t t,
                                     float** e_out, void* ws, size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = shard_check(n, m, row0, nnz_local, ws, ws_bytes);
    if (st != MAPI_OK) return st;
    if (m > 0 && (!row_ptr_local || (nnz_local > 0 && !col_idx_local)))
        return fail(MAPI_ERR_NULL, "row_ptr_local/col_idx_local is NULL");
    if (t < 0) return fail(MAPI_ERR_BAD_PARAM, "t (%d) must be >= 0", t);
    st = csr_shard_rows(n, m, row0, nnz_local, row_ptr_local, col_idx_local, t, e_out, ws,
                        static_cast<cudaStream_t>(stream), g_launches);
    if (st != MAPI_OK) return fail(st, "%s", csr_last_error());
    return MAPI_OK;
}

mapi_status mapi_rank_csr_shard_normalize(int64_t n, int64_t m, int64_t nnz_local, const float* cap, const float* bg,
                                          const float* b0, int32_t t, float tol, float* deltas, void* ws,
                                          size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = shard_check(n, m, 0, nnz_local, ws, ws_bytes);
    if (st != MAPI_OK) return st;
    if (!cap || !bg || !b0) return fail(MAPI_ERR_NULL, "a required pointer (cap/bg/b0) is NULL");
    if (t < 0) return fail(MAPI_ERR_BAD_PARAM, "t (%d) must be >= 0", t);
    if (!(tol >= 0.0f)) return fail(MAPI_ERR_BAD_PARAM, "tol (%g) must be >= 0", (double)tol);
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    st = csr_shard_normalize(n, m, nnz_local, cap, bg, b0, t, tol, deltas, ws, d.sms,
                             static_cast<cudaStream_t>(stream), g_launches);
    if (st != MAPI_OK) return fail(st, "%s", csr_last_error());
    return MAPI_OK;
}

mapi_status mapi_rank_csr_shard_finish(int64_t n, int64_t m, int64_t nnz_local, const float* b0, float* w_out,
                                       float* w_l2_out, int32_t* iters_done, int32_t* stopped, void* ws,
                                       size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = shard_check(n, m, 0, nnz_local, ws, ws_bytes);
    if (st != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (w_out) {
        if (!b0) return fail(MAPI_ERR_NULL, "b0 is NULL");
        Device d;
        if ((st = device_info(d)) != MAPI_OK) return st;
        st = csr_shard_output(n, m, nnz_local, b0, w_out, w_l2_out, ws, d.sms, s, g_launches);
        if (st != MAPI_OK) return fail(st, "%s", csr_last_error());
    }
    int32_t h[3] = {0, 0, 0};  // status, iterations done, stop flag
    cudaError_t e = cudaMemcpyAsync(h, ws, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(MAPI_ERR_CUDA, "status read-back: %s", cudaGetErrorString(e));
    if (iters_done) *iters_done = h[1];
    if (stopped) *stopped = h[2];
    st = (mapi_status)h[0];
    if (st == MAPI_ERR_NEGATIVE) return fail(st, "b0 has a negative entry");
    if (st == MAPI_ERR_DEGENERATE) return fail(st, "||G (+) w_t||_1 == 0");
    if (st == MAPI_ERR_NONFINITE) return fail(st, "||G (+) w_t||_1 is not finite");
    return st;
}

mapi_status mapi_csr_reorder(int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* col_idx, int32_t* perm_out,
                             int32_t* row_ptr_out, int32_t* col_idx_out, void* ws, size_t ws_bytes,
                             mapi_stream_t stream) {
    if (n < 1) return fail(MAPI_ERR_SHAPE, "n (%lld) must be >= 1", (long long)n);
    // same bounds as mapi_csr_prepare / mapi_rank_csr: (int)(n + 1) items feed the CUB scan
    if (nnz < 0 || nnz >= INT32_MAX) return fail(MAPI_ERR_SHAPE, "nnz (%lld) out of the int32 index range", (long long)nnz);
    if (n >= INT32_MAX) return fail(MAPI_ERR_SHAPE, "n (%lld) out of the int32 index range", (long long)n);
    if (!row_ptr || !perm_out || !row_ptr_out || (nnz > 0 && (!col_idx || !col_idx_out)))
        return fail(MAPI_ERR_NULL, "row_ptr / col_idx / perm_out / row_ptr_out / col_idx_out is NULL");
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    const size_t need = reorder_ws_bytes(n);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    mapi_status st = device_info(d);
    if (st != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* p = static_cast<char*>(ws);
    auto take = [&](size_t bytes) {
        char* r = p;
        p += align256(bytes);
        return r;
    };
    uint32_t* deg = reinterpret_cast<uint32_t*>(take(4 * (size_t)n));
    uint32_t* key = reinterpret_cast<uint32_t*>(take(4 * (size_t)n));
    uint32_t* key_out = reinterpret_cast<uint32_t*>(take(4 * (size_t)n));
    int32_t* ids = reinterpret_cast<int32_t*>(take(4 * (size_t)n));
    int32_t* order = reinterpret_cast<int32_t*>(take(4 * (size_t)n));
    int32_t* len = reinterpret_cast<int32_t*>(take(4 * (size_t)(n + 1)));
    size_t tmp_bytes = reorder_cub_bytes(n);
    void* tmp = take(tmp_bytes);
    const int grid = d.sms * 8;
    MAPI_CUDA(cudaMemsetAsync(deg, 0, 4 * (size_t)n, s));
    if (nnz > 0) k_reorder_outdeg<<<grid, 256, 0, s>>>(nnz, col_idx, deg);
    k_reorder_keys<<<grid, 256, 0, s>>>(n, deg, key, ids);
    MAPI_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key_out, ids, order, (int)n, 0, 32, s));
    k_reorder_perm<<<grid, 256, 0, s>>>(n, order, row_ptr, perm_out, len);
    tmp_bytes = reorder_cub_bytes(n);
    MAPI_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, len, row_ptr_out, (int)(n + 1), s));
    if (nnz > 0) k_reorder_copy<<<grid, 256, 0, s>>>(n, order, row_ptr, col_idx, perm_out, row_ptr_out, col_idx_out);
    g_launches.fetch_add(6, std::memory_order_relaxed);
    MAPI_CUDA(cudaGetLastError());
    return MAPI_OK;
}

mapi_status mapi_csr_permute(int64_t n, const int32_t* perm, const float* x, float* out, int32_t to_new,
                             mapi_stream_t stream) {
    if (n < 1) return fail(MAPI_ERR_SHAPE, "n (%lld) must be >= 1", (long long)n);
    if (!perm || !x || !out) return fail(MAPI_ERR_NULL, "perm / x / out is NULL");
    if (x == out) return fail(MAPI_ERR_BAD_PARAM, "x and out must not alias");
    Device d;
    mapi_status st = device_info(d);
    if (st != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    k_permute<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)d.sms * 8), 256, 0, s>>>(n, perm, x, out,
                                                                                            to_new ? 1 : 0);
    MAPI_LAUNCHED();
    MAPI_CUDA(cudaGetLastError());
    return MAPI_OK;
}

mapi_status mapi_center_rows(const float* V, int64_t M, int64_t N, int64_t ldv, float* Vc, int64_t ldvc,
                             float* mean_out, mapi_stream_t stream) {
    if (M < 0 || N < 1) return fail(MAPI_ERR_SHAPE, "M (%lld) must be >= 0 and N (%lld) >= 1", (long long)M, (long long)N);
    if (ldv < N || ldvc < N) return fail(MAPI_ERR_SHAPE, "ldv (%lld) / ldvc (%lld) < N (%lld)", (long long)ldv,
                                         (long long)ldvc, (long long)N);
    if (M == 0) return MAPI_OK;
    if (!V || !Vc || !mean_out) return fail(MAPI_ERR_NULL, "V, Vc or mean_out is NULL");
    Device d;
    mapi_status st;
    if ((st = device_info(d)) != MAPI_OK) return st;
    k_center_rows<<<(unsigned)((M + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(V, M, N, ldv, Vc, ldvc,
                                                                                            mean_out);
    MAPI_LAUNCHED();
    return MAPI_OK;
}

mapi_status mapi_mavp_deflate(int32_t op, const float* C, int64_t M, int64_t ldc, const float* w, float* D,
                              int64_t ldd, void* ws, size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = check_op(op, true);
    if (st != MAPI_OK) return st;
    if (M < 1 || M > kOuterMaxM) return fail(MAPI_ERR_SHAPE, "M (%lld) must be in [1, %d]", (long long)M, kOuterMaxM);
    if (ldc < M || ldd < M) return fail(MAPI_ERR_SHAPE, "ldc (%lld) / ldd (%lld) < M (%lld)", (long long)ldc,
                                        (long long)ldd, (long long)M);
    if (!C || !w || !D) return fail(MAPI_ERR_NULL, "C, w or D is NULL");
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    const size_t need = outer_ws_bytes(M, M, 1, 0);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Timer timer(s);
    timer.start();
    st = outer_run(op, w, M, 1, 1, C, M, ldc, true, nullptr, D, ldd, static_cast<char*>(ws), s);
    timer.stop();
    if (st != MAPI_OK) return st;
    if (timer.on) {
        MAPI_CUDA(cudaStreamSynchronize(s));
        timer.harvest();
    }
    return MAPI_OK;
}

mapi_status mapi_mavp_reconstruct(int32_t op, const float* W, int64_t M, int32_t r, int64_t ldw, const float* V,
                                  int64_t N, int64_t ldv, float* Vhat, int64_t ldvh, float* mean_out, void* ws,
                                  size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = check_op(op, true);
    if (st != MAPI_OK) return st;
    if (M < 1 || M > kOuterMaxM) return fail(MAPI_ERR_SHAPE, "M (%lld) must be in [1, %d]", (long long)M, kOuterMaxM);
    if (r < 1 || ldw < r) return fail(MAPI_ERR_SHAPE, "r (%d) must be >= 1 and ldw (%lld) >= r", r, (long long)ldw);
    if (N < 1 || ldv < N || ldvh < N)
        return fail(MAPI_ERR_SHAPE, "N (%lld) must be >= 1 with ldv, ldvh >= N", (long long)N);
    if (!W || !V || !Vhat) return fail(MAPI_ERR_NULL, "W, V or Vhat is NULL");
    if (!ws) return fail(MAPI_ERR_WORKSPACE, "workspace is NULL");
    const size_t need = outer_ws_bytes(M, N, r, N);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    char* p = static_cast<char*>(ws);
    float* Xc = reinterpret_cast<float*>(p + outer_ws_bytes(M, N, r, N) - align256(sizeof(float) * (size_t)M * N));
    if (!mean_out) return fail(MAPI_ERR_NULL, "mean_out is NULL (it is added back in step 8)");
    k_center_rows<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(V, M, N, ldv, Xc, N, mean_out);
    MAPI_LAUNCHED();
    return outer_run(op, W, M, r, ldw, Xc, N, N, false, mean_out, Vhat, ldvh, p, s);
}

mapi_status mapi_normalize(int32_t op, const float* y, int64_t n, float* w, float* s_out, float* delta_out,
                           int32_t* status_out, mapi_stream_t stream) {
    mapi_status st = check_op(op, true);
    if (st != MAPI_OK) return st;
    if (n < 1) return fail(MAPI_ERR_SHAPE, "n (%lld) must be >= 1", (long long)n);
    if (!y || !w) return fail(MAPI_ERR_NULL, "y or w is NULL");
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    k_normalize_full<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(n, y, w, op == MAPI_OP_DOT ? 1 : 0, s_out,
                                                                        delta_out, status_out);
    MAPI_LAUNCHED();
    return MAPI_OK;
}

// ---------------------------------------------------------------------------- fused P2P sharding
size_t mapi_p2p_exchange_bytes(int64_t n, int32_t world) {
    if (n < 0 || world < 1) return 0;
    return p2p_exchange_bytes(n, world);
}

mapi_status mapi_p2p_alloc(size_t bytes, void** ptr_out) {
    if (!ptr_out) return fail(MAPI_ERR_NULL, "ptr_out is NULL");
    *ptr_out = nullptr;
    if (bytes == 0) return fail(MAPI_ERR_BAD_PARAM, "bytes must be > 0");
    MAPI_CUDA(cudaMalloc(ptr_out, bytes));
    MAPI_CUDA(cudaMemset(*ptr_out, 0, bytes));
    return MAPI_OK;
}

mapi_status mapi_p2p_free(void* ptr) {
    if (ptr) MAPI_CUDA(cudaFree(ptr));
    return MAPI_OK;
}

mapi_status mapi_ipc_get_handle(const void* ptr, void* handle_out) {
    if (!ptr || !handle_out) return fail(MAPI_ERR_NULL, "ptr / handle_out is NULL");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    MAPI_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
    memcpy(handle_out, &h, sizeof(h));
    return MAPI_OK;
}

mapi_status mapi_ipc_open_handle(const void* handle, void** ptr_out) {
    if (!handle || !ptr_out) return fail(MAPI_ERR_NULL, "handle / ptr_out is NULL");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    MAPI_CUDA(cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return MAPI_OK;
}

mapi_status mapi_ipc_close_handle(void* ptr) {
    if (ptr) MAPI_CUDA(cudaIpcCloseMemHandle(ptr));
    return MAPI_OK;
}

static mapi_status p2p_common_checks(int32_t rank, int32_t world, int32_t grid) {
    if (world < 1 || world > kP2pMaxWorld || rank < 0 || rank >= world)
        return fail(MAPI_ERR_BAD_PARAM, "rank %d / world %d (world in [1, %d])", rank, world, kP2pMaxWorld);
    if (grid < 0 || grid > kP2pMaxGrid)
        return fail(MAPI_ERR_BAD_PARAM, "grid (%d) must be in [0, %d]", grid, kP2pMaxGrid);
    if (world > 1 && grid == 0)
        return fail(MAPI_ERR_BAD_PARAM, "world > 1 needs an explicit grid agreed by every rank (e.g. the min SM count)");
    return MAPI_OK;
}
static mapi_status p2p_device_checks(int32_t grid, Device& d) {
    mapi_status st = device_info(d);
    if (st != MAPI_OK) return st;
    if (grid > d.sms) return fail(MAPI_ERR_BAD_PARAM, "grid (%d) exceeds the device's %d SMs", grid, d.sms);
    return MAPI_OK;
}

static mapi_status p2p_finish(const int32_t* status, cudaStream_t s, Timer& timer, int32_t* iters_done,
                              int32_t* published_out) {
    int32_t h[2] = {0, 0};
    MAPI_CUDA(cudaMemcpyAsync(h, status, sizeof(h), cudaMemcpyDeviceToHost, s));
    MAPI_CUDA(cudaStreamSynchronize(s));
    timer.harvest();
    if (iters_done) *iters_done = h[1];
    // iterations that reached the exchange: the completed ones, plus the one a degenerate s stopped
    // (a timed-out exchange leaves the buffers inconsistent: the caller must discard the exchange)
    if (published_out) *published_out = h[1] + ((h[0] == kStDegenerate || h[0] == kStNonfinite) ? 1 : 0);
    if (h[0] == kStP2pTimeout)
        return fail(MAPI_ERR_CUDA, "peer exchange timed out at iteration %d (a rank did not arrive)", h[1]);
    if (h[0] != 0) return fail((mapi_status)h[0], "degenerate / non-finite norm at iteration %d", h[1]);
    return MAPI_OK;
}

mapi_status mapi_iterate_sharded(int32_t op, const float* A_local, int64_t m, int64_t n, int64_t lda, int64_t row0,
                                 const float* b0, int32_t iters, float tol, int32_t rank, int32_t world,
                                 const uint64_t* peers, uint64_t epoch0, uint64_t flag_base, int32_t grid_in,
                                 float* w_out, float* norms, float* deltas, int32_t* iters_done,
                                 int32_t* published_out, int32_t* grid_out, void* ws, size_t ws_bytes,
                                 mapi_stream_t stream) {
    mapi_status st = check_op(op, true);
    if (st != MAPI_OK) return st;
    if (!A_local || !b0 || !peers || !w_out || !ws) return fail(MAPI_ERR_NULL, "a required pointer is NULL");
    if ((st = p2p_common_checks(rank, world, grid_in)) != MAPI_OK) return st;
    if (n < 256 || m < 1 || m > n || row0 < 0 || row0 + m > n)
        return fail(MAPI_ERR_SHAPE, "rows [%lld, %lld) of n = %lld (n >= 256 required)", (long long)row0,
                    (long long)(row0 + m), (long long)n);
    if (lda < n) return fail(MAPI_ERR_SHAPE, "lda (%lld) < n (%lld)", (long long)lda, (long long)n);
    if (vec_width(A_local, lda) != 8) return fail(MAPI_ERR_SHAPE, "A_local rows must be 32 B-aligned (lda %% 8 == 0)");
    if (iters < 1) return fail(MAPI_ERR_BAD_PARAM, "iters (%d) must be >= 1", iters);
    if (!(tol >= 0.0f)) return fail(MAPI_ERR_BAD_PARAM, "tol must be >= 0");
    if (ws_bytes < sharded_ws_bytes()) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < %zu", ws_bytes, sharded_ws_bytes());
    Device d;
    if ((st = p2p_device_checks(grid_in, d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nw = coop_warps(n);
    const int grid = grid_in > 0 ? grid_in : (int)std::min<int64_t>({(int64_t)d.sms, (int64_t)kP2pMaxGrid});
    const size_t smem = p2p_smem_bytes(m, n, grid, nw);
    if (smem > (size_t)d.smem_optin) return fail(MAPI_ERR_SHAPE, "n (%lld) too large for the staged w", (long long)n);
    int32_t* status = static_cast<int32_t*>(ws);
    MAPI_CUDA(cudaMemsetAsync(ws, 0, 256, s));
    P2PArgs a;
    a.A = A_local; a.m = m; a.n = n; a.lda = lda; a.row0 = row0; a.b0 = b0; a.iters = iters; a.tol = tol;
    a.rank = rank; a.world = world; a.peers = reinterpret_cast<const unsigned long long*>(peers);
    a.epoch0 = epoch0; a.flag_base = flag_base; a.w_out = w_out; a.norms = norms; a.deltas = deltas;
    a.status = status;
    a.bar = reinterpret_cast<unsigned int*>(static_cast<char*>(ws) + 64);
    a.cslots = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
    const int pol = load_policy(d, m, lda);
    Timer timer(s);
    with_op(op, [&](auto OPc) {
        return with_pol(pol, [&](auto POLc) {
            constexpr int OP = decltype(OPc)::value, POL = decltype(POLc)::value;
            auto kern = nw == 32 ? k_iterate_p2p<OP, POL, 32> : k_iterate_p2p<OP, POL, 16>;
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e == cudaSuccess) {
                void* args[] = {&a};
                timer.start();
                e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(nw * 32), args, smem, s);
                timer.stop();
                g_launches.fetch_add(1, std::memory_order_relaxed);
            }
            if (e != cudaSuccess) st = fail(MAPI_ERR_CUDA, "sharded launch (grid %d): %s", grid, cudaGetErrorString(e));
            return 0;
        });
    });
    if (st != MAPI_OK) return st;
    if (grid_out) *grid_out = grid;
    return p2p_finish(status, s, timer, iters_done, published_out);
}

// ---- K2sp: K2s with the task list split over the ranks (p2p.cuh)
static inline void sym_shard_tasks(int64_t n, int32_t rank, int32_t world, int64_t& tlo, int64_t& thi) {
    const int64_t T = sym_task_start(sym_nb(n), sym_nc(n));
    tlo = T * rank / world;
    thi = T * (rank + 1) / world;
}

mapi_status mapi_sym_shard_rows(int64_t n, int32_t rank, int32_t world, int64_t* row_lo, int64_t* row_hi,
                                int64_t* task_lo, int64_t* task_hi) {
    if (n < 1) return fail(MAPI_ERR_SHAPE, "n (%lld) must be >= 1", (long long)n);
    if (world < 1 || world > kP2pMaxWorld || rank < 0 || rank >= world)
        return fail(MAPI_ERR_BAD_PARAM, "rank %d / world %d (world in [1, %d])", rank, world, kP2pMaxWorld);
    int64_t tlo, thi, r0, r1;
    sym_shard_tasks(n, rank, world, tlo, thi);
    sym_shard_rows(n, tlo, thi, r0, r1);
    if (row_lo) *row_lo = r0;
    if (row_hi) *row_hi = r1;
    if (task_lo) *task_lo = tlo;
    if (task_hi) *task_hi = thi;
    return MAPI_OK;
}

mapi_status mapi_sym_shard_valid(int64_t n, int32_t rank, int32_t world, int64_t j, int64_t* out4) {
    if (n < 1 || j < 0 || j >= n || !out4) return fail(MAPI_ERR_SHAPE, "bad n / j / out");
    if (world < 1 || world > kP2pMaxWorld || rank < 0 || rank >= world)
        return fail(MAPI_ERR_BAD_PARAM, "rank %d / world %d", rank, world);
    int64_t tlo, thi;
    sym_shard_tasks(n, rank, world, tlo, thi);
    const SymValid v = sym_valid(j, n, tlo, thi);
    out4[0] = v.c_lo; out4[1] = v.c_hi; out4[2] = v.b_lo; out4[3] = v.b_hi;
    return MAPI_OK;
}

mapi_status mapi_iterate_sym_sharded(int32_t op, const float* A_local, int64_t row_lo, int64_t row_hi, int64_t n,
                                     int64_t lda, const float* b0, int32_t iters, float tol, int32_t rank,
                                     int32_t world, const uint64_t* peers, uint64_t epoch0, uint64_t flag_base,
                                     int32_t grid_in, float* w_out, float* norms, float* deltas,
                                     int32_t* iters_done, int32_t* published_out, int32_t* grid_out, void* ws,
                                     size_t ws_bytes, mapi_stream_t stream) {
    mapi_status st = check_op(op, true);
    if (st != MAPI_OK) return st;
    if (!A_local || !b0 || !peers || !w_out || !ws) return fail(MAPI_ERR_NULL, "a required pointer is NULL");
    if ((st = p2p_common_checks(rank, world, grid_in)) != MAPI_OK) return st;
    if (n < 8 || n % 8 != 0) return fail(MAPI_ERR_SHAPE, "n (%lld) must be a positive multiple of 8", (long long)n);
    int64_t tlo, thi, r0, r1;
    sym_shard_tasks(n, rank, world, tlo, thi);
    sym_shard_rows(n, tlo, thi, r0, r1);
    if (row_lo != r0 || row_hi != r1)
        return fail(MAPI_ERR_SHAPE, "rank %d holds rows [%lld, %lld); mapi_sym_shard_rows gives [%lld, %lld)", rank,
                    (long long)row_lo, (long long)row_hi, (long long)r0, (long long)r1);
    if (lda < n || lda % 8 != 0 || (reinterpret_cast<uintptr_t>(A_local) & 31) != 0)
        return fail(MAPI_ERR_SHAPE, "A_local needs lda >= n, lda %% 8 == 0 and 32 B-aligned rows");
    if (iters < 1) return fail(MAPI_ERR_BAD_PARAM, "iters (%d) must be >= 1", iters);
    if (!(tol >= 0.0f)) return fail(MAPI_ERR_BAD_PARAM, "tol must be >= 0");
    const size_t need = mapi_workspace_size(MAPI_WS_ITERATE_SYM, n, 0, 0);
    if (ws_bytes < need) return fail(MAPI_ERR_WORKSPACE, "ws_bytes (%zu) < required (%zu)", ws_bytes, need);
    Device d;
    if ((st = p2p_device_checks(grid_in, d)) != MAPI_OK) return st;
    if (sym_smem_bytes(n) > (size_t)d.smem_optin) return fail(MAPI_ERR_SHAPE, "symmetric kernel smem too large");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int grid = grid_in > 0 ? grid_in : (int)std::min<int64_t>({(int64_t)d.sms, n, (int64_t)kP2pMaxGrid});
    IterWs W = carve_iterate(ws, n);
    float* partials = reinterpret_cast<float*>(static_cast<char*>(ws) + iterate_ws_bytes(n));
    MAPI_CUDA(cudaMemsetAsync(W.bar, 0, 256, s));
    MAPI_CUDA(cudaMemsetAsync(W.y, 0, sizeof(unsigned long long) * 2 * (size_t)n, s));
    SymShardArgs x;
    SymArgs& a = x.sa;
    a.it.A = A_local; a.it.n = n; a.it.lda = lda; a.it.b0 = b0; a.it.iters = iters; a.it.tol = tol;
    a.it.w_out = w_out; a.it.norms = norms; a.it.deltas = deltas; a.it.y = W.y; a.it.slots = W.slots;
    a.it.bar = W.bar; a.it.status = W.status;
    a.prow = partials;
    a.pcol = partials + (size_t)sym_nc(n) * (size_t)((n + 31) & ~int64_t(31));
    a.wtag = reinterpret_cast<unsigned long long*>(W.y);
    a.yg = W.w;
    a.prefetch_rows = 0;
    x.row0 = r0; x.tlo = tlo; x.thi = thi; x.rank = rank; x.world = world;
    x.peers = reinterpret_cast<const unsigned long long*>(peers);
    x.epoch0 = epoch0; x.flag_base = flag_base;
    using KernT = void (*)(SymShardArgs);
    KernT kern = op == 2 ? k_iterate_sym_sharded<2> : (op == 1 ? k_iterate_sym_sharded<1> : k_iterate_sym_sharded<0>);
    const size_t smem = sym_smem_bytes(n);
    MAPI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    Timer timer(s);
    void* args[] = {&x};
    timer.start();
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kSymThreads), args, smem, s);
    timer.stop();
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e != cudaSuccess)
        return fail(MAPI_ERR_CUDA, "sharded symmetric launch (grid %d): %s", grid, cudaGetErrorString(e));
    if (grid_out) *grid_out = grid;
    return p2p_finish(W.status, s, timer, iters_done, published_out);
}

mapi_status mapi_matvec_normalized(int32_t op, const float* A, int64_t n_rows, int64_t n_cols, int64_t lda,
                                   const float* y_prev, const float* w_prev, float* w_next, float* y_out,
                                   float* s_out, float* delta_out, int32_t* status_out, mapi_stream_t stream) {
    mapi_status st = check_op(op, true);
    if (st != MAPI_OK) return st;
    if (n_rows < 0 || n_cols < 1) return fail(MAPI_ERR_SHAPE, "n_rows (%lld) >= 0 and n_cols (%lld) >= 1 required",
                                              (long long)n_rows, (long long)n_cols);
    if (lda < n_cols) return fail(MAPI_ERR_SHAPE, "lda (%lld) < n_cols (%lld)", (long long)lda, (long long)n_cols);
    if (!y_prev || !w_prev || !w_next || (n_rows > 0 && (!A || !y_out)))
        return fail(MAPI_ERR_NULL, "a required pointer (A/y_prev/w_prev/w_next/y_out) is NULL");
    const size_t smem = sizeof(float) * (size_t)n_cols;
    if (smem > 200 * 1024) return fail(MAPI_ERR_SHAPE, "n_cols (%lld) too large for the staged x", (long long)n_cols);
    Device d;
    if ((st = device_info(d)) != MAPI_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int vec = vec_width(A ? A : y_prev, lda);
    const int pol = load_policy(d, n_rows, lda);
    with_op(op, [&](auto OPc) {
        return with_vec(vec, [&](auto VECc) {
            return with_pol(pol, [&](auto POLc) {
                constexpr int OP = decltype(OPc)::value, VEC = decltype(VECc)::value, POL = decltype(POLc)::value;
                auto kern = k_matvec_norm<OP, VEC, POL, unroll_for(VEC)>;
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                int occ = 1;
                if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 512, smem);
                if (e != cudaSuccess) {
                    st = fail(MAPI_ERR_CUDA, "matvec_normalized setup: %s", cudaGetErrorString(e));
                    return 0;
                }
                const int64_t want = std::max<int64_t>(1, (n_rows + 15) / 16);
                const int grid = (int)std::min<int64_t>((int64_t)std::max(occ, 1) * d.sms, want);
                kern<<<grid, 512, smem, s>>>(A, n_rows, n_cols, lda, y_prev, w_prev, w_next, y_out, s_out, delta_out,
                                            status_out);
                g_launches.fetch_add(1, std::memory_order_relaxed);
                e = cudaGetLastError();
                if (e != cudaSuccess) st = fail(MAPI_ERR_CUDA, "matvec_normalized launch: %s", cudaGetErrorString(e));
                return 0;
            });
        });
    });
    return st;
}

}  // extern "C"
