// reorder.cuh — node relabelling for the CSR ranking path (mapi_csr_reorder / permute / unpermute).
//
// The ranking step's cost is the gather of v over the edges' sources (Eq. 13; K3).
// Relabelling nodes by DESCENDING out-degree (ties by ascending id) puts the most gathered sources at the
// lowest ids, where the persistent gather kernel (K3h) keeps a shared-memory copy of v (on cfg5 the
// first 40,960 ids then carry 56% of the edges instead of 17%).  The relabelled graph is the same graph:
// new row i' = the in-edges of old node order[i'], sources renamed through perm (perm[order[i']] = i').
// Preparation, off the iteration loop: out-degree histogram (integer atomics: order-independent), a
// stable radix sort of (max - outdeg, id) (CUB, deterministic), a prefix sum of the relabelled row
// lengths, and one warp per row copying + renaming its sources (kept in their original order).
#pragma once
#include <cstdint>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

namespace mapi {

__global__ void k_reorder_outdeg(int64_t nnz, const int32_t* __restrict__ col_idx, uint32_t* __restrict__ deg) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(deg + col_idx[k], 1u);
}
// sort key: larger out-degree first; ids carried along (stable sort keeps ties in ascending id)
__global__ void k_reorder_keys(int64_t n, const uint32_t* __restrict__ deg, uint32_t* __restrict__ key,
                               int32_t* __restrict__ ids) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        key[j] = 0xffffffffu - deg[j];
        ids[j] = (int32_t)j;
    }
}
// perm[order[i]] = i; new row lengths len[i] = indeg(order[i]) (len[n] = 0 for the exclusive scan)
__global__ void k_reorder_perm(int64_t n, const int32_t* __restrict__ order, const int32_t* __restrict__ row_ptr,
                               int32_t* __restrict__ perm, int32_t* __restrict__ len) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n) {
            const int32_t o = order[i];
            perm[o] = (int32_t)i;
            len[i] = row_ptr[o + 1] - row_ptr[o];
        } else {
            len[n] = 0;
        }
    }
}
// one warp per new row: col_out[row_ptr_out[i] + t] = perm[col_idx[row_ptr[order[i]] + t]]
__global__ void k_reorder_copy(int64_t n, const int32_t* __restrict__ order, const int32_t* __restrict__ row_ptr,
                               const int32_t* __restrict__ col_idx, const int32_t* __restrict__ perm,
                               const int32_t* __restrict__ row_ptr_out, int32_t* __restrict__ col_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const int32_t o = order[i];
        const int32_t s0 = row_ptr[o], len = row_ptr[o + 1] - s0, d0 = row_ptr_out[i];
        for (int32_t t = lane; t < len; t += 32) col_out[d0 + t] = perm[col_idx[s0 + t]];
    }
}
// x_new[perm[j]] = x_old[j] (to_new) or x_old[j] = x_new[perm[j]] (back)
__global__ void k_permute(int64_t n, const int32_t* __restrict__ perm, const float* __restrict__ in,
                          float* __restrict__ out, int to_new) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        if (to_new) out[perm[j]] = in[j];
        else out[j] = in[perm[j]];
    }
}

inline size_t reorder_cub_bytes(int64_t n) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr, (const int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr, (int)(n + 1));
    return a > b ? a : b;
}
// [deg n u32][key n u32][key_out n u32][ids n i32][order n i32][len n+1 i32][cub temp]
inline size_t reorder_ws_bytes(int64_t n) {
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    return 5 * al(4 * (size_t)n) + al(4 * (size_t)(n + 1)) + al(reorder_cub_bytes(n));
}

}  // namespace mapi
