// packed.cuh — symmetric packed storage for the end-to-end host path (mapi_iterate_host_many_packed).
//
// MAPI's dense inputs are covariance matrices (Eq. 2 / Eq. 5), symmetric by construction.
// A host can send such a matrix in packed upper-triangular form (row j holds A[j][j..n-1], LAPACK's
// "packed" layout in row-major order): n(n+1)/2 floats instead of n^2, halving the PCIe bytes of the
// end-to-end path.  k_unpack_sym rebuilds the full row-major matrix on the device, bitwise: every
// A[j][k] (k >= j) is copied, every A[k][j] (k > j) is the same fp32 value mirrored.
//
// Layout: packed offset of row j = j n - j (j - 1) / 2, element (j, k >= j) at offset(j) + (k - j).
// Grid: one CTA per 32 x 32 upper tile (bi <= bj), tiles enumerated row-major over the upper triangle;
// a tile is read row-wise (coalesced along k) into shared memory, written to A[bi][bj] and, transposed,
// to A[bj][bi] (for diagonal tiles only the k > j part of the transpose).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mapi {

constexpr int kPackTile = 32;

__host__ __device__ inline int64_t packed_floats(int64_t n) { return n * (n + 1) / 2; }
__host__ __device__ inline int64_t packed_row_offset(int64_t n, int64_t j) { return j * n - j * (j - 1) / 2; }

// tile index t -> (bi, bj) over the upper triangle of an nb x nb tile grid, row-major
__device__ inline void upper_tile(int64_t t, int64_t nb, int64_t& bi, int64_t& bj) {
    // row bi starts at s(bi) = bi nb - bi (bi - 1) / 2; invert with a float estimate + correction
    const double b = 2.0 * (double)nb + 1.0;
    int64_t r = (int64_t)((b - sqrt(b * b - 8.0 * (double)t)) / 2.0);
    if (r < 0) r = 0;
    if (r >= nb) r = nb - 1;
    auto start = [&](int64_t x) { return x * nb - x * (x - 1) / 2; };
    while (r > 0 && start(r) > t) --r;
    while (r + 1 < nb && start(r + 1) <= t) ++r;
    bi = r;
    bj = r + (t - start(r));
}

__global__ void __launch_bounds__(256) k_unpack_sym(const float* __restrict__ P, int64_t n, float* __restrict__ A,
                                                     int64_t lda) {
    __shared__ float tile[kPackTile][kPackTile + 1];
    const int64_t nb = (n + kPackTile - 1) / kPackTile;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int64_t t = blockIdx.x; t < nb * (nb + 1) / 2; t += gridDim.x) {
        int64_t bi, bj;
        upper_tile(t, nb, bi, bj);
        const int64_t j0 = bi * kPackTile, k0 = bj * kPackTile;
        for (int r = ty; r < kPackTile; r += 8) {
            const int64_t j = j0 + r, k = k0 + tx;
            float v = 0.0f;
            if (j < n && k < n && k >= j) {
                v = P[packed_row_offset(n, j) + (k - j)];
                A[j * lda + k] = v;  // upper part, in place
            }
            tile[r][tx] = v;
        }
        __syncthreads();
        // mirrored part: A[k][j] = tile[j - j0][k - k0] for k > j
        for (int r = ty; r < kPackTile; r += 8) {
            const int64_t k = k0 + r, j = j0 + tx;
            if (k < n && j < n && k > j) A[k * lda + j] = tile[tx][r];
        }
        __syncthreads();
    }
}

}  // namespace mapi
