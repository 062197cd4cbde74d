// deflate.cuh — K5: L2 deflation for mapi_pca_topk (BASELINE configs[1]).
//
//   p_i = w_i / ||w_i||_2                       (fp64, from the fp32 MAPI output)      k_l2_to_p
//   r_i = p_i^T C   (row vector, fp64 accumulate, column reduction)                    k_colsum_*
//   D_i = (I - sum_{m<i} p_m p_m^T) C = C - sum_{m<i} p_m r_m^T, fp64 per element,
//         rounded ONCE to fp32                                                        k_build_deflated
// Streaming, HBM/L2-bound work off the per-iteration MAVP loop (the fp64 multiplies here are the
// deflation's own arithmetic; the MAVP loop itself stays multiplication-free).
#pragma once
#include "mapi_common.cuh"

namespace mapi {

// One CTA: p = w / ||w||_2 in fp64 (fixed-order sum of squares), p32 = fp32(p).
__global__ void __launch_bounds__(1024) k_l2_to_p(int64_t n, const float* __restrict__ w,
                                                  double* __restrict__ p64, float* __restrict__ p32) {
    __shared__ double red[33];
    double part = 0.0;
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const double v = (double)w[k];
        part = fma(v, v, part);
    }
    const double l2 = sqrt(block_sum(part, red));
    for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
        const double v = l2 > 0.0 ? (double)w[k] / l2 : 0.0;
        p64[k] = v;
        p32[k] = (float)v;
    }
}

// Column-reduction partials: part[s][c] = sum_{l in chunk s} p[l] * C[l][c] (l ascending).
// grid = (ceil(n/256), S); CTA (bx, s) owns columns [256 bx, 256 bx + 256) and row chunk s.
__global__ void __launch_bounds__(256) k_colsum_partial(const float* __restrict__ C, int64_t n,
                                                        int64_t ldc, const double* __restrict__ p,
                                                        double* __restrict__ part, int64_t rows_per) {
    const int64_t c = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int64_t l0 = (int64_t)blockIdx.y * rows_per, l1 = min(n, l0 + rows_per);
    if (c >= n) return;
    double acc = 0.0;
    for (int64_t l = l0; l < l1; ++l) acc = fma(p[l], (double)__ldg(C + l * ldc + c), acc);
    part[(int64_t)blockIdx.y * n + c] = acc;
}

__global__ void __launch_bounds__(256) k_colsum_final(int64_t n, int S, const double* __restrict__ part,
                                                      double* __restrict__ r) {
    const int64_t c = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (c >= n) return;
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc += part[(int64_t)s * n + c];
    r[c] = acc;
}

// D[row][c] = fp32( C[row][c] - sum_{m<i} P[m][row] * R[m][c] ), m ascending, fp64.
__global__ void __launch_bounds__(256) k_build_deflated(const float* __restrict__ C, int64_t n, int64_t ldc,
                                                        const double* __restrict__ P,
                                                        const double* __restrict__ R, int i,
                                                        float* __restrict__ D) {
    for (int64_t row = blockIdx.y; row < n; row += gridDim.y) {
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
             c += (int64_t)gridDim.x * blockDim.x) {
            double v = (double)__ldg(C + row * ldc + c);
            for (int m = 0; m < i; ++m) v = fma(-P[(int64_t)m * n + row], R[(int64_t)m * n + c], v);
            D[row * n + c] = (float)v;
        }
    }
}

}  // namespace mapi
