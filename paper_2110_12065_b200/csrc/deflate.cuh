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
    // the same sequential order (s ascending); loads issued 16 at a time instead of one per dependent add
    double acc = 0.0;
    int s = 0;
    for (; s + 16 <= S; s += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = part[(int64_t)(s + u) * n + c];
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += v[u];
    }
    for (; s < S; ++s) acc += part[(int64_t)s * n + c];
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

// Vectorised form for i <= 8 components (the BASELINE k = 8): thread owns 4 consecutive columns of a
// 1024-column strip and a run of rows; r_m for its columns stays in registers (i x 4 doubles), C is
// read and D written as float4, p_m[row] comes from L1 (warp broadcast).  Same per-element fp64
// sequence as k_build_deflated (v = C; v = fma(-p_m[row], r_m[c], v) for m = 0..i-1; one rounding),
// so the two are bitwise identical.  Requires n % 4 == 0, ldc % 4 == 0, 16 B-aligned C and D.
constexpr int kDeflRows = 16;  // rows per CTA
template <int I>
__global__ void __launch_bounds__(256) k_build_deflated_v4(const float* __restrict__ C, int64_t n, int64_t ldc,
                                                           const double* __restrict__ P,
                                                           const double* __restrict__ R,
                                                           float* __restrict__ D) {
    const int64_t c = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4;
    if (c >= n) return;
    double r[I][4];
#pragma unroll
    for (int m = 0; m < I; ++m) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(R + (int64_t)m * n + c));
        const double2 b = __ldg(reinterpret_cast<const double2*>(R + (int64_t)m * n + c) + 1);
        r[m][0] = a.x; r[m][1] = a.y; r[m][2] = b.x; r[m][3] = b.y;
    }
    const int64_t row0 = (int64_t)blockIdx.y * kDeflRows, row1 = min(n, row0 + kDeflRows);
#pragma unroll 4
    for (int64_t row = row0; row < row1; ++row) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(C + row * ldc + c));
        double v[4] = {(double)x.x, (double)x.y, (double)x.z, (double)x.w};
#pragma unroll
        for (int m = 0; m < I; ++m) {
            const double pm = -__ldg(P + (int64_t)m * n + row);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = fma(pm, r[m][j], v[j]);
        }
        reinterpret_cast<float4*>(D + row * n)[c >> 2] = make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
    }
}

}  // namespace mapi
