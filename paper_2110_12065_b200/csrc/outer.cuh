// outer.cuh — K9: Alg. 2's MAVP outer-product operator
//
//   Y = Q X   or   Y = X - Q X,   Q = W (op) W^T,   Q[i][j] = sum_c term(W[i][c], W[j][c])
//
// Step 6 is D = C - (w1 (+) w1^T) C (r = 1, X = C, subtract), step 8 is
// v_hat = (W (+) W^T)(v - m) + m (r = 2, X = the centred images, + m).  Q X is a REGULAR matrix product
// (S:269-277), an M^3 operation if Q is materialised.  For one component w (a = |w|, s = sign w) the
// min1 term is s_i s_j min(a_i, a_j), so with u_j = s_j X[j][k] and the rows ordered by (a, index):
//   sum_j min(a_i, a_j) u_j = sum_{rank j <= rank i} a_j u_j + a_i sum_{rank j > rank i} u_j
// exactly (ties: a_j = a_i either way) — an O(M) prefix scan per column instead of an O(M^2) product
// (reading R10).  min2 (Eq. 4) splits the rows into the positive / negative groups (zero
// rows contribute and receive nothing); dot is the rank-1 product w_i (w^T X).
// Kernels: k_outer_sort (one CTA bitonic sort of (bits(a_j), j) per component, M <= 16384),
// k_outer_blocksum (fp64 sums of a u and u per (row block, column)), k_outer_apply (each (row block,
// column) thread adds the sums of the preceding blocks in block order, walks its rows in sorted order,
// and writes Y).  Column-per-thread: every global access is a coalesced row segment.  fp64 scans.
#pragma once
#include "mapi_common.cuh"

namespace mapi {

constexpr int kOuterMaxM = 16384;   // single-CTA bitonic sort in shared memory (8 B keys)
constexpr int kOuterRB = 256;       // rows per scan block
constexpr int kOuterThreads = 256;  // columns per CTA

inline int64_t outer_blocks(int64_t M) { return (M + kOuterRB - 1) / kOuterRB; }

// (bits(|w_j|) << 32 | j) sorted ascending -> idx[t], a[t] = |w|, s[t] = sign(w) (+1, -1, 0)
__global__ void __launch_bounds__(1024) k_outer_sort(const float* __restrict__ W, int64_t M, int64_t ldw,
                                                     int32_t* __restrict__ idx, float* __restrict__ a_sorted,
                                                     float* __restrict__ s_sorted) {
    extern __shared__ unsigned long long keys[];
    const int c = blockIdx.x;
    int P = 1;
    while (P < M) P <<= 1;
    for (int t = threadIdx.x; t < P; t += blockDim.x) {
        if (t < M) {
            const float w = W[(int64_t)t * ldw + c];
            keys[t] = ((unsigned long long)__float_as_uint(fabsf(w)) << 32) | (unsigned)t;
        } else {
            keys[t] = ~0ull;
        }
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < P; t += blockDim.x) {
                const int l = t ^ j;
                if (l > t) {
                    const unsigned long long x = keys[t], y = keys[l];
                    const bool up = (t & k) == 0;
                    if ((x > y) == up) {
                        keys[t] = y;
                        keys[l] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < M; t += blockDim.x) {
        const int j = (int)(keys[t] & 0xffffffffu);
        const float w = W[(int64_t)j * ldw + c];
        idx[(int64_t)c * M + t] = j;
        a_sorted[(int64_t)c * M + t] = fabsf(w);
        s_sorted[(int64_t)c * M + t] = w > 0.0f ? 1.0f : (w < 0.0f ? -1.0f : 0.0f);
    }
}

// Per (component c, row block b, column k): G groups of {sum a u, sum u} over the block's sorted rows.
// min1: one group, u = s X.  min2: group 0 = positive rows, group 1 = negative rows, u = X.
// dot: one group, u = w X (only sum a u is used, with a := w).
template <int OP>
__global__ void __launch_bounds__(kOuterThreads) k_outer_blocksum(const float* __restrict__ X, int64_t M, int64_t q,
                                                                 int64_t ldx, const int32_t* __restrict__ idx,
                                                                 const float* __restrict__ a_sorted,
                                                                 const float* __restrict__ s_sorted, int c,
                                                                 double* __restrict__ part) {
    constexpr int G = OP == 1 ? 2 : 1;
    const int64_t k = (int64_t)blockIdx.x * kOuterThreads + threadIdx.x;
    const int64_t b = blockIdx.y, nb = gridDim.y;
    if (k >= q) return;
    const int64_t t0 = b * kOuterRB, t1 = min(M, t0 + kOuterRB);
    double sa[G], su[G];
#pragma unroll
    for (int g = 0; g < G; ++g) sa[g] = su[g] = 0.0;
    const int32_t* id = idx + (int64_t)c * M;
    const float* as = a_sorted + (int64_t)c * M;
    const float* ss = s_sorted + (int64_t)c * M;
#pragma unroll 4
    for (int64_t t = t0; t < t1; ++t) {
        const double x = (double)__ldg(X + (int64_t)id[t] * ldx + k);
        const double a = (double)as[t], s = (double)ss[t];
        if constexpr (OP == 0) {
            const double u = s * x;
            sa[0] += a * u;
            su[0] += u;
        } else if constexpr (OP == 1) {
            if (s > 0.0) { sa[0] += a * x; su[0] += x; }
            else if (s < 0.0) { sa[1] += a * x; su[1] += x; }
        } else {
            sa[0] += (s * a) * x;  // w_j X[j][k]
        }
    }
    double* out = part + ((((int64_t)c * nb + b) * q + k) * G) * 2;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        out[2 * g] = sa[g];
        out[2 * g + 1] = su[g];
    }
}

// Y[i][k] (+)= [X[i][k] - ] sigma_i (L + a_i (T - U)) [+ bias_i] over the rows of block b in sorted order.
// accumulate: add to Y (second component); subtract: Y = X - Q X; bias (nullable): + bias[i].
template <int OP>
__global__ void __launch_bounds__(kOuterThreads) k_outer_apply(const float* __restrict__ X, int64_t M, int64_t q,
                                                              int64_t ldx, const int32_t* __restrict__ idx,
                                                              const float* __restrict__ a_sorted,
                                                              const float* __restrict__ s_sorted, int c,
                                                              const double* __restrict__ part, float* __restrict__ Y,
                                                              int64_t ldy, int accumulate, int subtract,
                                                              const float* __restrict__ bias) {
    constexpr int G = OP == 1 ? 2 : 1;
    const int64_t k = (int64_t)blockIdx.x * kOuterThreads + threadIdx.x;
    const int64_t b = blockIdx.y, nb = gridDim.y;
    if (k >= q) return;
    // prefix over the preceding blocks (block order) and totals
    double L[G], U[G], T[G];
#pragma unroll
    for (int g = 0; g < G; ++g) L[g] = U[g] = T[g] = 0.0;
    for (int64_t bb = 0; bb < nb; ++bb) {
        const double* pp = part + ((((int64_t)c * nb + bb) * q + k) * G) * 2;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if (bb < b) {
                L[g] += pp[2 * g];
                U[g] += pp[2 * g + 1];
            }
            T[g] += OP == 2 ? pp[2 * g] : pp[2 * g + 1];
        }
    }
    const int64_t t0 = b * kOuterRB, t1 = min(M, t0 + kOuterRB);
    const int32_t* id = idx + (int64_t)c * M;
    const float* as = a_sorted + (int64_t)c * M;
    const float* ss = s_sorted + (int64_t)c * M;
#pragma unroll 2
    for (int64_t t = t0; t < t1; ++t) {
        const int64_t i = id[t];
        const double x = (double)__ldg(X + i * ldx + k);
        const double a = (double)as[t], s = (double)ss[t];
        double qx;
        if constexpr (OP == 0) {
            const double u = s * x;
            L[0] += a * u;
            U[0] += u;
            qx = s * (L[0] + a * (T[0] - U[0]));
        } else if constexpr (OP == 1) {
            if (s > 0.0) {
                L[0] += a * x;
                U[0] += x;
                qx = L[0] + a * (T[0] - U[0]);
            } else if (s < 0.0) {
                L[1] += a * x;
                U[1] += x;
                qx = L[1] + a * (T[1] - U[1]);
            } else {
                qx = 0.0;
            }
        } else {
            qx = (s * a) * T[0];  // w_i (w^T X)[k]
        }
        float* yp = Y + i * ldy + k;
        double v = subtract ? x - qx : qx;
        if (accumulate) v += (double)*yp;
        if (bias) v += (double)bias[i];
        *yp = (float)v;
    }
}

// Alg. 2 step 3: m_i = mean_j V[i][j] (fp64, j in order), Xc = V - m.  One thread per row.
__global__ void k_center_rows(const float* __restrict__ V, int64_t M, int64_t N, int64_t ldv, float* __restrict__ Xc,
                              int64_t ldx, float* __restrict__ mean) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    double s = 0.0;
    for (int64_t j = 0; j < N; ++j) s += (double)V[i * ldv + j];
    const double m = s / (double)N;
    for (int64_t j = 0; j < N; ++j) Xc[i * ldx + j] = (float)((double)V[i * ldv + j] - m);
    mean[i] = (float)m;
}

}  // namespace mapi
