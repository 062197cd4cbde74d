// mapi_common.cuh — sm_100a device primitives shared by the MAPI kernels.
//
// The MAVP term (Eq. 3)  sign(a*w) * min(|a|,|w|)  is ONE instruction on sm_100a:
// PTX `min.xorsign.abs.f32` -> SASS `FMNMX.XORSIGN Rd, |Ra|, |Rb|` (the sign of the result is
// sign(a) XOR sign(w), its magnitude min(|a|,|w|); a zero operand yields +-0, which adds like 0,
// i.e. sign(0) = 0 as in reading Q1).  No multiply is involved anywhere in the MAVP loops (P:5).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mapi {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------------------------
// MAVP term. OP 0 = min1 (Eq. 3), OP 1 = min2 (Eq. 4: 1(sign a = sign w) min(|a|,|w|)).
// OP 2 = the regular product a*w of Eq. (1): the RPI comparator, the only
// operator with a multiply; it is never used by the MAVP entry points' default path.
template <int OP>
__device__ __forceinline__ float mavp_term(float a, float w) {
    if constexpr (OP == 2) {
        return a * w;
    } else {
        float d;
        asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(w));
        if constexpr (OP == 1) d = fmaxf(d, 0.0f);  // opposite signs -> 0 (indicator false)
        return d;
    }
}

// Per-element contribution to the normalisation and its finish: l1 for MAVP (Eq. 8),
// l2 for the regular product (Eq. 1).  Accumulated in fp64.
template <int OP>
__device__ __forceinline__ double norm_part(float v) {
    if constexpr (OP == 2) return (double)v * (double)v;
    else return (double)fabsf(v);
}
template <int OP>
__device__ __forceinline__ double norm_final(double s) {
    if constexpr (OP == 2) return sqrt(s);
    else return s;
}

// ---------------------------------------------------------------------------------------------
// Streaming loads of the matrix. POL 0: L2 evict-first (matrix >> L2, read once per iteration);
// POL 1: default L2 policy (matrix may stay L2-resident across iterations). L1 no-allocate.
template <int VEC, int POL>
__device__ __forceinline__ void ld_stream(const float* p, float (&v)[VEC]) {
    if constexpr (VEC == 8) {
        if constexpr (POL == 0)
            asm volatile(
                "ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                  "=f"(v[7])
                : "l"(p));
        else
            asm volatile(
                "ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                  "=f"(v[7])
                : "l"(p));
    } else if constexpr (VEC == 4) {
        // (the .L2::evict_first qualifier exists only for 256-bit loads; narrower paths are
        //  the unaligned fallbacks and use the default L2 policy)
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
                     : "l"(p));
    } else {
        asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v[0]) : "l"(p));
    }
}

// The iterate vector: from shared memory (WG = false) or global memory through L1 (WG = true).
template <int VEC, bool WG>
__device__ __forceinline__ void ld_vec(const float* p, float (&v)[VEC]) {
    if constexpr (VEC == 8) {
        float4 a, b;
        if constexpr (WG) {
            a = __ldg(reinterpret_cast<const float4*>(p));
            b = __ldg(reinterpret_cast<const float4*>(p) + 1);
        } else {
            a = reinterpret_cast<const float4*>(p)[0];
            b = reinterpret_cast<const float4*>(p)[1];
        }
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else if constexpr (VEC == 4) {
        float4 a = WG ? __ldg(reinterpret_cast<const float4*>(p)) : reinterpret_cast<const float4*>(p)[0];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
        v[0] = WG ? __ldg(p) : p[0];
    }
}

// ---------------------------------------------------------------------------------------------
// Deterministic reductions (fixed order for a fixed launch shape; no float atomics).

// Butterfly: every lane ends with the same bit pattern (fp add is commutative).
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Block sum; `scratch` holds >= 32 floats; result broadcast to all threads.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();  // scratch reuse guard
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        T x = lane < nw ? scratch[lane] : T(0);
        x = warp_sum(x);
        if (lane == 0) scratch[32] = x;
    }
    __syncthreads();
    return scratch[32];
}

// Pairwise tree over a small register array (fixed shape).
template <int N>
__device__ __forceinline__ float tree_sum(const float (&a)[N]) {
    if constexpr (N == 1) {
        return a[0];
    } else if constexpr (N == 2) {
        return a[0] + a[1];
    } else if constexpr (N == 4) {
        return (a[0] + a[1]) + (a[2] + a[3]);
    } else {
        static_assert(N == 8, "tree_sum supports 1, 2, 4, 8");
        return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
}

// ---------------------------------------------------------------------------------------------
// Grid barrier for cooperative (co-resident) launches: a monotonically increasing arrival
// counter; the epoch-th barrier waits until counter >= epoch * gridDim.x.  The counter is
// zeroed by the host (stream-ordered memset) before each launch.  Targets are taken modulo
// 2^32 and compared wrap-safely (a signed difference), so runs longer than 2^32 / gridDim.x
// barriers stay correct: the counter never leads a waiter's target by 2^31 or more.
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
        unsigned int v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        } while ((int)(v - target) < 0);
        __threadfence();
    }
    __syncthreads();
}

// L2-coherent load of data written by other CTAs of the same launch (bypasses L1).
__device__ __forceinline__ float ld_cg(const float* p) { return __ldcg(p); }

}  // namespace mapi
