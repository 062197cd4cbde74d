// probe_tmem.cu — investigation only: can TMEM (256 KB/SM) + shared memory hold a mid-size MAPI matrix
// on chip, and how fast can the MAVP row pass read it back?
//
// One CTA of 512 threads per SM (cfg2's D_i: 4096 x 4096 fp32 = 64 MiB = 148 x ~453 KB).  Thread
// (quarter q = warp % 4, lane l) owns the 32 columns [32L, 32L + 32) with L = 32q + l of every row it
// touches; warp group s = warp / 4 owns 4 TMEM rows (TMEM columns [128s, 128s + 128) of its 32 lanes)
// and 3 shared-memory rows.  Modes (cycles per pass, all 16 warps, one __syncthreads per pass):
//   0: TMEM read only (4 x tcgen05.ld 32x32b.x32 per warp = 256 KB per SM per pass) + 1 FADD per value
//   1: shared-memory rows only (3 rows x 8 LDS.128 per thread = 192 KB per SM per pass) + MAVP terms
//   2: both, the full on-chip MAVP pass (4 TMEM rows + 3 smem rows, 224 terms per thread)
//   3: registers only (224 terms from register-resident A): the ALU floor of the pass
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float term(float a, float w) {
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(w));
    return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long pack2(float x, float y) {
    return (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(y) << 32);
}
__device__ __forceinline__ void tmem_ld32(uint32_t ta, float (&v)[32]) {
    uint32_t* r = reinterpret_cast<uint32_t*>(v);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta));
}
__device__ __forceinline__ void tmem_st32(uint32_t ta, const float (&v)[32]) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

// 32 terms of one row chunk against the thread's 32 w values -> one partial (4 chains, pairwise)
__device__ __forceinline__ float row32(const float (&a)[32], const float (&w)[32]) {
    unsigned long long p0 = 0, p1 = 0;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        p0 = fadd2(p0, pack2(term(a[4 * m], w[4 * m]), term(a[4 * m + 1], w[4 * m + 1])));
        p1 = fadd2(p1, pack2(term(a[4 * m + 2], w[4 * m + 2]), term(a[4 * m + 3], w[4 * m + 3])));
    }
    return (__uint_as_float((uint32_t)p0) + __uint_as_float((uint32_t)(p0 >> 32))) +
           (__uint_as_float((uint32_t)p1) + __uint_as_float((uint32_t)(p1 >> 32)));
}

template <int MODE, int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_probe(int passes, float* out, long long* cyc) {
    constexpr int SUBS = NW / 4, TR = 16 / SUBS, SR = 12 / SUBS;  // TMEM / smem rows per warp group
    extern __shared__ __align__(16) float sm[];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, q = warp & 3, s = warp >> 2;
    const int L = 32 * q + lane;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + 32u * TR * s;
    // fill: smem rows 12 x 4096, TMEM 16 rows x 32 columns per lane, w
    for (int i = tid; i < 12 * 4096; i += NW * 32) sm[i] = (float)((i * 2654435761u) >> 20) * 1e-3f - 2.0f;
    float w[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) w[k] = 1e-3f * (float)((L * 32 + k) % 97) - 0.04f;
    {
        float v[32];
#pragma unroll
        for (int r = 0; r < TR; ++r) {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[k] = (float)((r * 7 + k + L) % 13) - 6.0f;
            tmem_st32(ta + 32u * r, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    float areg[2][32];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < 32; ++k) areg[r][k] = (float)((r * 5 + k * 3 + L) % 11) - 5.0f;
    __syncthreads();
    float tot = 0.0f;
    long long t0 = clock64();
    for (int p = 0; p < passes; ++p) {
        float part[TR + SR];
        if constexpr (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int r = 0; r < TR; ++r) {
                float a[32];
                tmem_ld32(ta + 32u * r, a);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if constexpr (MODE == 0) {
                    float x = 0.0f;
#pragma unroll
                    for (int k = 0; k < 32; ++k) x += a[k];
                    part[r] = x;
                } else {
                    part[r] = row32(a, w);
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < TR; ++r) part[r] = 0.0f;
        }
        if constexpr (MODE == 1 || MODE == 2) {
#pragma unroll
            for (int r = 0; r < SR; ++r) {
                const float4* rp = reinterpret_cast<const float4*>(sm + (size_t)(s * SR + r) * 4096) + 8 * L;
                float a[32];
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    const int c = (m + lane) & 7;  // rotated chunk order: conflict-free LDS.128
                    const float4 v = rp[c];
                    a[4 * m] = v.x; a[4 * m + 1] = v.y; a[4 * m + 2] = v.z; a[4 * m + 3] = v.w;
                }
                part[TR + r] = row32(a, w);
            }
        } else if constexpr (MODE == 3) {
#pragma unroll
            for (int r = 0; r < TR + SR; ++r) part[r] = row32(areg[r & 1], w);
        } else {
#pragma unroll
            for (int r = 0; r < SR; ++r) part[TR + r] = 0.0f;
        }
        float x = 0.0f;
#pragma unroll
        for (int r = 0; r < TR + SR; ++r) x += part[r];
        tot += x;
#pragma unroll
        for (int k = 0; k < 32; ++k) w[k] = __int_as_float(__float_as_int(w[k]) ^ (__float_as_int(x) & 0x80000000));
        __syncthreads();
    }
    long long t1 = clock64();
    out[blockIdx.x * 512 + tid] = tot;
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int MODE, int NW>
void run(int sms, float* out, long long* cyc, const char* name0) {
    char name[128];
    snprintf(name, sizeof name, "%s [%d warps]", name0, NW);
    const int smem = 12 * 4096 * 4 + 1024;
    cudaFuncSetAttribute(k_probe<MODE, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int passes = 2000;
    k_probe<MODE, NW><<<sms, NW * 32, smem>>>(passes, out, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_probe<MODE, NW><<<sms, NW * 32, smem>>>(passes, out, cyc);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long h[1024];
    cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%-34s %8.0f cycles/pass (max over SMs)  %6.3f us/pass (events)\n", name, mx / passes, 1e3 * ms / passes);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, 4 * 512 * sms);
    cudaMalloc(&cyc, 8 * sms);
    run<0, 16>(sms, out, cyc, "TMEM read 256 KB/SM");
    run<1, 16>(sms, out, cyc, "smem rows 192 KB/SM + terms");
    run<2, 16>(sms, out, cyc, "TMEM + smem full pass");
    run<3, 16>(sms, out, cyc, "register-only terms (same count)");
    run<0, 8>(sms, out, cyc, "TMEM read 256 KB/SM");
    run<1, 8>(sms, out, cyc, "smem rows 192 KB/SM + terms");
    run<2, 8>(sms, out, cyc, "TMEM + smem full pass");
    run<3, 8>(sms, out, cyc, "register-only terms (same count)");
    return 0;
}
