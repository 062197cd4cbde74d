// probe_bulk_hbm.cu — investigation: HBM read rate of 1 KB row chunks streamed by (a) LDG.256 per lane
// (K2s's task pattern, register double buffer) vs (b) per-warp cp.async.bulk rings in shared memory
// (TMA engine, no registers held), over a 4 GiB buffer, one pass; 148 CTAs x 512 threads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) k_ldg(const float* __restrict__ A, int64_t chunks, float* out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 5), W = (int64_t)gridDim.x * 16;
    float acc = 0.f;
    for (int64_t c = gw; c < chunks; c += W * 4) {
        float v[4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t cc = c + u * W;
            const float* p = A + cc * 256 + 8 * lane;
            if (cc < chunks)
                asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=f"(v[u][0]), "=f"(v[u][1]), "=f"(v[u][2]), "=f"(v[u][3]), "=f"(v[u][4]), "=f"(v[u][5]),
                               "=f"(v[u][6]), "=f"(v[u][7])
                             : "l"(p));
            else
                for (int e = 0; e < 8; ++e) v[u][e] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc += v[u][e];
    }
    if (acc == 1234.5f) out[0] = acc;
}

template <int SLOTS>
__global__ void __launch_bounds__(512, 1) k_bulk(const float* __restrict__ A, int64_t chunks, float* out) {
    extern __shared__ __align__(128) float ring[];  // 16 warps x SLOTS x 256 floats
    __shared__ __align__(8) uint64_t bars[16 * SLOTS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * 16 + warp, W = (int64_t)gridDim.x * 16;
    float* my = ring + (size_t)warp * SLOTS * 256;
    uint64_t* mb = bars + warp * SLOTS;
    if (lane == 0)
        for (int s = 0; s < SLOTS; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t mine = gw < chunks ? (chunks - 1 - gw) / W + 1 : 0;  // this warp's chunks gw, gw + W, ...
    auto issue = [&](int64_t i) {
        if (lane == 0 && i < mine) {
            const int s = (int)(i % SLOTS);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 1024;" ::"r"(smem_u32(mb + s)) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];" ::"r"(
                             smem_u32(my + s * 256)),
                         "l"(A + (gw + i * W) * 256), "r"(smem_u32(mb + s))
                         : "memory");
        }
    };
    for (int64_t i = 0; i < SLOTS; ++i) issue(i);
    float acc = 0.f;
    for (int64_t i = 0; i < mine; ++i) {
        const int s = (int)(i % SLOTS);
        const uint32_t ph = (uint32_t)((i / SLOTS) & 1);
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                         : "=r"(ok)
                         : "r"(smem_u32(mb + s)), "r"(ph)
                         : "memory");
        const float4* q = reinterpret_cast<const float4*>(my + s * 256) + 2 * lane;
        const float4 x = q[0], y = q[1];
        acc += ((x.x + x.y) + (x.z + x.w)) + ((y.x + y.y) + (y.z + y.w));
        __syncwarp();
        issue(i + SLOTS);
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    const int64_t bytes = 4ll << 30, chunks = bytes / 1024;
    float *A, *out;
    cudaMalloc(&A, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(A, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b);
        cudaError_t e = cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-40s %7.3f TB/s %s\n", name, bytes * 5 / (ms * 1e-3) / 1e12, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    timeit("LDG.256, 4 chunks in flight per warp", [&]() { k_ldg<<<sms, 512>>>(A, chunks, out); });
    cudaFuncSetAttribute(k_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 8 * 1024);
    timeit("bulk ring, 8 x 1 KB slots per warp", [&]() { k_bulk<8><<<sms, 512, 16 * 8 * 1024>>>(A, chunks, out); });
    cudaFuncSetAttribute(k_bulk<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 12 * 1024);
    timeit("bulk ring, 12 x 1 KB slots per warp", [&]() { k_bulk<12><<<sms, 512, 16 * 12 * 1024>>>(A, chunks, out); });
    return 0;
}
