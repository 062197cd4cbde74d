// probe_task_shape.cu — investigation for K2s: HBM read rate of warp tasks of R rows x (CW x 1 KB) columns of a
// 32768 x 32768 fp32 matrix (row stride 128 KB), every lane loading 32 B per row piece with LDG.256
// evict-first, 8 loads in flight per lane (K2s's register double buffer), 148 CTAs x 16 warps, tasks dealt
// round-robin (static) or from a counter (dynamic).  R x CW = 128 always (128 KB per task, K2s's size).
// Question: does a wider contiguous run per row (2 / 4 / 8 KB instead of K2s's 1 KB) raise the DRAM rate?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld8(float (&v)[8], const float* p) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}

// CW: 1 KB pieces per row of a task; R = 128 / CW rows.  Task t: row block t / (n / (256 CW)) ... row-major
// over (row block, column block).  DYN: tasks from a global counter.
template <int CW, bool DYN>
__global__ void __launch_bounds__(512, 1) k_tasks(const float* __restrict__ A, int64_t n, int64_t ntasks,
                                                  unsigned long long* counter, float* out) {
    constexpr int R = 128 / CW;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 5), W = (int64_t)gridDim.x * 16;
    const int64_t cblocks = n / (256 * CW);
    float acc = 0.f;
    int64_t t = gw;
    if (DYN) {
        unsigned long long x = 0;
        if (lane == 0) x = atomicAdd(counter, 1ull);
        t = (int64_t)__shfl_sync(0xffffffffu, x, 0);
    }
    while (t < ntasks) {
        const int64_t rb = t / cblocks, cb = t % cblocks;
        const float* base = A + rb * R * n + cb * 256 * CW + 8 * lane;
        // pieces of the task in row-major order: piece q -> row q / CW, 1 KB piece q % CW; 4 pieces per batch,
        // two batches in flight
        float v[2][4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) ld8(v[0][u], base + (int64_t)(u / CW) * n + (u % CW) * 256);
#pragma unroll 1
        for (int q = 4; q < 128; q += 8) {
#pragma unroll
            for (int u = 0; u < 4; ++u) ld8(v[1][u], base + (int64_t)((q + u) / CW) * n + ((q + u) % CW) * 256);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc += v[0][u][e];
            if (q + 4 < 128) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    ld8(v[0][u], base + (int64_t)((q + 4 + u) / CW) * n + ((q + 4 + u) % CW) * 256);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc += v[1][u][e];
        }
        if (DYN) {
            unsigned long long x = 0;
            if (lane == 0) x = atomicAdd(counter, 1ull);
            t = (int64_t)__shfl_sync(0xffffffffu, x, 0);
        } else {
            t += W;
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    const int64_t n = 32768, bytes = n * n * 4, ntasks = bytes / (128 * 1024);
    float *A, *out;
    unsigned long long* counter;
    cudaMalloc(&A, bytes);
    cudaMalloc(&out, 4);
    cudaMalloc(&counter, 8);
    cudaMemset(A, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        float best = 1e9f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(counter, 0, 8);
            launch();
            cudaDeviceSynchronize();
            cudaMemset(counter, 0, 8);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (e != cudaSuccess) printf("%s: %s\n", name, cudaGetErrorString(e));
            best = ms < best ? ms : best;
        }
        printf("%-52s %7.3f TB/s (%.3f ms per 4 GiB pass)\n", name, bytes / (best * 1e-3) / 1e12, best);
    };
#define RUN(CW)                                                                                                   \
    timeit("static  tasks " #CW " KB x (128/" #CW ") rows",                                                       \
           [&]() { k_tasks<CW, false><<<sms, 512>>>(A, n, ntasks, counter, out); });                               \
    timeit("dynamic tasks " #CW " KB x (128/" #CW ") rows",                                                       \
           [&]() { k_tasks<CW, true><<<sms, 512>>>(A, n, ntasks, counter, out); });
    RUN(1)
    RUN(2)
    RUN(4)
    RUN(8)
    RUN(32)
    RUN(128)
    return 0;
}
