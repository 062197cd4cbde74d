// probe_fp64.cu — measured fp64 issue rates on this B200 (DADD, DFMA, F2F.F64.F32 + DADD as in K3s's node pass).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int R = 8, ITERS = 4096;
__global__ void k_dadd(double* out, double s) {
    double x[R]; for (int i = 0; i < R; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < R; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[i]) : "d"(s));
    }
    double a = 0; for (int i = 0; i < R; ++i) a += x[i]; if (a == 1.2345) out[0] = a;
}
__global__ void k_dfma(double* out, double s) {
    double x[R]; for (int i = 0; i < R; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < R; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(x[i]) : "d"(s));
    }
    double a = 0; for (int i = 0; i < R; ++i) a += x[i]; if (a == 1.2345) out[0] = a;
}
__global__ void k_cvt_dadd(double* out, float s) {
    double x[R]; float f[R]; for (int i = 0; i < R; ++i) { x[i] = i; f[i] = threadIdx.x * 1e-3f + i; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < R; ++i) { double d; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f[i])); asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[i]) : "d"(d)); f[i] += s; }
    }
    double a = 0; for (int i = 0; i < R; ++i) a += x[i]; if (a == 1.2345) out[0] = a;
}
__global__ void k_cvt(double* out, float s) {
    double x[R]; float f[R]; for (int i = 0; i < R; ++i) { x[i] = i; f[i] = threadIdx.x * 1e-3f + i; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < R; ++i) { asm volatile("cvt.f64.f32 %0, %1;" : "=d"(x[i]) : "f"(f[i])); f[i] += s; }
    }
    double a = 0; for (int i = 0; i < R; ++i) a += x[i]; if (a == 1.2345) out[0] = a;
}
template <typename K, typename T>
void run(K k, const char* name, T s, int sms, int khz) {
    double* out; cudaMalloc(&out, 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) { cudaEventRecord(a); k<<<sms * 4, 512>>>(out, s); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms; }
    double lanes = (double)sms * 4 * 512 * ITERS * R;
    printf("%-20s %8.3f ms  %7.1f lane-ops/clk/SM at %d MHz\n", name, best, lanes / (best / 1e3) / sms / (khz * 1e3), khz / 1000);
}
int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); int khz = 0; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    printf("%s, %d SMs, %d kHz\n", p.name, p.multiProcessorCount, khz);
    run(k_dadd, "DADD", 0.5, p.multiProcessorCount, khz);
    run(k_dfma, "DFMA", 0.5, p.multiProcessorCount, khz);
    run(k_cvt, "F2F.F64.F32", 0.5f, p.multiProcessorCount, khz);
    run(k_cvt_dadd, "F2F + DADD", 0.5f, p.multiProcessorCount, khz);
    return 0;
}
