// probe_k2r.cu — per-phase cycle breakdown of the K2r on-chip-resident iteration (investigation only):
// compiled with -DMAPI_RES_TRACE so CTA 0 / thread 0 stamps clock64 at: iteration start, pass done,
// after the first __syncthreads, y published, y gathered, s_t known, quotients done, delta_t known.
// n = 4096 (cfg2 size), random data, 200 iterations; warp counts, register rows (RR), cluster-pair epilogue (CL).
#include <cstdio>
#include <vector>
#include "../paper_2110_12065_b200/csrc/resident.cuh"
using namespace mapi;

template <int NW, int CL, int RR = 0>
void run(float* A, float* b0, float* w, float* y, float* norms, float* deltas, double* slots, unsigned* bar, int* st,
         int n, int T, int grid) {
    auto kern = k_iterate_resident<0, NW, CL, RR>;
    const size_t smem = resident_smem_bytes(kResSmemRows - (NW / 4) * RR);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    IterArgs a{};
    a.A = A; a.n = n; a.lda = n; a.b0 = b0; a.iters = T; a.tol = 0; a.w_out = w; a.norms = norms; a.deltas = deltas;
    a.y = y; a.slots = reinterpret_cast<float*>(slots); a.bar = bar; a.status = st;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 256);
        cudaMemset(y, 0, 16 * n);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(NW * 32); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = CL; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 2;
        cudaEventRecord(e0);
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
        cudaEventRecord(e1);
        if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return; }
        if ((e = cudaDeviceSynchronize()) != cudaSuccess) { printf("sync: %s\n", cudaGetErrorString(e)); return; }
        cudaEventElapsedTime(&ms, e0, e1);
    }
    std::vector<long long> h(8 * 512);
    cudaMemcpyFromSymbol(h.data(), g_res_trace, 8 * 8 * 512);
    double ph[7] = {0, 0, 0, 0, 0, 0, 0}, tot = 0;
    const int ord[8] = {0, 1, 2, 3, 4, 5, 7, 6};  // stamp order within an iteration
    int cnt = 0;
    for (int t = 20; t < T - 1; ++t, ++cnt) {
        for (int k = 0; k < 7; ++k) ph[k] += h[t * 8 + ord[k + 1]] - h[t * 8 + ord[k]];
        tot += h[(t + 1) * 8] - h[t * 8];
    }
    {
        std::vector<int> pr(148 * 512);
        cudaMemcpyFromSymbol(pr.data(), g_res_polls, 4 * 148 * 512);
        double m0 = 0, mall = 0; int mx = 0;
        for (int t = 20; t < T - 1; ++t) {
            m0 += pr[t];
            for (int c = 0; c < grid; ++c) { mall += pr[c * 512 + t]; mx = pr[c * 512 + t] > mx ? pr[c * 512 + t] : mx; }
        }
        printf("  poll rounds: CTA0 mean %.2f, all-CTA mean %.2f, max %d\n", m0 / (T - 21), mall / (T - 21) / grid, mx);
    }
    printf("K2r NW=%d CL=%d RR=%d: %.2f us/iteration (events, incl. staging) | cycles: pass %.0f | reduce+sync %.0f | "
           "publish %.0f | gather y %.0f | |y| partial + sync %.0f | s, 1/s, quotients, delta partial %.0f | "
           "delta reduce + sync %.0f | total %.0f\n",
           NW, CL, RR, 1e3 * ms / T, ph[0] / cnt, ph[1] / cnt, ph[2] / cnt, ph[3] / cnt, ph[4] / cnt,
           ph[5] / cnt, ph[6] / cnt, tot / cnt);
}

__global__ void k_dfma(double* out, int reps) {
    double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9, d = a + 1, e = a + 2, f = a + 3;
    for (int i = 0; i < reps; ++i) {
        a = fma(a, b, c); d = fma(d, b, c); e = fma(e, b, c); f = fma(f, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f;
}
__global__ void k_ddiv(double* out, int reps) {
    double a = threadIdx.x * 1e-3 + 1.0, r = 0;
    for (int i = 0; i < reps; ++i) { r += 1.0 / a; a += 1e-7; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    const int n = 4096, T = 200;
    std::vector<float> hA((size_t)n * n), hb(n, 1.0f / 64);
    unsigned s = 1;
    for (auto& x : hA) { s = s * 1664525u + 1013904223u; x = ((s >> 8) / 16777216.0f - 0.5f); }
    for (int i = 0; i < n; ++i) hA[(size_t)i * n + i] += 4.0f;
    float *A, *b0, *w, *y, *norms, *deltas; double* slots; unsigned* bar; int* st;
    cudaMalloc(&A, 4ull * n * n); cudaMalloc(&b0, 4 * n); cudaMalloc(&w, 4 * n); cudaMalloc(&y, 16 * n);
    cudaMalloc(&norms, 4 * T); cudaMalloc(&deltas, 4 * T); cudaMalloc(&slots, 8 * 4096); cudaMalloc(&bar, 256);
    cudaMalloc(&st, 8);
    cudaMemcpy(A, hA.data(), 4ull * n * n, cudaMemcpyHostToDevice);
    cudaMemcpy(b0, hb.data(), 4 * n, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    {
        double* o; cudaMalloc(&o, 8 * 148 * 1024 * 4);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
        k_dfma<<<sms * 2, 1024>>>(o, 1000);
        cudaEventRecord(e0); k_dfma<<<sms * 2, 1024>>>(o, 10000); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("DFMA: %.1f lane-ops/clk/SM at 1965 MHz\n", 4.0 * 10000 * sms * 2 * 1024 / (ms * 1e-3) / sms / 1.965e9);
        k_ddiv<<<sms * 2, 1024>>>(o, 1000);
        cudaEventRecord(e0); k_ddiv<<<sms * 2, 1024>>>(o, 10000); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("1.0/x (DDIV): %.2f lane-ops/clk/SM at 1965 MHz\n", 1.0 * 10000 * sms * 2 * 1024 / (ms * 1e-3) / sms / 1.965e9);
    }
    run<8, 1, 0>(A, b0, w, y, norms, deltas, slots, bar, st, n, T, sms);
    run<8, 1, 1>(A, b0, w, y, norms, deltas, slots, bar, st, n, T, sms);
    run<8, 1, 2>(A, b0, w, y, norms, deltas, slots, bar, st, n, T, sms);
    run<8, 2, 2>(A, b0, w, y, norms, deltas, slots, bar, st, n, T, sms);
    run<16, 1, 0>(A, b0, w, y, norms, deltas, slots, bar, st, n, T, sms);
    return 0;
}
