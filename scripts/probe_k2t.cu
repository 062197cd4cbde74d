// probe_k2t.cu — per-phase cycle breakdown of the K2t bulk-ring iteration (investigation only):
// compiled with -DMAPI_BULK_TRACE so CTA 0 / thread 0 stamps clock64 at: iteration start, its warp's
// items done, all warps' items done (__syncthreads), after the grid barrier, after s_t, after delta.
// n = 4096 (cfg2 size), random data, 60 iterations.
#include <cstdio>
#include <vector>
#include "../paper_2110_12065_b200/csrc/bulk.cuh"
using namespace mapi;

int main() {
    const int n = 4096, T = 60;
    std::vector<float> hA((size_t)n * n), hb(n, 1.0f / 64);
    unsigned s = 1;
    for (auto& x : hA) { s = s * 1664525u + 1013904223u; x = ((s >> 8) / 16777216.0f - 0.5f); }
    for (int i = 0; i < n; ++i) hA[(size_t)i * n + i] += 4.0f;
    float *A, *b0, *w, *y, *norms, *deltas; double* slots; unsigned* bar; int* st;
    cudaMalloc(&A, 4ull * n * n); cudaMalloc(&b0, 4 * n); cudaMalloc(&w, 4 * n); cudaMalloc(&y, 8 * n);
    cudaMalloc(&norms, 4 * T); cudaMalloc(&deltas, 4 * T); cudaMalloc(&slots, 8 * 4096); cudaMalloc(&bar, 256);
    cudaMalloc(&st, 8);
    cudaMemcpy(A, hA.data(), 4ull * n * n, cudaMemcpyHostToDevice);
    cudaMemcpy(b0, hb.data(), 4 * n, cudaMemcpyHostToDevice);
    int sms, optin;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    const int grid = sms;
    const size_t fixed = bulk_fixed_smem(n, (n + grid - 1) / grid);
    int slotsN = (int)std::min<size_t>(kBulkMaxSlots, (optin - fixed) / (4 * kBulkChunk));
    slotsN = slotsN / kBulkNC * kBulkNC;
    const size_t smem = fixed + 4ull * kBulkChunk * slotsN;
    cudaFuncSetAttribute(k_iterate_bulk<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    IterArgs a{};
    a.A = A; a.n = n; a.lda = n; a.b0 = b0; a.iters = T; a.tol = 0; a.w_out = w; a.norms = norms; a.deltas = deltas;
    a.y = y; a.slots = reinterpret_cast<float*>(slots); a.bar = bar; a.status = st;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 256);
        void* args[] = {&a, &slotsN};
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_iterate_bulk<0>, dim3(grid), dim3(kBulkThreads),
                                                    args, smem, 0);
        if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
        if ((e = cudaDeviceSynchronize()) != cudaSuccess) { printf("sync: %s\n", cudaGetErrorString(e)); return 1; }
    }
    std::vector<long long> h(6 * 512);
    cudaMemcpyFromSymbol(h.data(), g_bulk_trace, 8 * 6 * 512);
    double ph[5] = {0, 0, 0, 0, 0}, tot = 0;
    int cnt = 0;
    for (int t = 10; t < T - 1; ++t, ++cnt) {
        for (int k = 0; k < 5; ++k) ph[k] += h[t * 6 + k + 1] - h[t * 6 + k];
        tot += h[(t + 1) * 6] - h[t * 6];
    }
    printf("K2t n=4096 slots=%d cycles/iteration: own items %.0f | wait other warps %.0f | rows+blocksum+grid barrier %.0f"
           " | s_t (+y loads) %.0f | w + delta %.0f | total %.0f\n",
           slotsN, ph[0] / cnt, ph[1] / cnt, ph[2] / cnt, ph[3] / cnt, ph[4] / cnt, tot / cnt);
    return 0;
}
