// probe_hub.cu — investigation: would a shared-memory cache of the highest out-degree sources cut the
// CSR ranking gather (cfg5)?  Relabels source ids by descending out-degree (host), then compares the
// gather-sum over all nonzeros: original ids / relabelled ids / relabelled + the first K v values in
// shared memory (persistent grid, one CTA per SM loads them once per launch).
// Input: the cfg5 col_idx dumped by scripts/dump_cfg5.py.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void gather_plain(const int* __restrict__ col, long long nnz, const float* __restrict__ v, float* out) {
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; k0 < nnz; k0 += stride * 8) {
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = (k0 + u * stride < nnz) ? __ldg(col + k0 + u * stride) : -1;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += c[u] >= 0 ? __ldg(v + c[u]) : 0.f;
    }
    if (acc == 1234.5f) out[0] = acc;
}

template <int K>
__global__ void __launch_bounds__(1024, 1) gather_hub(const int* __restrict__ col, long long nnz, const float* __restrict__ v,
                                                      float* out) {
    extern __shared__ float hub[];
    for (int i = threadIdx.x; i < K; i += blockDim.x) hub[i] = v[i];
    __syncthreads();
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; k0 < nnz; k0 += stride * 8) {
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = (k0 + u * stride < nnz) ? __ldg(col + k0 + u * stride) : -1;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += c[u] < 0 ? 0.f : (c[u] < K ? hub[c[u]] : __ldg(v + c[u]));
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "/tmp/cfg5_col.bin";
    FILE* f = fopen(path, "rb");
    if (!f) { printf("no %s\n", path); return 1; }
    fseek(f, 0, SEEK_END);
    const long long nnz = ftell(f) / 4;
    fseek(f, 0, SEEK_SET);
    std::vector<int> col(nnz);
    if (fread(col.data(), 4, nnz, f) != (size_t)nnz) return 1;
    fclose(f);
    const int n = 1 << 22;
    std::vector<int> deg(n, 0);
    for (long long k = 0; k < nnz; ++k) deg[col[k]]++;
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return deg[a] > deg[b]; });
    std::vector<int> perm(n);
    for (int i = 0; i < n; ++i) perm[order[i]] = i;
    std::vector<int> col2(nnz);
    for (long long k = 0; k < nnz; ++k) col2[k] = perm[col[k]];
    long long cum = 0;
    for (int K : {8192, 16384, 32768, 49152}) {
        cum = 0;
        for (int i = 0; i < K; ++i) cum += deg[order[i]];
        printf("top %d sources: %.3f of the edges\n", K, (double)cum / nnz);
    }
    int *dc, *dc2; float *dv, *dout;
    CK(cudaMalloc(&dc, 4 * nnz)); CK(cudaMalloc(&dc2, 4 * nnz)); CK(cudaMalloc(&dv, 4ll * n)); CK(cudaMalloc(&dout, 4));
    CK(cudaMemcpy(dc, col.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dc2, col2.data(), 4 * nnz, cudaMemcpyHostToDevice));
    std::vector<float> hv(n);
    for (int i = 0; i < n; ++i) hv[i] = 1e-7f * (1 + (i % 13));
    CK(cudaMemcpy(dv, hv.data(), 4ll * n, cudaMemcpyHostToDevice));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) launch();
        cudaEventRecord(b);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-48s %8.1f us\n", name, 1e3 * ms / 10);
    };
    timeit("gather, original ids", [&]() { gather_plain<<<sms * 8, 256>>>(dc, nnz, dv, dout); });
    timeit("gather, relabelled by out-degree", [&]() { gather_plain<<<sms * 8, 256>>>(dc2, nnz, dv, dout); });
    auto hubrun = [&](auto kern, int K, const char* name) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * K));
        timeit(name, [&]() { kern<<<sms, 1024, 4 * K>>>(dc2, nnz, dv, dout); });
    };
    hubrun(gather_hub<16384>, 16384, "relabelled + 16K hub values in smem");
    hubrun(gather_hub<32768>, 32768, "relabelled + 32K hub values in smem");
    hubrun(gather_hub<49152>, 49152, "relabelled + 48K hub values in smem");
    return 0;
}
