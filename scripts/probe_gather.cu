// probe_gather.cu — ceiling of the CSR ranking step's gather on THIS graph: sum over all nonzeros of
// v[col_idx[k]] (coalesced col_idx stream + scattered 4-byte gathers from a 16 MB vector), vs the
// col_idx stream alone.  Investigation tool; input: the cfg5 col_idx dumped by scripts/dump_cfg5.py.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int U>
__global__ void gather_sum(const int* __restrict__ col, long long nnz, const float* __restrict__ v, float* out) {
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride * U) {
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = (k + u * stride < nnz) ? __ldg(col + k + u * stride) : -1;
#pragma unroll
        for (int u = 0; u < U; ++u) acc += c[u] >= 0 ? __ldg(v + c[u]) : 0.f;
    }
    if (acc == 1234.5f) out[0] = acc;
}
template <int U>
__global__ void stream_only(const int* __restrict__ col, long long nnz, float* out) {
    int acc = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) if (k + u * stride < nnz) acc += __ldg(col + k + u * stride);
    }
    if (acc == 12345) out[0] = (float)acc;
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
    }
    return best;
}

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "/tmp/cfg5_col.bin";
    const long long n = argc > 2 ? atoll(argv[2]) : (1LL << 22);
    FILE* f = fopen(path, "rb");
    if (!f) { printf("cannot open %s\n", path); return 1; }
    fseek(f, 0, SEEK_END); long long nnz = ftell(f) / 4; fseek(f, 0, SEEK_SET);
    std::vector<int> h(nnz);
    if (fread(h.data(), 4, nnz, f) != (size_t)nnz) { printf("short read\n"); return 1; }
    fclose(f);
    int *col; float *v, *out;
    CK(cudaMalloc(&col, 4 * nnz)); CK(cudaMalloc(&v, 4 * n)); CK(cudaMalloc(&out, 64));
    CK(cudaMemcpy(col, h.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemset(v, 0, 4 * n));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("nnz %lld  n %lld\n", nnz, n);
    for (int g : {4, 8, 16}) {
        float t1 = timeit([&] { gather_sum<8><<<sms * g, 256>>>(col, nnz, v, out); });
        printf("gather_sum U8 grid %dx256: %8.1f us  %6.2f Ggather/s  col stream %6.0f GB/s\n", sms * g, t1 * 1e3,
               nnz / (t1 / 1e3) / 1e9, 4.0 * nnz / (t1 / 1e3) / 1e9);
    }
    float t2 = timeit([&] { stream_only<8><<<sms * 8, 256>>>(col, nnz, out); });
    printf("col_idx stream only:          %8.1f us  %6.0f GB/s\n", t2 * 1e3, 4.0 * nnz / (t2 / 1e3) / 1e9);
    return 0;
}
