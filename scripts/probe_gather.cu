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

// hot-prefix replication: v[0..H) is stored R times; SM s gathers from copy s % R (spreads the
// hottest lines of a power-law graph over R different L2 slices)
template <int U>
__global__ void gather_sum_rep(const int* __restrict__ col, long long nnz, const float* __restrict__ v,
                               const float* __restrict__ rep, int H, int R, float* out) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    const float* my = rep + (size_t)(smid % R) * H;
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride * U) {
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = (k + u * stride < nnz) ? __ldg(col + k + u * stride) : -1;
#pragma unroll
        for (int u = 0; u < U; ++u) acc += c[u] >= 0 ? __ldg((c[u] < H ? my : v) + c[u]) : 0.f;
    }
    if (acc == 1234.5f) out[0] = acc;
}
template <int U>
__global__ void stream_v4(const int4* __restrict__ col, long long n4, float* out) {
    int acc = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n4; k += stride * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) if (k + u * stride < n4) { int4 q = __ldg(col + k + u * stride); acc += q.x ^ q.y ^ q.z ^ q.w; }
    }
    if (acc == 12345) out[0] = (float)acc;
}

// col_idx read as int4 (4 consecutive columns per thread), 2 int4 = 8 gathers in flight per trip
__global__ void gather_sum_v4(const int4* __restrict__ col, long long n4, const float* __restrict__ v, float* out) {
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n4; k += 2 * stride) {
        int4 a = __ldg(col + k);
        int4 b = (k + stride < n4) ? __ldg(col + k + stride) : make_int4(-1, -1, -1, -1);
        const int c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += c[u] >= 0 ? __ldg(v + c[u]) : 0.f;
    }
    if (acc == 1234.5f) out[0] = acc;
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
    float t3 = timeit([&] { stream_v4<4><<<sms * 8, 256>>>((const int4*)col, nnz / 4, out); });
    printf("col_idx stream int4:          %8.1f us  %6.0f GB/s\n", t3 * 1e3, 4.0 * nnz / (t3 / 1e3) / 1e9);
    // edge share of the hottest prefixes
    for (int H : {1024, 8192, 65536}) {
        long long c = 0;
        for (long long k = 0; k < nnz; ++k) c += h[k] < H;
        printf("edges with col < %6d: %5.1f%%\n", H, 100.0 * c / nnz);
    }
    for (int g : {8, 16}) {
        float t5 = timeit([&] { gather_sum_v4<<<sms * g, 256>>>((const int4*)col, nnz / 4, v, out); });
        printf("gather_sum_v4 grid %dx256:    %8.1f us  %6.2f Ggather/s\n", sms * g, t5 * 1e3, nnz / (t5 / 1e3) / 1e9);
    }
    float* rep;
    CK(cudaMalloc(&rep, 4ll * 65536 * 32));
    CK(cudaMemset(rep, 0, 4ll * 65536 * 32));
    for (int H : {1024, 8192, 65536})
        for (int R : {4, 16, 32}) {
            float t4 = timeit([&] { gather_sum_rep<8><<<sms * 16, 256>>>(col, nnz, v, rep, H, R, out); });
            printf("gather_sum_rep H %6d R %2d:   %8.1f us  %6.2f Ggather/s\n", H, R, t4 * 1e3, nnz / (t4 / 1e3) / 1e9);
        }
    return 0;
}
