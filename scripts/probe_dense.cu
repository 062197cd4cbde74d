// probe_dense.cu — variant sweep of the persistent MAPI kernel at cfg3 size (n = 32768, 4 GiB) and
// a read-only streaming ceiling.  Investigation tool (not part of the library); prints one line per
// variant: ms per 100 iterations, GB/s, and whether w matches the reference variant bitwise.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2110_12065_b200/csrc/dense.cuh"
using namespace mapi;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void fill(float* A, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)(i * 2654435761u) ^ (uint32_t)(i >> 17);
        h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
        float v = ((h & 0xffff) / 65536.0f - 0.5f) * 0.01f;
        int64_t r = i / n, c = i % n;
        A[i] = (r == c) ? 5.0f + v : v;
    }
}

template <int U>
__global__ void __launch_bounds__(512, 1) read_probe(const float* A, int64_t total, float* out) {
    float acc = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8 * U;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < total; i += stride) {
        float v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) if (i + (int64_t)u * gridDim.x * blockDim.x * 8 < total) ld_stream<8, 0>(A + i + (int64_t)u * gridDim.x * blockDim.x * 8, v[u]); else for (int k = 0; k < 8; ++k) v[u][k] = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) for (int k = 0; k < 8; ++k) acc += v[u][k];
    }
    if (acc == 1234.5f) out[0] = acc;
}

// warp-per-row streaming (the K2 access pattern), no compute dependency beyond a sum
template <int U>
__global__ void __launch_bounds__(512, 1) read_rows_warp(const float* A, int64_t n, float* out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * 16 + (threadIdx.x >> 5), tw = (int64_t)gridDim.x * 16;
    float acc = 0.f;
    for (int64_t row = gw; row < n; row += tw) {
        const float* a = A + row * n;
        for (int64_t c = lane * 8; c < n; c += 256 * U) {
            float v[U][8];
#pragma unroll
            for (int u = 0; u < U; ++u) ld_stream<8, 0>(a + c + u * 256, v[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) for (int k = 0; k < 8; ++k) acc += v[u][k];
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}
// CTA-cooperative rows: CTA c streams rows c, c+G, ... with its 16 warps on 16 column segments
template <int U>
__global__ void __launch_bounds__(512, 1) read_rows_cta(const float* A, int64_t n, float* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t seg = n / 16;
    float acc = 0.f;
    for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
        const float* a = A + row * n + warp * seg;
        for (int64_t c = lane * 8; c < seg; c += 256 * U) {
            float v[U][8];
#pragma unroll
            for (int u = 0; u < U; ++u) ld_stream<8, 0>(a + c + u * 256, v[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) for (int k = 0; k < 8; ++k) acc += v[u][k];
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

template <typename K>
float time_plain(K kern, const char* name, int grid, int threads, const float* A, int64_t n, float* out) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        kern<<<grid, threads>>>(A, n, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    printf("%-40s grid %4d x %4d  %8.3f ms  %7.1f GB/s\n", name, grid, threads, best, 4.0 * n * n / (best / 1e3) / 1e9);
    return best;
}

template <typename K>
float run_iter(K kern, const char* name, int threads, const float* A, int64_t n, const float* b0, float* w, void* ws, int iters, std::vector<float>& ref, int reps = 3, size_t smem_override = 0) {
    size_t smem = smem_override ? smem_override : sizeof(float) * ((n + 3) & ~3) + sizeof(double) * 33;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int grid = occ * sms;
    char* p = (char*)ws;
    IterArgs a;
    a.A = A; a.n = n; a.lda = n; a.b0 = b0; a.iters = iters; a.tol = 0.f; a.w_out = w; a.norms = nullptr; a.deltas = nullptr;
    a.bar = (unsigned*)p; a.status = (int*)(p + 64); a.slots = (float*)(p + 256); a.y = (float*)(p + 256 + 8192);
    void* args[] = {&a};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps + 1; ++r) {
        CK(cudaMemset(ws, 0, 256));
        cudaEventRecord(e0);
        CK(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(threads), args, smem, 0));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    std::vector<float> h(n);
    CK(cudaMemcpy(h.data(), w, 4 * n, cudaMemcpyDeviceToHost));
    bool same = true;
    if (ref.empty()) ref = h; else for (int64_t i = 0; i < n; ++i) if (h[i] != ref[i]) { same = false; break; }
    double gbs = (4.0 * n * n + 8.0 * n) * iters / (best / 1e3) / 1e9;
    printf("%-40s grid %4d x %4d  %8.3f ms  %8.1f it/s  %7.1f GB/s  bitwise_same=%d\n", name, grid, threads, best, iters / (best / 1e3), gbs, same);
    return best;
}

int main() {
    const int64_t n = 32768;
    float *A, *b0, *w, *out;
    void* ws;
    CK(cudaMalloc(&A, 4 * n * n));
    CK(cudaMalloc(&b0, 4 * n));
    CK(cudaMalloc(&w, 4 * n));
    CK(cudaMalloc(&out, 64));
    CK(cudaMalloc(&ws, 256 + 8192 + 8 * n + 4096));
    fill<<<4096, 256>>>(A, n);
    std::vector<float> hb(n, 1.0f / 181.01933598375618f);
    CK(cudaMemcpy(b0, hb.data(), 4 * n, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    // read-only ceiling
    {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        for (int U : {2, 4, 8}) {
            float best = 1e30f;
            for (int r = 0; r < 6; ++r) {
                cudaEventRecord(e0);
                if (U == 2) read_probe<2><<<sms * 2, 512>>>(A, n * n, out);
                if (U == 4) read_probe<4><<<sms * 2, 512>>>(A, n * n, out);
                if (U == 8) read_probe<8><<<sms * 2, 512>>>(A, n * n, out);
                cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (r > 0 && ms < best) best = ms;
            }
            printf("read_probe U=%d (2x512/SM, LDG.256 evict-first)   %8.3f ms  %7.1f GB/s\n", U, best, 4.0 * n * n / (best / 1e3) / 1e9);
        }
    }
    {
        int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        time_plain(read_rows_warp<4>, "read rows/warp U4", sms, 512, A, n, out);
        time_plain(read_rows_warp<2>, "read rows/warp U2", sms, 512, A, n, out);
        time_plain(read_rows_cta<4>, "read rows/cta U4", sms, 512, A, n, out);
        time_plain(read_rows_cta<8>, "read rows/cta U8", sms, 512, A, n, out);
        time_plain(read_rows_cta<4>, "read rows/cta U4 2cta", 2 * sms, 512, A, n, out);
    }
    const int iters = 20;
    std::vector<float> ref;
    {
        std::vector<float> ref2, ref2b;
        run_iter(k_iterate_coop<0, 0, 32, 2>, "coop NW32 D2 (production)", 1024, A, n, b0, w, ws, iters, ref2, 3, coop_smem_bytes(n, 148, 32));
        run_iter(k_iterate_coop<0, 0, 32, 3>, "coop NW32 D3", 1024, A, n, b0, w, ws, iters, ref2, 3, coop_smem_bytes(n, 148, 32));
        run_iter(k_iterate_coop<0, 0, 16, 4>, "coop NW16 D4", 512, A, n, b0, w, ws, iters, ref2b, 3, coop_smem_bytes(n, 148, 16));
        run_iter(k_iterate_coop<0, 0, 16, 6>, "coop NW16 D6", 512, A, n, b0, w, ws, iters, ref2b, 3, coop_smem_bytes(n, 148, 16));
        // cfg2-size (n = 4096, 64 MiB: may stay L2-resident)
        const int64_t n2 = 4096;
        std::vector<float> ref3, ref4, ref5;
        run_iter(k_iterate_persistent<0, 8, 1, 4, 0, 0>, "n4096 rows U4 L2-normal", 512, A, n2, b0, w, ws, 100, ref3);
        run_iter(k_iterate_persistent<0, 8, 1, 2, 0, 0, 2>, "n4096 rows U2 2CTA/SM", 512, A, n2, b0, w, ws, 100, ref3);
        run_iter(k_iterate_persistent<0, 8, 1, 4, 0, 0, 2>, "n4096 rows U4 2CTA/SM", 512, A, n2, b0, w, ws, 100, ref3);
        run_iter(k_iterate_persistent<0, 8, 1, 1, 0, 0, 2>, "n4096 rows U1 2CTA/SM", 512, A, n2, b0, w, ws, 100, ref3);
        run_iter(k_iterate_persistent<0, 4, 1, 4, 0, 0, 2>, "n4096 rows V4 U4 2CTA/SM", 512, A, n2, b0, w, ws, 100, ref3);
        run_iter(k_iterate_persistent<0, 8, 1, 8, 0, 0, 1>, "n4096 rows V8 U8 1CTA/SM", 512, A, n2, b0, w, ws, 100, ref3);
        run_iter(k_iterate_persistent<0, 4, 1, 16, 0, 0, 1>, "n4096 rows V4 U16 1CTA/SM", 512, A, n2, b0, w, ws, 100, ref3);
        run_iter(k_iterate_persistent<0, 4, 1, 8, 0, 0, 1>, "n4096 rows V4 U8 1CTA/SM", 512, A, n2, b0, w, ws, 100, ref3);
        run_iter(k_iterate_persistent<0, 8, 1, 2, 0, 0, 2>, "n4096 rows V8 U2 2CTA/SM", 512, A, n2, b0, w, ws, 100, ref3);
        const int64_t n3 = 8192;
        std::vector<float> ref6;
        run_iter(k_iterate_persistent<0, 8, 1, 4, 0, 0>, "n8192 rows U4", 512, A, n3, b0, w, ws, 100, ref6);
        run_iter(k_iterate_coop<0, 1, 16, 2>, "n8192 coop NW16", 512, A, n3, b0, w, ws, 100, ref6, 3, coop_smem_bytes(n3, 148, 16));
        run_iter(k_iterate_coop<0, 1, 32, 2>, "n8192 coop NW32", 1024, A, n3, b0, w, ws, 100, ref6, 3, coop_smem_bytes(n3, 148, 32));
        run_iter(k_iterate_coop<0, 1, 16, 2>, "n4096 coop NW16 D2", 512, A, n2, b0, w, ws, 100, ref4, 3, coop_smem_bytes(n2, 148, 16));
        run_iter(k_iterate_coop<0, 1, 16, 4>, "n4096 coop NW16 D4", 512, A, n2, b0, w, ws, 100, ref4, 3, coop_smem_bytes(n2, 148, 16));
        run_iter(k_iterate_coop<0, 1, 16, 8>, "n4096 coop NW16 D8", 512, A, n2, b0, w, ws, 100, ref4, 3, coop_smem_bytes(n2, 148, 16));
        run_iter(k_iterate_coop<0, 1, 16, 12>, "n4096 coop NW16 D12", 512, A, n2, b0, w, ws, 100, ref4, 3, coop_smem_bytes(n2, 148, 16));
        run_iter(k_iterate_coop<0, 0, 16, 8>, "n4096 coop NW16 D8 evict-first", 512, A, n2, b0, w, ws, 100, ref4, 3, coop_smem_bytes(n2, 148, 16));
        run_iter(k_iterate_coop<0, 1, 32, 2>, "n4096 coop NW32 D2", 1024, A, n2, b0, w, ws, 100, ref5, 3, coop_smem_bytes(n2, 148, 32));
        run_iter(k_iterate_coop<0, 1, 32, 3>, "n4096 coop NW32 D3", 1024, A, n2, b0, w, ws, 100, ref5, 3, coop_smem_bytes(n2, 148, 32));
    }
    return 0;
}
