// probe_k2s.cu — per-phase cycle breakdown of the K2s symmetric iteration (investigation only): compiled
// with -DMAPI_SYM_TRACE, CTA 0 / thread 0 stamps clock64 at: iteration start, own tasks done, after grid
// barrier 1, partial reduction + block sum done, after grid barrier 2, (next iteration start).
// n = 32768 symmetric synthetic matrix generated on the device, 20 iterations.
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../paper_2110_12065_b200/csrc/sym.cuh"
using namespace mapi;

__global__ void k_fill_sym(float* A, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i / n, k = i % n, lo = j < k ? j : k, hi = j < k ? k : j;
        uint32_t h = (uint32_t)(lo * 2654435761u) ^ (uint32_t)(hi * 40503u + 12345u);
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        A[i] = (float)(h & 0xffff) / 65536.0f - 0.5f + (j == k ? 8.0f : 0.0f);
    }
}

int main() {
    const int64_t n = 32768;
    const int T = 20;
    float *A, *b0, *w, *y, *nr, *dl, *part; double* sl; unsigned* bar; int* st;
    cudaMalloc(&A, 4ull * n * n); cudaMalloc(&b0, 4 * n); cudaMalloc(&w, 4 * n); cudaMalloc(&y, 16 * n);
    cudaMalloc(&nr, 4 * T); cudaMalloc(&dl, 4 * T); cudaMalloc(&sl, 8 * 4096); cudaMalloc(&bar, 256); cudaMalloc(&st, 8);
    cudaMalloc(&part, sym_partials_bytes(n));
    unsigned long long* wtag; float* yg;
    cudaMalloc(&wtag, 16 * n); cudaMalloc(&yg, 4 * n);
    k_fill_sym<<<4096, 256>>>(A, n);
    std::vector<float> hb(n, 1.0f / 181.0f);
    cudaMemcpy(b0, hb.data(), 4 * n, cudaMemcpyHostToDevice);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = sym_smem_bytes(n);
    cudaFuncSetAttribute(k_iterate_sym<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    SymArgs a{};
    a.it.A = A; a.it.n = n; a.it.lda = n; a.it.b0 = b0; a.it.iters = T; a.it.tol = 0; a.it.w_out = w;
    a.it.norms = nr; a.it.deltas = dl; a.it.y = y; a.it.slots = reinterpret_cast<float*>(sl); a.it.bar = bar;
    a.it.status = st; a.prow = part; a.pcol = part + sym_nc(n) * ((n + 31) & ~int64_t(31));
    a.wtag = wtag; a.yg = yg;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(bar, 0, 256);
        cudaMemset(wtag, 0, 16 * n);
        void* args[] = {&a};
        cudaEventRecord(e0);
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_iterate_sym<0>, dim3(sms), dim3(kSymThreads), args, smem, 0);
        cudaEventRecord(e1);
        if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
        if ((e = cudaDeviceSynchronize()) != cudaSuccess) { printf("sync: %s\n", cudaGetErrorString(e)); return 1; }
        cudaEventElapsedTime(&ms, e0, e1);
    }
    std::vector<long long> h(6 * 512);
    cudaMemcpyFromSymbol(h.data(), g_sym_trace, 8 * 6 * 512);
    double ph[5] = {0, 0, 0, 0, 0}, tot = 0;
    int cnt = 0;
    for (int t = 3; t < T - 1; ++t, ++cnt) {
        for (int k = 0; k < 4; ++k) ph[k] += h[t * 6 + k + 1] - h[t * 6 + k];
        ph[4] += h[(t + 1) * 6] - h[t * 6 + 4];
        tot += h[(t + 1) * 6] - h[t * 6];
    }
    {
        std::vector<long long> g(2 * 256 * 32);
        cudaMemcpyFromSymbol(g.data(), g_sym_cta, 8 * g.size());
        // task-phase end per CTA relative to the earliest end, averaged over iterations 3..T-2
        std::vector<double> endrel(sms, 0.0), dur(sms, 0.0);
        for (int t = 3; t < T - 1 && t < 32; ++t) {
            long long mn = 1LL << 62;
            for (int c = 0; c < sms; ++c) mn = std::min(mn, g[((t * 256) + c) * 2 + 1]);
            for (int c = 0; c < sms; ++c) {
                endrel[c] += (g[((t * 256) + c) * 2 + 1] - mn) / 1e3;
                dur[c] += (g[((t * 256) + c) * 2 + 1] - g[((t * 256) + c) * 2 + 0]) / 1e3;
            }
        }
        const int it = std::min(T - 1, 32) - 3;
        double mx = 0, avg = 0, dmx = 0, dmn = 1e30;
        for (int c = 0; c < sms; ++c) {
            endrel[c] /= it; dur[c] /= it;
            mx = std::max(mx, endrel[c]); avg += endrel[c] / sms;
            dmx = std::max(dmx, dur[c]); dmn = std::min(dmn, dur[c]);
        }
        printf("task phase: end spread over CTAs max %.1f us (mean %.1f us after the earliest); duration min %.1f max %.1f us\n",
               mx, avg, dmn, dmx);
        printf("  slowest CTAs:");
        for (int k = 0; k < 6; ++k) {
            int bi = 0;
            for (int c = 0; c < sms; ++c) if (endrel[c] > endrel[bi]) bi = c;
            printf(" %d(+%.1f)", bi, endrel[bi]);
            endrel[bi] = -1;
        }
        printf("\n");
    }
    printf("K2s n=%lld: %.1f us/iteration (events) | cycles: own tasks %.0f | barrier 1 %.0f | partial reduction %.0f | "
           "barrier 2 %.0f | s, w publish, delta partial %.0f | total %.0f\n", (long long)n, 1e3 * ms / T, ph[0] / cnt, ph[1] / cnt,
           ph[2] / cnt, ph[3] / cnt, ph[4] / cnt, tot / cnt);
    return 0;
}
