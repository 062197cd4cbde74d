// probe_k6.cu — per-phase cycle breakdown of the K6 cluster iteration (investigation only).
// A copy of k_iterate_cluster<0>'s loop with clock64 stamps (CTA rank 0, thread 0) at: iteration
// start, rows done (before cluster barrier), after cluster barrier, after warp-0 epilogue (thread 0
// is in warp 0), after __syncthreads.  n = 256 (cfg1 shape), random data, 60 iterations.
#include <cstdio>
#include <vector>
#include "../paper_2110_12065_b200/csrc/dense.cuh"
using namespace mapi;

__global__ void __launch_bounds__(kClusterThreads, 1) k6_probe(IterArgs p, long long* stamps) {
    extern __shared__ __align__(16) float sm[];
    const int64_t n = p.n, np = cluster_ld(n);
    const int64_t R = cluster_rows_per_cta(n);
    float* As = sm;
    float* w_s = sm + R * np;
    float* ybuf = w_s + np;
    const uint32_t rank = cluster_ctarank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kClusterThreads / 32;
    const int64_t r0 = (int64_t)rank * R, r1 = min(n, r0 + R);
    for (int64_t q = tid; q < R * np; q += kClusterThreads) {
        const int64_t r = q / np, c = q - r * np;
        As[q] = (r0 + r < n && c < n) ? p.A[(r0 + r) * p.lda + c] : 0.0f;
    }
    for (int64_t k = tid; k < np; k += kClusterThreads) w_s[k] = k < n ? p.b0[k] : 0.0f;
    cluster_sync_all();
    __shared__ int32_t s_flag[2];
    const bool rec = rank == 0 && tid == 0;
    for (int32_t t = 0; t < p.iters; ++t) {
        if (rec) stamps[t * 5 + 0] = clock64();
        float* yb = ybuf + (t & 1) * np;
        for (int64_t r = r0 + warp; r < r1; r += nw) {
            const float v = cluster_row<0>(As + (r - r0) * np, w_s, np, lane);
            if (rec) stamps[1000 + t] = clock64();
            if (lane < kClusterCtas) st_cluster(yb + r, (uint32_t)lane, v);
        }
        if (rec) stamps[t * 5 + 1] = clock64();
        cluster_sync_all();
        if (rec) stamps[t * 5 + 2] = clock64();
        if (warp == 0) {
            double ap = 0.0;
            for (int64_t k = lane; k < n; k += 32) ap += norm_part<0>(yb[k]);
            const double sd = norm_final<0>(warp_sum(ap));
            double dp = 0.0;
            for (int64_t k = lane; k < n; k += 32) {
                const float wn = (float)((double)yb[k] / sd);
                dp += (double)fabsf(wn - w_s[k]);
                w_s[k] = wn;
            }
            const double delta = warp_sum(dp);
            if (lane == 0) {
                s_flag[0] = 0;
                if (rank == 0 && p.norms) p.norms[t] = (float)sd;
                if (rank == 0 && p.deltas) p.deltas[t] = (float)delta;
            }
        }
        if (rec) stamps[t * 5 + 3] = clock64();
        __syncthreads();
        if (rec) stamps[t * 5 + 4] = clock64();
    }
    cluster_sync_all();
}

int main() {
    const int n = 256, T = 60;
    std::vector<float> hA(n * n), hb(n, 1.0f / 16);
    unsigned s = 1;
    for (auto& x : hA) { s = s * 1664525u + 1013904223u; x = ((s >> 8) / 16777216.0f - 0.5f); }
    float *A, *b0, *w, *y, *norms, *deltas; double* slots; unsigned* bar; int* st; long long* stamps;
    cudaMalloc(&A, 4 * n * n); cudaMalloc(&b0, 4 * n); cudaMalloc(&w, 4 * n); cudaMalloc(&y, 8 * n);
    cudaMalloc(&norms, 4 * T); cudaMalloc(&deltas, 4 * T); cudaMalloc(&slots, 8 * 4096); cudaMalloc(&bar, 256);
    cudaMalloc(&st, 8); cudaMalloc(&stamps, 8 * 2000);
    cudaMemcpy(A, hA.data(), 4 * n * n, cudaMemcpyHostToDevice);
    cudaMemcpy(b0, hb.data(), 4 * n, cudaMemcpyHostToDevice);
    IterArgs a{};
    a.A = A; a.n = n; a.lda = n; a.b0 = b0; a.iters = T; a.tol = 0; a.w_out = w; a.norms = norms; a.deltas = deltas;
    a.y = y; a.slots = reinterpret_cast<float*>(slots); a.bar = bar; a.status = st;
    const size_t smem = cluster_smem_bytes(n);
    cudaFuncSetAttribute(k6_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kClusterCtas); cfg.blockDim = dim3(kClusterThreads); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kClusterCtas; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    for (int rep = 0; rep < 3; ++rep) {
        cudaError_t e = cudaLaunchKernelEx(&cfg, k6_probe, a, stamps);
        if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("sync: %s\n", cudaGetErrorString(e)); return 1; }
    }
    std::vector<long long> h(5 * T);
    cudaMemcpy(h.data(), stamps, 8 * 5 * T, cudaMemcpyDeviceToHost);
    double ph[4] = {0, 0, 0, 0}, tot = 0;
    int cnt = 0;
    for (int t = 10; t < T - 1; ++t, ++cnt) {
        for (int k = 0; k < 4; ++k) ph[k] += h[t * 5 + k + 1] - h[t * 5 + k];
        tot += h[(t + 1) * 5] - h[t * 5];
    }
    std::vector<long long> h2(T);
    cudaMemcpy(h2.data(), stamps + 1000, 8 * T, cudaMemcpyDeviceToHost);
    double rc = 0;
    for (int t = 10; t < T - 1; ++t) rc += h2[t] - h[t * 5];
    printf("  of rows: compute (start -> before DSMEM stores) %.0f cycles\n", rc / cnt);
    printf("K6 n=256 cycles/iteration: rows %.0f  cluster-barrier %.0f  epilogue(warp0) %.0f  syncthreads %.0f  total %.0f\n",
           ph[0] / cnt, ph[1] / cnt, ph[2] / cnt, ph[3] / cnt, tot / cnt);
    return 0;
}
