#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 1) k(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int coop; cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, 0);
    printf("SMs %d coop %d\n", sms, coop);
    for (int smem : {150 * 1024, 200 * 1024}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
            cfg.attrs = a; cfg.numAttrs = 1;
            int nc = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
            printf("smem %d KB cluster %2d: max active clusters %d (%d CTAs) %s\n", smem / 1024, cs, nc, nc * cs, cudaGetErrorString(e));
        }
    }
    // cooperative + cluster launch
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 150 * 1024;
    cudaLaunchAttribute a[2]; a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    a[1].id = cudaLaunchAttributeCooperative; a[1].val.cooperative = 1;
    cfg.attrs = a; cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, (int*)nullptr);
    printf("coop+cluster2 grid 148: %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(cudaDeviceSynchronize()));
    a[0].val.clusterDim.x = 4;
    e = cudaLaunchKernelEx(&cfg, k, (int*)nullptr);
    printf("coop+cluster4 grid 148: %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
