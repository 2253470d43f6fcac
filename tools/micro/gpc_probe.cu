// How many thread-block clusters of each size can be co-resident (one CTA per SM: max smem)?
// Reveals the GPC structure that bounds the cluster column kernel.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { if (p) p[0] = 1; }
int main() {
    int dev = 0, sms = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    printf("sms %d optin %d\n", sms, optin);
    for (int cb = 1; cb <= 16; ++cb) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cb);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = optin;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cb; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %2d: %3d clusters = %3d SMs %s\n", cb, n, n * cb, e ? cudaGetErrorString(e) : "");
    }
    return 0;
}
