// How many clusters of 1/2/4/8 CTAs can be co-resident for a kernel shaped
// like k_umma_f4 (256 threads, ~216 KB of dynamic shared memory, one CTA per
// SM)? Clusters live inside one GPC, so larger clusters may strand SMs.
//   nvcc -arch=sm_100a -o /tmp/probe_clusters tools/probe_clusters.cu && /tmp/probe_clusters
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 1) k_dummy(int *p) {
    extern __shared__ unsigned char s[];
    if (p) p[0] = s[0];
}
int main() {
    const int smem = 220416;
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    printf("%s: %d SMs\n", pr.name, pr.multiProcessorCount);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(pr.multiProcessorCount / cs * cs);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
        printf("cluster %2d: max active clusters %d -> %d CTAs co-resident (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    return 0;
}
