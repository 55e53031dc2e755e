// How many thread-block clusters of a given size can be co-resident with the torus kernel's
// per-CTA resources (one 512-thread CTA per SM): probes the GPC structure that decides
// whether a fused launch of clusters fits in one wave.  nvcc -arch=sm_100a -o /tmp/co tools/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) k_probe(int *p) { if (p) p[threadIdx.x] = 0; }
int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = 150 * 1024;  // one CTA per SM, as the torus kernel (110 registers x 512 threads)
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    printf("SMs %d\n", nsm);
    for (int cs : {1, 2, 3, 4, 6, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int nc = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k_probe, &cfg);
        printf("cluster %2d: max active clusters %4d (CTAs %4d) %s\n", cs, nc, nc * cs, cudaGetErrorString(e));
    }
    return 0;
}
