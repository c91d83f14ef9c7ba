// Probe: how many clusters of a given shape can be co-resident (GPC packing), B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int *p) { if (p) p[threadIdx.x] = 0; }
int main() {
    struct C { int threads, smem_kb, cl; } cs[] = {{256, 93, 8}, {256, 93, 4}, {256, 93, 2}, {512, 200, 8},
                                                    {512, 200, 4}, {512, 200, 2}, {128, 110, 2}, {256, 100, 2},
                                                    {256, 200, 8}, {256, 200, 16}};
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (auto c : cs) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(c.cl * 64);
        cfg.blockDim = dim3(c.threads);
        cfg.dynamicSmemBytes = (size_t)c.smem_kb * 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, dummy, c.threads, cfg.dynamicSmemBytes);
        printf("threads %d smem %d KB cluster %d: max active clusters %d (CTAs %d of %d SMs x %d) %s\n", c.threads,
               c.smem_kb, c.cl, n, n * c.cl, sms, per, cudaGetErrorString(e));
    }
}
