// How many thread-block clusters of size k can be co-resident with one 544-thread,
// ~227-KB-smem CTA per SM (the executor's footprint), and does a cooperative
// launch with clusters work?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_clusters tools/probe_clusters.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k(int* out) {
    extern __shared__ char sm[];
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) {
        sm[0] = 1;
        out[blockIdx.x] = static_cast<int>(cl.block_rank());
    }
    cl.sync();
    cg::this_grid().sync();
}

int main() {
    int dev = 0, nsm = 0, smem = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    smem -= 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int* out;
    cudaMalloc(&out, 4096 * 4);
    printf("SMs %d smem %d\n", nsm, smem);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nsm / cs * cs);
        cfg.blockDim = dim3(544);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
        cfg.numAttrs = 2;
        cudaError_t e2 = cudaSuccess;
        int grid = 0;
        if (e == cudaSuccess && ncl > 0) {
            grid = ncl * cs;
            cfg.gridDim = dim3(grid);
            e2 = cudaLaunchKernelEx(&cfg, k, out);
            if (e2 == cudaSuccess) e2 = cudaDeviceSynchronize();
        }
        printf("cluster %2d: max active clusters %d (%s) -> %d CTAs; coop launch: %s\n", cs, ncl,
               cudaGetErrorString(e), ncl * cs, cudaGetErrorString(e2));
        cudaGetLastError();
    }
    return 0;
}
