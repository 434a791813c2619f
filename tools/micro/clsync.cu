// Microbenchmark: cost of cluster.sync() (barrier.cluster arrive.release + wait.acquire) for
// 1/2/4/8-CTA clusters of 256 threads, split arrive/wait, and of __syncthreads.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int mode, long long* out) {
    cg::cluster_group cl = cg::this_cluster();
    const int R = 1000;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) {
        for (int r = 0; r < R; r++) cl.sync();
    } else if (mode == 1) {
        for (int r = 0; r < R; r++) __syncthreads();
    } else {
        for (int r = 0; r < R; r++) {
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / R;
}
int main() {
    long long* d; cudaMalloc(&d, 64);
    for (int cs : {1, 2, 4, 8}) {
        for (int mode = 0; mode < 3; mode++) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs); cfg.blockDim = dim3(256);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k, mode, d);
            cudaLaunchKernelEx(&cfg, k, mode, d);
            long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("cs=%d %s: %lld cycles\n", cs, mode == 0 ? "cluster.sync" : mode == 1 ? "__syncthreads" : "arrive.release+wait.acquire", h);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
