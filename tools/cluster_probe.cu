// cluster_probe.cu -- latency of the synchronisation primitives the LU
// panel uses: __syncthreads, cluster barrier (cs = 2..16), DSMEM
// round trip, grid-wide cooperative barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/cluster_probe tools/cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int IT = 2000;

__global__ void k_cluster_sync(int *out) {
    cg::cluster_group cl = cg::this_cluster();
    for (int i = 0; i < IT; ++i) cl.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}

__global__ void k_cluster_sync_dsmem(int *out) {
    __shared__ double box[64];
    cg::cluster_group cl = cg::this_cluster();
    double acc = 0;
    if (threadIdx.x < 64) box[threadIdx.x] = threadIdx.x;
    for (int i = 0; i < IT; ++i) {
        if (threadIdx.x < 32) box[threadIdx.x + (i & 1) * 32] = acc + i;
        cl.sync();
        if (threadIdx.x < 32) {
            const double *r = cl.map_shared_rank(box, (i + threadIdx.x) % cl.num_blocks());
            acc += r[threadIdx.x + (i & 1) * 32];
        }
    }
    if (acc == 1.2345) out[0] = 1;
}

__global__ void k_syncthreads(int *out) {
    for (int i = 0; i < IT; ++i) __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}

__global__ void k_grid_sync(int *out) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < IT / 10; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1;
}

int main() {
    int *d;
    cudaMalloc(&d, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_cluster_sync_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int threads : {256, 512}) {
        k_syncthreads<<<1, threads>>>(d);
        cudaEventRecord(e0);
        k_syncthreads<<<1, threads>>>(d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"probe\": \"syncthreads\", \"threads\": %d, \"ns\": %.1f}\n", threads, ms * 1e6 / IT);
        for (int cs : {2, 4, 8, 16}) {
            for (int which = 0; which < 2; ++which) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs);
                cfg.blockDim = dim3(threads);
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaError_t err = which ? cudaLaunchKernelEx(&cfg, k_cluster_sync_dsmem, d)
                                        : cudaLaunchKernelEx(&cfg, k_cluster_sync, d);
                cudaDeviceSynchronize();
                cudaEventRecord(e0);
                err = which ? cudaLaunchKernelEx(&cfg, k_cluster_sync_dsmem, d) : cudaLaunchKernelEx(&cfg, k_cluster_sync, d);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                printf("{\"probe\": \"%s\", \"cs\": %d, \"threads\": %d, \"ns\": %.1f, \"err\": \"%s\"}\n",
                       which ? "cluster_sync+dsmem" : "cluster_sync", cs, threads, ms * 1e6 / IT,
                       cudaGetErrorString(err));
            }
        }
    }
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int blocks : {16, 64, 148}) {
        void *args[] = {&d};
        cudaLaunchCooperativeKernel((void *)k_grid_sync, blocks, 256, args, 0, 0);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void *)k_grid_sync, blocks, 256, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"probe\": \"grid_sync\", \"blocks\": %d, \"ns\": %.1f}\n", blocks, ms * 1e6 / (IT / 10));
    }
    return 0;
}
