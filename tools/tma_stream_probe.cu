// tma_stream_probe.cu -- streaming throughput of the batched config's access
// pattern (per instance, 16 chunks of 8 rows x 128 columns of a column-major
// 128 x 128 f64 matrix = 64-byte column segments) through a 4-stage shared
// ring: (a) one TMA tensor copy per chunk (cp.async.bulk.tensor.2d, box
// 8 x 128), (b) per-thread 16-byte cp.async (512 threads).  Consumers only
// wait and release.  Prints GB/s over 148 persistent CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_stream_probe tools/tma_stream_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

constexpr int N = 128, KC = 8, ST = 4;

__device__ __forceinline__ unsigned saddr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(unsigned long long *b, unsigned ph) {
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                     saddr(b)),
                 "r"(ph)
                 : "memory");
}

__global__ void __launch_bounds__(512, 1) k_tma(const __grid_constant__ CUtensorMap tm, int64_t batch, double *sink) {
    extern __shared__ __align__(1024) unsigned char dyn[];
    double(*ring)[2][N * KC] = reinterpret_cast<double(*)[2][N * KC]>(dyn);  // A and B chunk per stage
    __shared__ __align__(8) unsigned long long full[ST], empty[ST];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t G = gridDim.x, J = (batch - blockIdx.x + G - 1) / G, total = J * (N / KC);
    if (tid == 0) {
        for (int q = 0; q < ST; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&full[q])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;" ::"r"(saddr(&empty[q])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t g) {
        const int s = (int)(g % ST);
        const int64_t inst = blockIdx.x + (g / (N / KC)) * G;
        const int k0 = (int)(g % (N / KC)) * KC;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&full[s])),
                     "r"(2 * N * KC * 8)
                     : "memory");
        // two operands = two row bands of the same tensor (A at column block inst, B at inst + batch)
        for (int op = 0; op < 2; ++op) {
            const int c0 = k0, c1 = (int)((inst + op * batch) * N);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    saddr(&ring[s][op][0])),
                "l"(&tm), "r"(c0), "r"(c1), "r"(saddr(&full[s]))
                : "memory");
        }
    };
    if (tid == 0)
        for (int64_t g = 0; g < ST && g < total; ++g) issue(g);
    double acc = 0;
    for (int64_t g = 0; g < total; ++g) {
        const int s = (int)(g % ST);
        mwait(&full[s], (unsigned)((g / ST) & 1));
        acc += ring[s][warp & 1][lane];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&empty[s])) : "memory");
        if (tid == 0 && g + ST < total) {
            mwait(&empty[s], (unsigned)((g / ST) & 1));
            issue(g + ST);
        }
    }
    if (acc == 1.2345) sink[0] = acc;
}

__global__ void __launch_bounds__(512, 1) k_cpa(const double *X, int64_t batch, double *sink) {
    extern __shared__ __align__(1024) unsigned char dyn[];
    double(*ring)[2][N * (KC + 4)] = reinterpret_cast<double(*)[2][N * (KC + 4)]>(dyn);
    const int tid = threadIdx.x;
    const int64_t G = gridDim.x, J = (batch - blockIdx.x + G - 1) / G, total = J * (N / KC), nn = N * N;
    auto issue = [&](int64_t g) {
        const int s = (int)(g % ST);
        const int64_t inst = blockIdx.x + (g / (N / KC)) * G;
        const int k0 = (int)(g % (N / KC)) * KC;
        const int col = tid >> 2, piece = tid & 3;
        for (int op = 0; op < 2; ++op) {
            const double *src = X + (inst + op * batch) * nn + (int64_t)col * N + k0 + piece * 2;
            const unsigned d = saddr(&ring[s][op][col * (KC + 4) + piece * 2]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src));
        }
        asm volatile("cp.async.commit_group;");
    };
    for (int64_t g = 0; g < ST - 1; ++g) issue(g);
    double acc = 0;
    for (int64_t g = 0; g < total; ++g) {
        asm volatile("cp.async.wait_group 2;");
        __syncthreads();
        if (g + ST - 1 < total) issue(g + ST - 1);
        else asm volatile("cp.async.commit_group;");
        acc += ring[g % ST][tid & 1][tid >> 1];
    }
    if (acc == 1.2345) sink[0] = acc;
}

int main() {
    const int64_t batch = 20000;
    const size_t bytes = (size_t)2 * batch * N * N * 8;
    double *X, *sink;
    cudaMalloc(&X, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(X, 0, bytes);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    // 2D view: dim0 = row within a column (128, contiguous), dim1 = column index over all instances
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)(2 * batch * N)};
    cuuint64_t strides[1] = {(cuuint64_t)N * 8};
    cuuint32_t box[2] = {(cuuint32_t)KC, (cuuint32_t)N};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
    }
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_cpa, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0);
        k_tma<<<nsm, 512, ST * 2 * N * KC * 8>>>(tm, batch, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("TMA 2D box 8x128: %.1f GB/s (%s)\n", bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(e0);
        k_cpa<<<nsm, 512, ST * 2 * N * (KC + 4) * 8>>>(X, batch, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cp.async 16 B x 512 threads: %.1f GB/s (%s)\n", bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
