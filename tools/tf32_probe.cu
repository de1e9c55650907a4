// tf32_probe.cu -- legacy mma.sync.m16n8k8.tf32 and FFMA throughput on B200 (3xTF32 design input).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tf32_probe tools/tf32_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
__global__ void k(float *out, float a) {
    float c[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
    unsigned av[4], bv[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) av[i] = __float_as_uint(a + threadIdx.x + i);
    bv[0] = __float_as_uint(a - threadIdx.x); bv[1] = __float_as_uint(a * 2);
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                         : "r"(av[0]), "r"(av[1]), "r"(av[2]), "r"(av[3]), "r"(bv[0]), "r"(bv[1]));
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 1.2345f) out[0] = s;
}
__global__ void kf(float *out, float a) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, 1e-7f);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 1.2345f) out[0] = s;
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float *d; cudaMalloc(&d, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int wps : {8, 16, 32}) {
        k<<<nsm, wps * 32>>>(d, 1.0001f); cudaDeviceSynchronize();
        cudaEventRecord(e0); k<<<nsm, wps * 32>>>(d, 1.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("tf32 mma.sync m16n8k8 warps/SM %d: %.1f TFLOP/s\n", wps, 2.0 * 16 * 8 * 8 * 8 * (double)ITERS * wps * nsm / ms / 1e9);
        kf<<<nsm * 4, wps * 32>>>(d, 1.0001f); cudaDeviceSynchronize();
        cudaEventRecord(e0); kf<<<nsm * 4, wps * 32>>>(d, 1.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("ffma warps/SM %d: %.1f TFLOP/s\n", wps * 4, 2.0 * 16 * (double)ITERS * wps * 32 * nsm * 4 / ms / 1e9);
    }
    return 0;
}
