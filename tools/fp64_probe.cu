// fp64_probe.cu -- measures the FP64 ceilings the roofline needs and
// MEASURED_PEAKS.json lacks: DFMA, DMUL+DADD (the exact-order update the
// LU and solves use) and DMMA (mma.sync.m8n8k4.f64) throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double *out, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_mul_add(double *out, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __dsub_rn(x[i], __dmul_rn(a, b + i));
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_dmma(double *out, double a, double b) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    double av = a + threadIdx.x, bv = b - threadIdx.x;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(av), "d"(bv));
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = 256;
    const int blocks = nsm * 8;
    auto run = [&](const char *name, void (*k)(double *, double, double), double flops_per_thread_iter) {
        k<<<blocks, threads>>>(d, 1.0000001, 1e-9);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(d, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 5.0 * blocks * threads * (double)ITERS * flops_per_thread_iter;
        printf("{\"probe\": \"%s\", \"tflops\": %.3f, \"ms\": %.3f}\n", name, flops / (ms * 1e-3) / 1e12, ms);
    };
    run("dfma", k_dfma, 8 * 2.0);             // 8 FMAs = 16 flops
    run("dmul+dsub", k_mul_add, 8 * 2.0);     // 8 mul + 8 sub = 16 flops (2 instructions per MAC)
    run("dmma_m8n8k4", k_dmma, 8 * 512.0 / 32.0);  // per warp-mma 8*8*4*2 = 512 flops, per thread /32
    printf("{\"probe\": \"info\", \"sms\": %d, \"err\": \"%s\"}\n", nsm, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
