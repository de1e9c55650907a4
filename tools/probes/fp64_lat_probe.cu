// Latency of dependent FP64 operations on the B200 (cycles per op,
// one warp): DFMA/DMUL/DADD chains, __ddiv_rn, __drcp_rn, SHFL (64-bit).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double *out, long long *cyc, double a0, double b0, int iters) {
    double a = a0 + threadIdx.x * 1e-9, b = b0;
    __syncwarp();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (OP == 0) a = fma(a, b, 1e-30);
        if (OP == 1) a = __dmul_rn(a, b);
        if (OP == 2) a = __dadd_rn(a, b);
        if (OP == 3) a = __ddiv_rn(a, b);
        if (OP == 4) a = __drcp_rn(a);
        if (OP == 5) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31);
        if (OP == 6) a = __dsub_rn(a, __dmul_rn(a, b));
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8);
    const char *names[] = {"DFMA", "DMUL", "DADD", "ddiv_rn", "drcp_rn", "SHFL f64", "DMUL+DSUB"};
    const int iters = 4096;
    for (int op = 0; op < 7; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
            case 0: chain<0><<<1, 32>>>(out, cyc, 1.0, 0.9999999, iters); break;
            case 1: chain<1><<<1, 32>>>(out, cyc, 1.0, 0.9999999, iters); break;
            case 2: chain<2><<<1, 32>>>(out, cyc, 1.0, 1e-9, iters); break;
            case 3: chain<3><<<1, 32>>>(out, cyc, 1.0, 1.0000001, iters); break;
            case 4: chain<4><<<1, 32>>>(out, cyc, 1.5, 1.0, iters); break;
            case 5: chain<5><<<1, 32>>>(out, cyc, 1.5, 1.0, iters); break;
            case 6: chain<6><<<1, 32>>>(out, cyc, 1.5, 1e-3, iters); break;
            }
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-10s %6.1f cycles per dependent op\n", names[op], (double)h / iters);
    }
    return 0;
}
