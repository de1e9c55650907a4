// Cycles per step of barrier / division / shuffle chains at different CTA
// sizes (calibrates the latency model of the one-CTA panel kernels).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void steps(double *out, long long *cyc, double y, int iters) {
    __shared__ double sh[64];
    double x = 1.0 + threadIdx.x * 1e-7;
    if (threadIdx.x < 64) sh[threadIdx.x] = x;
    __syncthreads();
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        if (MODE & 1) __syncthreads();
        if (MODE & 2) x = x / y;
        if (MODE & 4) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
        if (MODE & 8) x = fma(x, y, sh[k & 63]);
        if (MODE & 16) {
            if ((threadIdx.x & 7) == (k & 7)) x = x / y;
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8);
    const int iters = 1024;
    const int modes[] = {1, 2, 4, 8, 3, 7, 15, 16, 21, 29};
    const char *names[] = {"bar", "div", "shfl", "lds+fma", "bar+div", "bar+div+shfl", "bar+div+shfl+fma",
                           "div(1/8 lanes)", "bar+div1/8+shfl", "bar+div1/8+fma+shfl"};
    for (int nt : {32, 64, 512}) {
        for (int mi = 0; mi < 10; ++mi) {
            for (int rep = 0; rep < 2; ++rep) {
                switch (modes[mi]) {
#define M(v) case v: steps<v><<<1, nt>>>(out, cyc, 1.0000001, iters); break;
                    M(1) M(2) M(4) M(8) M(3) M(7) M(15) M(16) M(21) M(29)
                }
                cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            }
            printf("threads %3d  %-22s %7.1f cycles/step\n", nt, names[mi], (double)h / iters);
        }
    }
    return 0;
}
