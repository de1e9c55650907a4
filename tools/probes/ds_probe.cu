// Streaming-kernel variants for the 4096^2 f64 diag_scale shape (128 MB in,
// 128 MB out): which structure reaches the copy ceiling.  nvcc -O3 -arch=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct alignas(32) V4 { double v[4]; };
__device__ __forceinline__ V4 ld32(const double *p) {
    V4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
    return r;
}
__device__ __forceinline__ void st32(double *p, const V4 &x) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(x.v[0]), "d"(x.v[1]), "d"(x.v[2]), "d"(x.v[3]) : "memory");
}
__device__ __forceinline__ void st32wb(double *p, const V4 &x) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(x.v[0]), "d"(x.v[1]), "d"(x.v[2]), "d"(x.v[3]) : "memory");
}

template <int U, bool CS>
__global__ void __launch_bounds__(256) cols32(const double *d, const double *b, double *out, int64_t rows, int64_t cols, int gx) {
    const int slots = gridDim.x / gx, slot = blockIdx.x / gx;
    const int64_t i = ((int64_t)(blockIdx.x - slot * gx) * blockDim.x + threadIdx.x) * 4;
    if (i >= rows || slot >= slots) return;
    double dl[4];
    for (int l = 0; l < 4; ++l) dl[l] = d[i + l];
    const double *bp = b + i + slot * rows;
    double *op = out + i + slot * rows;
    const int64_t sb = (int64_t)slots * rows;
    int64_t j = slot;
    for (; j + (U - 1) * (int64_t)slots < cols; j += U * (int64_t)slots) {
        V4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld32(bp + u * sb);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            V4 r;
#pragma unroll
            for (int l = 0; l < 4; ++l) r.v[l] = __dmul_rn(dl[l], x[u].v[l]);
            if (CS) st32(op + u * sb, r); else st32wb(op + u * sb, r);
        }
        bp += U * sb;
        op += U * sb;
    }
    for (; j < cols; j += slots) {
        V4 x = ld32(bp), r;
        for (int l = 0; l < 4; ++l) r.v[l] = __dmul_rn(dl[l], x.v[l]);
        st32(op, r);
        bp += sb;
        op += sb;
    }
}

template <int U>
__global__ void __launch_bounds__(256, 8) cols32_lb(const double *d, const double *b, double *out, int64_t rows, int64_t cols, int gx) {
    const int slots = gridDim.x / gx, slot = blockIdx.x / gx;
    const int64_t i = ((int64_t)(blockIdx.x - slot * gx) * blockDim.x + threadIdx.x) * 4;
    if (i >= rows || slot >= slots) return;
    double dl[4];
    for (int l = 0; l < 4; ++l) dl[l] = d[i + l];
    const double *bp = b + i + slot * rows;
    double *op = out + i + slot * rows;
    const int64_t sb = (int64_t)slots * rows;
    int64_t j = slot;
    for (; j + (U - 1) * (int64_t)slots < cols; j += U * (int64_t)slots) {
        V4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld32(bp + u * sb);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            V4 r;
#pragma unroll
            for (int l = 0; l < 4; ++l) r.v[l] = __dmul_rn(dl[l], x[u].v[l]);
            st32(op + u * sb, r);
        }
        bp += U * sb;
        op += U * sb;
    }
    for (; j < cols; j += slots) {
        V4 x = ld32(bp), r;
        for (int l = 0; l < 4; ++l) r.v[l] = __dmul_rn(dl[l], x.v[l]);
        st32(op, r);
        bp += sb;
        op += sb;
    }
}

// contiguous column chunk per CTA
template <int U>
__global__ void __launch_bounds__(256) chunk32(const double *d, const double *b, double *out, int64_t rows, int64_t cols, int gx, int64_t cpb) {
    const int slot = blockIdx.x / gx;
    const int64_t i = ((int64_t)(blockIdx.x - slot * gx) * blockDim.x + threadIdx.x) * 4;
    if (i >= rows) return;
    double dl[4];
    for (int l = 0; l < 4; ++l) dl[l] = d[i + l];
    int64_t j = slot * cpb;
    const int64_t j1 = j + cpb < cols ? j + cpb : cols;
    const double *bp = b + i + j * rows;
    double *op = out + i + j * rows;
    for (; j + U <= j1; j += U) {
        V4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld32(bp + u * rows);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            V4 r;
#pragma unroll
            for (int l = 0; l < 4; ++l) r.v[l] = __dmul_rn(dl[l], x[u].v[l]);
            st32(op + u * rows, r);
        }
        bp += U * rows;
        op += U * rows;
    }
    for (; j < j1; ++j) {
        V4 x = ld32(bp), r;
        for (int l = 0; l < 4; ++l) r.v[l] = __dmul_rn(dl[l], x.v[l]);
        st32(op, r);
        bp += rows;
        op += rows;
    }
}

// flat: vector v -> rows via mask (rows power of two) -- the ceiling for a flat layout
template <int U>
__global__ void __launch_bounds__(256) flat32(const double *d, const double *b, double *out, uint32_t rmask, uint32_t nvec) {
    const uint32_t nth = gridDim.x * blockDim.x;
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + (U - 1) * nth < nvec; v += U * nth) {
        V4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld32(b + (size_t)(v + u * nth) * 4);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t i = ((v + u * nth) * 4) & rmask;
            const V4 dv = *reinterpret_cast<const V4 *>(d + i);
            V4 r;
#pragma unroll
            for (int l = 0; l < 4; ++l) r.v[l] = __dmul_rn(dv.v[l], x[u].v[l]);
            st32(out + (size_t)(v + u * nth) * 4, r);
        }
    }
}

// pure copy, flat, 16 B or 32 B vectors
template <int U>
__global__ void __launch_bounds__(256) copy32(const double *b, double *out, uint32_t nvec) {
    const uint32_t nth = gridDim.x * blockDim.x;
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + (U - 1) * nth < nvec; v += U * nth) {
        V4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld32(b + (size_t)(v + u * nth) * 4);
#pragma unroll
        for (int u = 0; u < U; ++u) st32(out + (size_t)(v + u * nth) * 4, x[u]);
    }
}
template <int U>
__global__ void __launch_bounds__(256) copy16(const double2 *b, double2 *out, uint32_t nvec) {
    const uint32_t nth = gridDim.x * blockDim.x;
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + (U - 1) * nth < nvec; v += U * nth) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcs(b + v + u * nth);
#pragma unroll
        for (int u = 0; u < U; ++u) __stcs(out + v + u * nth, x[u]);
    }
}

template <class F> float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms / 20 < best) best = ms / 20;
    }
    return best;
}

template <class K> int occ(K k) {
    int n = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 256, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    return n * sms;
}

int main() {
    for (int64_t n : {4096, 8192}) {
        const int64_t N = n * n;
        double *d, *b, *o;
        cudaMalloc(&d, n * 8);
        cudaMalloc(&b, N * 8);
        cudaMalloc(&o, N * 8);
        cudaMemset(b, 0, N * 8);
        cudaMemset(d, 0, n * 8);
        const double GB = 2.0 * N * 8 / 1e9;
        const int gx = (int)(n / 1024);
        auto rep = [&](const char *name, float ms) { printf("n=%lld %-28s %8.1f us %7.0f GB/s\n", (long long)n, name, ms * 1e3, GB / ms * 1e3); };
#define COLS(K, NAME) { int R = occ(K); int slots = R / gx; rep(NAME, timeit([&] { K<<<gx * slots, 256>>>(d, b, o, n, n, gx); })); }
        COLS((cols32<4, true>), "cols32 U4 cs");
        COLS((cols32<4, false>), "cols32 U4 wb");
        COLS((cols32<8, true>), "cols32 U8 cs");
        COLS((cols32<2, true>), "cols32 U2 cs");
        COLS((cols32_lb<4>), "cols32 U4 lb8");
        {
            int R = occ(cols32<4, true>);
            for (int mult : {2, 4, 8}) {
                int slots = R * mult / gx;
                char nm[64]; snprintf(nm, 64, "cols32 U4 cs x%d grid", mult);
                rep(nm, timeit([&] { cols32<4, true><<<gx * slots, 256>>>(d, b, o, n, n, gx); }));
            }
        }
        {
            int R = occ(cols32<4, true>);
            for (int mult : {16, 32}) {
                int slots = R * mult / gx;
                char nm[64]; snprintf(nm, 64, "cols32 U4 cs x%d grid", mult);
                rep(nm, timeit([&] { cols32<4, true><<<gx * slots, 256>>>(d, b, o, n, n, gx); }));
            }
            for (int cpb : {4, 8, 16, 32}) {
                int slots = (int)(n / cpb);
                char nm[64]; snprintf(nm, 64, "chunk32 U4 cpb=%d", cpb);
                rep(nm, timeit([&] { chunk32<4><<<gx * slots, 256>>>(d, b, o, n, n, gx, cpb); }));
            }
            int R2 = occ(flat32<4>);
            for (int mult : {2, 4, 8}) {
                char nm[64]; snprintf(nm, 64, "flat32 U4 x%d grid", mult);
                rep(nm, timeit([&] { flat32<4><<<R2 * mult, 256>>>(d, b, o, (uint32_t)(n - 1), (uint32_t)(N / 4)); }));
            }
        }
        { int R = occ(flat32<4>); rep("flat32 U4", timeit([&] { flat32<4><<<R, 256>>>(d, b, o, (uint32_t)(n - 1), (uint32_t)(N / 4)); })); }
        { int R = occ(flat32<2>); rep("flat32 U2", timeit([&] { flat32<2><<<R, 256>>>(d, b, o, (uint32_t)(n - 1), (uint32_t)(N / 4)); })); }
        { int R = occ(copy32<4>); rep("copy32 U4", timeit([&] { copy32<4><<<R, 256>>>(b, o, (uint32_t)(N / 4)); })); }
        { int R = occ(copy32<2>); rep("copy32 U2", timeit([&] { copy32<2><<<R, 256>>>(b, o, (uint32_t)(N / 4)); })); }
        { int R = occ(copy16<4>); rep("copy16 U4", timeit([&] { copy16<4><<<R, 256>>>((const double2 *)b, (double2 *)o, (uint32_t)(N / 2)); })); }
        { int R = occ(copy16<8>); rep("copy16 U8", timeit([&] { copy16<8><<<R, 256>>>((const double2 *)b, (double2 *)o, (uint32_t)(N / 2)); })); }
        rep("cudaMemcpyD2D", timeit([&] { cudaMemcpyAsync(o, b, N * 8, cudaMemcpyDeviceToDevice); }));
        cudaFree(d); cudaFree(b); cudaFree(o);
    }
    return 0;
}
