// tcgen05_tf32_probe.cu -- one 128 x 128 x 128 product D = A.T @ B (f32 in,
// column-major) on tcgen05.mma kind::tf32 with 3xTF32 (hi/lo split, TMEM
// accumulator), checked against a double-precision host product.  Design
// check for the f32 batched kernel: descriptors (K-major, no swizzle,
// 8 x 16 B core matrices), TMEM alloc / ld, commit -> mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tcgen05_tf32_probe tools/tcgen05_tf32_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int N = 128, KC = 8;  // K per chunk = one MMA's K

__device__ __forceinline__ unsigned saddr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(const void *p, unsigned lbo, unsigned sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr(p) >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // descriptor version (Blackwell)
    return d;         // base offset 0, SWIZZLE_NONE (layout type 0)
}

constexpr uint32_t kIdesc = (1u << 4)                 // D format F32
                            | (2u << 7) | (2u << 10)  // A, B format TF32
                            | (0u << 15) | (0u << 16) // A, B K-major
                            | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(N >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(acc), "r"(kIdesc));
}

__device__ __forceinline__ float tf32r(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// core-matrix offset (bytes) of row r, 16-byte K piece kc within a chunk
__device__ __forceinline__ int core_off(int r, int kc) { return (r >> 3) * 256 + kc * 128 + (r & 7) * 16; }

__global__ void k(const float *A, const float *B, float *D, int passes) {
    __shared__ __align__(1024) float ah[N * KC], al[N * KC], bh[N * KC], bl[N * KC];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_base)),
                     "r"(N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    unsigned phase = 0;
    for (int c = 0; c < N / KC; ++c) {
        // 256 (row, k-piece) pieces per operand, 4 floats each; 128 threads x 2
        for (int e = tid; e < 2 * N; e += blockDim.x) {
            const int r = e >> 1, kc = e & 1;
            const float4 va = *reinterpret_cast<const float4 *>(A + r * N + c * KC + kc * 4);
            const float4 vb = *reinterpret_cast<const float4 *>(B + r * N + c * KC + kc * 4);
            float4 h, l;
            if (passes == 4) {  // hi = raw f32 (the MMA reads it as TF32), lo = x - truncated x
                h = va;
                l.x = va.x - __uint_as_float(__float_as_uint(va.x) & 0xffffe000u);
                l.y = va.y - __uint_as_float(__float_as_uint(va.y) & 0xffffe000u);
                l.z = va.z - __uint_as_float(__float_as_uint(va.z) & 0xffffe000u);
                l.w = va.w - __uint_as_float(__float_as_uint(va.w) & 0xffffe000u);
            } else {
            h.x = tf32r(va.x); l.x = tf32r(va.x - h.x);
            h.y = tf32r(va.y); l.y = tf32r(va.y - h.y);
            h.z = tf32r(va.z); l.z = tf32r(va.z - h.z);
            h.w = tf32r(va.w); l.w = tf32r(va.w - h.w);
            }
            *reinterpret_cast<float4 *>(reinterpret_cast<char *>(ah) + core_off(r, kc)) = h;
            *reinterpret_cast<float4 *>(reinterpret_cast<char *>(al) + core_off(r, kc)) = l;
            if (passes == 4) {
                h = vb;
                l.x = vb.x - __uint_as_float(__float_as_uint(vb.x) & 0xffffe000u);
                l.y = vb.y - __uint_as_float(__float_as_uint(vb.y) & 0xffffe000u);
                l.z = vb.z - __uint_as_float(__float_as_uint(vb.z) & 0xffffe000u);
                l.w = vb.w - __uint_as_float(__float_as_uint(vb.w) & 0xffffe000u);
            } else {
            h.x = tf32r(vb.x); l.x = tf32r(vb.x - h.x);
            h.y = tf32r(vb.y); l.y = tf32r(vb.y - h.y);
            h.z = tf32r(vb.z); l.z = tf32r(vb.z - h.z);
            h.w = tf32r(vb.w); l.w = tf32r(vb.w - h.w);
            }
            *reinterpret_cast<float4 *>(reinterpret_cast<char *>(bh) + core_off(r, kc)) = h;
            *reinterpret_cast<float4 *>(reinterpret_cast<char *>(bl) + core_off(r, kc)) = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint64_t dah = sdesc(ah, 128, 256), dal = sdesc(al, 128, 256);
            const uint64_t dbh = sdesc(bh, 128, 256), dbl = sdesc(bl, 128, 256);
            if (passes >= 3) {
                mma_tf32(tmem, dah, dbl, c > 0);
                mma_tf32(tmem, dal, dbh, 1);
                mma_tf32(tmem, dah, dbh, 1);
            } else {
                mma_tf32(tmem, dah, dbh, c > 0);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                saddr(&bar))
                         : "memory");
        }
        // wait for the MMAs of this chunk before the buffers are rewritten
        asm volatile(
            "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                saddr(&bar)),
            "r"(phase)
            : "memory");
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows m), 128 columns (n)
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                       "=r"(v[7])
                     : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int m = 32 * warp + lane;
        for (int q = 0; q < 8; ++q) D[m + (c0 + q) * N] = __uint_as_float(v[q]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N));
}

__global__ void kt(float *out, int iters, long long *clk) {
    __shared__ __align__(1024) float ah[N * KC], bh[N * KC];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int e = tid; e < N * KC; e += blockDim.x) ah[e] = bh[e] = 0.5f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_base)),
                     "r"(N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const long long t0 = clock64();
        const uint64_t da = sdesc(ah, 128, 256), db = sdesc(bh, 128, 256);
        for (int i = 0; i < iters; ++i) mma_tf32(tmem, da, db, i > 0);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar))
                     : "memory");
        asm volatile(
            "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(
                saddr(&bar))
            : "memory");
        clk[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N));
}

int main() {
    std::vector<float> A(N * N), B(N * N), D(N * N);
    srand(1);
    for (auto &x : A) x = 2.f * rand() / RAND_MAX - 1.f;
    for (auto &x : B) x = 2.f * rand() / RAND_MAX - 1.f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, 4 * N * N);
    cudaMalloc(&dB, 4 * N * N);
    cudaMalloc(&dD, 4 * N * N);
    cudaMemcpy(dA, A.data(), 4 * N * N, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), 4 * N * N, cudaMemcpyHostToDevice);
    for (int passes : {1, 3, 4}) {
        cudaMemset(dD, 0, 4 * N * N);
        k<<<1, 128>>>(dA, dB, dD, passes);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error: %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(D.data(), dD, 4 * N * N, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxref = 0;
        for (int n = 0; n < N; ++n)
            for (int m = 0; m < N; ++m) {
                double ref = 0;
                for (int kk = 0; kk < N; ++kk) ref += (double)A[m * N + kk] * (double)B[n * N + kk];
                maxerr = fmax(maxerr, fabs(ref - D[m + n * N]));
                maxref = fmax(maxref, fabs(ref));
            }
        printf("passes %d: normwise error %.3e (max |ref| %.3f)\n", passes, maxerr / maxref, maxref);
    }
    {
        long long *dclk;
        cudaMalloc(&dclk, 8 * 148);
        for (int iters : {1, 3, 48, 1000}) {
            kt<<<1, 128>>>(dD, iters, dclk);
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, dclk, 8, cudaMemcpyDeviceToHost);
            printf("%d MMAs (128x128x8 tf32, no swizzle) back to back: %lld clk (%.1f clk/MMA, %.1f TF/s per SM at 1.965 GHz)\n",
                   iters, c, (double)c / iters, 2.0 * 128 * 128 * 8 * iters / (c / 1.965e9) / 1e12);
        }
    }
    return 0;
}
