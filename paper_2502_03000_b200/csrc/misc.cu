// misc.cu -- structure scan, data movement and the batched size-class
// kernel.
//
//  lm_analyze            <- _loops.py:15-34 (_analyze), exact integer result
//  lm_transpose_copy     <- _loops.py:391-396
//  lm_diag_materialise   <- _loops.py:399-407
//  lm_set_identity       <- kernels.py:296-297 (explicit_inverse's I)
//  lm_analyze_batched, lm_expr_atb_schur_trace_batched: batched configs
//
// The structure scan runs at REWRITE time for every solve on a leaf
// (rewrite.py:146-173) and is HBM-bound: 8 bytes per element read once.
// Square matrices are walked as tile pairs (I,J) / (J,I) with I <= J so
// the symmetry test A[i,j] == A[j,i] reads every element exactly once;
// the transposed tile is staged through shared memory.
#include "common.cuh"

namespace lm {

constexpr int kAT = 32;

template <class T>
__global__ void __launch_bounds__(256) analyze_tiles(View<const T> A, int square, int64_t npairs, int64_t tr,
                                                     unsigned long long *out /* lbw, ubw, asym */) {
    __shared__ T sT[kAT][kAT + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    unsigned long long lbw = 0, ubw = 0, asym = 0;
    const int64_t tc = ceil_div(A.cols, kAT);
    for (int64_t t = blockIdx.x; t < npairs; t += gridDim.x) {
        int64_t I, J;
        if (square) {
            // triangular pair index -> (I <= J)
            int64_t jj = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
            while ((jj + 1) * (jj + 2) / 2 <= t) ++jj;
            while (jj * (jj + 1) / 2 > t) --jj;
            J = jj;
            I = t - jj * (jj + 1) / 2;
        } else {
            I = t % tr;
            J = t / tr;
        }
        const int64_t i0 = I * kAT, j0 = J * kAT;
        // tile (I,J): element (i0+tx, j0+ty+8r)
        T v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t i = i0 + tx, j = j0 + ty + 8 * r;
            v[r] = (i < A.rows && j < A.cols) ? A(i, j) : T(0);
            if (v[r] != T(0)) {
                const int64_t d = i - j;
                if (d > 0) lbw = max(lbw, (unsigned long long)d);
                else if (-d > 0) ubw = max(ubw, (unsigned long long)(-d));
            }
        }
        if (square && I != J) {
            // tile (J,I): element (j0+tx, i0+ty+8r); stage transposed
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t i = j0 + tx, j = i0 + ty + 8 * r;
                const T w = (i < A.rows && j < A.cols) ? A(i, j) : T(0);
                sT[tx][ty + 8 * r] = w;  // sT[a][b] = A(j0+a, i0+b)
                if (w != T(0)) {
                    const int64_t d = i - j;
                    if (d > 0) lbw = max(lbw, (unsigned long long)d);
                    else if (-d > 0) ubw = max(ubw, (unsigned long long)(-d));
                }
            }
            __syncthreads();
            // compare A(i0+tx, j0+c) with A(j0+c, i0+tx) = sT[c][tx]
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int64_t i = i0 + tx, j = j0 + ty + 8 * r;
                if (i < A.rows && j < A.cols && v[r] != sT[ty + 8 * r][tx]) asym = 1;
            }
            __syncthreads();
        } else if (square) {
            // diagonal tile: compare within (i < j)
#pragma unroll
            for (int r = 0; r < 4; ++r) sT[ty + 8 * r][tx] = v[r];  // sT[jl][il] = A(i0+il, j0+jl)
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int il = tx, jl = ty + 8 * r;
                const int64_t i = i0 + il, j = j0 + jl;
                if (i < j && j < A.cols && i < A.rows && sT[jl][il] != sT[il][jl]) asym = 1;
            }
            __syncthreads();
        }
    }
    // reduce: warp max then one atomic per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lbw = max(lbw, __shfl_xor_sync(0xffffffffu, lbw, o));
        ubw = max(ubw, __shfl_xor_sync(0xffffffffu, ubw, o));
        asym |= __shfl_xor_sync(0xffffffffu, asym, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (lbw) atomicMax(&out[0], lbw);
        if (ubw) atomicMax(&out[1], ubw);
        if (asym) atomicOr(&out[2], 1ull);
    }
}

__global__ void analyze_finish(unsigned long long *out, int square) {
    if (threadIdx.x == 0) out[2] = (square && out[2] == 0) ? 1ull : 0ull;
}

template <class T> int analyze_impl(const lm_view &av, int square, int64_t *d_out, cudaStream_t s) {
    LM_CUDA(cudaMemsetAsync(d_out, 0, 3 * sizeof(int64_t), s));
    View<const T> A{(const T *)av.ptr, av.rows, av.cols, av.rs, av.cs};
    const int64_t tr = ceil_div(av.rows, kAT), tc = ceil_div(av.cols, kAT);
    const int64_t npairs = square ? tr * (tr + 1) / 2 : tr * tc;
    if (npairs > 0) {
        int64_t blocks = (int64_t)num_sms() * 8;
        if (blocks > npairs) blocks = npairs;
        analyze_tiles<T><<<(unsigned)blocks, 256, 0, s>>>(A, square, npairs, tr, (unsigned long long *)d_out);
        LM_LAUNCHED(1);
    }
    analyze_finish<<<1, 32, 0, s>>>((unsigned long long *)d_out, square);
    LM_LAUNCHED(1);
    return 0;
}

// ---- transpose / diag fill / identity ------------------------------------------

template <class T> __global__ void __launch_bounds__(256) transpose_tiles(View<const T> A, View<T> O) {
    __shared__ T sT[kAT][kAT + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * kAT, j0 = (int64_t)blockIdx.y * kAT;  // tile of A
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t i = i0 + tx, j = j0 + ty + 8 * r;
        sT[ty + 8 * r][tx] = (i < A.rows && j < A.cols) ? A(i, j) : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        // O(j, i) = A(i, j); write along O's rows j0+tx
        const int64_t oj = j0 + tx, oi = i0 + ty + 8 * r;
        if (oj < A.cols && oi < A.rows) O(oj, oi) = sT[tx][ty + 8 * r];
    }
}

template <class T> __global__ void diag_fill(Vec<const T> d, View<T> O, int ident) {
    const int64_t n = O.rows;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += nth) {
        const int64_t j = e / n, i = e - j * n;
        O(i, j) = (i == j) ? (ident ? T(1) : d[i]) : T(0);
    }
}


// ---- batched structure scan ---------------------------------------------------------

// One CTA per instance.  n <= 64: the instance is staged through shared
// memory once (coalesced), the symmetric partner is read from smem with an
// odd row stride (conflict-free); larger n read the partner from L1/L2.
template <class T>
__global__ void __launch_bounds__(256) analyze_batched_k(int64_t n, const T *__restrict__ A, int64_t *out) {
    __shared__ T sA[64 * 65];
    const T *a = A + (int64_t)blockIdx.x * n * n;
    unsigned long long lbw = 0, ubw = 0, asym = 0;
    if (n <= 64) {
        const int nn = (int)n, ld = nn + 1;
        for (int e = threadIdx.x; e < nn * nn; e += blockDim.x) {
            const int j = e / nn, i = e - j * nn;
            sA[j * ld + i] = __ldg(a + e);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nn * nn; e += blockDim.x) {
            const int j = e / nn, i = e - j * nn;
            const T v = sA[j * ld + i];
            if (v != T(0)) {
                const int d = i - j;
                if (d > 0) lbw = max(lbw, (unsigned long long)d);
                else if (-d > 0) ubw = max(ubw, (unsigned long long)(-d));
            }
            if (i < j && v != sA[i * ld + j]) asym = 1;
        }
    } else {
        for (int64_t e = threadIdx.x; e < n * n; e += blockDim.x) {
            const int64_t j = e / n, i = e - j * n;
            const T v = a[e];
            if (v != T(0)) {
                const int64_t d = i - j;
                if (d > 0) lbw = max(lbw, (unsigned long long)d);
                else if (-d > 0) ubw = max(ubw, (unsigned long long)(-d));
            }
            if (i < j && v != a[j + i * n]) asym = 1;
        }
    }
    __shared__ unsigned long long r[3];
    if (threadIdx.x == 0) r[0] = r[1] = r[2] = 0;
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lbw = max(lbw, __shfl_xor_sync(0xffffffffu, lbw, o));
        ubw = max(ubw, __shfl_xor_sync(0xffffffffu, ubw, o));
        asym |= __shfl_xor_sync(0xffffffffu, asym, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&r[0], lbw);
        atomicMax(&r[1], ubw);
        atomicOr(&r[2], asym);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[3 * blockIdx.x + 0] = (int64_t)r[0];
        out[3 * blockIdx.x + 1] = (int64_t)r[1];
        out[3 * blockIdx.x + 2] = r[2] ? 0 : 1;
    }
}

}  // namespace lm

using namespace lm;

extern "C" int lm_analyze(int dtype, lm_view a, int square, int64_t *d_out, void *stream) {
    clear_error();
    LM_REQUIRE(!square || a.rows == a.cols, "analyze: square flag on a non-square view");
    if (dtype == LM_F64) return analyze_impl<double>(a, square, d_out, as_stream(stream));
    if (dtype == LM_F32) return analyze_impl<float>(a, square, d_out, as_stream(stream));
    set_error("bad dtype");
    return -1;
}

extern "C" int lm_transpose_copy(int dtype, lm_view a, lm_view out, void *stream) {
    clear_error();
    LM_REQUIRE(out.rows == a.cols && out.cols == a.rows, "transpose_copy out shape mismatch");
    if (a.rows == 0 || a.cols == 0) return 0;
    dim3 grid((unsigned)ceil_div(a.rows, kAT), (unsigned)ceil_div(a.cols, kAT));
    cudaStream_t s = as_stream(stream);
    if (dtype == LM_F64)
        transpose_tiles<double><<<grid, 256, 0, s>>>(View<const double>{(const double *)a.ptr, a.rows, a.cols, a.rs, a.cs},
                                                    to_view<double>(out));
    else if (dtype == LM_F32)
        transpose_tiles<float><<<grid, 256, 0, s>>>(View<const float>{(const float *)a.ptr, a.rows, a.cols, a.rs, a.cs},
                                                   to_view<float>(out));
    else {
        set_error("bad dtype");
        return -1;
    }
    LM_LAUNCHED(1);
    return 0;
}

extern "C" int lm_diag_materialise(int dtype, lm_vec d, lm_view out, void *stream) {
    clear_error();
    LM_REQUIRE(out.rows == out.cols && d.n == out.rows, "diag_materialise shape mismatch");
    if (out.rows == 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int g = ew_grid(out.rows * out.rows);
    if (dtype == LM_F64)
        diag_fill<double><<<g, 256, 0, s>>>(Vec<const double>{(const double *)d.ptr, d.n, d.stride}, to_view<double>(out), 0);
    else if (dtype == LM_F32)
        diag_fill<float><<<g, 256, 0, s>>>(Vec<const float>{(const float *)d.ptr, d.n, d.stride}, to_view<float>(out), 0);
    else {
        set_error("bad dtype");
        return -1;
    }
    LM_LAUNCHED(1);
    return 0;
}

extern "C" int lm_set_identity(int dtype, lm_view out, void *stream) {
    clear_error();
    LM_REQUIRE(out.rows == out.cols, "set_identity needs a square output");
    if (out.rows == 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int g = ew_grid(out.rows * out.rows);
    if (dtype == LM_F64)
        diag_fill<double><<<g, 256, 0, s>>>(Vec<const double>{nullptr, 0, 0}, to_view<double>(out), 1);
    else if (dtype == LM_F32)
        diag_fill<float><<<g, 256, 0, s>>>(Vec<const float>{nullptr, 0, 0}, to_view<float>(out), 1);
    else {
        set_error("bad dtype");
        return -1;
    }
    LM_LAUNCHED(1);
    return 0;
}

// ---- synthetic data: U(lo, hi) from a counter-based hash of GLOBAL (i, j) ----
// Any rank can generate any slice of a distributed matrix consistently
// (config 5b: rank g needs rows of B and a column block of B).  Not on the
// evaluation path; bench/test data only.
namespace lm {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
template <class T>
__global__ void fill_hash_uniform(View<T> o, uint64_t seed, int64_t row0, int64_t col0, int64_t gld, double lo,
                                  double hi) {
    const int64_t n = o.rows * o.cols, nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += nth) {
        const int64_t j = e / o.rows, i = e - j * o.rows;
        const uint64_t g = (uint64_t)(row0 + i) + (uint64_t)(col0 + j) * (uint64_t)gld;
        const double u = (double)(mix64(seed ^ mix64(g)) >> 11) * (1.0 / 9007199254740992.0);
        o(i, j) = (T)(lo + (hi - lo) * u);
    }
}
}  // namespace lm

extern "C" int lm_fill_uniform(int dtype, lm_view out, uint64_t seed, int64_t row0, int64_t col0, int64_t global_rows,
                               double lo, double hi, void *stream) {
    clear_error();
    const int64_t n = out.rows * out.cols;
    if (n == 0) return 0;
    cudaStream_t s = as_stream(stream);
    if (dtype == LM_F64)
        fill_hash_uniform<double><<<ew_grid(n), 256, 0, s>>>(to_view<double>(out), seed, row0, col0, global_rows, lo, hi);
    else if (dtype == LM_F32)
        fill_hash_uniform<float><<<ew_grid(n), 256, 0, s>>>(to_view<float>(out), seed, row0, col0, global_rows, lo, hi);
    else {
        set_error("bad dtype");
        return -1;
    }
    LM_LAUNCHED(1);
    return 0;
}

extern "C" int lm_analyze_batched(int dtype, int64_t n, int64_t batch, const void *a, int64_t *d_out, void *stream) {
    clear_error();
    if (batch == 0) return 0;
    cudaStream_t s = as_stream(stream);
    if (dtype == LM_F64)
        analyze_batched_k<double><<<(unsigned)batch, 256, 0, s>>>(n, (const double *)a, d_out);
    else if (dtype == LM_F32)
        analyze_batched_k<float><<<(unsigned)batch, 256, 0, s>>>(n, (const float *)a, d_out);
    else {
        set_error("bad dtype");
        return -1;
    }
    LM_LAUNCHED(1);
    return 0;
}

