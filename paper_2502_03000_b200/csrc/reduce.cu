// reduce.cu -- R3 / R4 / R5 / R7 kernels: diagonal scaling and
// dot-reductions that never form a product.
//
//  lm_diag_scale       <- _loops.py:144-158 (_diag_scale_left/right), bit-exact
//  lm_trace_of_product <- _loops.py:179-188 (_trace_of_product)
//  lm_diag_of_product  <- _loops.py:161-176 (_diag_of_product)
//  lm_triple_diag_dot  <- _loops.py:191-197 (_triple_diag_dot)
//
// trace(A*B) = sum over all (i,k) of A[i,k]*B[k,i]: A is read along its
// columns and B along its rows, so each 32x32 tile of B is staged through
// shared memory (transposed, padded) while the matching tile of A streams
// from registers; both operands are read from HBM exactly once
// (2 * p * q * sizeof(T) algorithmic bytes).  The reduction tree is fixed
// (static tile -> block assignment, fixed warp/block trees, a final
// single-block pass over per-block partials in index order), so results
// are bitwise reproducible run to run; they differ from the reference's
// sequential sum only by reassociation (<= 1e-12 relative, north star).
#include "common.cuh"

namespace lm {

constexpr int kTile = 32;
constexpr int kRedThreads = 256;  // 32 x 8

// ---- diag_scale -----------------------------------------------------------------

template <class T, bool RIGHT>
__global__ void __launch_bounds__(256) diag_scale_flat(Vec<const T> d, const T *__restrict__ b, T *__restrict__ out,
                                                       int64_t rows, int64_t nvec, int64_t n) {
    using V = typename Vec16<T>::type;
    constexpr int VN = Vec16<T>::N;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += nth) {
        const V x = ld_stream(reinterpret_cast<const V *>(b) + v);
        int64_t e0 = v * VN;
        int64_t j = e0 / rows, i = e0 - j * rows;
        V r;
#pragma unroll
        for (int l = 0; l < VN; ++l) {
            const T bv = (&x.x)[l];
            (&r.x)[l] = RIGHT ? rmul(bv, d[j]) : rmul(d[i], bv);
            if (++i == rows) {
                i = 0;
                ++j;
            }
        }
        st_stream(reinterpret_cast<V *>(out) + v, r);
    }
    if (blockIdx.x == 0)
        for (int64_t e = nvec * VN + threadIdx.x; e < n; e += blockDim.x) {
            const int64_t j = e / rows, i = e - j * rows;
            out[e] = RIGHT ? rmul(b[e], d[j]) : rmul(d[i], b[e]);
        }
}

template <class T, bool RIGHT>
__global__ void __launch_bounds__(256) diag_scale_strided(Vec<const T> d, View<const T> b, View<T> out, int64_t n) {
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += nth) {
        const int64_t j = e / b.rows, i = e - j * b.rows;
        out(i, j) = RIGHT ? rmul(b(i, j), d[j]) : rmul(d[i], b(i, j));
    }
}


template <class T> int diag_scale_impl(const lm_vec &dv, const lm_view &bv, int side, const lm_view &ov, cudaStream_t s) {
    const int64_t n = bv.rows * bv.cols;
    if (n == 0) return 0;
    Vec<const T> d{reinterpret_cast<const T *>(dv.ptr), dv.n, dv.stride};
    const bool flat = is_linear(bv) && is_linear(ov) && (reinterpret_cast<uintptr_t>(bv.ptr) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(ov.ptr) & 15) == 0;
    if (flat) {
        constexpr int VN = Vec16<T>::N;
        const int64_t nvec = n / VN;
        if (side)
            diag_scale_flat<T, true><<<ew_grid(nvec), 256, 0, s>>>(d, (const T *)bv.ptr, (T *)ov.ptr, bv.rows, nvec, n);
        else
            diag_scale_flat<T, false><<<ew_grid(nvec), 256, 0, s>>>(d, (const T *)bv.ptr, (T *)ov.ptr, bv.rows, nvec, n);
    } else {
        View<const T> b{(const T *)bv.ptr, bv.rows, bv.cols, bv.rs, bv.cs};
        View<T> o = to_view<T>(ov);
        if (side)
            diag_scale_strided<T, true><<<ew_grid(n), 256, 0, s>>>(d, b, o, n);
        else
            diag_scale_strided<T, false><<<ew_grid(n), 256, 0, s>>>(d, b, o, n);
    }
    LM_LAUNCHED(1);
    return 0;
}

// ---- trace(A*B) ---------------------------------------------------------------------

// Per-block partial of sum_{i,k} A[i,k]*B[k,i] over a static set of
// 32x32 (i,k) tiles.  Register double-buffering keeps the next tile's
// 8 loads per thread in flight while the current one is consumed.
template <class T>
__global__ void __launch_bounds__(kRedThreads) trace_tiles(View<const T> A, View<const T> B, int64_t ntr, int64_t ntiles,
                                                           T *__restrict__ partials) {
    __shared__ T sB[kTile][kTile + 1];
    __shared__ T red[kRedThreads / 32];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t p = A.rows, q = A.cols;
    T acc = T(0);
    T ra[4], rb[4];
    auto load = [&](int64_t t) {
        const int64_t i0 = (t % ntr) * kTile, k0 = (t / ntr) * kTile;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t ia = i0 + tx, ka = k0 + ty + 8 * r;
            ra[r] = (ia < p && ka < q) ? A(ia, ka) : T(0);
            const int64_t kb = k0 + tx, ib = i0 + ty + 8 * r;
            rb[r] = (kb < q && ib < p) ? B(kb, ib) : T(0);
        }
    };
    int64_t t = blockIdx.x;
    if (t < ntiles) load(t);
    for (; t < ntiles; t += gridDim.x) {
        T ca[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            ca[r] = ra[r];
            sB[ty + 8 * r][tx] = rb[r];  // sB[i_local][k_local] = B[k0+k_local, i0+i_local]
        }
        __syncthreads();
        if (t + gridDim.x < ntiles) load(t + gridDim.x);
#pragma unroll
        for (int r = 0; r < 4; ++r) acc = radd(acc, rmul(ca[r], sB[tx][ty + 8 * r]));
        __syncthreads();
    }
    acc = block_sum<T, kRedThreads>(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

// Sum of `n` partials in index order, fixed tree; writes *out.
template <class T> __global__ void __launch_bounds__(1024) sum_partials(const T *__restrict__ part, int64_t n, T *out) {
    __shared__ T red[32];
    T acc = T(0);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc = radd(acc, part[i]);
    acc = block_sum<T, 1024>(acc, red);
    if (threadIdx.x == 0) *out = acc;
}

template <class T> int trace_impl(const lm_view &av, const lm_view &bv, void *d_result, cudaStream_t s) {
    const int64_t p = av.rows, q = av.cols;
    View<const T> A{(const T *)av.ptr, av.rows, av.cols, av.rs, av.cs};
    View<const T> B{(const T *)bv.ptr, bv.rows, bv.cols, bv.rs, bv.cs};
    const int64_t ntr = ceil_div(p, kTile), ntc = ceil_div(q, kTile), ntiles = ntr * ntc;
    int64_t blocks = (int64_t)num_sms() * 8;
    if (blocks > ntiles) blocks = ntiles;
    if (blocks < 1) blocks = 1;
    Scratch part;
    if (int rc = part.alloc(sizeof(T) * blocks, s)) return rc;
    if (ntiles > 0) {
        trace_tiles<T><<<(unsigned)blocks, kRedThreads, 0, s>>>(A, B, ntr, ntiles, part.as<T>());
        LM_LAUNCHED(1);
    } else {
        LM_CUDA(cudaMemsetAsync(part.p, 0, sizeof(T), s));
    }
    sum_partials<T><<<1, 1024, 0, s>>>(part.as<T>(), blocks, (T *)d_result);
    LM_LAUNCHED(1);
    return 0;
}

// ---- diag(A*B) ------------------------------------------------------------------------

// Block (row tile I, k chunk c): partial[c][i] = sum over its k tiles.
template <class T>
__global__ void __launch_bounds__(kRedThreads) diag_tiles(View<const T> A, View<const T> B, int64_t ktiles_per_chunk,
                                                          T *__restrict__ partials) {
    __shared__ T sB[kTile][kTile + 1];
    __shared__ T red[8][kTile + 1];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t p = A.rows, q = A.cols;
    const int64_t i0 = (int64_t)blockIdx.x * kTile;
    const int64_t kt0 = (int64_t)blockIdx.y * ktiles_per_chunk;
    const int64_t ntc = ceil_div(q, kTile);
    T acc = T(0);
    for (int64_t kt = kt0; kt < kt0 + ktiles_per_chunk && kt < ntc; ++kt) {
        const int64_t k0 = kt * kTile;
        T ra[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t ia = i0 + tx, ka = k0 + ty + 8 * r;
            ra[r] = (ia < p && ka < q) ? A(ia, ka) : T(0);
            const int64_t kb = k0 + tx, ib = i0 + ty + 8 * r;
            sB[ty + 8 * r][tx] = (kb < q && ib < p) ? B(kb, ib) : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 4; ++r) acc = radd(acc, rmul(ra[r], sB[tx][ty + 8 * r]));
        __syncthreads();
    }
    red[ty][tx] = acc;
    __syncthreads();
    if (ty == 0) {
        T v = red[0][tx];
#pragma unroll
        for (int w = 1; w < 8; ++w) v = radd(v, red[w][tx]);
        if (i0 + tx < p) partials[blockIdx.y * p + i0 + tx] = v;
    }
}

template <class T>
__global__ void __launch_bounds__(256) diag_finish(const T *__restrict__ part, int64_t p, int64_t nchunks, Vec<T> out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= p) return;
    T acc = part[i];
    for (int64_t c = 1; c < nchunks; ++c) acc = radd(acc, part[c * p + i]);
    out[i] = acc;
}

template <class T> int diag_of_product_impl(const lm_view &av, const lm_view &bv, const lm_vec &ov, cudaStream_t s) {
    const int64_t p = av.rows, q = av.cols;
    if (p == 0) return 0;
    View<const T> A{(const T *)av.ptr, av.rows, av.cols, av.rs, av.cs};
    View<const T> B{(const T *)bv.ptr, bv.rows, bv.cols, bv.rs, bv.cs};
    const int64_t ntr = ceil_div(p, kTile), ntc = ceil_div(q, kTile);
    int64_t want_chunks = ceil_div((int64_t)num_sms() * 8, ntr);
    if (want_chunks > ntc) want_chunks = ntc;
    if (want_chunks < 1) want_chunks = 1;
    const int64_t per = ceil_div(ntc > 0 ? ntc : 1, want_chunks);
    const int64_t nchunks = ntc > 0 ? ceil_div(ntc, per) : 1;
    Scratch part;
    if (int rc = part.alloc(sizeof(T) * p * nchunks, s)) return rc;
    if (ntc > 0) {
        diag_tiles<T><<<dim3((unsigned)ntr, (unsigned)nchunks), kRedThreads, 0, s>>>(A, B, per, part.as<T>());
        LM_LAUNCHED(1);
    } else {
        LM_CUDA(cudaMemsetAsync(part.p, 0, sizeof(T) * p, s));
    }
    diag_finish<T><<<(unsigned)ceil_div(p, 256), 256, 0, s>>>(part.as<T>(), p, nchunks, to_vec<T>(ov));
    LM_LAUNCHED(1);
    return 0;
}

// ---- triple_diag_dot --------------------------------------------------------------------

template <class T>
__global__ void __launch_bounds__(256) triple_partials(Vec<const T> a, Vec<const T> d, Vec<const T> c, T *part) {
    __shared__ T red[8];
    T acc = T(0);
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += nth)
        acc = radd(acc, rmul(rmul(a[i], d[i]), c[i]));
    acc = block_sum<T, 256>(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

template <class T>
int triple_impl(const lm_vec &av, const lm_vec &dv, const lm_vec &cv, void *d_result, cudaStream_t s) {
    int64_t blocks = ceil_div(av.n, 256);
    if (blocks > num_sms() * 4) blocks = num_sms() * 4;
    if (blocks < 1) blocks = 1;
    Scratch part;
    if (int rc = part.alloc(sizeof(T) * blocks, s)) return rc;
    Vec<const T> a{(const T *)av.ptr, av.n, av.stride}, d{(const T *)dv.ptr, dv.n, dv.stride},
        c{(const T *)cv.ptr, cv.n, cv.stride};
    triple_partials<T><<<(unsigned)blocks, 256, 0, s>>>(a, d, c, part.as<T>());
    LM_LAUNCHED(1);
    sum_partials<T><<<1, 1024, 0, s>>>(part.as<T>(), blocks, (T *)d_result);
    LM_LAUNCHED(1);
    return 0;
}

}  // namespace lm

using namespace lm;

#define LM_DTYPE_DISPATCH(dtype, CALL_F64, CALL_F32)         \
    do {                                                     \
        if ((dtype) == LM_F64) return CALL_F64;              \
        if ((dtype) == LM_F32) return CALL_F32;              \
        set_error("bad dtype %d", (int)(dtype));             \
        return -1;                                           \
    } while (0)

extern "C" int lm_diag_scale(int dtype, lm_vec d, lm_view b, int side, lm_view out, void *stream) {
    clear_error();
    LM_REQUIRE(out.rows == b.rows && out.cols == b.cols, "diag_scale out shape mismatch");
    LM_REQUIRE(side == 0 || side == 1, "diag_scale side must be 0 (left) or 1 (right)");
    LM_REQUIRE(d.n == (side ? b.cols : b.rows), "diag_scale d length %lld", (long long)d.n);
    LM_DTYPE_DISPATCH(dtype, diag_scale_impl<double>(d, b, side, out, as_stream(stream)),
                      diag_scale_impl<float>(d, b, side, out, as_stream(stream)));
}

extern "C" int lm_trace_of_product(int dtype, lm_view a, lm_view b, void *d_result, void *stream) {
    clear_error();
    LM_REQUIRE(b.rows == a.cols && b.cols == a.rows, "trace_of_product needs b of shape (%lld,%lld)",
               (long long)a.cols, (long long)a.rows);
    LM_DTYPE_DISPATCH(dtype, trace_impl<double>(a, b, d_result, as_stream(stream)),
                      trace_impl<float>(a, b, d_result, as_stream(stream)));
}

extern "C" int lm_diag_of_product(int dtype, lm_view a, lm_view b, lm_vec out, void *stream) {
    clear_error();
    LM_REQUIRE(b.rows == a.cols && b.cols == a.rows, "diag_of_product shape mismatch");
    LM_REQUIRE(out.n == a.rows, "diag_of_product out length");
    LM_DTYPE_DISPATCH(dtype, diag_of_product_impl<double>(a, b, out, as_stream(stream)),
                      diag_of_product_impl<float>(a, b, out, as_stream(stream)));
}

extern "C" int lm_triple_diag_dot(int dtype, lm_vec a, lm_vec d, lm_vec c, void *d_result, void *stream) {
    clear_error();
    LM_REQUIRE(d.n == a.n && c.n == a.n, "triple_diag_dot needs three equal-length vectors");
    LM_DTYPE_DISPATCH(dtype, triple_impl<double>(a, d, c, d_result, as_stream(stream)),
                      triple_impl<float>(a, d, c, d_result, as_stream(stream)));
}

// ---- sum of a strided vector (naive arm's trace of a materialised
// matrix, expr.py:371-377 -- np.sum(np.diagonal(x)) in the reference).
namespace lm {
template <class T> __global__ void __launch_bounds__(256) vec_partials(Vec<const T> v, T *part) {
    __shared__ T red[8];
    T acc = T(0);
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < v.n; i += nth) acc = radd(acc, v[i]);
    acc = block_sum<T, 256>(acc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
template <class T> int vec_sum_impl(const lm_vec &vv, void *d_result, cudaStream_t s) {
    int64_t blocks = ceil_div(vv.n, 256);
    if (blocks > num_sms() * 4) blocks = num_sms() * 4;
    if (blocks < 1) blocks = 1;
    Scratch part;
    if (int rc = part.alloc(sizeof(T) * blocks, s)) return rc;
    vec_partials<T><<<(unsigned)blocks, 256, 0, s>>>(Vec<const T>{(const T *)vv.ptr, vv.n, vv.stride}, part.as<T>());
    LM_LAUNCHED(1);
    sum_partials<T><<<1, 1024, 0, s>>>(part.as<T>(), blocks, (T *)d_result);
    LM_LAUNCHED(1);
    return 0;
}
}  // namespace lm

extern "C" int lm_vec_sum(int dtype, lm_vec v, void *d_result, void *stream) {
    clear_error();
    LM_DTYPE_DISPATCH(dtype, vec_sum_impl<double>(v, d_result, as_stream(stream)),
                      vec_sum_impl<float>(v, d_result, as_stream(stream)));
}
