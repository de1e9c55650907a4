// elementwise.cu -- the R1 fused element-wise family.
//
// Reference: lazymat/_loops.py:37-84 (_fused1.._fused4, _fused_axpy),
// wrapped by kernels.fused_axpby_n (kernels.py:32-62).  Per element the
// reference computes acc = c0*s0; acc = acc + ck*sk (k ascending), one
// rounding per multiply and per add, no FMA.  These kernels do exactly
// that (explicit __dmul_rn/__dadd_rn), so results are bit-identical.
//
// HBM-bound: algorithmic bytes = (nterms + 1) * n_elems * sizeof(T).
// Layout fast path: every operand enumerates its elements in F-order
// with unit step ("linear") -> one flat stream, 16-byte vector loads
// (ld.global.nc.L1::no_allocate), streaming stores, 2 vectors in flight
// per thread per source, grid = a multiple of the SM count.  Anything
// else (transposed / strided views, R2) takes the 2-D strided path.
#include "common.cuh"

namespace lm {

constexpr int kEwThreads = 256;
constexpr int kMaxTermsPerPass = 8;

template <class T> struct AxArgs {
    const T *src[kMaxTermsPerPass];
    double c[kMaxTermsPerPass];
    T *out;
};

template <class V> __device__ __forceinline__ auto &lane(V &v, int i) { return (&v.x)[i]; }

template <class T, int NT, bool FROM_OUT>
__device__ __forceinline__ T axpby_elem(const AxArgs<T> &a, const T (&x)[kMaxTermsPerPass], T prev) {
    T acc;
    int k0 = 0;
    if (FROM_OUT) {
        acc = prev;
    } else {
        acc = rmul(T(a.c[0]), x[0]);
        k0 = 1;
    }
#pragma unroll
    for (int k = k0; k < NT; ++k) acc = radd(acc, rmul(T(a.c[k]), x[k]));
    return acc;
}

// Flat (linear) path, 16-byte vectors, UNROLL vectors per thread per trip.
template <class T, int NT, bool FROM_OUT>
__global__ void __launch_bounds__(kEwThreads) axpby_flat_vec(AxArgs<T> a, int64_t nvec, int64_t n) {
    using V = typename Vec16<T>::type;
    constexpr int VN = Vec16<T>::N;
    constexpr int UNROLL = 2;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + (UNROLL - 1) * nth < nvec; v += UNROLL * nth) {
        V x[UNROLL][kMaxTermsPerPass];
        V o[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
#pragma unroll
            for (int k = 0; k < NT; ++k) x[u][k] = ld_stream(reinterpret_cast<const V *>(a.src[k]) + v + u * nth);
            if (FROM_OUT) o[u] = *(reinterpret_cast<const V *>(a.out) + v + u * nth);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            V r;
#pragma unroll
            for (int e = 0; e < VN; ++e) {
                T xs[kMaxTermsPerPass];
#pragma unroll
                for (int k = 0; k < NT; ++k) xs[k] = lane(x[u][k], e);
                lane(r, e) = axpby_elem<T, NT, FROM_OUT>(a, xs, FROM_OUT ? lane(o[u], e) : T(0));
            }
            st_stream(reinterpret_cast<V *>(a.out) + v + u * nth, r);
        }
    }
    for (; v < nvec; v += nth) {
        V x[kMaxTermsPerPass];
        V o;
#pragma unroll
        for (int k = 0; k < NT; ++k) x[k] = ld_stream(reinterpret_cast<const V *>(a.src[k]) + v);
        if (FROM_OUT) o = *(reinterpret_cast<const V *>(a.out) + v);
        V r;
#pragma unroll
        for (int e = 0; e < VN; ++e) {
            T xs[kMaxTermsPerPass];
#pragma unroll
            for (int k = 0; k < NT; ++k) xs[k] = lane(x[k], e);
            lane(r, e) = axpby_elem<T, NT, FROM_OUT>(a, xs, FROM_OUT ? lane(o, e) : T(0));
        }
        st_stream(reinterpret_cast<V *>(a.out) + v, r);
    }
    // scalar tail
    if (blockIdx.x == 0) {
        for (int64_t e = nvec * VN + threadIdx.x; e < n; e += blockDim.x) {
            T xs[kMaxTermsPerPass];
#pragma unroll
            for (int k = 0; k < NT; ++k) xs[k] = a.src[k][e];
            a.out[e] = axpby_elem<T, NT, FROM_OUT>(a, xs, FROM_OUT ? a.out[e] : T(0));
        }
    }
}

// Flat path without vector alignment.
template <class T, int NT, bool FROM_OUT>
__global__ void __launch_bounds__(kEwThreads) axpby_flat_scalar(AxArgs<T> a, int64_t n) {
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += nth) {
        T xs[kMaxTermsPerPass];
#pragma unroll
        for (int k = 0; k < NT; ++k) xs[k] = a.src[k][e];
        a.out[e] = axpby_elem<T, NT, FROM_OUT>(a, xs, FROM_OUT ? a.out[e] : T(0));
    }
}

struct Strides {
    int64_t rs[kMaxTermsPerPass], cs[kMaxTermsPerPass];
    int64_t ors, ocs;
};

// General strided 2-D path (R2 views): i fastest.
template <class T, int NT, bool FROM_OUT>
__global__ void __launch_bounds__(kEwThreads) axpby_strided(AxArgs<T> a, Strides st, int64_t rows, int64_t n) {
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += nth) {
        const int64_t j = e / rows, i = e - j * rows;
        T xs[kMaxTermsPerPass];
#pragma unroll
        for (int k = 0; k < NT; ++k) xs[k] = a.src[k][i * st.rs[k] + j * st.cs[k]];
        T &o = a.out[i * st.ors + j * st.ocs];
        o = axpby_elem<T, NT, FROM_OUT>(a, xs, FROM_OUT ? o : T(0));
    }
}

bool is_linear(const lm_view &v) {
    if (v.rows <= 1) return v.cols <= 1 || v.cs == 1;
    if (v.cols <= 1) return v.rs == 1;
    return v.rs == 1 && v.cs == v.rows;
}

int ew_grid(int64_t work_items) {
    int64_t blocks = ceil_div(work_items, kEwThreads);
    int64_t cap = (int64_t)num_sms() * 8;  // 8 x 256 threads resident per SM
    if (blocks > cap) blocks = cap;
    return (int)(blocks < 1 ? 1 : blocks);
}

template <class T, int NT, bool FROM_OUT>
int launch_axpby(const AxArgs<T> &a, const lm_view *srcs, const lm_view &out, bool flat, cudaStream_t s) {
    const int64_t n = out.rows * out.cols;
    if (n == 0) return 0;
    if (flat) {
        bool aligned = (reinterpret_cast<uintptr_t>(a.out) & 15) == 0;
        for (int k = 0; k < NT; ++k) aligned = aligned && (reinterpret_cast<uintptr_t>(a.src[k]) & 15) == 0;
        if (aligned) {
            constexpr int VN = Vec16<T>::N;
            const int64_t nvec = n / VN;
            axpby_flat_vec<T, NT, FROM_OUT><<<ew_grid(ceil_div(nvec, 2)), kEwThreads, 0, s>>>(a, nvec, n);
        } else {
            axpby_flat_scalar<T, NT, FROM_OUT><<<ew_grid(n), kEwThreads, 0, s>>>(a, n);
        }
    } else {
        Strides st{};
        for (int k = 0; k < NT; ++k) {
            st.rs[k] = srcs[k].rs;
            st.cs[k] = srcs[k].cs;
        }
        st.ors = out.rs;
        st.ocs = out.cs;
        axpby_strided<T, NT, FROM_OUT><<<ew_grid(n), kEwThreads, 0, s>>>(a, st, out.rows, n);
    }
    LM_LAUNCHED(1);
    return 0;
}

template <class T, bool FROM_OUT>
int dispatch_axpby(int nt, const AxArgs<T> &a, const lm_view *srcs, const lm_view &out, bool flat, cudaStream_t s) {
    switch (nt) {
    case 1: return launch_axpby<T, 1, FROM_OUT>(a, srcs, out, flat, s);
    case 2: return launch_axpby<T, 2, FROM_OUT>(a, srcs, out, flat, s);
    case 3: return launch_axpby<T, 3, FROM_OUT>(a, srcs, out, flat, s);
    case 4: return launch_axpby<T, 4, FROM_OUT>(a, srcs, out, flat, s);
    case 5: return launch_axpby<T, 5, FROM_OUT>(a, srcs, out, flat, s);
    case 6: return launch_axpby<T, 6, FROM_OUT>(a, srcs, out, flat, s);
    case 7: return launch_axpby<T, 7, FROM_OUT>(a, srcs, out, flat, s);
    case 8: return launch_axpby<T, 8, FROM_OUT>(a, srcs, out, flat, s);
    }
    set_error("axpby: bad term count %d", nt);
    return -1;
}

template <class T>
int fused_axpby_impl(int nterms, const double *coeffs, const lm_view *srcs, const lm_view &out, cudaStream_t s) {
    bool flat = is_linear(out);
    for (int k = 0; k < nterms; ++k) flat = flat && is_linear(srcs[k]);
    // Terms beyond the first pass continue accumulating into `out`, the
    // same per-element sequence as the reference's _fused_axpy chain
    // (kernels.py:59-62): storing the f64 accumulator is exact.
    for (int k0 = 0, nt = 0; k0 < nterms; k0 += nt) {
        nt = (nterms - k0) < kMaxTermsPerPass ? (nterms - k0) : kMaxTermsPerPass;
        AxArgs<T> a{};
        for (int k = 0; k < nt; ++k) {
            a.src[k] = reinterpret_cast<const T *>(srcs[k0 + k].ptr);
            a.c[k] = coeffs[k0 + k];
        }
        a.out = reinterpret_cast<T *>(out.ptr);
        int rc = (k0 == 0) ? dispatch_axpby<T, false>(nt, a, srcs + k0, out, flat, s)
                           : dispatch_axpby<T, true>(nt, a, srcs + k0, out, flat, s);
        if (rc) return rc;
    }
    return 0;
}

}  // namespace lm

using namespace lm;

extern "C" int lm_fused_axpby(int dtype, int nterms, const double *coeffs, const lm_view *srcs, lm_view out,
                              void *stream) {
    clear_error();
    LM_REQUIRE(nterms >= 1 && coeffs && srcs, "fused_axpby needs matching non-empty lists");
    for (int k = 0; k < nterms; ++k)
        LM_REQUIRE(srcs[k].rows == out.rows && srcs[k].cols == out.cols, "fused_axpby source %d shape mismatch", k);
    if (dtype == LM_F64) return fused_axpby_impl<double>(nterms, coeffs, srcs, out, as_stream(stream));
    if (dtype == LM_F32) return fused_axpby_impl<float>(nterms, coeffs, srcs, out, as_stream(stream));
    set_error("bad dtype %d", dtype);
    return -1;
}

// ---- plain copy (np.copyto in the reference executor, rewrite.py:653;
// the view-extraction copies of the naive arm).  No trace event, exact.
namespace lm {

template <class T>
__global__ void __launch_bounds__(256) copy_strided(View<const T> src, View<T> dst, int64_t n) {
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += nth) {
        const int64_t j = e / src.rows, i = e - j * src.rows;
        dst(i, j) = src(i, j);
    }
}

template <class T> int copy_impl(const lm_view &s, const lm_view &d, cudaStream_t st) {
    const int64_t n = s.rows * s.cols;
    if (n == 0) return 0;
    if (is_linear(s) && is_linear(d)) {
        LM_CUDA(cudaMemcpyAsync(d.ptr, s.ptr, sizeof(T) * n, cudaMemcpyDeviceToDevice, st));
        return 0;
    }
    copy_strided<T><<<ew_grid(n), 256, 0, st>>>(View<const T>{(const T *)s.ptr, s.rows, s.cols, s.rs, s.cs},
                                                to_view<T>(d), n);
    LM_LAUNCHED(1);
    return 0;
}

}  // namespace lm

extern "C" int lm_copy(int dtype, lm_view src, lm_view dst, void *stream) {
    clear_error();
    LM_REQUIRE(src.rows == dst.rows && src.cols == dst.cols, "copy shape mismatch");
    if (dtype == LM_F64) return copy_impl<double>(src, dst, as_stream(stream));
    if (dtype == LM_F32) return copy_impl<float>(src, dst, as_stream(stream));
    set_error("bad dtype %d", dtype);
    return -1;
}
