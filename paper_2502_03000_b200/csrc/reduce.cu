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

// Column-panel streaming kernel (F-order b and out: rs == 1): a thread owns
// VN consecutive rows and walks a chunk of columns, U vectors in flight;
// the row scale d[i..] is loaded once (left) or one d[j] per column
// (right, a broadcast).  No index division anywhere.
template <class T, bool RIGHT, bool VEC>
__global__ void __launch_bounds__(256) diag_scale_cols(Vec<const T> d, const T *__restrict__ b, int64_t ldb,
                                                       T *__restrict__ out, int64_t ldo, int64_t rows, int64_t cols,
                                                       int64_t cols_per_block) {
    using V = typename Vec16<T>::type;
    constexpr int VN = VEC ? Vec16<T>::N : 1;
    constexpr int U = 4;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * VN;
    if (i >= rows) return;
    const int64_t j0 = (int64_t)blockIdx.y * cols_per_block;
    const int64_t j1 = j0 + cols_per_block < cols ? j0 + cols_per_block : cols;
    T dl[VN];
    if (!RIGHT)
#pragma unroll
        for (int l = 0; l < VN; ++l) dl[l] = d[i + l];
    int64_t j = j0;
    for (; j + U <= j1; j += U) {
        T x[U][VN];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (VEC) {
                const V t = ld_stream(reinterpret_cast<const V *>(b + i + (j + u) * ldb));
#pragma unroll
                for (int l = 0; l < VN; ++l) x[u][l] = (&t.x)[l];
            } else {
                x[u][0] = b[i + (j + u) * ldb];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const T dj = RIGHT ? d[j + u] : T(0);
            if (VEC) {
                V r;
#pragma unroll
                for (int l = 0; l < VN; ++l) (&r.x)[l] = RIGHT ? rmul(x[u][l], dj) : rmul(dl[l], x[u][l]);
                st_stream(reinterpret_cast<V *>(out + i + (j + u) * ldo), r);
            } else {
                out[i + (j + u) * ldo] = RIGHT ? rmul(x[u][0], dj) : rmul(dl[0], x[u][0]);
            }
        }
    }
    for (; j < j1; ++j) {
        const T dj = RIGHT ? d[j] : T(0);
#pragma unroll
        for (int l = 0; l < VN; ++l) {
            const T bv = b[i + l + j * ldb];
            out[i + l + j * ldo] = RIGHT ? rmul(bv, dj) : rmul(dl[l], bv);
        }
    }
}

// 32-byte-vector column-chunk kernel: CTA c owns the row chunk (c % gx) of
// the 4 columns 4 * (c / gx) ..; all 4 loads are issued before the first
// store.  Many short CTAs beat a persistent one-wave grid here (measured on
// B200 for 128 MB - 2 GB operands, tools/probes/ds_probe.cu: 6.2-6.8 TB/s
// vs 5.6-5.9 TB/s).  The left scale d[i..i+VN) is loaded once per thread,
// the right scale d[j] once per column (a warp broadcast).
template <class T, bool RIGHT>
__global__ void __launch_bounds__(256) diag_scale_cols32(Vec<const T> d, const T *__restrict__ b, int64_t ldb,
                                                         T *__restrict__ out, int64_t ldo, int64_t rows, int64_t cols,
                                                         int gx) {
    pdl_wait();  // inputs may be the previous kernel's output (PDL)
    pdl_trigger();
    constexpr int VN = Vec32<T>::N;
    constexpr int U = 4;
    const int64_t chunk = blockIdx.x / gx;
    const int64_t i = ((int64_t)(blockIdx.x - chunk * gx) * blockDim.x + threadIdx.x) * VN;
    if (i >= rows) return;
    T dl[VN];
    if (!RIGHT)
#pragma unroll
        for (int l = 0; l < VN; ++l) dl[l] = d[i + l];
    const int64_t j0 = chunk * U;
    const T *bp = b + i + j0 * ldb;
    T *op = out + i + j0 * ldo;
    if (j0 + U <= cols) {
        Vec32<T> x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ld_stream32(bp + u * ldb);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const T dj = RIGHT ? d[j0 + u] : T(0);
            Vec32<T> r;
#pragma unroll
            for (int l = 0; l < VN; ++l) r.v[l] = RIGHT ? rmul(x[u].v[l], dj) : rmul(dl[l], x[u].v[l]);
            st_stream32(op + u * ldo, r);
        }
    } else {
        for (int u = 0; j0 + u < cols; ++u) {
            const Vec32<T> x = ld_stream32(bp + u * ldb);
            const T dj = RIGHT ? d[j0 + u] : T(0);
            Vec32<T> r;
#pragma unroll
            for (int l = 0; l < VN; ++l) r.v[l] = RIGHT ? rmul(x.v[l], dj) : rmul(dl[l], x.v[l]);
            st_stream32(op + u * ldo, r);
        }
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
    const bool cm = bv.rs == 1 && ov.rs == 1;  // column-major b and out (any leading dims)
    if (cm) {
        constexpr int VN = Vec16<T>::N;
        const int64_t ldb = bv.cols > 1 ? bv.cs : bv.rows, ldo = ov.cols > 1 ? ov.cs : ov.rows;
        constexpr int VN32 = Vec32<T>::N;
        if (bv.rows % VN32 == 0 && ldb % VN32 == 0 && ldo % VN32 == 0 && aligned32(bv.ptr) && aligned32(ov.ptr)) {
            const int gx = (int)ceil_div(bv.rows, 256 * VN32);
            const int64_t grid = gx * ceil_div(bv.cols, 4);
            if (grid <= 0x7fffffff) {
                auto kern = side ? diag_scale_cols32<T, true> : diag_scale_cols32<T, false>;
                LM_CUDA(launch_pdl(kern, dim3((unsigned)grid), dim3(256), 0, s, d, (const T *)bv.ptr, ldb, (T *)ov.ptr,
                                   ldo, bv.rows, bv.cols, gx));
                LM_LAUNCHED(1);
                return 0;
            }
        }
        const bool vec = bv.rows % VN == 0 && ldb % VN == 0 && ldo % VN == 0 &&
                         (reinterpret_cast<uintptr_t>(bv.ptr) & 15) == 0 && (reinterpret_cast<uintptr_t>(ov.ptr) & 15) == 0;
        const int64_t gx = ceil_div(bv.rows, 256 * (vec ? VN : 1));
        int64_t gy = ceil_div((int64_t)num_sms() * 8, gx);
        if (gy > bv.cols) gy = bv.cols;
        if (gy > 65535) gy = 65535;
        const int64_t cpb = ceil_div(bv.cols, gy);
        gy = ceil_div(bv.cols, cpb);
        dim3 grid((unsigned)gx, (unsigned)gy);
        const T *bp = (const T *)bv.ptr;
        T *op = (T *)ov.ptr;
        if (side && vec) diag_scale_cols<T, true, true><<<grid, 256, 0, s>>>(d, bp, ldb, op, ldo, bv.rows, bv.cols, cpb);
        else if (side) diag_scale_cols<T, true, false><<<grid, 256, 0, s>>>(d, bp, ldb, op, ldo, bv.rows, bv.cols, cpb);
        else if (vec) diag_scale_cols<T, false, true><<<grid, 256, 0, s>>>(d, bp, ldb, op, ldo, bv.rows, bv.cols, cpb);
        else diag_scale_cols<T, false, false><<<grid, 256, 0, s>>>(d, bp, ldb, op, ldo, bv.rows, bv.cols, cpb);
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
// 64x64 (i,k) tiles (persistent grid, one full wave).  Each thread holds
// 16 elements of the A tile (rows tx, tx+32; columns ty+8r) in registers
// and stages 16 elements of the B tile transposed through shared memory
// (row stride 65: conflict-free on both the store and the load); the next
// tile's 32 loads are issued before the current tile is consumed.
constexpr int kTr = 64;
template <class T, bool CONTIG>
__global__ void __launch_bounds__(kRedThreads, 2) trace_tiles(View<const T> A, View<const T> B, int64_t ntr,
                                                              int64_t ntiles, T *__restrict__ partials) {
    pdl_wait();  // inputs may be the previous kernel's output (PDL)
    pdl_trigger();
    __shared__ T sB[kTr][kTr + 1];
    __shared__ T red[kRedThreads / 32];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t p = A.rows, q = A.cols;
    T acc0 = T(0), acc1 = T(0);
    T ra[16], rb[16];
    auto load = [&](int64_t t) {
        const int64_t i0 = (t % ntr) * kTr, k0 = (t / ntr) * kTr;
        const bool full = i0 + kTr <= p && k0 + kTr <= q;
        if (CONTIG && full) {
            const T *pa = A.p + (i0 + tx) + (k0 + ty) * A.cs;
            const T *pb = B.p + (k0 + tx) + (i0 + ty) * B.cs;
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    ra[e * 8 + r] = __ldg(pa + 32 * e + 8 * r * A.cs);
                    rb[e * 8 + r] = __ldg(pb + 32 * e + 8 * r * B.cs);
                }
        } else {
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int64_t ia = i0 + tx + 32 * e, ka = k0 + ty + 8 * r;
                    ra[e * 8 + r] = (ia < p && ka < q) ? A(ia, ka) : T(0);
                    const int64_t kb = k0 + tx + 32 * e, ib = i0 + ty + 8 * r;
                    rb[e * 8 + r] = (kb < q && ib < p) ? B(kb, ib) : T(0);
                }
        }
    };
    int64_t t = blockIdx.x;
    if (t < ntiles) load(t);
    for (; t < ntiles; t += gridDim.x) {
        T ca[16];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                ca[e * 8 + r] = ra[e * 8 + r];
                sB[ty + 8 * r][tx + 32 * e] = rb[e * 8 + r];  // sB[i_local][k_local] = B[k0+k_local, i0+i_local]
            }
        __syncthreads();
        if (t + gridDim.x < ntiles) load(t + gridDim.x);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            acc0 = fma(ca[r], sB[tx][ty + 8 * r], acc0);
            acc1 = fma(ca[8 + r], sB[tx + 32][ty + 8 * r], acc1);
        }
        __syncthreads();
    }
    T acc = radd(acc0, acc1);
    acc = block_sum<T, kRedThreads>(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

// Register-blocked variant for column-major A, B with 4-aligned leading
// dimensions: each thread loads a 4x4 block of A (A[I..I+3, K..K+3], four
// 4-element column vectors) and the matching block of B (B[K..K+3, I..I+3])
// and pairs them in registers -- no shared-memory transpose.  Lane (a, b) =
// (lane % 4, lane / 4) takes I = 4a, K = 4b inside its warp's 16 x 32
// sub-tile, so every vector load instruction of a warp touches whole 128 B
// lines (A: 8 columns x 128 B, B: 4 columns x 256 B).  Per 16 B of input
// pairs: half a vector load and one FMA (the SMEM version issued ~4
// instructions per pair and was issue-bound below the HBM rate).
template <class T> struct Quad {
    T v[4];
};
__device__ __forceinline__ Quad<double> ld_quad(const double *p) {
    const Vec32<double> x = ld_stream32(p);
    return Quad<double>{{x.v[0], x.v[1], x.v[2], x.v[3]}};
}
__device__ __forceinline__ Quad<float> ld_quad(const float *p) {
    const float4 x = ld_stream(reinterpret_cast<const float4 *>(p));
    return Quad<float>{{x.x, x.y, x.z, x.w}};
}

template <class T, int MINB>
__global__ void __launch_bounds__(kRedThreads, MINB) trace_quads(View<const T> A, View<const T> B, int64_t ntr,
                                                             int64_t ntiles, T *__restrict__ partials,
                                                             unsigned *__restrict__ ticket, T *__restrict__ result) {
    __shared__ T red[kRedThreads / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int di = 16 * (w & 3) + 4 * (lane & 3);  // I offset in the 64 x 64 tile
    const int dk = 32 * (w >> 2) + 4 * (lane >> 2);  // K offset
    const int64_t p = A.rows, q = A.cols;
    T acc[4] = {T(0), T(0), T(0), T(0)};
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t i0 = (t % ntr) * kTr + di, k0 = (t / ntr) * kTr + dk;
        if (i0 + 4 <= p && k0 + 4 <= q) {
            Quad<T> a[4], b[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                a[c] = ld_quad(A.p + i0 + (k0 + c) * A.cs);  // A[i0.., k0+c]
                b[c] = ld_quad(B.p + k0 + (i0 + c) * B.cs);  // B[k0.., i0+c]
            }
#pragma unroll
            for (int l = 0; l < 4; ++l)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[l] = fma(a[c].v[l], b[l].v[c], acc[l]);  // A[i0+l,k0+c]*B[k0+c,i0+l]
        } else {
            for (int l = 0; l < 4; ++l)
                for (int c = 0; c < 4; ++c)
                    if (i0 + l < p && k0 + c < q) acc[l] = fma(A(i0 + l, k0 + c), B(k0 + c, i0 + l), acc[l]);
        }
    }
    T v = radd(radd(acc[0], acc[1]), radd(acc[2], acc[3]));
    v = block_sum<T, kRedThreads>(v, red);
    // the last CTA to finish sums the partials in index order (fixed tree)
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = v;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    T s = T(0);
    for (int64_t i = threadIdx.x; i < gridDim.x; i += kRedThreads) s = radd(s, __ldcg(partials + i));
    s = block_sum<T, kRedThreads>(s, red);
    if (threadIdx.x == 0) *result = s;
}

// Sum of `n` partials in index order, fixed tree; writes *out.
template <class T> __global__ void __launch_bounds__(1024) sum_partials(const T *__restrict__ part, int64_t n, T *out) {
    pdl_wait();  // inputs may be the previous kernel's output (PDL)
    pdl_trigger();
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
    const int64_t ntr = ceil_div(p, kTr), ntc = ceil_div(q, kTr), ntiles = ntr * ntc;
    const bool contig = av.rs == 1 && bv.rs == 1;
    const bool quads = contig && (av.cols <= 1 || av.cs % 4 == 0) && (bv.cols <= 1 || bv.cs % 4 == 0) &&
                       (reinterpret_cast<uintptr_t>(av.ptr) & (4 * sizeof(T) - 1)) == 0 &&
                       (reinterpret_cast<uintptr_t>(bv.ptr) & (4 * sizeof(T) - 1)) == 0;
    // Large operands (>= 512 MB read): the register-quad kernel with an
    // 8x oversubscribed grid (6.5-6.9 TB/s at 8192^2-16384^2 f64); below that
    // the shared-memory kernel's resident wave is faster (6.25 vs 5.9 TB/s at
    // 4096^2), measured with tools/bw_probe.py.
    if (quads && ntiles > 0 && 2.0 * p * q * sizeof(T) >= 512.0 * (1 << 20)) {
        static PerDevice<int> res_cache;
        int res = 0;
        res_cache.get(res, [](int &r) {
            r = resident_grid(trace_quads<T, 2>, kRedThreads);
            return 0;
        });
        int64_t blocks = (int64_t)res * 8;
        if (blocks > ntiles) blocks = ntiles;
        Scratch part;
        if (int rc = part.alloc(sizeof(T) * blocks + 16, s)) return rc;
        unsigned *ticket = reinterpret_cast<unsigned *>(part.as<char>() + sizeof(T) * blocks);
        LM_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), s));
        trace_quads<T, 2><<<(unsigned)blocks, kRedThreads, 0, s>>>(A, B, ntr, ntiles, part.as<T>(), ticket, (T *)d_result);
        LM_LAUNCHED(1);
        return 0;
    }
    auto kern = contig ? trace_tiles<T, true> : trace_tiles<T, false>;
    static PerDevice<int> grid_cache[2];
    int g = 0;
    grid_cache[contig ? 1 : 0].get(g, [&](int &v) {
        v = resident_grid(kern, kRedThreads);
        return 0;
    });
    int64_t blocks = g;
    if (blocks > ntiles) blocks = ntiles;
    if (blocks < 1) blocks = 1;
    Scratch part;
    if (int rc = part.alloc(sizeof(T) * blocks, s)) return rc;
    if (ntiles > 0) {
        LM_CUDA(launch_pdl(kern, dim3((unsigned)blocks), dim3(kRedThreads), 0, s, A, B, ntr, ntiles, part.as<T>()));
        LM_LAUNCHED(1);
    } else {
        LM_CUDA(cudaMemsetAsync(part.p, 0, sizeof(T), s));
    }
    LM_CUDA(launch_pdl(sum_partials<T>, dim3(1), dim3(1024), 0, s, (const T *)part.as<T>(), blocks, (T *)d_result));
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
