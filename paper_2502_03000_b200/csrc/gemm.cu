// gemm.cu -- products: GEMV (split-K), FP64 tensor-core GEMM (DMMA),
// SYRK (upper tiles + bitwise mirror).
//
//  lm_gemm <- _loops.py:87-98  (_gemm; planner emits it for every pair
//             product, rewrite.py:381-385; n x 1 / 1 x n outputs go to GEMV)
//  lm_gemv <- _loops.py:101-121 (_gemv, _gemv_t)
//  lm_syrk <- _loops.py:124-141 (_syrk)
//
// FP64 on sm_100a: tcgen05.mma has no f64 kind, so FP64 contractions use
// the legacy tensor path mma.sync.m8n8k4.f64 (SASS DMMA).  Tiles are
// staged global->shared with cp.async (16 B when the leading dimension
// allows), double buffered; the shared layout follows whichever
// dimension is contiguous in HBM (M or K for A, K or N for B), so the
// transposed views the planner hands over (A.T*B, A.T*A) are read in
// place, never copied -- the "transpose flag" of the north star.
// Shared rows are padded to LD = 4 (mod 16) doubles: the m8n8k4
// fragment loads are then bank-conflict free.
//
// Split-K (partials + an ordered reduction pass) keeps skinny products
// (100 x 8000 x 100, n x 1 GEMV) on all 148 SMs; the reduction order is
// fixed, so results are reproducible.  FP64 FMA accumulation: results
// match the reference's sequential sums to ~1e-15 normwise (north star:
// <= 1e-12).
#include "common.cuh"

namespace lm {

// ============================================================================
// GEMV:  y = M x  with M (p x q) a strided view
// ============================================================================

constexpr int kGvThreads = 256;

// Column-contiguous M (rs == 1): threads along rows, each block owns
// kGvRows rows x one K chunk; partial[chunk][row].
template <class T, int RPT>
__global__ void __launch_bounds__(kGvThreads) gemv_colmajor(View<const T> M, Vec<const T> x, int64_t kchunk,
                                                            T *__restrict__ part) {
    const int64_t p = M.rows, q = M.cols;
    const int64_t r0 = ((int64_t)blockIdx.x * kGvThreads + threadIdx.x) * RPT;
    const int64_t k0 = (int64_t)blockIdx.y * kchunk;
    int64_t k1 = k0 + kchunk;
    if (k1 > q) k1 = q;
    T acc[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) acc[r] = T(0);
    if (r0 + RPT <= p) {
        int64_t k = k0;
        for (; k + 4 <= k1; k += 4) {
            T v[4][RPT];
            T xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const T *col = &M(r0, k + u);
                if (RPT == 2) {
                    const double2 t = __ldg(reinterpret_cast<const double2 *>(col));
                    v[u][0] = t.x;
                    v[u][RPT - 1] = t.y;
                } else {
#pragma unroll
                    for (int r = 0; r < RPT; ++r) v[u][r] = __ldg(col + r);
                }
                xv[u] = x[k + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int r = 0; r < RPT; ++r) acc[r] = fma(v[u][r], xv[u], acc[r]);
        }
        for (; k < k1; ++k) {
            const T xk = x[k];
#pragma unroll
            for (int r = 0; r < RPT; ++r) acc[r] = fma(M(r0 + r, k), xk, acc[r]);
        }
    } else {
        for (int64_t k = k0; k < k1; ++k) {
            const T xk = x[k];
#pragma unroll
            for (int r = 0; r < RPT; ++r)
                if (r0 + r < p) acc[r] = fma(M(r0 + r, k), xk, acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r)
        if (r0 + r < p) part[blockIdx.y * p + r0 + r] = acc[r];
}

// Column-major M with 32 B-aligned columns: CTA (rowblock b, chunk c) owns
// rows [b*RB, b*RB+RB) x columns [c*KC, c*KC+KC).  A thread holds RPT = 32 B
// of one column (4 doubles / 8 floats); warp w of the CTA takes columns
// w, w+8, ... of the chunk, so every warp load is one contiguous 1 KB
// segment and 8 column loads are in flight per thread.  Warp partials are
// summed in warp order through shared memory into part[chunk][row];
// gemv_finish sums the chunks in order.  (A last-CTA-finishes ticket
// variant was no faster: its __threadfence per CTA cost what the second
// launch does.)
constexpr int kGv32Warps = 8;
constexpr int kGv32KC = 64;
template <class T>
__global__ void __launch_bounds__(kGv32Warps * 32, 3) gemv_cm32(const T *__restrict__ M, int64_t ld, int64_t p,
                                                              int64_t q, Vec<const T> x, T *__restrict__ part) {
    constexpr int RPT = Vec32<T>::N;
    constexpr int RB = 32 * RPT;  // rows per CTA
    constexpr int U = kGv32KC / kGv32Warps;  // columns per warp
    __shared__ T red[kGv32Warps][RB];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t rb = blockIdx.x, c = blockIdx.y;
    const int64_t r0 = rb * RB + lane * RPT;
    const int64_t k0 = c * kGv32KC + w;
    T acc[RPT];
#pragma unroll
    for (int l = 0; l < RPT; ++l) acc[l] = T(0);
    if (r0 < p) {  // p % RPT == 0: a thread's rows are all valid or all not
        Vec32<T> v[U];
        T xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = k0 + u * kGv32Warps;
            if (k < q) {
                v[u] = ld_stream32(M + r0 + k * ld);
                xv[u] = x[k];
            } else {
#pragma unroll
                for (int l = 0; l < RPT; ++l) v[u].v[l] = T(0);
                xv[u] = T(0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int l = 0; l < RPT; ++l) acc[l] = fma(v[u].v[l], xv[u], acc[l]);
    }
#pragma unroll
    for (int l = 0; l < RPT; ++l) red[w][lane * RPT + l] = acc[l];
    __syncthreads();
    for (int r = threadIdx.x; r < RB; r += blockDim.x) {
        T sum = red[0][r];
#pragma unroll
        for (int q2 = 1; q2 < kGv32Warps; ++q2) sum += red[q2][r];
        if (rb * RB + r < p) part[c * p + rb * RB + r] = sum;
    }
}

// Row-contiguous (or general) M: one warp per row, lanes along K.
template <class T>
__global__ void __launch_bounds__(kGvThreads) gemv_rowmajor(View<const T> M, Vec<const T> x, int64_t kchunk,
                                                            T *__restrict__ part) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (kGvThreads / 32) + (threadIdx.x >> 5);
    const int64_t p = M.rows, q = M.cols;
    if (row >= p) return;
    const int64_t k0 = (int64_t)blockIdx.y * kchunk;
    int64_t k1 = k0 + kchunk;
    if (k1 > q) k1 = q;
    T acc = T(0);
    for (int64_t k = k0 + lane; k < k1; k += 32) acc = fma(M(row, k), x[k], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) part[blockIdx.y * p + row] = acc;
}

// y[i] = sum over chunks c (ascending) of part[c][i]: 32 rows per CTA, warp w
// sums chunks w, w+8, ... (independent loads in flight), the 8 warp sums
// are added in warp order -- a fixed tree, reproducible run to run.
template <class T>
__global__ void __launch_bounds__(256) gemv_finish(const T *__restrict__ part, int64_t p, int64_t nchunks, Vec<T> y) {
    __shared__ T red[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    T acc = T(0);
    if (i < p) {
#pragma unroll 4
        for (int64_t c = w; c < nchunks; c += 8) acc += part[c * p + i];
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0 && i < p) {
        T s = red[0][lane];
#pragma unroll
        for (int q = 1; q < 8; ++q) s += red[q][lane];
        y[i] = s;
    }
}

template <class T> int gemv_impl(const lm_view &mv, const lm_vec &xv, const lm_vec &yv, cudaStream_t s) {
    const int64_t p = mv.rows, q = mv.cols;
    if (p == 0) return 0;
    View<const T> M{(const T *)mv.ptr, mv.rows, mv.cols, mv.rs, mv.cs};
    Vec<const T> x{(const T *)xv.ptr, xv.n, xv.stride};
    const int nsm = num_sms();
    constexpr int RPT32 = Vec32<T>::N;
    if (q > 0 && mv.rs == 1 && p % RPT32 == 0 && (mv.cols <= 1 || mv.cs % RPT32 == 0) && aligned32(mv.ptr) &&
        ceil_div(q, kGv32KC) <= 65535) {
        constexpr int RB = 32 * RPT32;
        const int64_t rowblocks = ceil_div(p, RB), chunks = ceil_div(q, kGv32KC);
        const int64_t ld = mv.cols > 1 ? mv.cs : p;
        Scratch part;
        if (int rc = part.alloc(sizeof(T) * p * chunks, s)) return rc;
        gemv_cm32<T><<<dim3((unsigned)rowblocks, (unsigned)chunks), kGv32Warps * 32, 0, s>>>((const T *)mv.ptr, ld, p,
                                                                                            q, x, part.as<T>());
        gemv_finish<T><<<(unsigned)ceil_div(p, 32), 256, 0, s>>>(part.as<T>(), p, chunks, to_vec<T>(yv));
        LM_LAUNCHED(2);
        return 0;
    }
    if (mv.rs == 1 || mv.cs != 1) {
        const bool vec2 = sizeof(T) == 8 && mv.rs == 1 && (mv.cs % 2 == 0) && ((uintptr_t)mv.ptr % 16 == 0);
        const int rpt = vec2 ? 2 : 1;
        const int64_t rowblocks = ceil_div(p, (int64_t)kGvThreads * rpt);
        // K chunks so that rowblocks * chunks ~ 4 waves of 148 SMs
        int64_t chunks = ceil_div((int64_t)nsm * 4, rowblocks);
        int64_t kchunk = ceil_div(q > 0 ? q : 1, chunks);
        kchunk = ((kchunk + 15) / 16) * 16;
        if (kchunk < 64) kchunk = 64;
        chunks = q > 0 ? ceil_div(q, kchunk) : 1;
        Scratch part;
        if (int rc = part.alloc(sizeof(T) * p * chunks, s)) return rc;
        if (q == 0) {
            LM_CUDA(cudaMemsetAsync(part.p, 0, sizeof(T) * p, s));
        } else if (vec2) {
            gemv_colmajor<T, 2><<<dim3((unsigned)rowblocks, (unsigned)chunks), kGvThreads, 0, s>>>(M, x, kchunk,
                                                                                                   part.as<T>());
            LM_LAUNCHED(1);
        } else {
            gemv_colmajor<T, 1><<<dim3((unsigned)rowblocks, (unsigned)chunks), kGvThreads, 0, s>>>(M, x, kchunk,
                                                                                                   part.as<T>());
            LM_LAUNCHED(1);
        }
        gemv_finish<T><<<(unsigned)ceil_div(p, 32), 256, 0, s>>>(part.as<T>(), p, chunks, to_vec<T>(yv));
        LM_LAUNCHED(1);
    } else {
        const int64_t rowblocks = ceil_div(p, kGvThreads / 32);
        int64_t chunks = ceil_div((int64_t)nsm * 4, rowblocks);
        int64_t kchunk = ceil_div(q > 0 ? q : 1, chunks);
        if (kchunk < 256) kchunk = 256;
        chunks = q > 0 ? ceil_div(q, kchunk) : 1;
        Scratch part;
        if (int rc = part.alloc(sizeof(T) * p * chunks, s)) return rc;
        if (q == 0) {
            LM_CUDA(cudaMemsetAsync(part.p, 0, sizeof(T) * p, s));
        } else {
            gemv_rowmajor<T><<<dim3((unsigned)rowblocks, (unsigned)chunks), kGvThreads, 0, s>>>(M, x, kchunk,
                                                                                               part.as<T>());
            LM_LAUNCHED(1);
        }
        gemv_finish<T><<<(unsigned)ceil_div(p, 32), 256, 0, s>>>(part.as<T>(), p, chunks, to_vec<T>(yv));
        LM_LAUNCHED(1);
    }
    return 0;
}

// ============================================================================
// FP64 GEMM on DMMA (mma.sync.m8n8k4.f64)
// ============================================================================

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int kGmThreads = 128;  // 4 warps, 2 x 2, warp tile 32 x 32
constexpr int LDM = BM + 4;      // smem row length (doubles) when M/N-contiguous
constexpr int LDK = BK + 4;      // when K-contiguous

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    const int n = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Operand tile loader.  CONTIG_OUTER: the tile's non-K dimension (M for
// A, N for B) is contiguous in HBM -> smem layout [BK][LDM]; otherwise K
// is contiguous -> smem layout [BM][LDK].  (outer index o, k index kk)
// element is X(o, kk) = ptr[o*so + kk*sk].
template <bool CONTIG_OUTER, bool VEC16>
__device__ __forceinline__ void load_tile(double *sm, const double *ptr, int64_t so, int64_t sk, int64_t o0, int64_t k0,
                                          int64_t no, int64_t nk) {
    constexpr int ELEMS = BM * BK;  // 1024
    if (CONTIG_OUTER) {
        // pairs along o
        constexpr int W = VEC16 ? 2 : 1;
        for (int e = threadIdx.x * W; e < ELEMS; e += kGmThreads * W) {
            const int kk = e / BM, oo = e % BM;
            const int64_t go = o0 + oo, gk = k0 + kk;
            double *dst = sm + kk * LDM + oo;
            const double *src = ptr + go * so + gk * sk;
            if (VEC16) {
                int bytes = 0;
                if (gk < nk) bytes = go + 1 < no ? 16 : (go < no ? 8 : 0);
                cp_async16(dst, bytes ? src : ptr, bytes);
            } else {
                const bool ok = gk < nk && go < no;
                cp_async8(dst, ok ? src : ptr, ok);
            }
        }
    } else {
        constexpr int W = VEC16 ? 2 : 1;
        for (int e = threadIdx.x * W; e < ELEMS; e += kGmThreads * W) {
            const int oo = e / BK, kk = e % BK;
            const int64_t go = o0 + oo, gk = k0 + kk;
            double *dst = sm + oo * LDK + kk;
            const double *src = ptr + go * so + gk * sk;
            if (VEC16) {
                int bytes = 0;
                if (go < no) bytes = gk + 1 < nk ? 16 : (gk < nk ? 8 : 0);
                cp_async16(dst, bytes ? src : ptr, bytes);
            } else {
                const bool ok = gk < nk && go < no;
                cp_async8(dst, ok ? src : ptr, ok);
            }
        }
    }
}

template <bool CONTIG_OUTER> __device__ __forceinline__ double frag(const double *sm, int o, int k) {
    return CONTIG_OUTER ? sm[k * LDM + o] : sm[o * LDK + k];
}

struct GemmArgs {
    const double *a;
    int64_t a_sm, a_sk;  // A(m,k) = a[m*a_sm + k*a_sk]
    const double *b;
    int64_t b_sk, b_sn;  // B(k,n) = b[k*b_sk + n*b_sn]
    double *c;
    int64_t c_sm, c_sn;
    int64_t M, N, K;
    int64_t kchunk;  // K range per blockIdx.z
    double *part;    // split-K partials [z][M*N] (F-order), or null
    int syrk;        // 1: only upper tiles (tile index -> (tm <= tn)), mirrored store
    int64_t tiles_n;
};

constexpr int kStageDoubles = (BK * LDM > BM * LDK ? BK * LDM : BM * LDK);

template <bool A_CM, bool B_CN, bool VA, bool VB>
__global__ void __launch_bounds__(kGmThreads) dgemm_dmma(GemmArgs g) {
    __shared__ __align__(16) double sA[2][kStageDoubles];
    __shared__ __align__(16) double sB[2][kStageDoubles];
    int64_t tm, tn;
    if (g.syrk) {
        // triangular tile index: idx -> (tm <= tn)
        const int64_t idx = blockIdx.x;
        int64_t t = (int64_t)((sqrt(8.0 * (double)idx + 1.0) - 1.0) * 0.5);
        while ((t + 1) * (t + 2) / 2 <= idx) ++t;
        while (t * (t + 1) / 2 > idx) --t;
        tn = t;
        tm = idx - t * (t + 1) / 2;
    } else {
        tm = blockIdx.x % ((g.M + BM - 1) / BM);
        tn = blockIdx.x / ((g.M + BM - 1) / BM);
    }
    const int64_t m0 = tm * BM, n0 = tn * BN;
    const int64_t kb = (int64_t)blockIdx.z * g.kchunk;
    int64_t ke = kb + g.kchunk;
    if (ke > g.K) ke = g.K;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    const int fr = lane >> 2, fc = lane & 3;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // A as (outer = m, k); B as (outer = n, k)
    auto issue = [&](int stage, int64_t k0) {
        load_tile<A_CM, VA>(sA[stage], g.a, g.a_sm, g.a_sk, m0, k0, g.M, ke);
        load_tile<B_CN, VB>(sB[stage], g.b, g.b_sn, g.b_sk, n0, k0, g.N, ke);
        cp_commit();
    };
    const int64_t nk = ke > kb ? (ke - kb + BK - 1) / BK : 0;
    if (nk > 0) issue(0, kb);
    for (int64_t it = 0; it < nk; ++it) {
        const int st = it & 1;
        if (it + 1 < nk) {
            issue(st ^ 1, kb + (it + 1) * BK);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const double *a_s = sA[st];
        const double *b_s = sB[st];
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = frag<A_CM>(a_s, wm + i * 8 + fr, kk + fc);
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = frag<B_CN>(b_s, wn + j * 8 + fr, kk + fc);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
        }
        __syncthreads();
    }
    // epilogue: C fragment (row fr, cols 2*fc, 2*fc+1)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t m = m0 + wm + i * 8 + fr, n = n0 + wn + j * 8 + 2 * fc + h;
                if (m >= g.M || n >= g.N) continue;
                const double v = acc[i][j][h];
                if (g.part) {
                    g.part[(int64_t)blockIdx.z * g.M * g.N + m + n * g.M] = v;
                } else if (g.syrk) {
                    if (tm == tn && m > n) continue;
                    g.c[m * g.c_sm + n * g.c_sn] = v;
                    g.c[n * g.c_sm + m * g.c_sn] = v;
                } else {
                    g.c[m * g.c_sm + n * g.c_sn] = v;
                }
            }
}

// out = sum over z of partials (fixed order); syrk: upper only + mirror.
__global__ void __launch_bounds__(256) splitk_finish(const double *__restrict__ part, int64_t M, int64_t N, int64_t nz,
                                                     double *c, int64_t c_sm, int64_t c_sn, int syrk) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= M * N) return;
    const int64_t n = e / M, m = e - n * M;
    if (syrk && m > n) return;
    double acc = part[e];
    for (int64_t z = 1; z < nz; ++z) acc += part[z * M * N + e];
    c[m * c_sm + n * c_sn] = acc;
    if (syrk) c[n * c_sm + m * c_sn] = acc;
}

template <bool A_CM, bool B_CN>
int launch_dgemm_layout(GemmArgs &g, bool va, bool vb, dim3 grid, cudaStream_t s) {
    if (va && vb)
        dgemm_dmma<A_CM, B_CN, true, true><<<grid, kGmThreads, 0, s>>>(g);
    else if (va)
        dgemm_dmma<A_CM, B_CN, true, false><<<grid, kGmThreads, 0, s>>>(g);
    else if (vb)
        dgemm_dmma<A_CM, B_CN, false, true><<<grid, kGmThreads, 0, s>>>(g);
    else
        dgemm_dmma<A_CM, B_CN, false, false><<<grid, kGmThreads, 0, s>>>(g);
    LM_LAUNCHED(1);
    return 0;
}

// A(m,k) strides (a_sm, a_sk), B(k,n) strides (b_sk, b_sn).
int dgemm(const double *a, int64_t a_sm, int64_t a_sk, const double *b, int64_t b_sk, int64_t b_sn, double *c,
          int64_t c_sm, int64_t c_sn, int64_t M, int64_t N, int64_t K, bool syrk, cudaStream_t s) {
    if (M == 0 || N == 0) return 0;
    GemmArgs g{};
    g.a = a;
    g.a_sm = a_sm;
    g.a_sk = a_sk;
    g.b = b;
    g.b_sk = b_sk;
    g.b_sn = b_sn;
    g.c = c;
    g.c_sm = c_sm;
    g.c_sn = c_sn;
    g.M = M;
    g.N = N;
    g.K = K;
    g.syrk = syrk ? 1 : 0;
    const int64_t tM = ceil_div(M, BM), tN = ceil_div(N, BN);
    const int64_t tiles = syrk ? tM * (tM + 1) / 2 : tM * tN;
    g.tiles_n = tN;
    // choose split-K so the grid covers >= ~2 waves of the machine
    const int64_t nsm = num_sms();
    int64_t splits = 1;
    if (K > 0) {
        const int64_t kt = ceil_div(K, BK);
        while (tiles * splits < nsm * 2 && splits * 2 <= kt / 8) splits *= 2;
    }
    g.kchunk = K > 0 ? ceil_div(ceil_div(K, splits), BK) * BK : BK;
    if (K > 0) splits = ceil_div(K, g.kchunk);
    Scratch part;
    if (K == 0) {
        // empty inner dimension: out = 0
        for (int64_t n = 0; n < N; ++n) {
            if (c_sm == 1)
                LM_CUDA(cudaMemsetAsync(c + n * c_sn, 0, sizeof(double) * M, s));
            else
                return -1;
        }
        return 0;
    }
    if (splits > 1) {
        if (int rc = part.alloc(sizeof(double) * M * N * splits, s)) return rc;
        g.part = part.as<double>();
    }
    const bool a_cm = (a_sm == 1);          // A contiguous along M
    const bool b_cn = (b_sn == 1 && b_sk != 1);  // B contiguous along N
    auto aligned16 = [](const void *p) { return ((uintptr_t)p & 15) == 0; };
    // 16-byte cp.async needs the contiguous dim unit-stride and the other
    // stride even (every pair starts 16-byte aligned).
    const bool va = aligned16(a) && (a_cm ? (a_sk % 2 == 0) : (a_sk == 1 && a_sm % 2 == 0));
    const bool vb = aligned16(b) && (b_cn ? (b_sk % 2 == 0) : (b_sk == 1 && b_sn % 2 == 0));
    dim3 grid((unsigned)tiles, 1, (unsigned)splits);
    int rc;
    if (a_cm && b_cn)
        rc = launch_dgemm_layout<true, true>(g, va, vb, grid, s);
    else if (a_cm)
        rc = launch_dgemm_layout<true, false>(g, va, vb && b_sk == 1, grid, s);
    else if (b_cn)
        rc = launch_dgemm_layout<false, true>(g, va && a_sk == 1, vb, grid, s);
    else
        rc = launch_dgemm_layout<false, false>(g, va && a_sk == 1, vb && b_sk == 1, grid, s);
    if (rc) return rc;
    if (splits > 1) {
        splitk_finish<<<(unsigned)ceil_div(M * N, 256), 256, 0, s>>>(g.part, M, N, splits, c, c_sm, c_sn, g.syrk);
        LM_LAUNCHED(1);
    }
    return 0;
}

// FP32 (batched-config extension) generic SIMT GEMM, FMA accumulate.
__global__ void __launch_bounds__(256) sgemm_simple(View<const float> A, View<const float> B, View<float> C) {
    __shared__ float sA[32][33], sB[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const int64_t m0 = (int64_t)blockIdx.x * 32, n0 = (int64_t)blockIdx.y * 32;
    float acc[4] = {0, 0, 0, 0};
    for (int64_t k0 = 0; k0 < A.cols; k0 += 32) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t m = m0 + tx, k = k0 + ty + 8 * r;
            sA[ty + 8 * r][tx] = (m < A.rows && k < A.cols) ? A(m, k) : 0.f;
            const int64_t kb = k0 + tx, n = n0 + ty + 8 * r;
            sB[ty + 8 * r][tx] = (kb < B.rows && n < B.cols) ? B(kb, n) : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < 32; ++kk)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[r] = fmaf(sA[kk][tx], sB[ty + 8 * r][kk], acc[r]);
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t m = m0 + tx, n = n0 + ty + 8 * r;
        if (m < C.rows && n < C.cols) C(m, n) = acc[r];
    }
}

}  // namespace lm

using namespace lm;

extern "C" int lm_gemv(int dtype, lm_view a, lm_vec x, lm_vec out, int trans, void *stream) {
    clear_error();
    lm_view m = a;
    if (trans) {
        m.rows = a.cols;
        m.cols = a.rows;
        m.rs = a.cs;
        m.cs = a.rs;
    }
    LM_REQUIRE(x.n == m.cols, "gemv x length %lld != %lld", (long long)x.n, (long long)m.cols);
    LM_REQUIRE(out.n == m.rows, "gemv out length %lld != %lld", (long long)out.n, (long long)m.rows);
    if (dtype == LM_F64) return gemv_impl<double>(m, x, out, as_stream(stream));
    if (dtype == LM_F32) return gemv_impl<float>(m, x, out, as_stream(stream));
    set_error("bad dtype");
    return -1;
}

extern "C" int lm_gemm(int dtype, lm_view a, lm_view b, lm_view out, void *stream) {
    clear_error();
    LM_REQUIRE(a.cols == b.rows, "gemm inner dimensions %lld != %lld", (long long)a.cols, (long long)b.rows);
    LM_REQUIRE(out.rows == a.rows && out.cols == b.cols, "gemm out shape mismatch");
    cudaStream_t s = as_stream(stream);
    if (out.rows == 0 || out.cols == 0) return 0;
    if (out.cols == 1 && a.rows > 1) {
        // n x 1 result: GEMV over a with x = b[:,0]
        lm_vec x{b.ptr, b.rows, b.rs};
        lm_vec y{out.ptr, out.rows, out.rs};
        return lm_gemv(dtype, a, x, y, 0, stream);
    }
    if (out.rows == 1 && b.cols > 1) {
        // 1 x n result: out[0,:] = b.T @ a[0,:]
        lm_vec x{a.ptr, a.cols, a.cs};
        lm_vec y{out.ptr, out.cols, out.cs};
        return lm_gemv(dtype, b, x, y, 1, stream);
    }
    if (dtype == LM_F64)
        return dgemm((const double *)a.ptr, a.rs, a.cs, (const double *)b.ptr, b.rs, b.cs, (double *)out.ptr, out.rs,
                     out.cs, a.rows, b.cols, a.cols, false, s);
    if (dtype == LM_F32) {
        View<const float> A{(const float *)a.ptr, a.rows, a.cols, a.rs, a.cs};
        View<const float> B{(const float *)b.ptr, b.rows, b.cols, b.rs, b.cs};
        sgemm_simple<<<dim3((unsigned)ceil_div(a.rows, 32), (unsigned)ceil_div(b.cols, 32)), 256, 0, s>>>(
            A, B, to_view<float>(out));
        LM_LAUNCHED(1);
        return 0;
    }
    set_error("bad dtype");
    return -1;
}

extern "C" int lm_syrk(int dtype, lm_view a, lm_view out, void *stream) {
    clear_error();
    LM_REQUIRE(out.rows == a.rows && out.cols == a.rows, "syrk out shape mismatch");
    LM_REQUIRE(dtype == LM_F64, "syrk: f64 only");
    // out = a @ a.T : A(m,k) = a(m,k), B(k,n) = a(n,k)
    return dgemm((const double *)a.ptr, a.rs, a.cs, (const double *)a.ptr, a.cs, a.rs, (double *)out.ptr, out.rs,
                 out.cs, a.rows, a.rows, a.cols, true, as_stream(stream));
}
