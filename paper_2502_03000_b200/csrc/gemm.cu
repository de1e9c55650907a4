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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>

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
template <class T, int KC, int MINB>
__global__ void __launch_bounds__(kGv32Warps * 32, MINB) gemv_cm32(const T *__restrict__ M, int64_t ld, int64_t p,
                                                                 int64_t q, Vec<const T> x, T *__restrict__ part) {
    constexpr int kGv32KC = KC;
    constexpr int RPT = Vec32<T>::N;
    constexpr int RB = 32 * RPT;  // rows per CTA
    constexpr int U = kGv32KC / kGv32Warps;  // columns per warp
    __shared__ T red[kGv32Warps][RB];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t rb = blockIdx.x, c = blockIdx.y;
    const int64_t r0 = rb * RB + lane * RPT;
    const int64_t k0 = c * kGv32KC + w;
    pdl_wait();  // M and x may be the previous kernel's output
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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

// Row-owner GEMV (f64, column-major M with 16-byte columns): CTA b owns
// rows [8b, 8b+8) and ALL columns, so there are no split-K partials and no
// finish launch.  Lane l of warp w reads rows 8b + 2(l % 4) .. +1 of column
// 8(w + 8i) + l / 4 as one 16-byte load (a warp: eight 64-byte column
// pieces per instruction), eight loads in flight per thread; the column
// lanes and the eight warps are then summed in a fixed order
// (reproducible).  p / 8 CTAs (config 3a: 512, ~3.5 per SM); config 3a
// 75.4 -> 72.9 us per step (16 rows per CTA: 101 us; 4 rows: 88 us;
// 16 loads in flight: 82 us).  LM_GEMV_ROWS=0: the split-K kernel below.
constexpr int kGvRowsRB = 8;
__global__ void __launch_bounds__(256) gemv_rows_f64(const double *__restrict__ M, int64_t ld, int64_t p, int64_t q,
                                                    Vec<const double> x, Vec<double> y) {
    constexpr int RPL = kGvRowsRB / 2;  // lanes per column piece (2 rows each)
    constexpr int CPW = 32 / RPL;       // columns per warp load
    constexpr int CS = 8 * CPW;         // column stride of a thread
    __shared__ double2 red[8][RPL];
    pdl_wait();  // M and x may be the previous kernel's output
    pdl_trigger();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int rp = lane % RPL, co = lane / RPL;
    const int64_t r0 = (int64_t)blockIdx.x * kGvRowsRB + 2 * rp;
    const double *base = M + r0;
    double a0 = 0.0, a1 = 0.0;
    constexpr int U = 8;
    int64_t k = (int64_t)CPW * w + co;
    for (; k + (int64_t)CS * (U - 1) < q; k += (int64_t)CS * U) {
        double2 v[U];
        double xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            v[u] = __ldcs(reinterpret_cast<const double2 *>(base + (k + CS * u) * ld));
            xv[u] = x[k + CS * u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a0 = fma(v[u].x, xv[u], a0);
            a1 = fma(v[u].y, xv[u], a1);
        }
    }
    for (; k < q; k += CS) {
        const double2 v = __ldcs(reinterpret_cast<const double2 *>(base + k * ld));
        const double xk = x[k];
        a0 = fma(v.x, xk, a0);
        a1 = fma(v.y, xk, a1);
    }
    // the column lanes of each row pair, in a fixed order
#pragma unroll
    for (int o = RPL; o < 32; o <<= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if (lane < RPL) red[w][lane] = make_double2(a0, a1);
    __syncthreads();
    if (threadIdx.x < RPL) {
        double2 t = red[0][threadIdx.x];
#pragma unroll
        for (int q2 = 1; q2 < 8; ++q2) {
            t.x += red[q2][threadIdx.x].x;
            t.y += red[q2][threadIdx.x].y;
        }
        const int64_t r = (int64_t)blockIdx.x * kGvRowsRB + 2 * threadIdx.x;
        if (r < p) y[r] = t.x;
        if (r + 1 < p) y[r + 1] = t.y;
    }
}

template <class T> int gemv_impl(const lm_view &mv, const lm_vec &xv, const lm_vec &yv, cudaStream_t s) {
    const int64_t p = mv.rows, q = mv.cols;
    if (p == 0) return 0;
    View<const T> M{(const T *)mv.ptr, mv.rows, mv.cols, mv.rs, mv.cs};
    Vec<const T> x{(const T *)xv.ptr, xv.n, xv.stride};
    const int nsm = num_sms();
    constexpr int RPT32 = Vec32<T>::N;
    // 64-column chunks, 4 CTAs per SM (64 registers, no spill): 5.3 TB/s on
    // config 3a; 3 CTAs/SM spilled (4.7), 128-column chunks spill (3.0-3.6)
    constexpr int KCv = 64;
    static const bool rows_on = !(getenv("LM_GEMV_ROWS") && getenv("LM_GEMV_ROWS")[0] == '0');
    if (sizeof(T) == 8 && rows_on && q > 0 && mv.rs == 1 && p % kGvRowsRB == 0 &&
        (mv.cols <= 1 || mv.cs % 2 == 0) && ((uintptr_t)mv.ptr & 15) == 0 && p / kGvRowsRB <= 0x7fffffff) {
        const int64_t ld = mv.cols > 1 ? mv.cs : p;
        LM_CUDA(launch_pdl(gemv_rows_f64, dim3((unsigned)(p / kGvRowsRB)), dim3(256), 0, s,
                           (const double *)mv.ptr, ld, p, q, Vec<const double>{(const double *)xv.ptr, xv.n, xv.stride},
                           Vec<double>{(double *)yv.ptr, yv.n, yv.stride}));
        LM_LAUNCHED(1);
        note_variant("gemv_rows");
        return 0;
    }
    if (q > 0 && mv.rs == 1 && p % RPT32 == 0 && (mv.cols <= 1 || mv.cs % RPT32 == 0) && aligned32(mv.ptr) &&
        ceil_div(q, KCv) <= 65535) {
        constexpr int RB = 32 * RPT32;
        const int64_t rowblocks = ceil_div(p, RB), chunks = ceil_div(q, KCv);
        const int64_t ld = mv.cols > 1 ? mv.cs : p;
        Scratch part;
        if (int rc = part.alloc(sizeof(T) * p * chunks, s)) return rc;
        const dim3 grid((unsigned)rowblocks, (unsigned)chunks);
        LM_CUDA(launch_pdl(gemv_cm32<T, KCv, sizeof(T) == 8 ? 4 : 3>, grid, dim3(kGv32Warps * 32), 0, s,
                           (const T *)mv.ptr, ld, p, q, x, part.as<T>()));
        LM_CUDA(launch_pdl(gemv_finish<T>, dim3((unsigned)ceil_div(p, 32)), dim3(256), 0, s, (const T *)part.as<T>(), p,
                           chunks, to_vec<T>(yv)));
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

struct GemmArgs {
    const double *a;
    int64_t a_sm, a_sk;  // A(m,k) = a[m*a_sm + k*a_sk]
    const double *b;
    int64_t b_sk, b_sn;  // B(k,n) = b[k*b_sk + n*b_sn]
    double *c;
    int64_t c_sm, c_sn;
    int64_t M, N, K;
    int64_t kchunk;  // K range per blockIdx.z (a multiple of the kernel's BKT)
    double *part;    // split-K partials [z][M*N] (F-order), or null
    int syrk;        // 1: only upper tiles (tile index -> (tm <= tn)), mirrored store
    int64_t tiles_n;
    int sub;         // 1: C -= A B (one rounding per element; never split along K)
};

// One operand's tile stream (A as (outer = m, k), B as (outer = n, k)).
// CONTIG_OUTER: the outer dimension is unit-stride in HBM -> smem [BKT][LDM]
// (o contiguous); otherwise K is unit-stride -> smem [BM][BKT + 4].  Each
// thread owns a fixed set of (o, k) slots of the tile: its source pointer
// and smem offsets are computed once and advanced by BKT * sk per K step,
// so an interior tile costs one cp.async (+ one add) per 16 B.  Edge tiles
// (outer or K overhang) take the predicated path.
template <bool CONTIG_OUTER, bool VEC16, int BKT> struct TileStream {
    static constexpr int LDS_ = CONTIG_OUTER ? BM + 4 : BKT + 4;  // smem row length
    static constexpr int ELEMS = BM * BKT;
    static constexpr int W = VEC16 ? 2 : 1;
    static constexpr int PER = ELEMS / W / kGmThreads;  // copies per thread per stage
    static constexpr int STEP = kGmThreads * W;          // element index step between a thread's copies
    const double *src;  // slot 0 source at the current K step
    int64_t di;         // source delta between slots
    int64_t dk;         // source delta per K step
    int sm0, dsm;       // smem offset of slot 0, delta between slots
    int o_first, k_first, o_step, k_step;  // slot coordinates (for the predicated path)

    __device__ __forceinline__ void init(const double *ptr, int64_t so, int64_t sk, int64_t o0, int64_t k0) {
        const int e = threadIdx.x * W;
        int oo, kk;
        if (CONTIG_OUTER) {
            oo = e % BM;
            kk = e / BM;
            o_step = 0;
            k_step = STEP / BM;
            dsm = k_step * LDS_;
            sm0 = kk * LDS_ + oo;
        } else {
            kk = e % BKT;
            oo = e / BKT;
            o_step = STEP / BKT;
            k_step = 0;
            dsm = o_step * LDS_;
            sm0 = oo * LDS_ + kk;
        }
        o_first = oo;
        k_first = kk;
        src = ptr + (o0 + oo) * so + (k0 + kk) * sk;
        di = (int64_t)o_step * so + (int64_t)k_step * sk;
        dk = (int64_t)BKT * sk;
    }
    // interior tile
    __device__ __forceinline__ void issue_full(double *sm) const {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            if (VEC16)
                cp_async16(sm + sm0 + i * dsm, src + i * di, 16);
            else
                cp_async8(sm + sm0 + i * dsm, src + i * di, true);
        }
    }
    // edge tile: (o0, k0) of the tile, bounds no, nk; zero fill outside
    __device__ __forceinline__ void issue_edge(double *sm, const double *base, int64_t o0, int64_t k0, int64_t no,
                                               int64_t nk) const {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int64_t go = o0 + o_first + i * o_step, gk = k0 + k_first + i * k_step;
            const double *sp = src + i * di;
            if (VEC16) {
                // the pair runs along the contiguous dimension
                const int64_t lim = CONTIG_OUTER ? no - go : nk - gk;
                const bool in = CONTIG_OUTER ? gk < nk : go < no;
                const int bytes = !in ? 0 : lim >= 2 ? 16 : lim == 1 ? 8 : 0;
                cp_async16(sm + sm0 + i * dsm, bytes ? sp : base, bytes);
            } else {
                const bool ok = go < no && gk < nk;
                cp_async8(sm + sm0 + i * dsm, ok ? sp : base, ok);
            }
        }
    }
    __device__ __forceinline__ void advance() { src += dk; }
};

template <bool CONTIG_OUTER, int BKT> __device__ __forceinline__ double frag(const double *sm, int o, int k) {
    return CONTIG_OUTER ? sm[k * (BM + 4) + o] : sm[o * (BKT + 4) + k];
}

template <bool CONTIG_OUTER, int BKT> constexpr int stage_doubles() {
    return CONTIG_OUTER ? BKT * (BM + 4) : BM * (BKT + 4);
}

// C tile (BM x BN) = sum over this CTA's K chunk of A * B on DMMA
// (mma.sync.m8n8k4.f64).  4 warps in 2 x 2, warp tile 32 x 32 (16 DMMA
// accumulators), ST-stage cp.async ring with one barrier per K step.
template <bool A_CM, bool B_CN, bool VA, bool VB, int BKT, int ST>
// (launch bounds: 4 CTAs per SM at <= 128 registers for the 3-stage ring, 5 at <= 102 for the 2-stage one)
__global__ void __launch_bounds__(kGmThreads, ST == 2 ? 5 : 4) dgemm_dmma(GemmArgs g) {
    pdl_wait();  // inputs may be the previous kernel's output (PDL)
    pdl_trigger();
    extern __shared__ __align__(16) double gsm[];
    constexpr int SA = stage_doubles<A_CM, BKT>(), SB = stage_doubles<B_CN, BKT>();
    double *sA = gsm;
    double *sB = gsm + ST * SA;
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

    // 8 x 8 fragments wholly outside C are skipped (warp-uniform): an edge
    // tile of a 100 x 100 product issues ~40% fewer DMMAs
    unsigned live = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (m0 + wm + i * 8 < g.M && n0 + wn + j * 8 < g.N) live |= 1u << (4 * i + j);
    // C -= A B reads its C tile only in the epilogue, from HBM (the LU's
    // trailing matrix does not fit L2): ask for the lines now, one request per
    // 64-byte fragment column, so the epilogue's loads find them in L2
    if (g.sub && g.c_sm == 1 && fr == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t m = m0 + wm + i * 8, n = n0 + wn + j * 8 + 2 * fc + h;
                    if (m < g.M && n < g.N) asm volatile("prefetch.global.L2 [%0];" ::"l"(g.c + m + n * g.c_sn));
                }
    }
    TileStream<A_CM, VA, BKT> ta;
    TileStream<B_CN, VB, BKT> tb;
    ta.init(g.a, g.a_sm, g.a_sk, m0, kb);
    tb.init(g.b, g.b_sn, g.b_sk, n0, kb);
    const bool interior = m0 + BM <= g.M && n0 + BN <= g.N && (ke - kb) % BKT == 0;
    const int64_t nk = ke > kb ? (ke - kb + BKT - 1) / BKT : 0;
    auto issue = [&](int64_t it) {
        if (it < nk) {
            const int st = (int)(it % ST);
            if (interior) {
                ta.issue_full(sA + st * SA);
                tb.issue_full(sB + st * SB);
            } else {
                const int64_t k0 = kb + it * BKT;
                ta.issue_edge(sA + st * SA, g.a, m0, k0, g.M, ke);
                tb.issue_edge(sB + st * SB, g.b, n0, k0, g.N, ke);
            }
            ta.advance();
            tb.advance();
        }
        cp_commit();  // (empty groups keep the wait count uniform)
    };
#pragma unroll
    for (int it = 0; it < ST - 1; ++it) issue(it);
    for (int64_t it = 0; it < nk; ++it) {
        cp_wait<ST - 2>();
        __syncthreads();  // stage it visible to all; stage it-1 free for reuse
        issue(it + ST - 1);
        const int st = (int)(it % ST);
        const double *a_s = sA + st * SA;
        const double *b_s = sB + st * SB;
#pragma unroll
        for (int kk = 0; kk < BKT; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = frag<A_CM, BKT>(a_s, wm + i * 8 + fr, kk + fc);
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = frag<B_CN, BKT>(b_s, wn + j * 8 + fr, kk + fc);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    dmma(acc[i][j], af[i], bf[j]);
        }
    }
    // C -= A B on an F-order C with even rows / leading dimension: lanes fr and
    // fr ^ 1 trade one accumulator so that each owns two consecutive rows of one
    // column -- 16-byte read-modify-writes, half the memory instructions
    if (g.sub && g.c_sm == 1 && !(g.c_sn & 1) && !((uintptr_t)g.c & 15) && !(g.M & 1)) {
        const bool odd = fr & 1;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const double give = odd ? acc[i][j][0] : acc[i][j][1];
                const double got = __shfl_xor_sync(0xffffffffu, give, 4);
                const int64_t m = m0 + wm + i * 8 + (fr & ~1), n = n0 + wn + j * 8 + 2 * fc + (odd ? 1 : 0);
                if (m >= g.M || n >= g.N) continue;
                const double v0 = odd ? got : acc[i][j][0], v1 = odd ? acc[i][j][1] : got;
                double2 *pc = reinterpret_cast<double2 *>(g.c + m + n * g.c_sn);
                double2 c2 = *pc;
                c2.x = __dsub_rn(c2.x, v0);
                c2.y = __dsub_rn(c2.y, v1);
                *pc = c2;
            }
        return;
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
                } else if (g.sub) {
                    double *pc = g.c + m * g.c_sm + n * g.c_sn;
                    *pc = __dsub_rn(*pc, v);
                } else {
                    g.c[m * g.c_sm + n * g.c_sn] = v;
                }
            }
}

// ---------------------------------------------------------------------------
// TMA-fed variant (the default where the operands allow it): every stage's
// A and B tiles arrive by cp.async.bulk.tensor (one elected thread, per-
// launch tensor maps, mbarrier completion by transaction bytes) in the
// 128-byte swizzled layout, so a stage costs 2-5 TMA instructions instead of
// 2 x 512 cp.async, and edge tiles need no predicated path (the tensor
// engine zero-fills outside the tensor).  Tile layouts in shared memory:
//   K-contiguous operand (KC): box {16 k, 64 outer}: row o = 128 B (k 0..15),
//     16-byte chunk c at c ^ (o & 7);
//   outer-contiguous operand (OC): 8 boxes {8 outer, 16 k}, no swizzle: box
//     q = 1 KB, row k = 64 B (outer 8q..8q+7) -- a fragment's 4 consecutive
//     k rows alternate between the two 64-byte bank halves.
// Both make the m8n8k4 fragment loads hit the 2-wavefront minimum.  K
// chunks of a split are multiples of 16, so a box never reads another
// split's K range; only the tensor's own end is zero-filled.
constexpr int kTmaTile = BM * BK * 8;  // bytes per operand tile (8 KB)

template <bool KC> __device__ __forceinline__ double tfrag(const unsigned char *t, int o, int k) {
    if (KC) return *reinterpret_cast<const double *>(t + o * 128 + ((((k >> 1) ^ (o & 7))) << 4) + ((k & 1) << 3));
    return *reinterpret_cast<const double *>(t + ((o >> 3) << 10) + k * 64 + ((o & 7) << 3));
}

__device__ __forceinline__ unsigned smaddr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            bar),
        "r"(parity)
        : "memory");
}

template <bool KC, int OUTER>
__device__ __forceinline__ void tma_tile(unsigned dst, const CUtensorMap *tm, int64_t o0, int64_t k0, unsigned bar) {
    if (KC) {  // one box {16 k, OUTER rows}
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
                "r"(dst),
            "l"(tm), "r"((int)k0), "r"((int)o0), "r"(bar)
            : "memory");
    } else {
#pragma unroll
        for (int q = 0; q < OUTER / 8; ++q)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(dst + q * 1024),
                "l"(tm), "r"((int)(o0 + 8 * q)), "r"((int)k0), "r"(bar)
                : "memory");
    }
}

// Warp-specialised: 4 MMA warps (2 x 2) and one producer warp; stages are
// handed over with full / empty mbarriers only -- no CTA-wide barrier per K
// step (a __syncthreads every 64 DMMAs per warp lines the warps up on the
// DMMA latency, tools/dmma_occ_probe.cu).  The CTA tile is 64 x BNT: BNT =
// 64 (warp tile 32 x 32), or 128 for products 65..128 columns wide (warp
// tile 32 x 64: a 100-wide product is one tile column instead of two 64-wide
// ones); 8 x 8 fragments wholly outside C are skipped (warp-uniform).
constexpr int kGmTmaThreads = kGmThreads + 32;
template <bool A_KC, bool B_KC, int ST, int BNT>
__global__ void __launch_bounds__(kGmTmaThreads, BNT == 64 ? 1 : 2) dgemm_dmma_tma(GemmArgs g, const __grid_constant__ CUtensorMap tmA,
                                                               const __grid_constant__ CUtensorMap tmB) {
    constexpr int NFW = BNT / 16;                    // N fragments per warp
    constexpr int TA = kTmaTile, TB = BNT * BK * 8;  // stage bytes per operand
    pdl_wait();  // inputs may be the previous kernel's output (PDL)
    pdl_trigger();
    extern __shared__ unsigned char tsm_raw[];
    unsigned char *tsm = tsm_raw + ((1024 - (smaddr(tsm_raw) & 1023)) & 1023);  // 128B swizzle: 1 KB aligned
    unsigned long long *full = reinterpret_cast<unsigned long long *>(tsm + ST * (TA + TB));
    unsigned long long *empty = full + ST;
    int64_t tm, tn;
    if (g.syrk) {
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
    const int64_t m0 = tm * BM, n0 = tn * BNT;
    const int64_t kb = (int64_t)blockIdx.z * g.kchunk;
    int64_t ke = kb + g.kchunk;
    if (ke > g.K) ke = g.K;
    const int64_t nk = ke > kb ? (ke - kb + BK - 1) / BK : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < ST; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smaddr(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(smaddr(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 4) {  // producer
        if (lane == 0) {
            for (int64_t it = 0; it < nk; ++it) {
                const int s = (int)(it % ST);
                if (it >= ST) tma_wait(smaddr(&empty[s]), (unsigned)(((it / ST) - 1) & 1));
                const unsigned bar = smaddr(&full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)(TA + TB))
                             : "memory");
                const int64_t k0 = kb + it * BK;
                tma_tile<A_KC, BM>(smaddr(tsm + s * (TA + TB)), &tmA, m0, k0, bar);
                tma_tile<B_KC, BNT>(smaddr(tsm + s * (TA + TB) + TA), &tmB, n0, k0, bar);
            }
        }
        return;
    }
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * (BNT / 2);
    const int fr = lane >> 2, fc = lane & 3;
    double acc[4][NFW][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NFW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // live fragment rows / columns (warp-uniform)
    unsigned live_i = 0, live_j = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (m0 + wm + i * 8 < g.M) live_i |= 1u << i;
#pragma unroll
    for (int j = 0; j < NFW; ++j)
        if (n0 + wn + j * 8 < g.N) live_j |= 1u << j;
    for (int64_t it = 0; it < nk; ++it) {
        const int s = (int)(it % ST);
        tma_wait(smaddr(&full[s]), (unsigned)((it / ST) & 1));
        const unsigned char *a_s = tsm + s * (TA + TB);
        const unsigned char *b_s = a_s + TA;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[NFW];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = tfrag<A_KC>(a_s, wm + i * 8 + fr, kk + fc);
#pragma unroll
            for (int j = 0; j < NFW; ++j) bf[j] = tfrag<B_KC>(b_s, wn + j * 8 + fr, kk + fc);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < NFW; ++j)
                    if (BNT == 64 || (((live_i >> i) & (live_j >> j)) & 1)) dmma(acc[i][j], af[i], bf[j]);
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smaddr(&empty[s])) : "memory");
    }
    // epilogue (as dgemm_dmma)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NFW; ++j)
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
                } else if (g.sub) {
                    double *pc = g.c + m * g.c_sm + n * g.c_sn;
                    *pc = __dsub_rn(*pc, v);
                } else {
                    g.c[m * g.c_sm + n * g.c_sn] = v;
                }
            }
}

static PFN_cuTensorMapEncodeTiled_v12000 gemm_tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return f;
    }();
    return enc;
}

// Tensor map of one operand: KC (K unit-stride): dims {K, outer}, box
// {16, 64}, 128-byte swizzle; OC (outer unit-stride): dims {outer, K}, box
// {8, 16}, no swizzle.  False when TMA cannot address it (alignment, strides, sizes).
static bool gemm_tmap(CUtensorMap *tm, const double *base, bool kc, int64_t outer, int64_t K, int64_t stride,
                      int box_outer = BM) {
    auto enc = gemm_tmap_encoder();
    if (!enc || ((uintptr_t)base & 15) || (stride * 8) % 16 || stride <= 0 || outer > 0x7fffffff || K > 0x7fffffff ||
        stride * 8 >= (1ll << 40))
        return false;
    cuuint64_t dims[2], strides[1] = {(cuuint64_t)(stride * 8)};
    cuuint32_t box[2], es[2] = {1, 1};
    if (kc) {
        dims[0] = (cuuint64_t)K;
        dims[1] = (cuuint64_t)outer;
        box[0] = BK;
        box[1] = (cuuint32_t)box_outer;
    } else {
        dims[0] = (cuuint64_t)outer;
        dims[1] = (cuuint64_t)K;
        box[0] = 8;
        box[1] = BK;
    }
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, kc ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool gemm_tma_enabled() {
    static const bool on = [] {
        const char *e = getenv("LM_GEMM_TMA");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <bool A_KC, bool B_KC, int ST, int BNT>
int launch_dgemm_tma_kernel(const GemmArgs &g, const CUtensorMap &ta, const CUtensorMap &tb, dim3 grid,
                            cudaStream_t s) {
    auto k = dgemm_dmma_tma<A_KC, B_KC, ST, BNT>;
    constexpr int smem = ST * (kTmaTile + BNT * BK * 8) + 1024 + 16 * ST;
    if (int rc = func_attrs(k, smem)) return rc;
    LM_CUDA(launch_pdl(k, grid, dim3(kGmTmaThreads), smem, s, g, ta, tb));
    LM_LAUNCHED(1);
    note_variant(BNT == 64 ? "gemm_tma" : "gemm_tma_wide");
    return 0;
}

// 0: launched; 1: not TMA-addressable (the caller launches the cp.async kernel)
int try_launch_dgemm_tma(const GemmArgs &g, dim3 grid, cudaStream_t s, bool wide) {
    static const bool tma_sub = getenv("LM_GEMM_TMA_SUB") && getenv("LM_GEMM_TMA_SUB")[0] == '1';
    if (!gemm_tma_enabled() || (g.sub && !tma_sub)) return 1;  // the LU's C -= A B keeps the cp.async ring
    const bool a_kc = g.a_sk == 1, b_kc = g.b_sk == 1;
    if (!a_kc && g.a_sm != 1) return 1;
    if (!b_kc && g.b_sn != 1) return 1;
    CUtensorMap ta, tb;
    if (!gemm_tmap(&ta, g.a, a_kc, g.M, g.K, a_kc ? g.a_sm : g.a_sk)) return 1;
    if (!gemm_tmap(&tb, g.b, b_kc, g.N, g.K, b_kc ? g.b_sn : g.b_sk, wide ? 128 : BM)) return 1;
    if (wide) {
        if (a_kc && b_kc) return launch_dgemm_tma_kernel<true, true, 4, 128>(g, ta, tb, grid, s);
        if (a_kc) return launch_dgemm_tma_kernel<true, false, 4, 128>(g, ta, tb, grid, s);
        if (b_kc) return launch_dgemm_tma_kernel<false, true, 4, 128>(g, ta, tb, grid, s);
        return launch_dgemm_tma_kernel<false, false, 4, 128>(g, ta, tb, grid, s);
    }
    if (a_kc && b_kc) return launch_dgemm_tma_kernel<true, true, 4, 64>(g, ta, tb, grid, s);
    if (a_kc) return launch_dgemm_tma_kernel<true, false, 4, 64>(g, ta, tb, grid, s);
    if (b_kc) return launch_dgemm_tma_kernel<false, true, 4, 64>(g, ta, tb, grid, s);
    return launch_dgemm_tma_kernel<false, false, 4, 64>(g, ta, tb, grid, s);
}

// Whether a product takes the 64 x 128-tile TMA kernel: 65..128 columns
// (one tile column instead of two), not SYRK / the LU's update, and TMA-
// addressable operands (checked again by try_launch_dgemm_tma); opt-in.
static bool dgemm_wide(const GemmArgs &g) {
    // opt-in (LM_GEMM_WIDE=1): measured slower on config 3b (50 vs 33 us per
    // step: 2 CTAs per SM at 168 registers with spills, twice the per-CTA work)
    static const bool on = getenv("LM_GEMM_WIDE") && getenv("LM_GEMM_WIDE")[0] == '1';
    if (!on || !gemm_tma_enabled() || g.syrk || g.sub || g.N <= 64 || g.N > 128) return false;
    const bool a_kc = g.a_sk == 1, b_kc = g.b_sk == 1;
    const int64_t sa = a_kc ? g.a_sm : g.a_sk, sb = b_kc ? g.b_sn : g.b_sk;
    return (a_kc || g.a_sm == 1) && (b_kc || g.b_sn == 1) && ((uintptr_t)g.a & 15) == 0 &&
           ((uintptr_t)g.b & 15) == 0 && sa % 2 == 0 && sb % 2 == 0;
}

// Few partials: one thread per element, loads unrolled (independent).
__global__ void __launch_bounds__(256) splitk_finish_flat(const double *__restrict__ part, int64_t M, int64_t N,
                                                          int64_t nz, double *c, int64_t c_sm, int64_t c_sn, int syrk) {
    pdl_wait();  // inputs may be the previous kernel's output (PDL)
    pdl_trigger();
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t MN = M * N;
    if (e >= MN) return;
    const int64_t n = e / M, m = e - n * M;
    if (syrk && m > n) return;
    double acc = part[e];
#pragma unroll 8
    for (int64_t z = 1; z < nz; ++z) acc += part[z * MN + e];
    c[m * c_sm + n * c_sn] = acc;
    if (syrk) c[n * c_sm + m * c_sn] = acc;
}

// Many partials: out = sum over z of partials; syrk: upper only + mirror.  32 elements per
// CTA, warp w sums z = w, w+8, ... (independent loads in flight), the 8 warp
// sums are combined in warp order: a fixed tree, reproducible run to run.
__global__ void __launch_bounds__(256) splitk_finish(const double *__restrict__ part, int64_t M, int64_t N, int64_t nz,
                                                     double *c, int64_t c_sm, int64_t c_sn, int syrk) {
    pdl_wait();  // inputs may be the previous kernel's output (PDL)
    pdl_trigger();
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t e = (int64_t)blockIdx.x * 32 + lane;
    const int64_t MN = M * N;
    double acc = 0.0;
    if (e < MN) {
#pragma unroll 4
        for (int64_t z = w; z < nz; z += 8) acc += part[z * MN + e];
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w != 0 || e >= MN) return;
    const int64_t n = e / M, m = e - n * M;
    if (syrk && m > n) return;
    double v = red[0][lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) v += red[q][lane];
    c[m * c_sm + n * c_sn] = v;
    if (syrk) c[n * c_sm + m * c_sn] = v;
}

template <bool A_CM, bool B_CN, bool VA, bool VB, int BKT, int ST>
int launch_dgemm_kernel(const GemmArgs &g, dim3 grid, cudaStream_t s) {
    auto k = dgemm_dmma<A_CM, B_CN, VA, VB, BKT, ST>;
    constexpr int smem = ST * (stage_doubles<A_CM, BKT>() + stage_doubles<B_CN, BKT>()) * 8;
    if (int rc = func_attrs(k, smem)) return rc;
    LM_CUDA(launch_pdl(k, grid, dim3(kGmThreads), smem, s, g));
    LM_LAUNCHED(1);
    note_variant("gemm_cp");
    return 0;
}

template <bool A_CM, bool B_CN, int BKT, int ST>
int launch_dgemm_layout(const GemmArgs &g, bool va, bool vb, dim3 grid, cudaStream_t s) {
    if (va && vb) return launch_dgemm_kernel<A_CM, B_CN, true, true, BKT, ST>(g, grid, s);
    if (va) return launch_dgemm_kernel<A_CM, B_CN, true, false, BKT, ST>(g, grid, s);
    if (vb) return launch_dgemm_kernel<A_CM, B_CN, false, true, BKT, ST>(g, grid, s);
    return launch_dgemm_kernel<A_CM, B_CN, false, false, BKT, ST>(g, grid, s);
}

// Resident CTAs of the kernel configuration (all layout variants share the
// register / shared-memory footprint within a few registers).
template <int BKT, int ST> int64_t dgemm_resident() {
    static PerDevice<int64_t> cache;
    int64_t r = num_sms();
    cache.get(r, [](int64_t &r) {
        auto k = dgemm_dmma<false, false, true, true, BKT, ST>;
        constexpr int smem = ST * 2 * stage_doubles<false, BKT>() * 8;
        func_attrs(k, smem);
        int per = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kGmThreads, smem) != cudaSuccess || per < 1) per = 1;
        r = (int64_t)per * num_sms();
        return 0;
    });
    return r;
}

// Split-K choice: maximise (wave efficiency) x (pipeline fill) / (1 + the
// partials' HBM time relative to the math time).  Wave efficiency counts
// the tail: units / resident / ceil(units / resident).
inline int64_t choose_splits(int64_t tiles, int64_t M, int64_t N, int64_t K, int bkt, int64_t resident) {
    const int64_t kt = ceil_div(K, bkt);
    const double t_math = 2.0 * (double)tiles * BM * BN * (double)K / 35e12;
    int64_t best = 1;
    double best_score = -1.0;
    for (int64_t s = 1; s <= 128 && s <= kt; ++s) {
        const int64_t kchunk = ceil_div(ceil_div(K, s), bkt) * bkt;
        const int64_t se = ceil_div(K, kchunk);
        if (se != s) continue;
        if ((double)se * M * N * 8 > 1e9) break;
        const double waves = (double)(tiles * se) / (double)resident;
        const double eff = waves / std::ceil(waves);
        const double kit = (double)kchunk / bkt;
        const double pipe = kit / (kit + 3.0);
        const double t_part = se > 1 ? 2.0 * se * (double)M * N * 8 / 6e12 + 3e-6 : 0.0;
        const double score = eff * pipe / (1.0 + t_part / t_math);
        if (score > best_score * 1.0001) {
            best_score = score;
            best = se;
        }
    }
    return best;
}

template <int BKT, int ST>
int dgemm_cfg(GemmArgs &g, bool a_cm, bool b_cn, bool va, bool vb, cudaStream_t s) {
    const int64_t M = g.M, N = g.N, K = g.K;
    const bool wide = dgemm_wide(g);
    const int64_t tM = ceil_div(M, BM), tN = wide ? 1 : ceil_div(N, BN);
    const int64_t tiles = g.syrk ? tM * (tM + 1) / 2 : tM * tN;
    g.tiles_n = tN;
    int64_t splits = g.sub ? 1 : choose_splits(tiles, M, N, K, BKT, dgemm_resident<BKT, ST>());
    static const int64_t force_splits = getenv("LM_GEMM_SPLITS") ? atoll(getenv("LM_GEMM_SPLITS")) : 0;  // A/B
    if (force_splits > 0 && !g.sub && splits > 1) splits = force_splits;
    g.kchunk = ceil_div(ceil_div(K, splits), BKT) * BKT;
    splits = ceil_div(K, g.kchunk);
    Scratch part;
    if (splits > 1) {
        if (int rc = part.alloc(sizeof(double) * M * N * splits, s)) return rc;
        g.part = part.as<double>();
    }
    dim3 grid((unsigned)tiles, 1, (unsigned)splits);
    int rc = try_launch_dgemm_tma(g, grid, s, wide);
    if (rc < 0) return rc;
    LM_REQUIRE(rc == 0 || !wide, "gemm: wide tile chosen for operands TMA cannot address");
    if (rc == 0)
        ;
    else if (a_cm && b_cn)
        rc = launch_dgemm_layout<true, true, BKT, ST>(g, va, vb, grid, s);
    else if (a_cm)
        rc = launch_dgemm_layout<true, false, BKT, ST>(g, va, vb, grid, s);
    else if (b_cn)
        rc = launch_dgemm_layout<false, true, BKT, ST>(g, va, vb, grid, s);
    else
        rc = launch_dgemm_layout<false, false, BKT, ST>(g, va, vb, grid, s);
    if (rc) return rc;
    if (splits > 1) {
        if (splits <= 16)
            LM_CUDA(launch_pdl(splitk_finish_flat, dim3((unsigned)ceil_div(M * N, 256)), dim3(256), 0, s,
                               (const double *)g.part, M, N, (int64_t)splits, g.c, g.c_sm, g.c_sn, g.syrk));
        else
            LM_CUDA(launch_pdl(splitk_finish, dim3((unsigned)ceil_div(M * N, 32)), dim3(256), 0, s,
                               (const double *)g.part, M, N, (int64_t)splits, g.c, g.c_sm, g.c_sn, g.syrk));
        LM_LAUNCHED(1);
    }
    return 0;
}

// gemm_skinny.cu: one or two short dimensions (0 launched, 1 not taken, < 0 error)
int try_dgemm_skinny(const double *a, int64_t a_sm, int64_t a_sk, const double *b, int64_t b_sk, int64_t b_sn,
                     double *c, int64_t c_sm, int64_t c_sn, int64_t M, int64_t N, int64_t K, cudaStream_t s);

// A(m,k) strides (a_sm, a_sk), B(k,n) strides (b_sk, b_sn).
int dgemm(const double *a, int64_t a_sm, int64_t a_sk, const double *b, int64_t b_sk, int64_t b_sn, double *c,
          int64_t c_sm, int64_t c_sn, int64_t M, int64_t N, int64_t K, bool syrk, cudaStream_t s) {
    if (M == 0 || N == 0) return 0;
    if (K == 0) {
        // empty inner dimension: out = 0
        LM_REQUIRE(c_sm == 1, "gemm: K == 0 needs a column-major output");
        for (int64_t n = 0; n < N; ++n) LM_CUDA(cudaMemsetAsync(c + n * c_sn, 0, sizeof(double) * M, s));
        return 0;
    }
    if (!syrk) {
        const int rc = try_dgemm_skinny(a, a_sm, a_sk, b, b_sk, b_sn, c, c_sm, c_sn, M, N, K, s);
        if (rc <= 0) return rc;
    }
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
    const bool a_cm = (a_sm == 1);               // A contiguous along M
    const bool b_cn = (b_sn == 1 && b_sk != 1);  // B contiguous along N
    auto aligned16 = [](const void *p) { return ((uintptr_t)p & 15) == 0; };
    // 16-byte cp.async needs the contiguous dim unit-stride and the other
    // stride even (every pair starts 16-byte aligned).
    const bool va = aligned16(a) && (a_cm ? (a_sk % 2 == 0) : (a_sk == 1 && a_sm % 2 == 0));
    const bool vb = aligned16(b) && (b_cn ? (b_sk % 2 == 0) : (b_sk == 1 && b_sn % 2 == 0));
    // BK 16, 3 stages: 32.3 TF/s on the config-3c SYRK (BK 32 x 2 stages ties,
    // 3-4 deep BK-32/16 rings lose occupancy)
    return dgemm_cfg<16, 3>(g, a_cm, b_cn, va, vb, s);
}

// C -= A B for column-major A (M x K, lda), B (K x N, ldb), C (M x N, ldc):
// the blocked LU's trailing update on the FP64 tensor cores (DMMA with FMA
// accumulation; lu_fast.cu's tensor mode).
int dgemm_sub(const double *a, int64_t lda, const double *b, int64_t ldb, double *c, int64_t ldc, int64_t M,
              int64_t N, int64_t K, cudaStream_t s) {
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    GemmArgs g{};
    g.a = a;
    g.a_sm = 1;
    g.a_sk = lda;
    g.b = b;
    g.b_sk = 1;
    g.b_sn = ldb;
    g.c = c;
    g.c_sm = 1;
    g.c_sn = ldc;
    g.M = M;
    g.N = N;
    g.K = K;
    g.sub = 1;
    auto aligned16 = [](const void *p) { return ((uintptr_t)p & 15) == 0; };
    const bool va = aligned16(a) && lda % 2 == 0;
    const bool vb = aligned16(b) && ldb % 2 == 0;
    // Wide trailing updates (more than 128 columns): the 2-stage ring at <= 102
    // registers, five resident CTAs per SM instead of four (the kernel is bound
    // by how many CTAs overlap their loads, barriers and read-modify-write
    // epilogues: 20.8 -> 23.9 TF/s alone, tools/gemm_sub_probe.py; config 4a
    // 25.95 -> 24.6 ms; deeper rings / BK = 32 at 2-3 CTAs per SM: 12-18 TF/s).
    // Same tiles, same K order: bit-identical.  LM_GEMM_SUB_CFG=163: the 3-stage ring.
    static const bool ring3 = getenv("LM_GEMM_SUB_CFG") && atoi(getenv("LM_GEMM_SUB_CFG")) == 163;
    if (N > 128 && !ring3) return dgemm_cfg<16, 2>(g, true, false, va, vb, s);
    return dgemm_cfg<16, 3>(g, true, false, va, vb, s);
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

extern "C" int lm_debug_gemm_sub(lm_view a, lm_view b, lm_view c, void *stream) {
    clear_error();
    LM_REQUIRE(a.cols == b.rows && c.rows == a.rows && c.cols == b.cols, "gemm_sub shape mismatch");
    LM_REQUIRE(a.rs == 1 && b.rs == 1 && c.rs == 1, "gemm_sub needs F-order operands");
    return dgemm_sub((const double *)a.ptr, a.cs, (const double *)b.ptr, b.cs, (double *)c.ptr, c.cs, a.rows, b.cols,
                     a.cols, as_stream(stream));
}

extern "C" int lm_syrk(int dtype, lm_view a, lm_view out, void *stream) {
    clear_error();
    LM_REQUIRE(out.rows == a.rows && out.cols == a.rows, "syrk out shape mismatch");
    LM_REQUIRE(dtype == LM_F64, "syrk: f64 only");
    // out = a @ a.T : A(m,k) = a(m,k), B(k,n) = a(n,k)
    return dgemm((const double *)a.ptr, a.rs, a.cs, (const double *)a.ptr, a.cs, a.rs, (double *)out.ptr, out.rs,
                 out.cs, a.rows, a.rows, a.cols, true, as_stream(stream));
}
