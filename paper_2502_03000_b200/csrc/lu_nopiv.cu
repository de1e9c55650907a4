// lu_nopiv.cu -- the blocked LU when partial pivoting provably never swaps.
//
// If A is strictly diagonally dominant by columns (|a_jj| > sum_{i != j}
// |a_ij| for every j), Gaussian elimination with partial pivoting performs
// no row interchanges: the diagonal entry is the unique maximum of its
// column, and every Schur complement stays column diagonally dominant
// (Golub & Van Loan, "Matrix Computations", diagonal dominance and GEPP).
// The reference's _lu_factor (lazymat/_loops.py:200-236) would therefore
// choose pivot k at every step; config 4a's A = U(-1,1) + 8192 I is such a
// matrix.  In tensor mode (values at residual level, pivots exact) the LU
// then needs no pivot search at all, and every step is GEMM-shaped:
//
//   per 64-column block J (right-looking, look-ahead of one block):
//     hi stream  diag_nopiv: A11 = L11 U11 in one CTA (shared memory), plus
//                L11^-1 and U11^-1 (column-parallel substitution);
//                L21 = A21 U11^-1 (DMMA GEMM), U12 of the NEXT block's
//                columns = L11^-1 A12, and that column panel's update
//     lo stream  U12 of the remaining columns, A22 -= L21 U12 (DMMA, the
//                bulk of the 2n^3/3 flops)
//
// The dominance test runs first (one pass over A, with a margin far above
// rounding so the reference's own rounded Schur complements keep the same
// strict maxima), and after the factorisation every multiplier is checked
// to be strictly inside (-1, 1) by the same margin (lower_absmax); if that
// ever failed, the original matrix (kept in a backup) is factored again by
// the pivoting path.  Pivots come back as the identity -- exactly what the
// reference computes for these matrices.
#include <chrono>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace lm {

int dgemm(const double *a, int64_t a_sm, int64_t a_sk, const double *b, int64_t b_sk, int64_t b_sn, double *c,
          int64_t c_sm, int64_t c_sn, int64_t M, int64_t N, int64_t K, bool syrk, cudaStream_t s);
int dgemm_sub(const double *a, int64_t lda, const double *b, int64_t ldb, double *c, int64_t ldc, int64_t M,
              int64_t N, int64_t K, cudaStream_t s);

namespace {

constexpr int NBD = 64;          // block width
constexpr int LDD = NBD + 1;     // shared-memory column length (odd: conflict-free column walks)
constexpr double kDomMargin = 1.001;   // |a_jj| > kDomMargin * sum_{i != j} |a_ij|
constexpr double kMulBound = 0.999;    // every multiplier |l_ij| < kMulBound (then the argmax is strict)

// one warp per column: flag columns that are not strictly dominant (or hold NaN / Inf)
__global__ void __launch_bounds__(256) coldom_check(const double *__restrict__ A, int64_t n, int64_t lda,
                                                   int *__restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = w; j < n; j += nw) {
        const double *col = A + j * lda;
        double s = 0.0;
        for (int64_t i = lane; i < n; i += 32)
            if (i != j) s += fabs(col[i]);
        s = warp_sum(s);
        if (lane == 0) {
            const double d = fabs(col[j]);
            if (!(d > kDomMargin * s) || !(s < 1e300)) atomicOr(flag, 1);
        }
    }
}

// A11 = L11 U11 (no pivoting) of the nb x nb block at A (nb <= NBD), in
// shared memory, FMA arithmetic (tensor mode), blocked by 8 columns: warp 0
// factors the 64 x 8 panel in registers (two rows per lane, the pivot row
// broadcast by shuffles, no barrier), 56 threads solve the panel's 8 rows of
// U against L11 (8 x 8), then all threads apply the rank-8 update -- three
// barriers per 8 columns.  (One rank-1 update and two barriers per column
// took 28-42 us per block on the panel chain, 5.3 ms per 8192 factorisation.)
// 128 threads at <= 128 registers and 33 KB: the CTA fits next to three
// resident trailing-update CTAs (46K registers, 170 KB) instead of waiting for
// two of them to finish.
constexpr int kDiagThreads = 128, kDiagSlices = kDiagThreads / NBD;
__global__ void __launch_bounds__(kDiagThreads) diag_nopiv(double *A, int64_t lda, int nb) {
    pdl_wait();  // launched with PDL: the previous chain kernel's output is the input
    pdl_trigger();
    __shared__ double a[NBD * LDD];  // (i, j) at a[j * LDD + i]; identity outside nb x nb
    constexpr int PB = 8;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tid & (NBD - 1), ty = tid >> 6;
#pragma unroll
    for (int c = ty; c < NBD; c += kDiagSlices)
        a[c * LDD + tx] = (tx < nb && c < nb) ? A[tx + (int64_t)c * lda] : (tx == c ? 1.0 : 0.0);
    __syncthreads();
#pragma unroll 1
    for (int c0 = 0; c0 < NBD; c0 += PB) {
        if (warp == 0) {
            // panel columns c0 .. c0 + 7, rows lane and lane + 32
            const int hk = c0 >> 5;  // the half holding the pivot rows (warp-uniform)
            double v[2][PB];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int q = 0; q < PB; ++q) v[h][q] = a[(c0 + q) * LDD + lane + 32 * h];
#pragma unroll
            for (int q = 0; q < PB; ++q) {
                const int k = c0 + q, lk = k & 31;
                double pv[PB];
#pragma unroll
                for (int q2 = q; q2 < PB; ++q2) pv[q2] = __shfl_sync(0xffffffffu, hk ? v[1][q2] : v[0][q2], lk);
                const double rp = __drcp_rn(pv[q]);  // tensor mode: multiply by the reciprocal
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (lane + 32 * h > k) {
                        const double l = v[h][q] * rp;
                        v[h][q] = l;
#pragma unroll
                        for (int q2 = q + 1; q2 < PB; ++q2) v[h][q2] = fma(-l, pv[q2], v[h][q2]);
                    }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int q = 0; q < PB; ++q) a[(c0 + q) * LDD + lane + 32 * h] = v[h][q];
        }
        __syncthreads();
        const int c1 = c0 + PB;
        if (c1 >= NBD) break;
        // rows c0 .. c0 + 7 of U over the columns right of the panel: L11 u = a (unit lower, 8 x 8)
        if (tid < NBD - c1) {
            double *col = a + (c1 + tid) * LDD + c0;
            double u[PB];
#pragma unroll
            for (int q = 0; q < PB; ++q) u[q] = col[q];
#pragma unroll
            for (int q = 0; q < PB; ++q)
#pragma unroll
                for (int q2 = q + 1; q2 < PB; ++q2) u[q2] = fma(-a[(c0 + q) * LDD + c0 + q2], u[q], u[q2]);
#pragma unroll
            for (int q = 0; q < PB; ++q) col[q] = u[q];
        }
        __syncthreads();
        // rank-8 update of the rows below the panel's, columns right of it
        if (tx >= c1) {
            double l[PB];
#pragma unroll
            for (int q = 0; q < PB; ++q) l[q] = a[(c0 + q) * LDD + tx];
            for (int c = c1 + ty; c < NBD; c += kDiagSlices) {
                const double *u = a + c * LDD + c0;
                double x = a[c * LDD + tx];
#pragma unroll
                for (int q = 0; q < PB; ++q) x = fma(-l[q], u[q], x);
                a[c * LDD + tx] = x;
            }
        }
        __syncthreads();
    }
    for (int c = ty; c < nb; c += kDiagSlices)
        if (tx < nb) A[tx + (int64_t)c * lda] = a[c * LDD + tx];
}

// The two triangular solves keep a thread's row (or column) SHIFTED in
// registers -- before step i, s[j] holds entry i + j -- so the step loop is
// rolled with static register indices (the fully unrolled 64 x 64 solve is
// ~8k instructions that every warp runs once: ncu showed 34% of the stalls
// waiting on instruction fetch).  The triangle sits in shared memory padded
// with zero columns so entry i + j never leaves it; the step loop runs in two
// halves -- steps 0..31 shift all 63 entries, steps 32..63 only the 31 that
// can still be non-zero -- so i + j <= 94: 95 columns, 49 KB.  That fits next
// to three resident trailing-update CTAs (the 128-column padding, 66.5 KB,
// had to wait for one of them to finish), and the second half does half the
// FMAs.
constexpr int HNB = NBD / 2;
constexpr int NPAD = NBD + HNB - 1;  // 95 columns (rows) of the padded triangle
constexpr int kTriSmem = NPAD * LDD * (int)sizeof(double);        // trsm_right_upper: [NPAD columns][LDD]
constexpr int kTriLowSmem = NBD * NPAD * (int)sizeof(double);     // trsm_left_lower_unit: [NBD columns][NPAD rows]

// L21 = A21 U11^-1 in place: one thread per row of A21 (rows [0, M),
// leading dimension lda), U11 (nb x nb at U).  Row-wise substitution
// x U = a:  x_i = s_i / u_ii;  s_j -= x_i u_ij (j > i)
__global__ void __launch_bounds__(64) trsm_right_upper(double *A21, int64_t lda, int64_t M, const double *U, int nb) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double tsm[];  // u_ij at tsm[j * LDD + i], j < NPAD (zero past nb)
    __shared__ double rinv[NBD];     // 1 / u_ii: tensor mode multiplies (a division is 126 cycles of chain)
    // the nb x nb block: all of a thread's 64 loads in flight at once (16 at a
    // time cost four L2 round trips on the panel chain), then the padding
    {
        const int i = threadIdx.x;  // blockDim.x == NBD
        double u[NBD];
#pragma unroll
        for (int j = 0; j < NBD; ++j) u[j] = (i < nb && j < nb) ? U[i + (int64_t)j * lda] : (i == j ? 1.0 : 0.0);
#pragma unroll
        for (int j = 0; j < NBD; ++j) tsm[j * LDD + i] = u[j];
#pragma unroll
        for (int j = NBD; j < NPAD; ++j) tsm[j * LDD + i] = 0.0;
        rinv[i] = i < nb ? 1.0 / U[i + (int64_t)i * lda] : 1.0;
    }
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= M) return;
    double *row = A21 + r;
    double sv[NBD];
#pragma unroll
    for (int c = 0; c < NBD; ++c) sv[c] = c < nb ? row[c * lda] : 0.0;
    const int n1 = nb < HNB ? nb : HNB;
#pragma unroll 1
    for (int i = 0; i < n1; ++i) {
        const double *ui = tsm + i;  // u_{i, i + j} at ui[(i + j) * LDD]
        const double x = sv[0] * rinv[i];
        row[i * lda] = x;
#pragma unroll
        for (int j = 1; j < NBD; ++j) sv[j - 1] = fma(-x, ui[(i + j) * LDD], sv[j]);
        sv[NBD - 1] = 0.0;
    }
#pragma unroll 1
    for (int i = HNB; i < nb; ++i) {  // entries i + j >= 64 do not exist: sv[32..] stays zero
        const double *ui = tsm + i;
        const double x = sv[0] * rinv[i];
        row[i * lda] = x;
#pragma unroll
        for (int j = 1; j < HNB; ++j) sv[j - 1] = fma(-x, ui[(i + j) * LDD], sv[j]);
        sv[HNB - 1] = 0.0;
    }
}

// U12 = L11^-1 A12 in place: one thread per column of A12 (nb rows, columns
// [0, N)), unit lower L11 (at L).  y_k final; y_i -= l_ik y_k (i > k)
__global__ void __launch_bounds__(64) trsm_left_lower_unit(double *A12, int64_t lda, int64_t N, const double *L,
                                                          int nb) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double tsm[];  // l_ik at tsm[k * LDD2 + i], i < NPAD (zero past nb / on and above the diagonal)
    constexpr int LDD2 = NPAD;  // 95: odd
    {
        const int i = threadIdx.x;  // blockDim.x == NBD: row i of L11, all loads in flight at once
        double l[NBD];
#pragma unroll
        for (int k = 0; k < NBD; ++k) l[k] = (i < nb && k < nb && i > k) ? L[i + (int64_t)k * lda] : 0.0;
#pragma unroll
        for (int k = 0; k < NBD; ++k) {
            tsm[k * LDD2 + i] = l[k];
            if (i < NPAD - NBD) tsm[k * LDD2 + NBD + i] = 0.0;
        }
    }
    __syncthreads();
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    double *col = A12 + c * lda;
    double y[NBD];
#pragma unroll
    for (int i = 0; i < NBD; ++i) y[i] = i < nb ? col[i] : 0.0;
    const int n1 = nb < HNB ? nb : HNB;
#pragma unroll 1
    for (int k = 0; k < n1; ++k) {
        const double yk = y[0];
        col[k] = yk;
        const double *lk = tsm + k * LDD2 + k;  // l_{k + j, k} at lk[j]
#pragma unroll
        for (int j = 1; j < NBD; ++j) y[j - 1] = fma(-lk[j], yk, y[j]);
        y[NBD - 1] = 0.0;
    }
#pragma unroll 1
    for (int k = HNB; k < nb; ++k) {  // rows k + j >= 64 do not exist: y[32..] stays zero
        const double yk = y[0];
        col[k] = yk;
        const double *lk = tsm + k * LDD2 + k;
#pragma unroll
        for (int j = 1; j < HNB; ++j) y[j - 1] = fma(-lk[j], yk, y[j]);
        y[HNB - 1] = 0.0;
    }
}

// U12 of a whole outer block in ONE launch (both inner blocks full): with
// L = [[L_aa, 0], [L_ba, L_bb]] (128 x 128 unit lower, at Lob), per column
//   y_a = L_aa^-1 a_a;   a_b -= L_ba y_a;   y_b = L_bb^-1 a_b
// -- what trsm_left_lower_unit, the 64 x N x 64 product and a second
// trsm_left_lower_unit did as three dependent launches on the panel chain.
// One thread per column; the three operators take turns in the same shared
// memory; y_a is re-read from the column (16 values at a time) for the
// middle step, so the footprint stays that of trsm_left_lower_unit.
__global__ void __launch_bounds__(64) trsm_left_lower_pair(double *A12, int64_t lda, int64_t N, const double *Lob) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double tsm[];
    constexpr int LDD2 = NPAD;
    const int t = threadIdx.x;  // blockDim.x == NBD
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + t;
    const bool live = c < N;
    double *col = A12 + (live ? c : 0) * lda;
    double y[NBD];
    // strictly lower part of the 64 x 64 block at L, zero-padded rows; CH loads
    // in flight at a time (32 while y is live: 64 + 2 x 64 registers spill)
    auto load_tri = [&](const double *L, auto ch) {
        constexpr int CH = decltype(ch)::value;
#pragma unroll
        for (int k0 = 0; k0 < NBD; k0 += CH) {
            double l[CH];
#pragma unroll
            for (int k = 0; k < CH; ++k) l[k] = t > k0 + k ? L[t + (int64_t)(k0 + k) * lda] : 0.0;
#pragma unroll
            for (int k = 0; k < CH; ++k) {
                tsm[(k0 + k) * LDD2 + t] = l[k];
                if (t < NPAD - NBD) tsm[(k0 + k) * LDD2 + NBD + t] = 0.0;
            }
        }
    };
    auto solve = [&](double *dst) {  // y <- L^-1 y, step by step into dst[0..63]
#pragma unroll 1
        for (int k = 0; k < HNB; ++k) {
            const double yk = y[0];
            dst[k] = yk;
            const double *lk = tsm + k * LDD2 + k;
#pragma unroll
            for (int j = 1; j < NBD; ++j) y[j - 1] = fma(-lk[j], yk, y[j]);
            y[NBD - 1] = 0.0;
        }
#pragma unroll 1
        for (int k = HNB; k < NBD; ++k) {
            const double yk = y[0];
            dst[k] = yk;
            const double *lk = tsm + k * LDD2 + k;
#pragma unroll
            for (int j = 1; j < HNB; ++j) y[j - 1] = fma(-lk[j], yk, y[j]);
            y[HNB - 1] = 0.0;
        }
    };
    load_tri(Lob, std::integral_constant<int, 32>{});
#pragma unroll
    for (int i = 0; i < NBD; ++i) y[i] = live ? col[i] : 0.0;
    __syncthreads();
    if (live) solve(col);
    __syncthreads();
    // L_ba (64 x 64, dense) -> tsm[k * NBD + i]; a_b - L_ba y_a -> y
#pragma unroll
    for (int k0 = 0; k0 < NBD; k0 += 32) {
        double l[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) l[k] = Lob[NBD + t + (int64_t)(k0 + k) * lda];
#pragma unroll
        for (int k = 0; k < 32; ++k) tsm[(k0 + k) * NBD + t] = l[k];
    }
    __syncthreads();
    // 32 outputs at a time (y_a, 16 values per batch, + 64 outputs + the
    // operator's values in flight would spill); the results go back to the
    // column and are re-read for the second solve
    if (live) {
#pragma unroll 1
        for (int h = 0; h < NBD; h += HNB) {
            double z[HNB];
#pragma unroll
            for (int i = 0; i < HNB; ++i) z[i] = col[NBD + h + i];
#pragma unroll 1
            for (int k0 = 0; k0 < NBD; k0 += 16) {
                double ya[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) ya[q] = col[k0 + q];  // (this thread's own stores)
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const double *lk = tsm + (k0 + q) * NBD + h;
#pragma unroll
                    for (int i = 0; i < HNB; ++i) z[i] = fma(-lk[i], ya[q], z[i]);
                }
            }
#pragma unroll
            for (int i = 0; i < HNB; ++i) col[NBD + h + i] = z[i];
        }
    }
    __syncthreads();
    load_tri(Lob + NBD + (int64_t)NBD * lda, std::integral_constant<int, 32>{});
#pragma unroll
    for (int i = 0; i < NBD; ++i) y[i] = live ? col[NBD + i] : 0.0;
    __syncthreads();
    if (live) solve(col + NBD);
}

// max |l_ij| over the strictly lower triangle of the n x n factor (bit pattern
// of a non-negative double orders like the value)
__global__ void __launch_bounds__(256) lower_absmax(const double *__restrict__ A, int64_t n, int64_t lda,
                                                   unsigned long long *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double m = 0.0;
    for (int64_t j = w; j < n; j += nw)
        for (int64_t i = j + 1 + lane; i < n; i += 32) {
            const double v = fabs(A[i + j * lda]);
            m = v > m || v != v ? (v != v ? 1e300 : v) : m;
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void iota_piv(int64_t *piv, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        piv[i] = i;
}

struct NoPivStreams {
    cudaStream_t hi = nullptr, lo = nullptr;
};

int nopiv_streams(NoPivStreams &st) {
    static PerDevice<NoPivStreams> cache;
    return cache.get(st, [](NoPivStreams &c) {
        int least = 0, greatest = 0;
        LM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        LM_CUDA(cudaStreamCreateWithPriority(&c.hi, cudaStreamNonBlocking, greatest));
        LM_CUDA(cudaStreamCreateWithPriority(&c.lo, cudaStreamNonBlocking, least));
        return 0;
    });
}

// The factorisation proper (A is known column-dominant).  Asynchronous on s.
int nopiv_factor(double *A, int64_t n, int64_t lda, cudaStream_t s) {
    NoPivStreams st;
    if (int rc = nopiv_streams(st)) return rc;
    if (int rc = func_attrs(trsm_right_upper, kTriSmem)) return rc;
    if (int rc = func_attrs(trsm_left_lower_unit, kTriLowSmem)) return rc;
    if (int rc = func_attrs(trsm_left_lower_pair, kTriLowSmem)) return rc;
    cudaEvent_t ev_fork, ev_l21, ev_rest, ev_join, ev_da, ev_ra, ev_db;
    LM_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_l21, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_rest, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_da, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_ra, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_db, cudaEventDisableTiming));
    struct EvGuard {
        cudaEvent_t e[7];
        ~EvGuard() {
            for (auto x : e) cudaEventDestroy(x);
        }
    } guard{{ev_fork, ev_l21, ev_rest, ev_join, ev_da, ev_ra, ev_db}};
    LM_CUDA(cudaEventRecord(ev_fork, s));
    LM_CUDA(cudaStreamWaitEvent(st.hi, ev_fork, 0));
    LM_CUDA(cudaStreamWaitEvent(st.lo, ev_fork, 0));
    // Look-ahead of one block.  Block J's trailing update on lo (columns
    // J2..n) overlaps block J+1's diagonal factor and L21 on hi; hi waits for
    // it only before touching those columns (block J+1's U12 of the next
    // panel and that panel's update).
    // LM_NOPIV_TRACE=1: per-phase device time on each stream (stderr)
    static const bool trace = getenv("LM_NOPIV_TRACE") != nullptr;
    std::vector<cudaEvent_t> evs;
    std::vector<int> tags;  // hi: 0 diag, 1 trsm_ru, 2 trsm_ll, 3 gemm, 4 wait for lo; lo: 6 wait, 7 U12, 8 update
    auto mark = [&](cudaStream_t str, int tag) {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, str);
        evs.push_back(e);
        tags.push_back(tag);
    };
    const auto h0 = std::chrono::steady_clock::now();
    mark(st.hi, -1);
    mark(st.lo, -2);
    // Outer blocks of OB = 2 x 64 columns (rank-128 trailing updates: the DMMA
    // GEMM runs at ~32 TF/s at K = 128, ~12 at K = 64), each factored as two
    // 64-column inner blocks a, b.
    constexpr int OB = 2 * NBD;
    auto trsm_ru = [&](double *A21, int64_t M, const double *U, int nb, cudaStream_t str) -> int {
        if (M <= 0) return 0;
        LM_CUDA(launch_pdl(trsm_right_upper, dim3((unsigned)ceil_div(M, 64)), dim3(64), kTriSmem, str, A21, lda, M, U, nb));
        LM_LAUNCHED(1);
        return 0;
    };
    auto trsm_ll = [&](double *A12, int64_t N, const double *L, int nb, cudaStream_t str) -> int {
        if (N <= 0) return 0;
        LM_CUDA(launch_pdl(trsm_left_lower_unit, dim3((unsigned)ceil_div(N, 64)), dim3(64), kTriLowSmem, str, A12,
                           lda, N, L, nb));
        LM_LAUNCHED(1);
        return 0;
    };
    bool rest_pending = false;
    // opt-in (LM_NOPIV_SPLIT=1): measured slower on config 4a, 28.6 vs 27.9 ms -- the
    // low-priority stream's GEMM work, not the panel chain's wait, bounds the step
    static const bool split_rest = getenv("LM_NOPIV_SPLIT") && getenv("LM_NOPIV_SPLIT")[0] == '1';
    // opt-in (LM_NOPIV_PAIR=1): measured neutral on config 4a (25.59 vs 25.51-25.54 ms)
    static const bool pair_u12 = getenv("LM_NOPIV_PAIR") && getenv("LM_NOPIV_PAIR")[0] == '1';
    // opt-in (LM_NOPIV_EARLY=1): measured neutral on config 4a (25.70 vs 25.71-25.79 ms)
    static const bool early_u12 = getenv("LM_NOPIV_EARLY") && getenv("LM_NOPIV_EARLY")[0] == '1';
    for (int64_t J0 = 0; J0 < n; J0 += OB) {
        const int na = (int)((n - J0) < NBD ? (n - J0) : NBD);
        const int64_t Ja = J0 + na;
        const int nbb = (int)((n - Ja) < NBD ? (n - Ja) : NBD);  // 0 at the very end
        const int64_t J1 = Ja + nbb, J2 = (J1 + OB) < n ? J1 + OB : n;
        const int nob = (int)(J1 - J0);
        double *Aaa = A + J0 + J0 * lda, *Abb = A + Ja + Ja * lda;
        // ---- factor the outer panel (columns J0..J1, rows J0..n) on hi.  The
        // low-priority stream's U12 solves of the remaining columns need only
        // the diagonal factors (and L_ba), not the whole L21: they are issued
        // as soon as those exist, so after ev_l21 only the trailing GEMM is
        // left on that stream (opt-in, LM_NOPIV_EARLY=1; default: all of it after ev_l21).
        const int64_t nn2 = n - J2;
        const bool early = early_u12 && nn2 > 0;
        LM_CUDA(launch_pdl(diag_nopiv, dim3(1), dim3(kDiagThreads), 0, st.hi, Aaa, lda, na));
        LM_LAUNCHED(1);
        mark(st.hi, 0);
        if (early) {
            LM_CUDA(cudaEventRecord(ev_da, st.hi));
            LM_CUDA(cudaStreamWaitEvent(st.lo, ev_da, 0));
            mark(st.lo, 6);
            if (int rc = trsm_ll(A + J0 + J2 * lda, nn2, Aaa, na, st.lo)) return rc;  // U12, rows of block a
            mark(st.lo, 7);
        }
        if (int rc = trsm_ru(A + Ja + J0 * lda, n - Ja, Aaa, na, st.hi)) return rc;  // L of block a, rows below a
        mark(st.hi, 1);
        if (nbb > 0) {
            if (early) {
                LM_CUDA(cudaEventRecord(ev_ra, st.hi));
                LM_CUDA(cudaStreamWaitEvent(st.lo, ev_ra, 0));
                mark(st.lo, 6);
                if (int rc = dgemm_sub(A + Ja + J0 * lda, lda, A + J0 + J2 * lda, lda, A + Ja + J2 * lda, lda, nbb, nn2,
                                       na, st.lo))
                    return rc;
                mark(st.lo, 7);
            }
            if (int rc = trsm_ll(A + J0 + Ja * lda, nbb, Aaa, na, st.hi)) return rc;  // U_ab
            mark(st.hi, 2);
            if (int rc = dgemm_sub(A + Ja + J0 * lda, lda, A + J0 + Ja * lda, lda, Abb, lda, n - Ja, nbb, na, st.hi))
                return rc;
            mark(st.hi, 3);
            LM_CUDA(launch_pdl(diag_nopiv, dim3(1), dim3(kDiagThreads), 0, st.hi, Abb, lda, nbb));
            LM_LAUNCHED(1);
            mark(st.hi, 0);
            if (early) {
                LM_CUDA(cudaEventRecord(ev_db, st.hi));
                LM_CUDA(cudaStreamWaitEvent(st.lo, ev_db, 0));
                mark(st.lo, 6);
                if (int rc = trsm_ll(A + Ja + J2 * lda, nn2, Abb, nbb, st.lo)) return rc;  // U12, rows of block b
                mark(st.lo, 7);
            }
            if (int rc = trsm_ru(A + J1 + Ja * lda, n - J1, Abb, nbb, st.hi)) return rc;  // L of block b
            mark(st.hi, 1);
        }
        LM_CUDA(cudaEventRecord(ev_l21, st.hi));
        if (J1 >= n) break;
        // ---- U12 of the outer block's rows over the columns [c0, c0 + nc), then
        // the rank-nob update of the rows below
        auto u12 = [&](int64_t c0, int64_t nc, cudaStream_t str, bool hi) -> int {
            const bool solved = !hi && early;  // the U12 solves were issued above
            const bool pair = !solved && pair_u12 && na == NBD && nbb == NBD;
            if (pair) {  // both solves and the product between them in one launch
                LM_CUDA(launch_pdl(trsm_left_lower_pair, dim3((unsigned)ceil_div(nc, 64)), dim3(64), kTriLowSmem, str,
                                   A + J0 + c0 * lda, lda, nc, Aaa));
                LM_LAUNCHED(1);
                mark(str, hi ? 2 : 7);
            }
            if (!solved && !pair) {
                if (int rc = trsm_ll(A + J0 + c0 * lda, nc, Aaa, na, str)) return rc;
                mark(str, hi ? 2 : 7);
            }
            if (nbb > 0 && !solved && !pair) {
                if (int rc = dgemm_sub(A + Ja + J0 * lda, lda, A + J0 + c0 * lda, lda, A + Ja + c0 * lda, lda, nbb, nc,
                                       na, str))
                    return rc;
                mark(str, hi ? 3 : 7);
                if (int rc = trsm_ll(A + Ja + c0 * lda, nc, Abb, nbb, str)) return rc;
                mark(str, hi ? 2 : 7);
            }
            // low-priority stream: the next outer panel's columns first, so the
            // panel chain (which waits on ev_rest) does not wait for the whole
            // trailing update
            const int64_t nfirst = (!hi && split_rest && nc > OB) ? OB : nc;
            if (int rc = dgemm_sub(A + J1 + J0 * lda, lda, A + J0 + c0 * lda, lda, A + J1 + c0 * lda, lda, n - J1,
                                   nfirst, nob, str))
                return rc;
            if (!hi) LM_CUDA(cudaEventRecord(ev_rest, str));
            if (nfirst < nc)
                if (int rc = dgemm_sub(A + J1 + J0 * lda, lda, A + J0 + (c0 + nfirst) * lda, lda,
                                       A + J1 + (c0 + nfirst) * lda, lda, n - J1, nc - nfirst, nob, str))
                    return rc;
            mark(str, hi ? 3 : 8);
            return 0;
        };
        // the remaining columns on the low-priority stream (after the previous
        // outer block's, which wrote the same columns)
        // the next outer panel's columns were last written by the first piece
        // of the previous block's trailing update (ev_rest, recorded inside
        // u12): the wait is enqueued before this block's update re-records it
        if (rest_pending) LM_CUDA(cudaStreamWaitEvent(st.hi, ev_rest, 0));
        mark(st.hi, 4);
        if (nn2 > 0) {
            LM_CUDA(cudaStreamWaitEvent(st.lo, ev_l21, 0));
            mark(st.lo, 6);
            if (int rc = u12(J2, nn2, st.lo, false)) return rc;
        }
        if (int rc = u12(J1, J2 - J1, st.hi, true)) return rc;
        rest_pending = nn2 > 0;
    }
    if (trace) {
        const double host_us =
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
        cudaDeviceSynchronize();
        double tot[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, last_hi = 0, last_lo = 0;
        float t;
        for (size_t i = 2; i < evs.size(); ++i) {
            const bool lo = tags[i] >= 5;
            cudaEventElapsedTime(&t, evs[0], evs[i]);
            double &last = lo ? last_lo : last_hi;
            tot[tags[i]] += t - last;
            last = t;
        }
        fprintf(stderr, "NOPIVTRACE host issue %.0f us | hi: diag %.2f ms, trsm_ru %.2f, trsm_ll %.2f, gemm %.2f, "
                        "wait for lo %.2f, end %.2f ms | lo: wait for hi %.2f, U12 solves + small gemm %.2f, "
                        "trailing gemm %.2f, end %.2f ms\n",
                host_us, tot[0], tot[1], tot[2], tot[3], tot[4], last_hi, tot[6], tot[7], tot[8], last_lo);
        for (auto e : evs) cudaEventDestroy(e);
    }
    LM_CUDA(cudaEventRecord(ev_rest, st.lo));  // everything on the low-priority stream
    LM_CUDA(cudaStreamWaitEvent(st.hi, ev_rest, 0));
    LM_CUDA(cudaEventRecord(ev_join, st.hi));
    LM_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    return 0;
}

}  // namespace

bool lu_nopiv_enabled() {
    static const bool on = [] {
        const char *e = getenv("LM_LU_NOPIV");
        return !(e && e[0] == '0');
    }();
    return on;
}

// 0: factored without swaps (piv = identity, *info = 0); 1: not applicable
// (A is not column-dominant, or a multiplier came out too close to 1 and A
// was restored) -- the caller runs the pivoting LU; < 0: error.
// Synchronises s twice (the dominance and the multiplier checks).  orig (may
// be null): an untouched copy of the matrix the caller still holds (leading
// dimension ldo) -- then no backup is made (a 537 MB copy at n = 8192).
int lu_factor_nopiv(double *A, int64_t n, int64_t lda, int64_t *piv, int32_t *info, cudaStream_t s, const double *orig,
                    int64_t ldo) {
    if (n < 2 || !lu_nopiv_enabled()) return 1;
    Scratch flags;
    if (int rc = flags.alloc(16, s)) return rc;
    int *d_flag = flags.as<int>();
    unsigned long long *d_max = reinterpret_cast<unsigned long long *>(flags.as<char>() + 8);
    LM_CUDA(cudaMemsetAsync(flags.p, 0, 16, s));
    coldom_check<<<(unsigned)(4 * num_sms()), 256, 0, s>>>(A, n, lda, d_flag);
    LM_LAUNCHED(1);
    int h_flag = 1;
    LM_CUDA(cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    LM_CUDA(cudaStreamSynchronize(s));
    if (h_flag) return 1;
    Scratch backup;  // the original matrix, in case the multiplier check fails
    if (!orig) {
        if (int rc = backup.alloc(sizeof(double) * (size_t)n * n, s)) return rc;
        LM_CUDA(cudaMemcpy2DAsync(backup.p, n * sizeof(double), A, lda * sizeof(double), n * sizeof(double), n,
                                  cudaMemcpyDeviceToDevice, s));
        orig = backup.as<double>();
        ldo = n;
    }
    if (int rc = nopiv_factor(A, n, lda, s)) return rc;
    lower_absmax<<<(unsigned)(4 * num_sms()), 256, 0, s>>>(A, n, lda, d_max);
    LM_LAUNCHED(1);
    unsigned long long h_max = 0;
    LM_CUDA(cudaMemcpyAsync(&h_max, d_max, sizeof(h_max), cudaMemcpyDeviceToHost, s));
    LM_CUDA(cudaStreamSynchronize(s));
    double mx;
    memcpy(&mx, &h_max, sizeof(mx));
    if (!(mx < kMulBound)) {  // not provably the reference's pivots: restore, let the caller pivot
        LM_CUDA(cudaMemcpy2DAsync(A, lda * sizeof(double), orig, ldo * sizeof(double), n * sizeof(double), n,
                                  cudaMemcpyDeviceToDevice, s));
        return 1;
    }
    iota_piv<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(piv, n);
    LM_LAUNCHED(1);
    LM_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
    return 0;
}

}  // namespace lm
