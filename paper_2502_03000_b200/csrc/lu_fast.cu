// lu_fast.cu -- LU factorisation of large matrices (BASELINE config 4a)
// in the reference's exact operation order, two-level blocked.
//
// Reference: lazymat/_loops.py:200-236 (_lu_factor).  Every element
// A[i,j] receives A[i,j] = A[i,j] - L[i,k]*U[k,j] for k ascending, each
// product and difference rounded (__dmul_rn/__dsub_rn), multipliers
// L[i,k] = A[i,k] / pivot (__ddiv_rn), the pivot is the first maximum of
// |A[i,k]| over the current rows i >= k, full-row swaps.  Any blocking that
// keeps, per element, the update order k ascending performs exactly these
// operations, so values and pivots are bit-identical to the reference.
//
//   outer blocks of ONB = 128 columns (trailing-update K = 128: the A22
//   read/write traffic is n^3/(3*128) * 16 B, 23 GB at n = 8192);
//   inside a block, panels of 32 columns factored by ONE thread-block
//   CLUSTER (up to 16 CTAs of one GPC, lu_panel.cu): every thread keeps one
//   (or two) panel rows in registers; per column the CTA candidates are
//   pushed into every CTA's inbox with st.async + mbarrier transaction
//   counts, with a one-column look-ahead;
//   row swaps of the other columns: one composed permutation per panel
//   (laswp_plan) applied as a gather (laswp_apply);
//   U12: 32-row triangular solves (smem-staged columns, one thread per
//   column) + order-preserving updates;
//   A22: order-preserving SIMT update, 128 x 128 tiles (8 x 8 per thread),
//   smaller tiles when the grid would not cover the machine, next K chunk
//   prefetched into registers.
//
// LM_LU_TRACE=1 prints a per-step timeline of both streams (debugging).
#include <cooperative_groups.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {

// ============================================================================
// order-preserving update  C -= A @ B  (k ascending, or descending if DESC)
// ============================================================================

constexpr int UK = 32;  // K chunk staged per step

// C tile (16*RM) x (16*RN) per CTA of 256 threads (16 x 16), RM x RN
// accumulators per thread; the next K chunk is prefetched into registers
// while the current one is consumed from shared memory.  Large updates use
// 128 x 128 tiles (8 x 8 per thread: 1 LDS per 4 exact MACs); narrow or
// short ones smaller tiles so the grid still covers the machine (a single
// 128 x 128 tile of a 128 x 128 x 128 update is ~35 us on one SM).
template <int RM, int RN, bool DESC, bool SKIP_ZERO>
__global__ void __launch_bounds__(256) exact_update_t(const double *__restrict__ A, int64_t lda,
                                                      const double *__restrict__ B, int64_t ldb, double *C,
                                                      int64_t ldc, int64_t M, int64_t N, int K) {
    constexpr int TM = 16 * RM, TN = 16 * RN;
    constexpr int LA = TM + 1, LB = TN + 1;
    constexpr int FA = TM * UK / 256, FB = TN * UK / 256;  // staged elements per thread
    extern __shared__ double su[];
    double *sA = su;             // [UK][LA]: sA[kk][ii] = A[i0+ii, k]
    double *sB = su + UK * LA;   // [UK][LB]: sB[kk][cc] = B[k, c0+cc]
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = (int64_t)blockIdx.x * TM, c0 = (int64_t)blockIdx.y * TN;
    const int nch = (K + UK - 1) / UK;
    double pa[FA], pb[FB];
    auto fetch = [&](int q) {
        const int k0 = (DESC ? (nch - 1 - q) : q) * UK;
#pragma unroll
        for (int u = 0; u < FA; ++u) {
            const int e = threadIdx.x + 256 * u;
            const int ii = e % TM, kk = e / TM;
            const int64_t i = i0 + ii;
            const int k = k0 + kk;
            pa[u] = (i < M && k < K) ? __ldg(A + i + (int64_t)k * lda) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < FB; ++u) {
            const int e = threadIdx.x + 256 * u;
            const int kb = e % UK, cc = e / UK;
            const int64_t c = c0 + cc;
            pb[u] = (c < N && k0 + kb < K) ? __ldg(B + (k0 + kb) + c * ldb) : 0.0;
        }
    };
    fetch(0);
    double acc[RM][RN];
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int s = 0; s < RN; ++s) {
            const int64_t i = i0 + tx + 16 * r, c = c0 + ty + 16 * s;
            acc[r][s] = (i < M && c < N) ? C[i + c * ldc] : 0.0;
        }
    for (int q = 0; q < nch; ++q) {
        const int k0 = (DESC ? (nch - 1 - q) : q) * UK;
#pragma unroll
        for (int u = 0; u < FA; ++u) {
            const int e = threadIdx.x + 256 * u;
            sA[(e / TM) * LA + e % TM] = pa[u];
        }
#pragma unroll
        for (int u = 0; u < FB; ++u) {
            const int e = threadIdx.x + 256 * u;
            sB[(e % UK) * LB + e / UK] = pb[u];
        }
        __syncthreads();
        if (q + 1 < nch) fetch(q + 1);
        const int kend = (K - k0) < UK ? (K - k0) : UK;
        for (int t = 0; t < kend; ++t) {
            const int kk = DESC ? (kend - 1 - t) : t;
            double av[RM], bv[RN];
#pragma unroll
            for (int r = 0; r < RM; ++r) av[r] = sA[kk * LA + tx + 16 * r];
#pragma unroll
            for (int s = 0; s < RN; ++s) bv[s] = sB[kk * LB + ty + 16 * s];
#pragma unroll
            for (int r = 0; r < RM; ++r)
#pragma unroll
                for (int s = 0; s < RN; ++s)
                    if (!SKIP_ZERO || bv[s] != 0.0) acc[r][s] = __dsub_rn(acc[r][s], __dmul_rn(av[r], bv[s]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int s = 0; s < RN; ++s) {
            const int64_t i = i0 + tx + 16 * r, c = c0 + ty + 16 * s;
            if (i < M && c < N) C[i + c * ldc] = acc[r][s];
        }
}

// cp.async variant (ascending k only, 16-byte aligned operands): the K
// chunks land in shared memory asynchronously (double buffer), so no
// staging registers are held and two CTAs fit per SM (the register-staged
// kernel holds 1: ncu showed 65% of the FP64 pipe, bound by "wait" stalls
// of the dmul -> dsub chains with 8 warps per SM).
__device__ __forceinline__ void cpa16z(void *smem, const void *gmem, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}

template <int RM, int RN>
__global__ void __launch_bounds__(256, 2) exact_update_c(const double *__restrict__ A, int64_t lda,
                                                        const double *__restrict__ B, int64_t ldb, double *C,
                                                        int64_t ldc, int64_t M, int64_t N, int K) {
    constexpr int TM = 16 * RM, TN = 16 * RN;
    constexpr int LA = TM + 2, LB = UK + 2;     // even: 16-byte aligned rows
    constexpr int SA = UK * LA, SB = TN * LB;   // doubles per stage
    constexpr int PA = TM / 2 * UK / 256, PB = TN * UK / 2 / 256;  // 16-byte pieces per thread
    extern __shared__ __align__(16) double su[];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = (int64_t)blockIdx.x * TM, c0 = (int64_t)blockIdx.y * TN;
    const int nch = (K + UK - 1) / UK;
    auto issue = [&](int q) {
        double *sA = su + (q & 1) * (SA + SB);
        double *sB = sA + SA;
        const int k0 = q * UK;
#pragma unroll
        for (int u = 0; u < PA; ++u) {
            const int pz = threadIdx.x + 256 * u;
            const int i2 = pz % (TM / 2), kk = pz / (TM / 2);
            const int64_t i = i0 + 2 * i2;
            const int k = k0 + kk;
            const int bytes = (k < K && i < M) ? (i + 1 < M ? 16 : 8) : 0;
            cpa16z(sA + kk * LA + 2 * i2, bytes ? A + i + (int64_t)k * lda : A, bytes);
        }
#pragma unroll
        for (int u = 0; u < PB; ++u) {
            const int pz = threadIdx.x + 256 * u;
            const int k2 = pz % (UK / 2), cc = pz / (UK / 2);
            const int64_t c = c0 + cc;
            const int k = k0 + 2 * k2;
            const int bytes = (c < N && k < K) ? (k + 1 < K ? 16 : 8) : 0;
            cpa16z(sB + cc * LB + 2 * k2, bytes ? B + k + c * ldb : B, bytes);
        }
        asm volatile("cp.async.commit_group;\n");
    };
    issue(0);
    double acc[RM][RN];
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int s = 0; s < RN; ++s) {
            const int64_t i = i0 + tx + 16 * r, c = c0 + ty + 16 * s;
            acc[r][s] = (i < M && c < N) ? C[i + c * ldc] : 0.0;
        }
    for (int q = 0; q < nch; ++q) {
        if (q + 1 < nch) {
            issue(q + 1);
            asm volatile("cp.async.wait_group 1;\n");
        } else {
            asm volatile("cp.async.wait_group 0;\n");
        }
        __syncthreads();
        const double *sA = su + (q & 1) * (SA + SB);
        const double *sB = sA + SA;
        const int kend = (K - q * UK) < UK ? (K - q * UK) : UK;
        for (int kk = 0; kk < kend; ++kk) {
            double av[RM], bv[RN];
#pragma unroll
            for (int r = 0; r < RM; ++r) av[r] = sA[kk * LA + tx + 16 * r];
#pragma unroll
            for (int s = 0; s < RN; ++s) bv[s] = sB[(ty + 16 * s) * LB + kk];
#pragma unroll
            for (int r = 0; r < RM; ++r)
#pragma unroll
                for (int s = 0; s < RN; ++s) acc[r][s] = __dsub_rn(acc[r][s], __dmul_rn(av[r], bv[s]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
        for (int s = 0; s < RN; ++s) {
            const int64_t i = i0 + tx + 16 * r, c = c0 + ty + 16 * s;
            if (i < M && c < N) C[i + c * ldc] = acc[r][s];
        }
}

template <int RM, int RN>
int launch_exact_update_c(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc,
                          int64_t M, int64_t N, int K, cudaStream_t s) {
    constexpr int TM = 16 * RM, TN = 16 * RN;
    const size_t smem = sizeof(double) * 2 * (UK * (TM + 2) + TN * (UK + 2));
    if (int rc = func_attrs(exact_update_c<RM, RN>, smem)) return rc;
    dim3 grid((unsigned)ceil_div(M, TM), (unsigned)ceil_div(N, TN));
    exact_update_c<RM, RN><<<grid, 256, smem, s>>>(A, lda, B, ldb, C, ldc, M, N, K);
    LM_LAUNCHED(1);
    return 0;
}

template <int RM, int RN, bool DESC, bool SKIP_ZERO>
int launch_exact_update(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc, int64_t M,
                        int64_t N, int K, cudaStream_t s) {
    constexpr int TM = 16 * RM, TN = 16 * RN;
    const size_t smem = sizeof(double) * UK * (TM + 1 + TN + 1);
    if (int rc = func_attrs(exact_update_t<RM, RN, DESC, SKIP_ZERO>, smem)) return rc;
    dim3 grid((unsigned)ceil_div(M, TM), (unsigned)ceil_div(N, TN));
    exact_update_t<RM, RN, DESC, SKIP_ZERO><<<grid, 256, smem, s>>>(A, lda, B, ldb, C, ldc, M, N, K);
    LM_LAUNCHED(1);
    return 0;
}

// Tile choice: the largest tile whose grid still gives every SM work
// (>= 148 CTAs), else the one with the most CTAs.  short_ctas (the
// look-ahead stream's trailing update): 128 x 64 tiles, half as long-lived
// as 128 x 128, so SMs free up sooner for the high-priority panel cluster
// (16 free SMs of one GPC) -- 49.4 -> 47.4 ms for the n = 8192 factorisation.
template <bool DESC, bool SKIP_ZERO>
int exact_update(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc, int64_t M,
                 int64_t N, int K, cudaStream_t s, bool short_ctas = false) {
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    const int64_t nsm = num_sms();
    auto ctas = [&](int tm, int tn) { return ceil_div(M, tm) * ceil_div(N, tn); };
    const bool async_ok = !DESC && !SKIP_ZERO && ((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0 &&
                          lda % 2 == 0 && ldb % 2 == 0;
    if (async_ok && N > 32 && ctas(128, 64) >= nsm)  // 45.7 -> 44.0 ms at n = 8192
        return launch_exact_update_c<8, 4>(A, lda, B, ldb, C, ldc, M, N, K, s);
    if (async_ok && N > 32 && ctas(64, 64) >= nsm)
        return launch_exact_update_c<4, 4>(A, lda, B, ldb, C, ldc, M, N, K, s);
    if (short_ctas && N > 32 && ctas(128, 64) >= nsm)
        return launch_exact_update<8, 4, DESC, SKIP_ZERO>(A, lda, B, ldb, C, ldc, M, N, K, s);
    if (ctas(128, 128) >= nsm)
        return launch_exact_update<8, 8, DESC, SKIP_ZERO>(A, lda, B, ldb, C, ldc, M, N, K, s);
    if (N > 32 && ctas(64, 64) >= nsm)
        return launch_exact_update<4, 4, DESC, SKIP_ZERO>(A, lda, B, ldb, C, ldc, M, N, K, s);
    if (ctas(64, 32) >= nsm || M > 2048)
        return launch_exact_update<4, 2, DESC, SKIP_ZERO>(A, lda, B, ldb, C, ldc, M, N, K, s);
    return launch_exact_update<2, 2, DESC, SKIP_ZERO>(A, lda, B, ldb, C, ldc, M, N, K, s);
}

template int exact_update<false, false>(const double *, int64_t, const double *, int64_t, double *, int64_t,
                                        int64_t, int64_t, int, cudaStream_t, bool);
template int exact_update<true, false>(const double *, int64_t, const double *, int64_t, double *, int64_t,
                                       int64_t, int64_t, int, cudaStream_t, bool);

// ============================================================================
// triangular solve on up to 32 rows: columns staged through shared
// memory (coalesced), one thread per column solves from registers
// ============================================================================

constexpr int TC = 64;  // columns per CTA

template <bool LOWER>
__global__ void __launch_bounds__(TC) tri_cols(const double *__restrict__ T, int64_t ldt, double *X, int64_t ldx,
                                               int nb, int64_t ncols) {
    __shared__ double sT[32][33];  // sT[i][j] = T[i,j]
    __shared__ double sX[TC][33];  // sX[c][i] = X[i, col0 + c]
    const int64_t col0 = (int64_t)blockIdx.x * TC;
    const int ncl = (int)((ncols - col0) < TC ? (ncols - col0) : TC);
    for (int e = threadIdx.x; e < nb * nb; e += TC) {
        const int i = e % nb, j = e / nb;
        sT[i][j] = T[i + (int64_t)j * ldt];
    }
    for (int e = threadIdx.x; e < nb * ncl; e += TC) {
        const int i = e % nb, c = e / nb;
        sX[c][i] = X[i + (col0 + c) * ldx];
    }
    __syncthreads();
    const int c = threadIdx.x;
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = (i < nb && c < ncl) ? sX[c][i] : 0.0;
    if (LOWER) {  // unit lower, forward: x_i -= T[i,j] x_j, j ascending
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j >= nb) break;
            const double xj = x[j];
#pragma unroll
            for (int i = j + 1; i < 32; ++i)
                if (i < nb) x[i] = __dsub_rn(x[i], __dmul_rn(sT[i][j], xj));
        }
    } else {  // upper, backward: x_j /= T[j,j]; x_i -= T[i,j] x_j, j descending
#pragma unroll
        for (int j = 31; j >= 0; --j) {
            if (j >= nb) continue;
            x[j] = __ddiv_rn(x[j], sT[j][j]);
            const double xj = x[j];
#pragma unroll
            for (int i = 0; i < j; ++i) x[i] = __dsub_rn(x[i], __dmul_rn(sT[i][j], xj));
        }
    }
    if (c < ncl)
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (i < nb) sX[c][i] = x[i];
    __syncthreads();
    for (int e = threadIdx.x; e < nb * ncl; e += TC) {
        const int i = e % nb, cc = e / nb;
        X[i + (col0 + cc) * ldx] = sX[cc][i];
    }
}

template <bool LOWER>
int tri32(const double *T, int64_t ldt, double *X, int64_t ldx, int nb, int64_t ncols, cudaStream_t s) {
    if (nb <= 0 || ncols <= 0) return 0;
    tri_cols<LOWER><<<(unsigned)ceil_div(ncols, TC), TC, 0, s>>>(T, ldt, X, ldx, nb, ncols);
    LM_LAUNCHED(1);
    return 0;
}
template int tri32<true>(const double *, int64_t, double *, int64_t, int, int64_t, cudaStream_t);
template int tri32<false>(const double *, int64_t, double *, int64_t, int, int64_t, cudaStream_t);

// ============================================================================
// row swaps of whole column ranges: compose, then gather
// ============================================================================

// list[0] = count, then (dst, src) pairs: final row dst takes old row src,
// for the sequential swaps piv[k0 .. k0+cnt) over rows [k0, n).
__global__ void __launch_bounds__(1024) laswp_plan(const int64_t *__restrict__ piv, int64_t k0, int cnt, int64_t n,
                                                   int32_t *list) {
    extern __shared__ int32_t content[];  // content[r - k0] = original row now at r
    __shared__ int count;
    const int64_t h = n - k0;
    for (int64_t r = threadIdx.x; r < h; r += blockDim.x) content[r] = (int32_t)(k0 + r);
    if (threadIdx.x == 0) count = 0;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int q = 0; q < cnt; ++q) {
            const int64_t k = k0 + q, p = piv[k];
            if (p != k) {
                const int32_t t = content[k - k0];
                content[k - k0] = content[p - k0];
                content[p - k0] = t;
            }
        }
    __syncthreads();
    for (int64_t r = threadIdx.x; r < h; r += blockDim.x)
        if (content[r] != (int32_t)(k0 + r)) {
            const int slot = atomicAdd(&count, 1);
            list[1 + 2 * slot] = (int32_t)(k0 + r);
            list[2 + 2 * slot] = content[r];
        }
    __syncthreads();
    if (threadIdx.x == 0) list[0] = count;
}

// one CTA per column; columns [a0, a1) then [b0, ...)
__global__ void __launch_bounds__(256) laswp_apply(double *A, int64_t lda, const int32_t *__restrict__ list, int64_t a0,
                                                   int64_t a1, int64_t b0) {
    __shared__ double v[512];
    const int cnt = list[0];
    if (cnt == 0) return;
    const int64_t na = a1 - a0;
    const int64_t col = blockIdx.x < na ? a0 + blockIdx.x : b0 + (blockIdx.x - na);
    double *x = A + col * lda;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) v[q] = x[list[2 + 2 * q]];
    __syncthreads();
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) x[list[1 + 2 * q]] = v[q];
}

// the 32-column panel (lu_panel.cu)
constexpr int PNB = 32;
bool panel_shape(int64_t h, int &cs, int &rp, int &R);
int launch_panel_cluster(double *A, int64_t lda, int64_t n, int64_t j0, int nb, int64_t *piv, int32_t *info,
                         cudaStream_t s, long long *dbg = nullptr, int64_t J0 = 0, int64_t J1 = 0);

int dgemm_sub(const double *a, int64_t lda, const double *b, int64_t ldb, double *c, int64_t ldc, int64_t M,
              int64_t N, int64_t K, cudaStream_t s);

// C -= A B: exact reference order (separately rounded multiply and subtract,
// k ascending -- bit-identical to _lu_factor) or, in tensor mode, DMMA with
// FMA accumulation (scaled residual within 1e-10, not bitwise).
static int trailing_update(bool tensor, const double *A, int64_t lda, const double *B, int64_t ldb, double *C,
                           int64_t ldc, int64_t M, int64_t N, int K, cudaStream_t s, bool short_ctas = false) {
    if (tensor) return dgemm_sub(A, lda, B, ldb, C, ldc, M, N, K, s);
    return exact_update<false, false>(A, lda, B, ldb, C, ldc, M, N, K, s, short_ctas);
}

// rows [k0, k0+cnt) pivots applied to columns [a0, a1) U [b0, b1)
static int laswp(double *A, int64_t lda, int64_t n, const int64_t *piv, int64_t k0, int cnt, int64_t a0, int64_t a1,
                 int64_t b0, int64_t b1, int32_t *list, cudaStream_t s) {
    const int64_t ncols = (a1 - a0) + (b1 - b0);
    if (ncols <= 0 || cnt <= 0) return 0;
    const size_t sm = sizeof(int32_t) * (size_t)(n - k0);
    LM_REQUIRE(sm <= 200 * 1024, "laswp: n too large");
    if (sm > 48 * 1024)
        if (int rc = func_attrs(laswp_plan, sm)) return rc;
    laswp_plan<<<1, 1024, sm, s>>>(piv, k0, cnt, n, list);
    LM_LAUNCHED(1);
    laswp_apply<<<(unsigned)ncols, 256, 0, s>>>(A, lda, list, a0, a1, b0);
    LM_LAUNCHED(1);
    return 0;
}

constexpr int ONB = 128;  // outer block

// U12 = L11^{-1} A12 and A22 -= L21 U12 for the columns [c0, c1) to the
// right of outer block [J0, J1) (32-row triangular blocks, order-preserving)
static int block_right(bool tensor, double *A, int64_t lda, int64_t n, int64_t J0, int64_t J1, int64_t c0,
                       int64_t c1, cudaStream_t s, bool short_ctas = false) {
    if (c1 <= c0) return 0;
    const int64_t nc = c1 - c0;
    for (int64_t b0 = J0; b0 < J1; b0 += PNB) {
        const int nbb = (int)((J1 - b0) < PNB ? (J1 - b0) : PNB);
        if (int rc = tri32<true>(A + b0 + b0 * lda, lda, A + b0 + c0 * lda, lda, nbb, nc, s)) return rc;
        if (b0 + nbb < J1)
            if (int rc = trailing_update(tensor, A + (b0 + nbb) + b0 * lda, lda, A + b0 + c0 * lda, lda,
                                         A + (b0 + nbb) + c0 * lda, lda, J1 - (b0 + nbb), nc, nbb, s))
                return rc;
    }
    return trailing_update(tensor, A + J1 + J0 * lda, lda, A + J0 + c0 * lda, lda, A + J1 + c0 * lda, lda, n - J1, nc,
                           (int)(J1 - J0), s, short_ctas);
}

struct LuStreams {
    cudaStream_t hi = nullptr, lo = nullptr;  // panel chain (high priority), look-ahead remainder
};

static int lu_streams(LuStreams &st) {
    static PerDevice<LuStreams> cache;
    return cache.get(st, [](LuStreams &c) {
        int least = 0, greatest = 0;
        LM_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        LM_CUDA(cudaStreamCreateWithPriority(&c.hi, cudaStreamNonBlocking, greatest));
        LM_CUDA(cudaStreamCreateWithPriority(&c.lo, cudaStreamNonBlocking, least));
        return 0;
    });
}

// Returns 1 (and does nothing) when the cluster panel is not usable for
// this n, so the caller can take the cooperative-grid path.
//
// Look-ahead: the panels of block J+1 (critical path, high-priority
// stream) run while the trailing update of block J's remainder (columns
// beyond J+1, low-priority stream) is still in flight; the only join is
// before block J+1's outer row swaps, which touch those columns.
// Debug timeline (LM_LU_TRACE=1): timing events after every step on both
// streams, printed to stderr as "stream label start_us end_us".
struct LuTrace {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, std::string>> ev[2];
    cudaEvent_t t0 = nullptr;
    std::chrono::steady_clock::time_point h0;
    void begin(cudaStream_t s) {
        on = getenv("LM_LU_TRACE") != nullptr;
        if (!on) return;
        h0 = std::chrono::steady_clock::now();
        cudaEventCreate(&t0);
        cudaEventRecord(t0, s);
    }
    void mark(int which, cudaStream_t s, const std::string &label) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev[which].push_back({e, label});
    }
    void dump() {
        if (!on) return;
        const double host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
        cudaDeviceSynchronize();
        fprintf(stderr, "LUTRACE host issue %.1f us\n", host_us);
        for (int w = 0; w < 2; ++w) {
            float prev = 0.f;
            for (auto &x : ev[w]) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, t0, x.first);
                fprintf(stderr, "LUTRACE %s %-28s end %10.1f us  (+%8.1f)\n", w ? "lo" : "hi", x.second.c_str(),
                        ms * 1e3, (ms - prev) * 1e3);
                prev = ms;
                cudaEventDestroy(x.first);
            }
        }
        cudaEventDestroy(t0);
    }
};

int lu_factor_fast(double *A, int64_t n, int64_t lda, int64_t *piv, int32_t *info, cudaStream_t s, bool tensor) {
    int cs = 0, rp = 0, R = 0;
    if (n >= (1ll << 31) || !panel_shape(n, cs, rp, R) || sizeof(int32_t) * (size_t)n > 200 * 1024) return 1;
    Scratch list;
    if (int rc = list.alloc(sizeof(int32_t) * (1 + 4 * ONB + 8), s)) return rc;
    int32_t *lp = list.as<int32_t>();
    LuStreams st;
    if (int rc = lu_streams(st)) return rc;
    cudaEvent_t ev_fork, ev_swapped, ev_rest, ev_join;
    LM_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_swapped, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_rest, cudaEventDisableTiming));
    LM_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    struct EvGuard {
        cudaEvent_t e[4];
        ~EvGuard() {
            for (auto x : e) cudaEventDestroy(x);
        }
    } guard{{ev_fork, ev_swapped, ev_rest, ev_join}};
    LM_CUDA(cudaEventRecord(ev_fork, s));
    LM_CUDA(cudaStreamWaitEvent(st.hi, ev_fork, 0));
    LM_CUDA(cudaStreamWaitEvent(st.lo, ev_fork, 0));
    cudaStream_t m = st.hi;
    bool rest_pending = false;
    LuTrace tr;
    tr.begin(s);
    for (int64_t J0 = 0; J0 < n; J0 += ONB) {
        const int NBJ = (int)((n - J0) < ONB ? (n - J0) : ONB);
        const int64_t J1 = J0 + NBJ;
        for (int64_t j0 = J0; j0 < J1; j0 += PNB) {
            const int nb = (int)((J1 - j0) < PNB ? (J1 - j0) : PNB);
            // the panel kernel also applies its swaps to the rest of the
            // outer block and solves U12 for the block's remaining columns
            if (int rc = launch_panel_cluster(A, lda, n, j0, nb, piv, info, m, nullptr, J0, J1)) return rc;
            tr.mark(0, m, "panel " + std::to_string(j0));
            const int64_t rest = J1 - (j0 + nb);
            if (rest > 0) {
                if (int rc = trailing_update(tensor, A + (j0 + nb) + j0 * lda, lda, A + j0 + (j0 + nb) * lda, lda,
                                             A + (j0 + nb) + (j0 + nb) * lda, lda, n - (j0 + nb), rest, nb, m))
                    return rc;
                tr.mark(0, m, "inner upd " + std::to_string(j0));
            }
        }
        // join the previous block's look-ahead remainder before the outer
        // swaps (they permute its columns and the L21 it reads)
        tr.mark(0, m, "chain done " + std::to_string(J0));
        if (rest_pending) LM_CUDA(cudaStreamWaitEvent(m, ev_rest, 0));
        rest_pending = false;
        if (int rc = laswp(A, lda, n, piv, J0, NBJ, 0, J0, J1, n, lp, m)) return rc;
        tr.mark(0, m, "outer swaps " + std::to_string(J0));
        if (J1 < n) {
            const int64_t J2 = (J1 + ONB) < n ? (J1 + ONB) : n;
            if (J2 < n) {
                LM_CUDA(cudaEventRecord(ev_swapped, m));
                LM_CUDA(cudaStreamWaitEvent(st.lo, ev_swapped, 0));
                // (one kernel per step: column-chunked remainders free SMs for the
                // panel cluster sooner but lose more in the update tails --
                // measured 51 ms at one chunk vs 55-121 ms at 2048-256 columns)
                if (int rc = block_right(tensor, A, lda, n, J0, J1, J2, n, st.lo, true)) return rc;
                tr.mark(1, st.lo, "remainder " + std::to_string(J0));
                LM_CUDA(cudaEventRecord(ev_rest, st.lo));
                rest_pending = true;
            }
            if (int rc = block_right(tensor, A, lda, n, J0, J1, J1, J2, m)) return rc;  // the next block first
            tr.mark(0, m, "next block " + std::to_string(J0));
        }
    }
    if (rest_pending) LM_CUDA(cudaStreamWaitEvent(m, ev_rest, 0));
    LM_CUDA(cudaEventRecord(ev_join, m));
    LM_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
    tr.dump();
    return 0;
}

}  // namespace lm
