// lu.cu -- R9/R10 solve family on the GPU, in the reference's EXACT
// operation order.
//
//  lm_lu_factor   <- _loops.py:200-236 (_lu_factor: right-looking getf2,
//                    strict-> pivot search, full-row swaps)
//  lm_lu_solve    <- _loops.py:239-259 (_lu_solve_inplace)
//  lm_tri_solve   <- _loops.py:363-388 (_tri_solve_inplace)
//  lm_band_solve  <- _loops.py:262-360 (_pack_band/_band_factor/_band_solve_inplace)
//  lm_lu_solve_batched: per-instance _lu_factor + _lu_solve_inplace
//
// Blocked, but bit-identical: every element A[i,j] of the reference
// receives its updates A[i,j] = A[i,j] - L[i,k]*U[k,j] one at a time in
// ascending k with the product and the difference each rounded
// (__dmul_rn / __dsub_rn, no FMA).  A right-looking blocked LU applies the
// same updates to the same values in the same order -- the panel in
// shared memory, U12 by an order-preserving triangular solve, A22 by an
// order-preserving "GEMM" -- and row swaps are pure permutations, so the
// pivots (and every value) equal the reference's on ANY matrix, not just
// diagonally dominant ones.  Cost: a multiply-add is 2 FP64 instructions
// (DMUL + DADD) instead of one DFMA.
//
// Panel: a cooperative kernel, one CTA per SM, each CTA holding a slice
// of the panel rows in shared memory; one grid-wide barrier per column
// (candidates and candidate rows are published to a double-buffered
// exchange area before the barrier, so the winner's row never needs a
// second round trip).  Row swaps of the columns outside the panel are
// done in the same step by all CTAs (the LAPACK laswp, fused).
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {

constexpr int kPanelThreads = 256;

struct PanelArgs {
    double *A;
    int64_t lda, n, j0;
    int nb, rp, P;
    int64_t *piv;
    int32_t *info;
    double *pub;  // [2][P][2 + nb]  (value, row-as-double, row values)
    double *pubk; // [2][nb]
};

// key for pivot candidates: larger |v| wins, ties -> lower row; NaN never
// wins unless it sits on the diagonal row k (the sequential loop starts
// from best = |A[k,k]| and only replaces on a strict >).
__device__ __forceinline__ bool better(double va, int64_t ia, double vb, int64_t ib) {
    if (ia < 0) return false;
    if (ib < 0) return true;
    if (va > vb) return true;
    if (va == vb) return ia < ib;
    return false;
}

__global__ void __launch_bounds__(kPanelThreads) lu_panel(PanelArgs a) {
    extern __shared__ double sm[];
    cg::grid_group grid = cg::this_grid();
    const int nb = a.nb, ld = nb + 1;
    double *sP = sm;                       // [rp][nb+1]
    double *sU = sP + (int64_t)a.rp * ld;  // [nb] pivot row
    __shared__ double redv[kPanelThreads / 32];
    __shared__ int64_t redi[kPanelThreads / 32];
    __shared__ int64_t s_p;
    __shared__ int s_w;

    const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t rbeg = a.j0 + (int64_t)c * a.rp;
    int64_t rend = rbeg + a.rp;
    if (rend > a.n) rend = a.n;
    const int nrow = rend > rbeg ? (int)(rend - rbeg) : 0;
    const int64_t gtid = (int64_t)c * kPanelThreads + tid, gth = (int64_t)a.P * kPanelThreads;
    const int64_t outside = a.n - nb;  // columns not in the panel

    for (int e = tid; e < nrow * nb; e += kPanelThreads) {
        const int r = e % nrow, j = e / nrow;
        sP[r * ld + j] = a.A[(rbeg + r) + (a.j0 + j) * a.lda];
    }
    __syncthreads();

    for (int kk = 0; kk < nb; ++kk) {
        const int64_t k = a.j0 + kk;
        const int par = kk & 1;
        double *pub = a.pub + (int64_t)par * a.P * (2 + nb);
        double *pubk = a.pubk + (int64_t)par * nb;
        // 1. local candidate over owned rows >= k
        double bv = -1.0;
        int64_t bi = -1;
        for (int r = tid; r < nrow; r += kPanelThreads) {
            const int64_t row = rbeg + r;
            if (row < k) continue;
            const double x = sP[r * ld + kk];
            double v = fabs(x);
            if (v != v) {
                if (row != k) continue;  // NaN off the diagonal never wins
                v = __longlong_as_double(0x7ff0000000000000LL);  // +inf: diagonal NaN keeps p = k
            }
            if (better(v, row, bv, bi)) {
                bv = v;
                bi = row;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (better(ov, oi, bv, bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            redv[wid] = bv;
            redi[wid] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < kPanelThreads / 32; ++w)
                if (better(redv[w], redi[w], bv, bi)) {
                    bv = redv[w];
                    bi = redi[w];
                }
            redv[0] = bv;
            redi[0] = bi;
            double *slot = pub + (int64_t)c * (2 + nb);
            slot[0] = bv;
            slot[1] = (double)bi;
        }
        __syncthreads();
        bi = redi[0];
        // publish candidate row and (if owned) row k
        if (bi >= 0)
            for (int j = tid; j < nb; j += kPanelThreads) pub[(int64_t)c * (2 + nb) + 2 + j] = sP[(bi - rbeg) * ld + j];
        if (k >= rbeg && k < rend)
            for (int j = tid; j < nb; j += kPanelThreads) pubk[j] = sP[(k - rbeg) * ld + j];
        grid.sync();

        // 2. global winner (every CTA computes the same answer)
        if (wid == 0) {
            double gv = -1.0;
            int64_t gi = -1;
            int gw = -1;
            for (int w = lane; w < a.P; w += 32) {
                const double v = pub[(int64_t)w * (2 + nb)];
                const int64_t i = (int64_t)pub[(int64_t)w * (2 + nb) + 1];
                if (better(v, i, gv, gi)) {
                    gv = v;
                    gi = i;
                    gw = w;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, gv, o);
                const int64_t oi = __shfl_xor_sync(0xffffffffu, gi, o);
                const int ow = __shfl_xor_sync(0xffffffffu, gw, o);
                if (better(ov, oi, gv, gi)) {
                    gv = ov;
                    gi = oi;
                    gw = ow;
                }
            }
            if (lane == 0) {
                s_p = gi;
                s_w = gw;
            }
        }
        __syncthreads();
        const int64_t p = s_p;
        const int w = s_w;
        for (int j = tid; j < nb; j += kPanelThreads) sU[j] = pub[(int64_t)w * (2 + nb) + 2 + j];
        __syncthreads();
        if (c == 0 && tid == 0) {
            a.piv[k] = p;
            if (sU[kk] == 0.0 && *a.info == 0) *a.info = (int32_t)(k + 1);
        }
        // 3. swaps: panel slice rows, then the outside columns (laswp)
        if (p != k) {
            if (p >= rbeg && p < rend)
                for (int j = tid; j < nb; j += kPanelThreads) sP[(p - rbeg) * ld + j] = pubk[j];
            if (k >= rbeg && k < rend)
                for (int j = tid; j < nb; j += kPanelThreads) sP[(k - rbeg) * ld + j] = sU[j];
            for (int64_t t = gtid; t < outside; t += gth) {
                const int64_t col = t < a.j0 ? t : t + nb;
                double *x = a.A + col * a.lda;
                const double u = x[k], v = x[p];
                x[k] = v;
                x[p] = u;
            }
        }
        __syncthreads();
        // 4. multipliers, then the rank-1 update of the panel columns
        const double pv = sU[kk];
        for (int r = tid; r < nrow; r += kPanelThreads)
            if (rbeg + r > k) sP[r * ld + kk] = rdiv(sP[r * ld + kk], pv);
        __syncthreads();
        const int ncol = nb - kk - 1;
        if (ncol > 0)
            for (int e = tid; e < nrow * ncol; e += kPanelThreads) {
                const int r = e % nrow, j = kk + 1 + e / nrow;
                if (rbeg + r > k) sP[r * ld + j] = rsub(sP[r * ld + j], rmul(sP[r * ld + kk], sU[j]));
            }
        __syncthreads();
    }
    for (int e = tid; e < nrow * nb; e += kPanelThreads) {
        const int r = e % nrow, j = e / nrow;
        a.A[(rbeg + r) + (a.j0 + j) * a.lda] = sP[r * ld + j];
    }
}

// Order-preserving triangular block solve on columns of X.
//   LOWER (unit diagonal, forward):  for j asc: xj = X[j]; X[i] -= T[i,j]*xj, i > j
//   UPPER (backward):  for j desc: X[j] /= T[j,j]; xj = X[j]; X[i] -= T[i,j]*xj, i < j
// SKIP_ZERO reproduces _tri_solve_inplace's `if xj != 0.0` guard.
// One CTA = nbj rows x CPB columns; T (nbj x nbj) staged in smem.
template <bool LOWER, bool SKIP_ZERO, int CPB>
__global__ void trsm_block(const double *__restrict__ T, int64_t ldt, double *X, int64_t ldx, int nbj, int64_t ncols,
                           int32_t *info) {
    extern __shared__ double sm[];
    double *sT = sm;                           // [nbj][nbj+1] (row i, col j) -> sT[j*(nbj+1) + i]
    double *sx = sT + (int64_t)nbj * (nbj + 1);  // [CPB]
    const int i = threadIdx.x % nbj;         // row within block
    const int cl = threadIdx.x / nbj;        // column within CTA
    const int64_t col = (int64_t)blockIdx.x * CPB + cl;
    for (int e = threadIdx.x; e < nbj * nbj; e += blockDim.x) {
        const int r = e % nbj, jj = e / nbj;
        sT[jj * (nbj + 1) + r] = T[r + jj * ldt];
    }
    const bool active = cl < CPB && col < ncols;
    double x = active ? X[i + col * ldx] : 0.0;
    __syncthreads();
    if (LOWER) {
        for (int j = 0; j < nbj; ++j) {
            if (active && i == j) sx[cl] = x;
            __syncthreads();
            const double xj = sx[cl];
            if (active && i > j && (!SKIP_ZERO || xj != 0.0)) x = rsub(x, rmul(sT[j * (nbj + 1) + i], xj));
            __syncthreads();
        }
    } else {
        for (int j = nbj - 1; j >= 0; --j) {
            if (active && i == j) {
                x = rdiv(x, sT[j * (nbj + 1) + j]);
                sx[cl] = x;
            }
            __syncthreads();
            const double xj = sx[cl];
            if (active && i < j && (!SKIP_ZERO || xj != 0.0)) x = rsub(x, rmul(sT[j * (nbj + 1) + i], xj));
            __syncthreads();
        }
    }
    if (active) X[i + col * ldx] = x;
}

// Order-preserving update  C[i,c] = C[i,c] - sum_k A[i,k]*B[k,c]  with the
// k sum applied term by term (ascending, or descending if DESC), each
// product and difference rounded.  64 x 64 output tile per CTA, 256
// threads, 4 x 4 register tile per thread (rows tx + 16*r, cols ty*4+s).
constexpr int kUpT = 64, kUpK = 16;
template <bool DESC, bool SKIP_ZERO>
__global__ void __launch_bounds__(256) exact_update(const double *__restrict__ A, int64_t lda,
                                                    const double *__restrict__ B, int64_t ldb, double *C, int64_t ldc,
                                                    int64_t M, int64_t N, int K) {
    __shared__ double sA[kUpK][kUpT + 1];  // sA[k][i]
    __shared__ double sB[kUpK][kUpT + 1];  // sB[k][c]
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = (int64_t)blockIdx.x * kUpT, c0 = (int64_t)blockIdx.y * kUpT;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int64_t i = i0 + tx + 16 * r, cc = c0 + ty * 4 + s;
            acc[r][s] = (i < M && cc < N) ? C[i + cc * ldc] : 0.0;
        }
    for (int kc = 0; kc < K; kc += kUpK) {
        // stage A[i0.., kc..] and B[kc.., c0..]  (chunk order follows DESC)
        const int kbase = DESC ? (K - kc - kUpK) : kc;
        for (int e = threadIdx.x; e < kUpK * kUpT; e += 256) {
            const int ii = e % kUpT, kk = e / kUpT;
            const int k = kbase + kk;
            const int64_t i = i0 + ii;
            sA[kk][ii] = (k >= 0 && k < K && i < M) ? A[i + (int64_t)k * lda] : 0.0;
        }
        for (int e = threadIdx.x; e < kUpK * kUpT; e += 256) {
            const int kk = e % kUpK, cc = e / kUpK;
            const int k = kbase + kk;
            const int64_t col = c0 + cc;
            sB[kk][cc] = (k >= 0 && k < K && col < N) ? B[k + col * ldb] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int q = 0; q < kUpK; ++q) {
            const int kk = DESC ? (kUpK - 1 - q) : q;
            const int k = kbase + kk;
            if (k < 0 || k >= K) continue;
            double av[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) av[r] = sA[kk][tx + 16 * r];
#pragma unroll
            for (int s = 0; s < 4; ++s) bv[s] = sB[kk][ty * 4 + s];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    if (!SKIP_ZERO || bv[s] != 0.0) acc[r][s] = rsub(acc[r][s], rmul(av[r], bv[s]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int64_t i = i0 + tx + 16 * r, cc = c0 + ty * 4 + s;
            if (i < M && cc < N) C[i + cc * ldc] = acc[r][s];
        }
}

template <bool DESC, bool SKIP_ZERO>
int launch_update(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc, int64_t M,
                  int64_t N, int K, cudaStream_t s) {
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    dim3 grid((unsigned)ceil_div(M, kUpT), (unsigned)ceil_div(N, kUpT));
    exact_update<DESC, SKIP_ZERO><<<grid, 256, 0, s>>>(A, lda, B, ldb, C, ldc, M, N, K);
    LM_LAUNCHED(1);
    return 0;
}

template <bool LOWER, bool SKIP_ZERO>
int launch_trsm(const double *T, int64_t ldt, double *X, int64_t ldx, int nbj, int64_t ncols, cudaStream_t s) {
    if (nbj <= 0 || ncols <= 0) return 0;
    constexpr int CPB = 4;
    const size_t smem = sizeof(double) * ((size_t)nbj * (nbj + 1) + CPB);
    if (smem > 48 * 1024)
        if (int rc = func_attrs(trsm_block<LOWER, SKIP_ZERO, CPB>, smem)) return rc;
    trsm_block<LOWER, SKIP_ZERO, CPB><<<(unsigned)ceil_div(ncols, CPB), nbj * CPB, smem, s>>>(T, ldt, X, ldx, nbj, ncols,
                                                                                           nullptr);
    LM_LAUNCHED(1);
    return 0;
}

constexpr int kLuNb = 64;

int lu_factor_fast(double *A, int64_t n, int64_t lda, int64_t *piv, int32_t *info, cudaStream_t s, bool tensor);
int lu_factor_nopiv(double *A, int64_t n, int64_t lda, int64_t *piv, int32_t *info, cudaStream_t s, const double *orig,
                    int64_t ldo);
int lu_solve_wavefront(const double *LU, int64_t n, int64_t lda, double *X, int64_t ldx, int64_t m, cudaStream_t s,
                       const int *only_if);
int lu_solve_tensor(const double *LU, int64_t n, int64_t lda, double *X, int64_t ldx, int64_t m, cudaStream_t s);
template <bool DESC, bool SKIP_ZERO>
int exact_update(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc, int64_t M,
                 int64_t N, int K, cudaStream_t s, bool short_ctas = false);
template <bool LOWER>
int tri32(const double *T, int64_t ldt, double *X, int64_t ldx, int nb, int64_t ncols, cudaStream_t s);

// Trailing-update arithmetic of the blocked LU (lm_lu_factor_mode):
// exact reference order below LU_TENSOR_MIN_N (values and pivots bitwise equal
// to _lu_factor, what the reference-generated goldens pin), the FP64 tensor
// cores (DMMA, FMA accumulation) from there on, where the north star asks a
// scaled residual <= 1e-10 and the same pivot indices.  LM_LU_MODE=exact /
// tensor overrides the automatic choice.
constexpr int64_t LU_TENSOR_MIN_N = 2048;
static bool lu_tensor_mode(int mode, int64_t n) {
    if (mode == LM_LU_EXACT) return false;
    if (mode == LM_LU_TENSOR) return true;
    static const int env = [] {
        const char *e = getenv("LM_LU_MODE");
        if (!e) return 0;
        return e[0] == 'e' ? 1 : e[0] == 't' ? 2 : 0;
    }();
    if (env) return env == 2;
    return n >= LU_TENSOR_MIN_N;
}

int lu_factor_impl(double *A, int64_t n, int64_t lda, int64_t *piv, int32_t *info, cudaStream_t s, int mode,
                   const double *orig = nullptr, int64_t ldo = 0) {
    LM_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
    if (n == 0) return 0;
    // two-level blocked LU with a thread-block-cluster panel (lu_fast.cu);
    // returns 1 when the panel does not fit a cluster -> cooperative path
    // (exact order only)
    const bool tensor = lu_tensor_mode(mode, n);
    // tensor mode, column diagonally dominant A: partial pivoting provably
    // never swaps -> the pivot-free, all-GEMM factorisation (lu_nopiv.cu)
    if (tensor)
        if (int rc = lu_factor_nopiv(A, n, lda, piv, info, s, orig, ldo); rc != 1) return rc;
    if (int rc = lu_factor_fast(A, n, lda, piv, info, s, tensor); rc != 1) return rc;
    const int nsm = num_sms();
    Scratch pub;
    const int maxP = nsm;
    if (int rc = pub.alloc(sizeof(double) * (2 * (size_t)maxP * (2 + kLuNb) + 2 * kLuNb), s)) return rc;
    for (int64_t j0 = 0; j0 < n; j0 += kLuNb) {
        const int nb = (int)((n - j0) < kLuNb ? (n - j0) : kLuNb);
        const int64_t h = n - j0;
        // rows per CTA: at least 16, at most what shared memory allows
        int P = (int)ceil_div(h, 16);
        if (P > maxP) P = maxP;
        int rp = (int)ceil_div(h, P);
        P = (int)ceil_div(h, rp);
        size_t smem = sizeof(double) * ((size_t)rp * (nb + 1) + nb);
        LM_REQUIRE(smem <= 200 * 1024, "lu panel: n too large for the panel slice (%lld)", (long long)n);
        if (int rc = func_attrs(lu_panel, smem)) return rc;
        PanelArgs a{A, lda, n, j0, nb, rp, P, piv, info, pub.as<double>(), pub.as<double>() + 2 * (size_t)maxP * (2 + kLuNb)};
        void *args[] = {&a};
        LM_CUDA(cudaLaunchCooperativeKernel((const void *)lu_panel, dim3(P), dim3(kPanelThreads), args, smem, s));
        count_launch(1);
        const int64_t j1 = j0 + nb, rest = n - j1;
        if (rest > 0) {
            // U12 = L11^{-1} A12 (order-preserving), then A22 -= L21 U12
            if (int rc = launch_trsm<true, false>(A + j0 + j0 * lda, lda, A + j0 + j1 * lda, lda, nb, rest, s)) return rc;
            if (int rc = launch_update<false, false>(A + j1 + j0 * lda, lda, A + j0 + j1 * lda, lda, A + j1 + j1 * lda,
                                                     lda, rest, rest, nb, s))
                return rc;
        }
    }
    return 0;
}

// perm[i] = source row of final row i after the sequential swaps piv.
// Two steps: every warp composes the 32 swaps of one pivot group into a
// permutation of the (<= 64) positions they touch (lane k tracks position
// g*32 + k; positions below the group found with a ballot); then one warp
// applies the groups in order as gathers on the permutation in shared
// memory.  (The sequential single-thread loop took ~0.45 ms at n = 8192.)
__global__ void __launch_bounds__(256) perm_groups(const int64_t *__restrict__ piv, int64_t n, int32_t *keys,
                                                   int32_t *srcs, int32_t *counts) {
    const int lane = threadIdx.x & 31;
    const int64_t g = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int64_t k0 = g * 32;
    if (k0 >= n) return;
    const int cnt = (int)((n - k0) < 32 ? (n - k0) : 32);
    int top_src = (int)(k0 + lane), bkey = -1, bsrc = 0, nbot = 0;
    for (int k = 0; k < cnt; ++k) {
        const int64_t p = piv[k0 + k];
        if (p == k0 + k) continue;
        const int a_src = __shfl_sync(0xffffffffu, top_src, k);
        int b_src;
        if (p < k0 + cnt) {
            const int pl = (int)(p - k0);
            b_src = __shfl_sync(0xffffffffu, top_src, pl);
            if (lane == pl) top_src = a_src;
        } else {
            const unsigned m = __ballot_sync(0xffffffffu, bkey == (int)p);
            if (m) {
                const int j = __ffs(m) - 1;
                b_src = __shfl_sync(0xffffffffu, bsrc, j);
                if (lane == j) bsrc = a_src;
            } else {
                b_src = (int)p;
                if (lane == nbot) {
                    bkey = (int)p;
                    bsrc = a_src;
                }
                ++nbot;
            }
        }
        if (lane == k) top_src = b_src;
    }
    int32_t *kg = keys + g * 64, *sg = srcs + g * 64;
    if (lane < cnt) {
        kg[lane] = (int32_t)(k0 + lane);
        sg[lane] = top_src;
    }
    if (lane < nbot) {
        kg[cnt + lane] = bkey;
        sg[cnt + lane] = bsrc;
    }
    if (lane == 0) counts[g] = cnt + nbot;
}

__global__ void __launch_bounds__(1024) perm_apply(int64_t n, int64_t ngroups, const int32_t *__restrict__ keys,
                                                   const int32_t *__restrict__ srcs, const int32_t *__restrict__ counts,
                                                   int32_t *perm) {
    extern __shared__ int32_t sp[];
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sp[i] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        for (int64_t g = 0; g < ngroups; ++g) {
            const int cnt = counts[g];
            const int32_t *kg = keys + g * 64, *sg = srcs + g * 64;
            int32_t v0 = 0, v1 = 0, k0 = -1, k1 = -1;
            if (lane < cnt) {
                k0 = kg[lane];
                v0 = sp[sg[lane]];
            }
            if (lane + 32 < cnt) {
                k1 = kg[lane + 32];
                v1 = sp[sg[lane + 32]];
            }
            __syncwarp();
            if (k0 >= 0) sp[k0] = v0;
            if (k1 >= 0) sp[k1] = v1;
            __syncwarp();
        }
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) perm[i] = sp[i];
}

__global__ void gather_rows(const double *__restrict__ src, int64_t ld_src, const int32_t *__restrict__ perm, int64_t n,
                            int64_t m, double *dst, int64_t ld_dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * m) return;
    const int64_t c = e / n, i = e - c * n;
    dst[i + c * ld_dst] = src[perm[i] + c * ld_src];
}

constexpr int kSolveNb = 64;

int lu_solve_impl(const double *LU, int64_t n, int64_t lda, const int64_t *piv, double *X, int64_t ldx, int64_t m,
                  cudaStream_t s, int mode) {
    if (n == 0 || m == 0) return 0;
    // 1. sequential row swaps == one gather by the composed permutation
    Scratch perm, tmp;
    if (int rc = perm.alloc(sizeof(int32_t) * n, s)) return rc;
    if (int rc = tmp.alloc(sizeof(double) * n * m, s)) return rc;
    const size_t psm = sizeof(int32_t) * n;
    LM_REQUIRE(psm <= 200 * 1024, "lu_solve: n too large for the permutation kernel");
    if (psm > 48 * 1024)
        if (int rc = func_attrs(perm_apply, psm)) return rc;
    const int64_t ngroups = ceil_div(n, 32);
    Scratch groups;
    if (int rc = groups.alloc(sizeof(int32_t) * ngroups * (64 + 64 + 1), s)) return rc;
    int32_t *gk = groups.as<int32_t>(), *gs = gk + ngroups * 64, *gc = gs + ngroups * 64;
    perm_groups<<<(unsigned)ceil_div(ngroups, 8), 256, 0, s>>>(piv, n, gk, gs, gc);
    perm_apply<<<1, 1024, psm, s>>>(n, ngroups, gk, gs, gc, perm.as<int32_t>());
    LM_LAUNCHED(2);
    // X -> tmp (one strided copy), then the permuted gather back into X
    LM_CUDA(cudaMemcpy2DAsync(tmp.as<double>(), sizeof(double) * n, X, sizeof(double) * ldx, sizeof(double) * n, m,
                              cudaMemcpyDeviceToDevice, s));
    gather_rows<<<(unsigned)ceil_div(n * m, 256), 256, 0, s>>>(tmp.as<double>(), n, perm.as<int32_t>(), n, m, X, ldx);
    LM_LAUNCHED(1);
    // 2./3. tensor mode: both sweeps as DMMA products with inverted diagonal
    // blocks (lu_solve_tc.cu; residual-level, falls back on device)
    if (lu_tensor_mode(mode, n))
        if (int rc = lu_solve_tensor(LU, n, lda, X, ldx, m, s); rc != 1) return rc;
    // exact order: one cooperative wavefront kernel for both sweeps (lu_solve.cu)
    if (int rc = lu_solve_wavefront(LU, n, lda, X, ldx, m, s, nullptr); rc != 1) return rc;
    // otherwise: forward, unit lower: 32-row block (one thread per rhs
    // column), then the rows below (order-preserving update, k ascending)
    constexpr int SB = 32;
    for (int64_t j0 = 0; j0 < n; j0 += SB) {
        const int nbj = (int)((n - j0) < SB ? (n - j0) : SB);
        if (int rc = tri32<true>(LU + j0 + j0 * lda, lda, X + j0, ldx, nbj, m, s)) return rc;
        const int64_t j1 = j0 + nbj;
        if (int rc = exact_update<false, false>(LU + j1 + j0 * lda, lda, X + j0, ldx, X + j1, ldx, n - j1, m, nbj, s))
            return rc;
    }
    // 3. backward, upper: blocks from the bottom, then rows above (k descending)
    for (int64_t jend = n; jend > 0; jend -= SB) {
        const int64_t j0 = jend > SB ? jend - SB : 0;
        const int nbj = (int)(jend - j0);
        if (int rc = tri32<false>(LU + j0 + j0 * lda, lda, X + j0, ldx, nbj, m, s)) return rc;
        if (int rc = exact_update<true, false>(LU + j0 * lda, lda, X + j0, ldx, X, ldx, j0, m, nbj, s)) return rc;
    }
    return 0;
}

// ---- triangular solve (R10:TRIU/TRIL) ------------------------------------------

__global__ void diag_zero_check(const double *A, int64_t lda, int64_t n, int32_t *info) {
    // first zero on the diagonal (reference checks all before solving)
    __shared__ int64_t first;
    if (threadIdx.x == 0) first = n;
    __syncthreads();
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x)
        if (A[j + j * lda] == 0.0) atomicMin((unsigned long long *)&first, (unsigned long long)j);
    __syncthreads();
    if (threadIdx.x == 0) *info = first < n ? (int32_t)(first + 1) : 0;
}

// Exact triangular solve, one CTA per RHS column, one thread per row chunk.
// Column-oriented exactly like the reference; O(n) barriers per column.
template <bool UPPER>
__global__ void __launch_bounds__(1024) tri_solve_col(const double *__restrict__ A, int64_t lda, int64_t n, double *X,
                                                      int64_t ldx, const int32_t *info) {
    if (*info != 0) return;
    double *x = X + (int64_t)blockIdx.x * ldx;
    __shared__ double xj_s;
    for (int64_t step = 0; step < n; ++step) {
        const int64_t j = UPPER ? (n - 1 - step) : step;
        if (threadIdx.x == 0) {
            const double v = rdiv(x[j], A[j + j * lda]);
            x[j] = v;
            xj_s = v;
        }
        __syncthreads();
        const double xj = xj_s;
        if (xj != 0.0) {
            if (UPPER) {
                for (int64_t i = threadIdx.x; i < j; i += blockDim.x) x[i] = rsub(x[i], rmul(A[i + j * lda], xj));
            } else {
                for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x) x[i] = rsub(x[i], rmul(A[i + j * lda], xj));
            }
        }
        __syncthreads();
    }
}

// ---- band solve (R10:BAND): exact sequential band LU, single CTA ----------------

__global__ void __launch_bounds__(256) band_solve_kernel(View<const double> A, double *AB, int64_t ldab, int64_t kl,
                                                         int64_t ku, int64_t *piv, int32_t *info, double *X,
                                                         int64_t ldx, int64_t m) {
    const int64_t n = A.rows, kv = kl + ku;
    const int tid = threadIdx.x, nt = blockDim.x;
#define AB_(r, c) AB[(int64_t)(r) + (int64_t)(c) * ldab]
    // pack (_loops.py:262-283)
    for (int64_t e = tid; e < ldab * n; e += nt) AB[e] = 0.0;
    __syncthreads();
    for (int64_t e = tid; e < n * n; e += nt) {
        const int64_t j = e / n, i = e - j * n;
        if (i >= j - ku && i <= j + kl) AB_(kv + i - j, j) = A(i, j);
    }
    __syncthreads();
    // factor (_loops.py:286-330)
    __shared__ int64_t s_jp, s_ju;
    __shared__ int s_fail;
    if (tid == 0) {
        s_ju = 0;
        s_fail = 0;
    }
    __syncthreads();
    for (int64_t j = 0; j < n; ++j) {
        const int64_t km = kl < n - 1 - j ? kl : n - 1 - j;
        if (tid == 0) {
            int64_t jp = 0;
            double best = fabs(AB_(kv, j));
            for (int64_t t = 1; t <= km; ++t) {
                const double v = fabs(AB_(kv + t, j));
                if (v > best) {
                    best = v;
                    jp = t;
                }
            }
            piv[j] = j + jp;
            if (AB_(kv + jp, j) == 0.0) {
                *info = (int32_t)(j + 1);
                s_fail = 1;
            }
            int64_t cand = j + ku + jp;
            int64_t ju = s_ju;
            if (cand > ju) ju = cand;
            if (ju > n - 1) ju = n - 1;
            s_ju = ju;
            s_jp = jp;
        }
        __syncthreads();
        if (s_fail) return;
        const int64_t jp = s_jp, ju = s_ju;
        if (jp != 0)
            for (int64_t jj = j + tid; jj <= ju; jj += nt) {
                const double t1 = AB_(kv + j - jj, jj);
                AB_(kv + j - jj, jj) = AB_(kv + j + jp - jj, jj);
                AB_(kv + j + jp - jj, jj) = t1;
            }
        __syncthreads();
        if (km > 0) {
            const double pv = AB_(kv, j);
            for (int64_t t = 1 + tid; t <= km; t += nt) AB_(kv + t, j) = rdiv(AB_(kv + t, j), pv);
            __syncthreads();
            // each (jj) column update is independent; t ascending inside
            for (int64_t jj = j + 1 + tid; jj <= ju; jj += nt) {
                const double f = AB_(kv + j - jj, jj);
                if (f != 0.0)
                    for (int64_t t = 1; t <= km; ++t)
                        AB_(kv + j - jj + t, jj) = rsub(AB_(kv + j - jj + t, jj), rmul(AB_(kv + t, j), f));
            }
        }
        __syncthreads();
    }
    if (tid == 0) *info = 0;
    // substitution (_loops.py:333-360), one thread per RHS column
    for (int64_t c = tid; c < m; c += nt) {
        double *x = X + c * ldx;
        for (int64_t j = 0; j < n; ++j) {
            const int64_t p = piv[j];
            if (p != j) {
                const double t1 = x[j];
                x[j] = x[p];
                x[p] = t1;
            }
            const int64_t km = kl < n - 1 - j ? kl : n - 1 - j;
            const double xj = x[j];
            if (xj != 0.0)
                for (int64_t t = 1; t <= km; ++t) x[j + t] = rsub(x[j + t], rmul(AB_(kv + t, j), xj));
        }
        for (int64_t j = n - 1; j >= 0; --j) {
            const int64_t u = kv < n - 1 - j ? kv : n - 1 - j;
            double acc = x[j];
            for (int64_t t = 1; t <= u; ++t) acc = rsub(acc, rmul(AB_(kv - t, j + t), x[j + t]));
            x[j] = rdiv(acc, AB_(kv, j));
        }
    }
#undef AB_
}

}  // namespace lm

using namespace lm;

extern "C" int lm_lu_factor(int dtype, lm_view lu, int64_t *d_piv, int32_t *d_info, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "lu_factor: f64 only");
    LM_REQUIRE(lu.rows == lu.cols, "lu_factor needs a square matrix");
    LM_REQUIRE(lu.rs == 1 && (lu.cs >= lu.rows || lu.rows <= 1), "lu_factor needs F-order storage");
    return lu_factor_impl((double *)lu.ptr, lu.rows, lu.cs > 0 ? lu.cs : 1, d_piv, d_info, as_stream(stream),
                          LM_LU_AUTO);
}

extern "C" int lm_lu_factor_mode(int dtype, lm_view lu, int64_t *d_piv, int32_t *d_info, int mode, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "lu_factor: f64 only");
    LM_REQUIRE(mode == LM_LU_AUTO || mode == LM_LU_EXACT || mode == LM_LU_TENSOR, "lu_factor: bad mode %d", mode);
    LM_REQUIRE(lu.rows == lu.cols, "lu_factor needs a square matrix");
    LM_REQUIRE(lu.rs == 1 && (lu.cs >= lu.rows || lu.rows <= 1), "lu_factor needs F-order storage");
    return lu_factor_impl((double *)lu.ptr, lu.rows, lu.cs > 0 ? lu.cs : 1, d_piv, d_info, as_stream(stream), mode);
}

extern "C" int lm_lu_factor_from(int dtype, lm_view src, lm_view lu, int64_t *d_piv, int32_t *d_info, int mode,
                                 void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "lu_factor: f64 only");
    LM_REQUIRE(mode == LM_LU_AUTO || mode == LM_LU_EXACT || mode == LM_LU_TENSOR, "lu_factor: bad mode %d", mode);
    LM_REQUIRE(lu.rows == lu.cols && src.rows == lu.rows && src.cols == lu.cols, "lu_factor needs square matrices of one size");
    LM_REQUIRE(lu.rs == 1 && (lu.cs >= lu.rows || lu.rows <= 1), "lu_factor needs F-order storage");
    LM_REQUIRE(src.rs == 1 && (src.cs >= src.rows || src.rows <= 1), "lu_factor_from needs an F-order source");
    LM_REQUIRE(src.ptr != lu.ptr, "lu_factor_from: source and workspace must differ");
    cudaStream_t s = as_stream(stream);
    const int64_t n = lu.rows, lda = lu.cs > 0 ? lu.cs : 1, ldo = src.cs > 0 ? src.cs : 1;
    if (n > 0)
        LM_CUDA(cudaMemcpy2DAsync(lu.ptr, lda * sizeof(double), src.ptr, ldo * sizeof(double), n * sizeof(double), n,
                                  cudaMemcpyDeviceToDevice, s));
    return lu_factor_impl((double *)lu.ptr, n, lda, d_piv, d_info, s, mode, (const double *)src.ptr, ldo);
}

extern "C" int lm_lu_solve(int dtype, lm_view lu, const int64_t *d_piv, lm_view x, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "lu_solve: f64 only");
    LM_REQUIRE(lu.rows == lu.cols && x.rows == lu.rows, "lu_solve shape mismatch");
    LM_REQUIRE(lu.rs == 1 && (x.rs == 1 || x.rows <= 1), "lu_solve needs F-order operands");
    const int64_t ldx = x.cols > 1 ? x.cs : (x.rows > 0 ? x.rows : 1);
    return lu_solve_impl((const double *)lu.ptr, lu.rows, lu.cs > 0 ? lu.cs : 1, d_piv, (double *)x.ptr, ldx, x.cols,
                         as_stream(stream), LM_LU_EXACT);
}

extern "C" int lm_lu_solve_mode(int dtype, lm_view lu, const int64_t *d_piv, lm_view x, int mode, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "lu_solve: f64 only");
    LM_REQUIRE(mode == LM_LU_AUTO || mode == LM_LU_EXACT || mode == LM_LU_TENSOR, "lu_solve: bad mode %d", mode);
    LM_REQUIRE(lu.rows == lu.cols && x.rows == lu.rows, "lu_solve shape mismatch");
    LM_REQUIRE(lu.rs == 1 && (x.rs == 1 || x.rows <= 1), "lu_solve needs F-order operands");
    const int64_t ldx = x.cols > 1 ? x.cs : (x.rows > 0 ? x.rows : 1);
    return lu_solve_impl((const double *)lu.ptr, lu.rows, lu.cs > 0 ? lu.cs : 1, d_piv, (double *)x.ptr, ldx, x.cols,
                         as_stream(stream), mode);
}

extern "C" int lm_tri_solve(int dtype, lm_view a, lm_view x, int upper, int32_t *d_info, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "tri_solve: f64 only");
    LM_REQUIRE(a.rows == a.cols && x.rows == a.rows, "tri_solve shape mismatch");
    LM_REQUIRE(a.rs == 1 && (x.rs == 1 || x.rows <= 1), "tri_solve needs F-order operands");
    cudaStream_t s = as_stream(stream);
    const int64_t n = a.rows, lda = a.cs > 0 ? a.cs : 1;
    const int64_t ldx = x.cols > 1 ? x.cs : (x.rows > 0 ? x.rows : 1);
    diag_zero_check<<<1, 1024, 0, s>>>((const double *)a.ptr, lda, n, d_info);
    LM_LAUNCHED(1);
    if (n == 0 || x.cols == 0) return 0;
    if (upper)
        tri_solve_col<true><<<(unsigned)x.cols, 256, 0, s>>>((const double *)a.ptr, lda, n, (double *)x.ptr, ldx, d_info);
    else
        tri_solve_col<false><<<(unsigned)x.cols, 256, 0, s>>>((const double *)a.ptr, lda, n, (double *)x.ptr, ldx, d_info);
    LM_LAUNCHED(1);
    return 0;
}

extern "C" int lm_band_solve(int dtype, lm_view a, lm_view x, int64_t kl, int64_t ku, void *ab_work, int64_t *d_piv,
                             int32_t *d_info, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "band_solve: f64 only");
    LM_REQUIRE(a.rows == a.cols && x.rows == a.rows, "band_solve shape mismatch");
    LM_REQUIRE(kl >= 0 && ku >= 0, "band_solve bandwidths");
    LM_REQUIRE(x.rs == 1 || x.rows <= 1, "band_solve needs F-order x");
    cudaStream_t s = as_stream(stream);
    const int64_t ldx = x.cols > 1 ? x.cs : (x.rows > 0 ? x.rows : 1);
    LM_CUDA(cudaMemsetAsync(d_info, 0, sizeof(int32_t), s));
    if (a.rows == 0) return 0;
    View<const double> A{(const double *)a.ptr, a.rows, a.cols, a.rs, a.cs};
    band_solve_kernel<<<1, 256, 0, s>>>(A, (double *)ab_work, 2 * kl + ku + 1, kl, ku, d_piv, d_info, (double *)x.ptr,
                                        ldx, x.cols);
    LM_LAUNCHED(1);
    return 0;
}

