// lu_batched.cu -- many independent small LU solves (BASELINE config 4b):
// per instance exactly the reference's _lu_factor + _lu_solve_inplace
// (lazymat/_loops.py:200-259), bit-identical values and pivots.
//
// One CTA of N threads per system (N = 16/32/64, instances padded with an
// identity block, which leaves the leading block's factorisation and
// pivots untouched).  Thread t keeps ORIGINAL row t of the matrix in N
// registers for the whole factorisation; the k and j loops are fully
// unrolled so every register index is static.  Row swaps never move
// data: every thread tracks the current position of its row, so the
// reference's "full-row swap" is two integer assignments.  Per column k
// one barrier: each warp finds its best candidate (|value| desc, position
// asc -- the reference's strict-> scan) with three redux.sync
// instructions and publishes it with the candidate's row; every thread
// then picks the global winner and reads the pivot row U[k, k+1:] as
// shared-memory broadcasts.  Multipliers and updates use __ddiv_rn /
// __dmul_rn / __dsub_rn in the reference order.
//
// Traffic per instance: A read once (N*N*8 B), b read, x written; the LU
// factors / pivots are written only when requested.
#include "common.cuh"

namespace lm {

template <int N, bool CLASSIFY>
__global__ void __launch_bounds__(N) lu_batched_rows(int64_t n, int64_t batch, const double *__restrict__ A,
                                                     double *__restrict__ X, double *__restrict__ LU,
                                                     int64_t *__restrict__ piv, int32_t *__restrict__ info,
                                                     int32_t *__restrict__ cls) {
    constexpr int W = N / 32 > 0 ? N / 32 : 1;  // warps per system
    constexpr unsigned MASK = N >= 32 ? 0xffffffffu : ((1u << N) - 1u);
    __shared__ double cand_row[2][W][N];        // published candidate rows (double-buffered by k parity)
    __shared__ unsigned cand_h[2][W], cand_l[2][W];
    __shared__ int cand_pos[2][W], cand_t[2][W];
    __shared__ double xb[N];   // substitution broadcast
    __shared__ int s_fail;

    const int t = threadIdx.x, w = t >> 5;
    const int64_t b = blockIdx.x;
    const double *Ab = A + b * n * n;
    double r[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        if (t < n && j < n)
            r[j] = __ldg(Ab + t + (int64_t)j * n);
        else
            r[j] = (t == j) ? 1.0 : 0.0;  // identity padding
    }
    double xv = t < n ? __ldg(X + b * n + t) : 0.0;
    int pos = t;  // current position of the row this thread owns
    if (t == 0) s_fail = 0;
    if constexpr (CLASSIFY) {
        // the R10 structure ladder of this instance (lazymat/rewrite.py:146-173
        // over _analyze, lazymat/_loops.py:15-34), from the registers: lower /
        // upper bandwidth over nonzeros, exact symmetry through a transposed
        // shared-memory copy
        __shared__ double sAt[N][N + 1];
        __shared__ unsigned s_lb[W], s_ub[W], s_as[W];
        unsigned lb = 0, ub = 0, asym = 0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (t < n && j < n) {
                sAt[t][j] = r[j];
                if (r[j] != 0.0) {
                    if (t > j) lb = max(lb, (unsigned)(t - j));
                    if (j > t) ub = max(ub, (unsigned)(j - t));
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < N; ++j)
            if (t < n && j < n && j > t && !(r[j] == sAt[j][t])) asym = 1;
        constexpr unsigned MASK = N >= 32 ? 0xffffffffu : ((1u << N) - 1u);
        lb = __reduce_max_sync(MASK, lb);
        ub = __reduce_max_sync(MASK, ub);
        asym = __reduce_or_sync(MASK, asym);
        if ((t & 31) == 0) {
            s_lb[t >> 5] = lb;
            s_ub[t >> 5] = ub;
            s_as[t >> 5] = asym;
        }
        __syncthreads();
        if (t == 0) {
#pragma unroll
            for (int q = 1; q < W; ++q) {
                lb = max(lb, s_lb[q]);
                ub = max(ub, s_ub[q]);
                asym |= s_as[q];
            }
            const unsigned lim = (unsigned)(n / 4 > 4 ? n / 4 : 4);
            int c = 0;  // general
            if (lb + ub <= lim) c = 1;        // band
            else if (lb == 0) c = 2;          // upper triangular
            else if (ub == 0) c = 3;          // lower triangular
            else if (!asym) c = 4;            // symmetric (still LU)
            cls[b] = c;
        }
    }
    __syncthreads();

#pragma unroll
    for (int k = 0; k < N; ++k) {
        const int par = k & 1;
        // --- first maximum of |r[k]| over positions >= k: (|v| bits desc,
        // position asc) with three redux.sync instructions per warp
        unsigned hk = 0u, lk = 0u;
        if (pos >= k) {
            double v = fabs(r[k]);
            bool ok = true;
            if (v != v) {
                ok = (pos == k);  // NaN never wins off the diagonal; on it, it keeps p = k
                v = __longlong_as_double(0x7ff0000000000000LL);
            }
            if (ok) {
                const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
                hk = (unsigned)(bits >> 32) + 1u;
                lk = (unsigned)bits;
            }
        }
        const unsigned H = __reduce_max_sync(MASK, hk);
        const unsigned L = __reduce_max_sync(MASK, hk == H ? lk : 0u);
        const unsigned P = __reduce_min_sync(MASK, (hk != 0u && hk == H && lk == L) ? (unsigned)pos : 0xffffffffu);
        // the warp winner publishes its key and its row (columns >= k)
        if (hk != 0u && (unsigned)pos == P) {
            cand_h[par][w] = H;
            cand_l[par][w] = L;
            cand_pos[par][w] = (int)P;
            cand_t[par][w] = t;
#pragma unroll
            for (int j = k; j < N; ++j) cand_row[par][w][j] = r[j];
        }
        if (W > 1 && H == 0u && (t & 31) == 0) cand_h[par][w] = 0u;  // no rows >= k in this warp
        __syncthreads();
        // global winner among the W published candidates
        int win = 0;
#pragma unroll
        for (int q = 1; q < W; ++q)
            if (cand_h[par][q] > cand_h[par][win] ||
                (cand_h[par][q] == cand_h[par][win] &&
                 (cand_l[par][q] > cand_l[par][win] ||
                  (cand_l[par][q] == cand_l[par][win] && cand_pos[par][q] < cand_pos[par][win]))))
                win = q;
        const int p = cand_pos[par][win];   // pivot position (reference's p)
        const int pt = cand_t[par][win];    // the thread holding it
        const double *U = cand_row[par][win];
        const double pvv = U[k];
        if (t == 0) {
            if (piv && k < n) piv[b * n + k] = p;
            if (pvv == 0.0 && s_fail == 0 && k < n) s_fail = k + 1;
        }
        // full-row swap of positions k and p == exchange of two positions
        if (p != k) {
            if (t == pt)
                pos = k;
            else if (pos == k)
                pos = p;
        }
        // multipliers and the rank-1 update of the rows below the pivot
        if (pos > k) {
            const double m = __ddiv_rn(r[k], pvv);
            r[k] = m;
#pragma unroll
            for (int j = k + 1; j < N; ++j) r[j] = __dsub_rn(r[j], __dmul_rn(m, U[j]));
        }
    }
    __syncthreads();
    const int fail = s_fail;
    if (t == 0) info[b] = fail;
    if (fail) return;
    // ---- solve: x held by position; swaps already applied via pos (the
    // sequential swaps of _lu_solve_inplace compose to "position pos[t]
    // holds original row t").
    // forward (unit lower), positions ascending
#pragma unroll
    for (int j = 0; j < N; ++j) {
        if (pos == j) xb[j] = xv;
        __syncthreads();
        if (pos > j) xv = __dsub_rn(xv, __dmul_rn(r[j], xb[j]));
    }
    // backward (upper), positions descending
#pragma unroll
    for (int j = N - 1; j >= 0; --j) {
        if (pos == j) {
            xv = __ddiv_rn(xv, r[j]);
            xb[j] = xv;
        }
        __syncthreads();
        if (pos < j) xv = __dsub_rn(xv, __dmul_rn(r[j], xb[j]));
    }
    if (pos < n) X[b * n + pos] = xv;
    if (LU && pos < n)
#pragma unroll
        for (int j = 0; j < N; ++j)
            if (j < n) LU[b * n * n + pos + (int64_t)j * n] = r[j];
}

}  // namespace lm

using namespace lm;

template <bool CLASSIFY>
static int launch_batched(int64_t n, int64_t batch, const double *A, double *X, double *LU, int64_t *d_piv,
                          int32_t *d_info, int32_t *d_cls, cudaStream_t s) {
    if (n <= 16)
        lu_batched_rows<16, CLASSIFY><<<(unsigned)batch, 16, 0, s>>>(n, batch, A, X, LU, d_piv, d_info, d_cls);
    else if (n <= 32)
        lu_batched_rows<32, CLASSIFY><<<(unsigned)batch, 32, 0, s>>>(n, batch, A, X, LU, d_piv, d_info, d_cls);
    else
        lu_batched_rows<64, CLASSIFY><<<(unsigned)batch, 64, 0, s>>>(n, batch, A, X, LU, d_piv, d_info, d_cls);
    LM_LAUNCHED(1);
    return 0;
}

extern "C" int lm_lu_solve_batched(int dtype, int64_t n, int64_t batch, const void *a, void *x, void *lu_out,
                                   int64_t *d_piv, int32_t *d_info, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "lu_solve_batched: f64 only");
    LM_REQUIRE(n >= 1 && n <= 64, "lu_solve_batched: 1 <= n <= 64 (got %lld)", (long long)n);
    if (batch == 0) return 0;
    LM_REQUIRE(batch <= 0x7fffffff, "lu_solve_batched: batch too large");
    return launch_batched<false>(n, batch, (const double *)a, (double *)x, (double *)lu_out, d_piv, d_info, nullptr,
                                 as_stream(stream));
}

extern "C" int lm_solve_batched_classified(int dtype, int64_t n, int64_t batch, const void *a, void *x,
                                           int32_t *d_cls, int32_t *d_info, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "solve_batched_classified: f64 only");
    LM_REQUIRE(n >= 1 && n <= 64, "solve_batched_classified: 1 <= n <= 64 (got %lld)", (long long)n);
    if (batch == 0) return 0;
    LM_REQUIRE(batch <= 0x7fffffff, "solve_batched_classified: batch too large");
    return launch_batched<true>(n, batch, (const double *)a, (double *)x, nullptr, nullptr, d_info, d_cls,
                                as_stream(stream));
}
