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
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// Solve-only variant (no LU factors requested): the same per-instance
// arithmetic in a compact, ROLLED column loop.
//
// The fully unrolled kernel above is ~21k instructions (its column loop
// is unrolled over k and j so that every register index is static); with
// six CTAs per SM at different columns the instruction cache thrashes
// (ncu: "no instruction" stalls, 30% issue).  Here each thread's row is
// kept SHIFTED: before step k, r[i] holds column k + i, so the pivot
// column is always r[0] and the update writes its result one slot down,
// r[i-1] = r[i] - m * U[k, k+i] -- the shift costs nothing.  The column
// loop is rolled inside blocks of KB columns; block kb's code updates a
// static N - kb*KB slots (slots past the live columns hold stale values
// and only ever feed stale slots).  The right-hand side is eliminated on
// the fly with the same multipliers, in the same order as
// _lu_solve_inplace's forward sweep (b_i -= L[i,k] * y_k, k ascending,
// lazymat/_loops.py:250-253); each pivot row is copied to shared memory
// (U[k, k:]) for the back sweep (:254-258), which one warp runs with
// shuffles instead of block barriers.
template <int N, int KB, bool CLASSIFY>
__global__ void __launch_bounds__(N, N == 64 ? 6 : 1)
    lu_batched_shift(int64_t n, int64_t batch, const double *__restrict__ A, double *__restrict__ X,
                     int64_t *__restrict__ piv, int32_t *__restrict__ info, int32_t *__restrict__ cls) {
    constexpr int W = N / 32 > 0 ? N / 32 : 1;  // warps per system
    constexpr int R = (N + 31) / 32;            // back-sweep positions per lane
    constexpr unsigned MASK = N >= 32 ? 0xffffffffu : ((1u << N) - 1u);
    __shared__ __align__(16) double cand_row[2][W][N];  // published candidate rows (by k parity)
    __shared__ double cand_x[2][W];
    __shared__ unsigned cand_h[2][W], cand_l[2][W];
    __shared__ int cand_pos[2][W], cand_t[2][W];
    __shared__ __align__(16) double Us[N * (N + 1)];  // U[k, k+i] at Us[k*N + i]; aliased by the classify transpose
    __shared__ double xs[N];
    __shared__ int s_fail;

    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
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
    int pos = t;
    if (t == 0) s_fail = 0;
    if constexpr (CLASSIFY) {
        // lazymat/rewrite.py:146-173 over _analyze (lazymat/_loops.py:15-34)
        double(*sAt)[N + 1] = reinterpret_cast<double(*)[N + 1]>(Us);
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
        lb = __reduce_max_sync(MASK, lb);
        ub = __reduce_max_sync(MASK, ub);
        asym = __reduce_or_sync(MASK, asym);
        if (lane == 0) {
            s_lb[w] = lb;
            s_ub[w] = ub;
            s_as[w] = asym;
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
            int c = 0;
            if (lb + ub <= lim) c = 1;
            else if (lb == 0) c = 2;
            else if (ub == 0) c = 3;
            else if (!asym) c = 4;
            cls[b] = c;
        }
    }
    __syncthreads();

#pragma unroll
    for (int kb = 0; kb < N / KB; ++kb) {
        const int L = N - kb * KB;  // static after unrolling: slots this block's code updates
#pragma unroll 1
        for (int kk = 0; kk < KB; ++kk) {
            const int k = kb * KB + kk;
            if (k >= n) break;
            const int par = k & 1;
            // first maximum of |A[i,k]| over positions >= k (lazymat/_loops.py:212-218)
            unsigned hk = 0u, lk = 0u;
            if (pos >= k) {
                double v = fabs(r[0]);
                bool ok = true;
                if (v != v) {
                    ok = (pos == k);
                    v = __longlong_as_double(0x7ff0000000000000LL);
                }
                if (ok) {
                    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
                    hk = (unsigned)(bits >> 32) + 1u;
                    lk = (unsigned)bits;
                }
            }
            const unsigned H = __reduce_max_sync(MASK, hk);
            const unsigned Lo = __reduce_max_sync(MASK, hk == H ? lk : 0u);
            const unsigned P =
                __reduce_min_sync(MASK, (hk != 0u && hk == H && lk == Lo) ? (unsigned)pos : 0xffffffffu);
            if (hk != 0u && (unsigned)pos == P) {
                cand_h[par][w] = H;
                cand_l[par][w] = Lo;
                cand_pos[par][w] = (int)P;
                cand_t[par][w] = t;
                cand_x[par][w] = xv;
                double2 *dst = reinterpret_cast<double2 *>(cand_row[par][w]);
#pragma unroll
                for (int i = 0; i < L; i += 2) dst[i >> 1] = make_double2(r[i], i + 1 < L ? r[i + 1] : 0.0);
            }
            if (W > 1 && H == 0u && lane == 0) cand_h[par][w] = 0u;
            __syncthreads();
            int win = 0;
#pragma unroll
            for (int q = 1; q < W; ++q)
                if (cand_h[par][q] > cand_h[par][win] ||
                    (cand_h[par][q] == cand_h[par][win] &&
                     (cand_l[par][q] > cand_l[par][win] ||
                      (cand_l[par][q] == cand_l[par][win] && cand_pos[par][q] < cand_pos[par][win]))))
                    win = q;
            const int p = cand_pos[par][win];
            const int pt = cand_t[par][win];
            const double *U = cand_row[par][win];
            const double pvv = U[0];
            if (t == 0) {
                if (piv) piv[b * n + k] = p;
                if (pvv == 0.0 && s_fail == 0) s_fail = k + 1;
            }
            if (t < L) Us[k * N + t] = U[t];  // pivot row U[k, k:] for the back sweep
            if (p != k) {
                if (t == pt)
                    pos = k;
                else if (pos == k)
                    pos = p;
            }
            if (pos > k) {
                const double m = __ddiv_rn(r[0], pvv);
                const double2 *U2 = reinterpret_cast<const double2 *>(U);
#pragma unroll
                for (int i = 1; i < L; ++i) {
                    const double2 u = U2[i >> 1];
                    r[i - 1] = __dsub_rn(r[i], __dmul_rn(m, (i & 1) ? u.y : u.x));
                }
                xv = __dsub_rn(xv, __dmul_rn(m, cand_x[par][win]));
            }
        }
    }
    if (pos < N) xs[pos] = xv;
    __syncthreads();
    const int fail = s_fail;
    if (t == 0) info[b] = fail;
    if (fail || w != 0) return;
    // back sweep (lazymat/_loops.py:254-258) by warp 0: lane l holds
    // positions l, l + 32, ...
    double c[R];
#pragma unroll
    for (int q = 0; q < R; ++q) c[q] = (q * 32 + lane < n) ? xs[q * 32 + lane] : 0.0;
#pragma unroll 1
    for (int j = (int)n - 1; j >= 0; --j) {
        const int jq = j >> 5, src = j & 31;
        double cj = c[0];
#pragma unroll
        for (int q = 1; q < R; ++q)
            if (jq == q) cj = c[q];
        cj = __shfl_sync(MASK, cj, src);
        const double xj = __ddiv_rn(cj, Us[j * N]);
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int i = q * 32 + lane;
            if (i == j) c[q] = xj;
            else if (i < j) c[q] = __dsub_rn(c[q], __dmul_rn(Us[i * N + (j - i)], xj));
        }
    }
#pragma unroll
    for (int q = 0; q < R; ++q)
        if (q * 32 + lane < n) X[b * n + q * 32 + lane] = c[q];
}

}  // namespace lm

using namespace lm;

static bool use_shift_kernel() {
    static const bool off = [] {
        const char *e = getenv("LM_BATCHED_LU_UNROLLED");
        return e && e[0] == '1';
    }();
    return !off;
}

template <bool CLASSIFY>
static int launch_batched(int64_t n, int64_t batch, const double *A, double *X, double *LU, int64_t *d_piv,
                          int32_t *d_info, int32_t *d_cls, cudaStream_t s) {
    if (LU == nullptr && use_shift_kernel()) {
        if (n <= 16)
            lu_batched_shift<16, 8, CLASSIFY><<<(unsigned)batch, 16, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls);
        else if (n <= 32)
            lu_batched_shift<32, 8, CLASSIFY><<<(unsigned)batch, 32, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls);
        else
            lu_batched_shift<64, 8, CLASSIFY><<<(unsigned)batch, 64, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls);
    } else if (n <= 16)
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
