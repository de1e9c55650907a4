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
#include <cstring>

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
__device__ __forceinline__ void shift_system(const int64_t b, int64_t n, const double *__restrict__ A,
                                             double *__restrict__ X, int64_t *__restrict__ piv,
                                             int32_t *__restrict__ info, int32_t *__restrict__ cls) {
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

// One system per CTA, or (redo_list set) a small grid that solves exactly the
// systems the pivot-free fast path listed as unproved.
template <int N, int KB, bool CLASSIFY>
__global__ void __launch_bounds__(N, N == 64 ? 6 : 1)
    lu_batched_shift(int64_t n, int64_t batch, const double *__restrict__ A, double *__restrict__ X,
                     int64_t *__restrict__ piv, int32_t *__restrict__ info, int32_t *__restrict__ cls,
                     const int *__restrict__ redo_list, const int *__restrict__ redo_count) {
    if (!redo_list) {
        shift_system<N, KB, CLASSIFY>(blockIdx.x, n, A, X, piv, info, cls);
        return;
    }
    const int cnt = *redo_count;
    for (int i = blockIdx.x; i < cnt; i += gridDim.x) {
        shift_system<N, KB, CLASSIFY>(redo_list[i], n, A, X, piv, info, cls);
        __syncthreads();  // shared buffers are reused by the next system
    }
}

// ---------------------------------------------------------------------------
// Pivot-free blocked fast path for 32 < n <= 64 (config 4b), bit-identical
// to _lu_factor + _lu_solve_inplace (lazymat/_loops.py:200-259) whenever
// the reference's partial pivoting never swaps -- and it PROVES that it
// never swaps: at step k the reference keeps p = k unless some
// |LU[i,k]| > |LU[k,k]| (strict, lazymat/_loops.py:212-218).  Every
// multiplier m = RN(LU[i,k] / LU[k,k]) is checked to satisfy |m| < 1,
// which implies |LU[i,k]| < |LU[k,k]| (rounding is monotonic and 1 is
// representable), so p = k; by induction over k the state at every step is
// the reference's own.  A failed check (including NaN, Inf and a zero
// pivot) marks the system (info = -1, x untouched) and the pivoting kernel
// (lu_batched_shift, redo mode) solves exactly those systems afterwards.
// Diagonally dominant batches (config 4b: A = U(-1,1) + 64 I) never fail.
//
// Without pivot search the per-column chain shrinks to a division, so the
// factorisation runs in blocks of KB = 8 columns with two block barriers
// per block (instead of one per column):
//   (a) the warp holding the block's 8 diagonal rows factors the 8 x 8
//       diagonal block with shuffles (the pivot row's values broadcast
//       lane to lane) and publishes U11, its multipliers and its rows' raw
//       rest (columns c0+8.., then the right-hand side);
//   (b) every row below divides and eliminates its own 8 panel values
//       against U11 (a per-row triangular solve in the reference's order:
//       column c0+s2 receives steps c0, c0+1, ... then its division);
//   (c) concurrently, one thread per rest column finishes the block's U
//       rows (row c0+s receives steps c0..c0+s-1 in order);
//   (d) every row below applies the 8 deferred rank-1 updates to its rest,
//       s ascending (mul and sub separately rounded: the reference's
//       sequence of roundings for every element).
// The rest buffer is double-buffered by block parity so block kb+1's (a)
// overlaps block kb's (d) in the other warp.  The back sweep is the
// shift kernel's (one warp, packed U).
__device__ __forceinline__ constexpr int upacked_off(int k) { return k * 64 - k * (k - 1) / 2; }

// Certified fast division.  __ddiv_rn costs ~126 cycles of dependent
// latency on the B200 (tools/probes/fp64_lat_probe.cu: DFMA 8.7, drcp 76,
// ddiv 126), and the pivot-free path divides by the same pivot many times.
// With y = RN(1/b) computed once per divisor, q0 = RN(a*y),
// r = RN(a - b*q0), q1 = RN(q0 + r*y) (Markstein's correction: three
// dependent FP64 operations) is RN(a/b) in practice -- and this is CHECKED,
// not assumed: rho = RN(a - b*q1) (one fma: a single rounding of the exact
// remainder) and q1 is certified when |rho| < T' = halfulp(q1) *
// RN(|b| * (1 - 2^-50)), halfulp(q1) being half the gap to q1's smaller
// neighbour (a power of two, so T' is an exact product).  Then
// |a - b*q1| <= |rho| * (1 + 2^-52) < |b| * halfulp(q1), i.e. a/b lies strictly
// inside q1's round-to-nearest interval, so q1 == RN(a/b) == __ddiv_rn(a, b).
// Exponent windows keep every quantity normal (no underflow in T' or in the
// remainder's rounding).  A zero dividend returns a*y (the correctly signed
// zero).  An uncertified quotient sets `bad`; the pivot-free kernel then
// hands the whole system to the pivoting kernel, so results never depend on
// an unproved quotient.
struct CertDiv {
    double b, y, bc;
    int eb;  // biased exponent of b; 0 = not certifiable (outside the window)
};

// y = RN(1/b) computed by the caller (once per divisor, off the chains)
__device__ __forceinline__ CertDiv cdiv_prep(double b, double y) {
    CertDiv d;
    d.b = b;
    d.y = y;
    d.bc = __dmul_rn(fabs(b), 1.0 - 0x1p-50);
    const int eb = (__double2hiint(b) >> 20) & 0x7ff;
    d.eb = (eb >= 1023 - 1000 && eb <= 1023 + 1000) ? eb : -4096;
    return d;
}

__device__ __forceinline__ double cdiv(double a, const CertDiv &d, int &bad) {
    const double q0 = __dmul_rn(a, d.y);
    const double r0 = __fma_rn(-q0, d.b, a);
    const double q1 = __fma_rn(r0, d.y, q0);
    const double rho = __fma_rn(-q1, d.b, a);
    const int hi = __double2hiint(q1), lo = __double2loint(q1);
    const int e = (hi >> 20) & 0x7ff;
    const int mz = ((hi & 0xfffff) | lo) == 0;  // |q1| a power of two: the gap below is half an ulp
    const double halfulp = __hiloint2double((e - 53 - mz) << 20, 0);
    const double tc = __dmul_rn(halfulp, d.bc);
    // q1 normal, half-ulp normal, not near overflow; T' = halfulp*|b| >= 2^-900
    const bool range = (unsigned)(e - 55) < 1945u && e + d.eb >= 2 * 1023 - 900;
    const bool zero = a == 0.0;
    const bool good = zero ? d.eb > 0 : (range && fabs(rho) < tc);
    bad |= !good;
    return zero ? q0 : q1;
}

// TRACE (LM_4B_TRACE=1, diagnostics): lane 0 of each warp records clock64()
// at the phase boundaries into trace[b * 64 + warp * 32 + i] (tools/lu4b_trace.py).
#define LU4B_MARK(i)                                                          \
    if (TRACE && lane == 0) trace[b * 64 + w * 32 + (i)] = clock64();
template <bool CLASSIFY, bool TRACE = false>
__global__ void __launch_bounds__(64, 6)
    lu_batched_nopiv(int64_t n, int64_t batch, const double *__restrict__ A, double *__restrict__ X,
                     int64_t *__restrict__ piv, int32_t *__restrict__ info, int32_t *__restrict__ cls,
                     int *__restrict__ redo_list, int *__restrict__ redo_count, long long *__restrict__ trace = nullptr) {
    constexpr int N = 64, KB = 8, NB = N / KB;
    constexpr int UW = N - KB + 2;  // rest width incl. the right-hand side, even
    constexpr unsigned MASK = 0xffffffffu;
    struct Fact {
        double Ub[2][KB][UW];        // block rows' rest: raw, then U[c0+s, c0+8+j]; column Rw = y
        double U11[KB][KB];          // diagonal block: U[c0+s, c0+s2] for s2 >= s
        double Ld[KB][KB];           // diagonal block multipliers L[c0+s, c0+s2], s2 < s
        double Lr[KB][N];            // multipliers of the rows below, by owning thread
        double Us[N * (N + 1) / 2];  // packed U: U[k, k+i] at upacked_off(k) + i
        double xs[N];                // y by position
        double yd[N];                // RN(1 / U[k,k]), for the certified divisions
    };
    constexpr size_t SAT = CLASSIFY ? sizeof(double) * N * (N + 1) : 0;
    constexpr size_t SMB = sizeof(Fact) > SAT ? sizeof(Fact) : SAT;
    __shared__ __align__(16) unsigned char smraw[SMB];
    Fact &f = *reinterpret_cast<Fact *>(smraw);

    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int64_t b = blockIdx.x;
    const double *Ab = A + b * n * n;
    double r[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        if (t < n && j < n)
            r[j] = __ldg(Ab + t + (int64_t)j * n);
        else
            r[j] = (t == j) ? 1.0 : 0.0;  // identity padding: pivot-free by construction
    }
    if (TRACE && lane == 0) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        trace[b * 64 + w * 32 + 31] = sm;
    }
    LU4B_MARK(0)
    double xv = t < n ? __ldg(X + b * n + t) : 0.0;
    int bad = 0;  // a multiplier with !(|m| < 1) seen by this thread
    if constexpr (CLASSIFY) {
        // lazymat/rewrite.py:146-173 over _analyze (lazymat/_loops.py:15-34)
        double(*sAt)[N + 1] = reinterpret_cast<double(*)[N + 1]>(smraw);
        __shared__ unsigned s_lb[2], s_ub[2], s_as[2];
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
            lb = max(lb, s_lb[1]);
            ub = max(ub, s_ub[1]);
            asym |= s_as[1];
            const unsigned lim = (unsigned)(n / 4 > 4 ? n / 4 : 4);
            int c = 0;
            if (lb + ub <= lim) c = 1;
            else if (lb == 0) c = 2;
            else if (ub == 0) c = 3;
            else if (!asym) c = 4;
            cls[b] = c;
        }
        __syncthreads();  // the transpose aliases the factorisation's buffers
    }

#pragma unroll
    for (int kb = 0; kb < NB; ++kb) {
        const int c0 = kb * KB, par = kb & 1;
        const int Rw = N - c0 - KB;  // rest columns right of the block (static)
        LU4B_MARK(1 + 3 * kb)
        // (a) the diagonal block, by the warp that holds rows c0..c0+7
        if (w == (c0 >> 5)) {
            const int ls = t - c0;  // 0..7 on the diagonal rows
            const bool diag = (unsigned)ls < (unsigned)KB;
#pragma unroll
            for (int s = 0; s < KB; ++s) {
                // the pivot row of step c0+s is final: its owner publishes it
                // (U11 row s) and the warp reads it back as broadcasts
                if (ls == s) {
#pragma unroll
                    for (int s2 = s; s2 < KB; ++s2) f.U11[s][s2] = r[c0 + s2];
                }
                __syncwarp();
                const double pv = f.U11[s][s];
                double u[KB];
#pragma unroll
                for (int s2 = s + 1; s2 < KB; ++s2) u[s2] = f.U11[s][s2];
                // branch-free: every lane divides, only the block's rows
                // below the pivot keep the result
                const bool act = diag && ls > s;
                const double m = __ddiv_rn(r[c0 + s], pv);
                bad |= act & !(fabs(m) < 1.0);
                if (act) f.Ld[ls][s] = m;
#pragma unroll
                for (int s2 = s + 1; s2 < KB; ++s2) {
                    const double v = __dsub_rn(r[c0 + s2], __dmul_rn(m, u[s2]));
                    r[c0 + s2] = act ? v : r[c0 + s2];
                }
            }
            if (diag) {
                double ukk = r[c0];
#pragma unroll
                for (int s2 = 1; s2 < KB; ++s2)
                    if (ls == s2) ukk = r[c0 + s2];
                f.yd[c0 + ls] = __drcp_rn(ukk);  // U[k,k] is final: its reciprocal for (b) and the back sweep
#pragma unroll
                for (int s2 = 0; s2 < KB; ++s2)
                    if (s2 >= ls) f.Us[upacked_off(c0 + ls) + s2 - ls] = r[c0 + s2];
                double2 *dst = reinterpret_cast<double2 *>(f.Ub[par][ls]);
#pragma unroll
                for (int j = 0; j < Rw; j += 2) dst[j >> 1] = make_double2(r[c0 + KB + j], r[c0 + KB + j + 1]);
                f.Ub[par][ls][Rw] = xv;
            }
        }
        __syncthreads();
        LU4B_MARK(2 + 3 * kb)
        // (c) U rows of the block, one thread per rest column (the last one is y)
        if (t <= Rw) {
#pragma unroll
            for (int s = 0; s < KB; ++s) {
                double u = f.Ub[par][s][t];
#pragma unroll
                for (int s2 = 0; s2 < s; ++s2) u = __dsub_rn(u, __dmul_rn(f.Ld[s][s2], f.Ub[par][s2][t]));
                f.Ub[par][s][t] = u;  // this thread's column only: read back by later s
                if (t < Rw)
                    f.Us[upacked_off(c0 + s) + KB - s + t] = u;
                else
                    f.xs[c0 + s] = u;
            }
        }
        if (TRACE && lane == 0 && kb < 4) trace[b * 64 + w * 32 + 27 + kb] = clock64();  // (c) done
        // (b) the rows below: divide and eliminate the own panel values
        if (t >= c0 + KB) {
#pragma unroll
            for (int s = 0; s < KB; ++s) {
                const CertDiv dv = cdiv_prep(f.U11[s][s], f.yd[c0 + s]);
                const double m = cdiv(r[c0 + s], dv, bad);
                bad |= !(fabs(m) < 1.0);
                f.Lr[s][t] = m;
#pragma unroll
                for (int s2 = s + 1; s2 < KB; ++s2) r[c0 + s2] = __dsub_rn(r[c0 + s2], __dmul_rn(m, f.U11[s][s2]));
            }
        }
        __syncthreads();
        LU4B_MARK(3 + 3 * kb)
        // (d) the block's deferred updates of the rows below, in step order
        if (t >= c0 + KB) {
#pragma unroll 1
            for (int s = 0; s < KB; ++s) {
                const double l = f.Lr[s][t];
                const double2 *U2 = reinterpret_cast<const double2 *>(f.Ub[par][s]);
#pragma unroll
                for (int j = 0; j < Rw; j += 2) {
                    const double2 u = U2[j >> 1];
                    r[c0 + KB + j] = __dsub_rn(r[c0 + KB + j], __dmul_rn(l, u.x));
                    r[c0 + KB + j + 1] = __dsub_rn(r[c0 + KB + j + 1], __dmul_rn(l, u.y));
                }
                xv = __dsub_rn(xv, __dmul_rn(l, f.Ub[par][s][Rw]));
            }
        }
    }
    if (__syncthreads_or(bad)) {  // pivoting could swap somewhere: the pivoting kernel redoes this system
        if (t == 0) {
            info[b] = -1;
            redo_list[atomicAdd(redo_count, 1)] = (int)b;
        }
        return;
    }
    // back sweep (lazymat/_loops.py:254-258) by warp 0 alone, no block
    // barrier: lane l holds positions l and l + 32; per step j (descending)
    // the owner divides (certified quotient, reciprocal of U[j,j] from (a)),
    // one shuffle hands x_j to the warp, every position above j subtracts
    // U[i,j] x_j -- each c_i sees j = n-1, ..., i+1 in the reference's order.
    LU4B_MARK(25)
    double c0v = 0.0, c1v = 0.0;
    if (w == 0) {
        const int i0 = lane, i1 = lane + 32;
        const CertDiv d0 = cdiv_prep(i0 < n ? f.Us[upacked_off(i0)] : 1.0, i0 < n ? f.yd[i0] : 1.0);
        const CertDiv d1 = cdiv_prep(i1 < n ? f.Us[upacked_off(i1)] : 1.0, i1 < n ? f.yd[i1] : 1.0);
        const int off0 = upacked_off(i0) - i0, off1 = upacked_off(i1) - i1;  // U[i, j] at off + j
        c0v = i0 < n ? f.xs[i0] : 0.0;
        c1v = i1 < n ? f.xs[i1] : 0.0;
#pragma unroll 1
        for (int j = (int)n - 1; j >= 32; --j) {  // owner in the upper half
            int bq = 0;
            const double q = cdiv(c1v, d1, bq);
            bad |= (i1 == j) & bq;
            const double xj = __shfl_sync(MASK, q, j - 32);
            const double up1 = __dsub_rn(c1v, __dmul_rn(f.Us[off1 + j], xj));
            c1v = i1 == j ? xj : (i1 < j ? up1 : c1v);
            c0v = __dsub_rn(c0v, __dmul_rn(f.Us[off0 + j], xj));  // every lower position is above j
        }
#pragma unroll 1
        for (int j = min((int)n, 32) - 1; j >= 0; --j) {
            int bq = 0;
            const double q = cdiv(c0v, d0, bq);
            bad |= (i0 == j) & bq;
            const double xj = __shfl_sync(MASK, q, j);
            const double up0 = __dsub_rn(c0v, __dmul_rn(f.Us[off0 + j], xj));
            c0v = i0 == j ? xj : (i0 < j ? up0 : c0v);
        }
    }
    if (__syncthreads_or(bad)) {  // an uncertified quotient: the pivoting kernel redoes the system
        if (t == 0) {
            info[b] = -1;
            redo_list[atomicAdd(redo_count, 1)] = (int)b;
        }
        return;
    }
    LU4B_MARK(26)
    if (w != 0) return;
    if (lane == 0) info[b] = 0;
    if (piv) {
        if (lane < n) piv[b * n + lane] = lane;
        if (lane + 32 < n) piv[b * n + lane + 32] = lane + 32;
    }
    if (lane < n) X[b * n + lane] = c0v;
    if (lane + 32 < n) X[b * n + lane + 32] = c1v;
}
#undef LU4B_MARK

// ---------------------------------------------------------------------------
// Pivot-free WAVEFRONT kernel for 32 < n <= 64 (config 4b; default).  The
// same proof of the reference's identity pivots (every multiplier
// |m| < 1, else the pivoting kernel redoes the system) as lu_batched_nopiv
// above, but the elimination is the unblocked right-looking loop of the
// reference itself, with no block barrier at all: thread t owns row t
// (shifted registers, rolled in blocks of 8 columns like lu_batched_shift);
// row k is final once its owner has applied step k-1, and the owner
// publishes it (U[k, k:] and y_k) to shared memory right then.  Consumers
// in the same warp see it after a __syncwarp; warp 1 waits for warp 0's
// rows (k < 32) on a per-row flag, and warp 0 leaves the loop once all its
// rows are final (k >= 31).  The back sweep is the mirror image: the owner
// of position j divides (certified quotient with the reciprocal of U[j,j]
// computed off the chain), shuffles x_j to its warp and, for j >= 32, hands
// it to warp 0 through a flag.  Per step the chain is the division and the
// owner's own update; the update of the rest of the row overlaps the next
// rows' steps in the other warp.
template <bool CLASSIFY>
__global__ void __launch_bounds__(64, 6)
    lu_batched_wave(int64_t n, int64_t batch, const double *__restrict__ A, double *__restrict__ X,
                    int64_t *__restrict__ piv, int32_t *__restrict__ info, int32_t *__restrict__ cls,
                    int *__restrict__ redo_list, int *__restrict__ redo_count) {
    constexpr int N = 64, KB = 8;
    constexpr unsigned MASK = 0xffffffffu;
    constexpr size_t SAT = CLASSIFY ? sizeof(double) * N * (N + 1) : 0;
    constexpr size_t SU = sizeof(double) * N * N;
    constexpr size_t SMB = SU > SAT ? SU : SAT;
    __shared__ __align__(16) unsigned char smraw[SMB];
    __shared__ double ys[N], xb[N];
    __shared__ int rflag[N], xflag[N];
    double *Us = reinterpret_cast<double *>(smraw);  // row k: U[k, k + i] at Us[k * N + i]

    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int64_t b = blockIdx.x;
    const double *Ab = A + b * n * n;
    double r[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        if (t < n && j < n)
            r[j] = __ldg(Ab + t + (int64_t)j * n);
        else
            r[j] = (t == j) ? 1.0 : 0.0;  // identity padding: pivot-free by construction
    }
    double xv = t < n ? __ldg(X + b * n + t) : 0.0;
    int bad = 0;
    rflag[t] = 0;
    xflag[t] = 0;
    if constexpr (CLASSIFY) {
        // lazymat/rewrite.py:146-173 over _analyze (lazymat/_loops.py:15-34)
        double(*sAt)[N + 1] = reinterpret_cast<double(*)[N + 1]>(smraw);
        __shared__ unsigned s_lb[2], s_ub[2], s_as[2];
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
            lb = max(lb, s_lb[1]);
            ub = max(ub, s_ub[1]);
            asym |= s_as[1];
            const unsigned lim = (unsigned)(n / 4 > 4 ? n / 4 : 4);
            int c = 0;
            if (lb + ub <= lim) c = 1;
            else if (lb == 0) c = 2;
            else if (ub == 0) c = 3;
            else if (!asym) c = 4;
            cls[b] = c;
        }
    }
    __syncthreads();  // flags cleared (and the transpose done) before anything is published
    // row 0 is final from the start
    if (t == 0) {
        double2 *dst = reinterpret_cast<double2 *>(Us);
#pragma unroll
        for (int i = 0; i < N; i += 2) dst[i >> 1] = make_double2(r[i], r[i + 1]);
        ys[0] = xv;
        __threadfence_block();
        *reinterpret_cast<volatile int *>(&rflag[0]) = 1;
    }
#pragma unroll
    for (int kb = 0; kb < N / KB; ++kb) {
        constexpr int dummy = 0;
        (void)dummy;
        const int L = N - kb * KB;  // static after unrolling: slots this block's code updates
        if (w == 0 && kb * KB >= 32) break;  // every row of warp 0 is final
#pragma unroll 1
        for (int kk = 0; kk < KB; ++kk) {
            const int k = kb * KB + kk;
            if (w == 0 && k >= 31) break;
            if (w == 1 && k < 32) {  // row k lives in warp 0: wait for its flag
                while (*reinterpret_cast<volatile int *>(&rflag[k]) == 0) {
                }
                __threadfence_block();
            }
            __syncwarp();
            if (t > k) {
                const double *Uk = Us + k * N;
                const double2 *U2 = reinterpret_cast<const double2 *>(Uk);
                const double m = __ddiv_rn(r[0], Uk[0]);
                bad |= !(fabs(m) < 1.0);
#pragma unroll
                for (int i = 1; i < L; ++i) {
                    const double2 u = U2[i >> 1];
                    r[i - 1] = __dsub_rn(r[i], __dmul_rn(m, (i & 1) ? u.y : u.x));
                }
                xv = __dsub_rn(xv, __dmul_rn(m, ys[k]));
                if (t == k + 1) {  // this row is final now: publish U[k+1, k+1:] and y_{k+1}
                    double2 *dst = reinterpret_cast<double2 *>(Us + (k + 1) * N);
#pragma unroll
                    for (int i = 0; i < L; i += 2) dst[i >> 1] = make_double2(r[i], r[i + 1]);
                    ys[k + 1] = xv;
                    __threadfence_block();
                    *reinterpret_cast<volatile int *>(&rflag[k + 1]) = 1;
                }
            }
        }
    }
    if (__syncthreads_or(bad)) {  // pivoting could swap somewhere: the pivoting kernel redoes this system
        if (t == 0) {
            info[b] = -1;
            redo_list[atomicAdd(redo_count, 1)] = (int)b;
        }
        return;
    }
    // back sweep (lazymat/_loops.py:254-258): thread t holds position t
    const double utt = t < n ? Us[t * N] : 1.0;
    const CertDiv dd = cdiv_prep(utt, __drcp_rn(utt));
    double c = xv;  // y_t
    const int nn = (int)n;
    if (w == 1) {
#pragma unroll 1
        for (int j = nn - 1; j >= 32; --j) {
            int bq = 0;
            const double q = cdiv(c, dd, bq);
            bad |= (t == j) & bq;
            const double xj = __shfl_sync(MASK, q, j & 31);
            if (t == j) {
                c = xj;
                xb[j] = xj;
                __threadfence_block();
                *reinterpret_cast<volatile int *>(&xflag[j]) = 1;
            } else if (t < j) {
                c = __dsub_rn(c, __dmul_rn(Us[t * N + (j - t)], xj));
            }
        }
    } else {
#pragma unroll 1
        for (int j = nn - 1; j >= 0; --j) {
            double xj;
            if (j >= 32) {
                while (*reinterpret_cast<volatile int *>(&xflag[j]) == 0) {
                }
                __threadfence_block();
                xj = xb[j];
            } else {
                int bq = 0;
                const double q = cdiv(c, dd, bq);
                bad |= (t == j) & bq;
                xj = __shfl_sync(MASK, q, j & 31);
            }
            if (t == j)
                c = xj;
            else if (t < j)
                c = __dsub_rn(c, __dmul_rn(Us[t * N + (j - t)], xj));
        }
    }
    if (__syncthreads_or(bad)) {  // an uncertified quotient: the pivoting kernel redoes the system
        if (t == 0) {
            info[b] = -1;
            redo_list[atomicAdd(redo_count, 1)] = (int)b;
        }
        return;
    }
    if (t == 0) info[b] = 0;
    if (piv && t < n) piv[b * n + t] = t;
    if (t < n) X[b * n + t] = c;
}

}  // namespace lm

using namespace lm;

// Solve-only kernels: for 32 < n <= 64 the pivot-free fast path
// ("nopiv", default; "wave" = LM_BATCHED_LU=wave, the unblocked wavefront
// variant, 278 vs 257 us) followed by the pivoting kernel on the systems it
// could not prove; "shift" (LM_BATCHED_LU=shift: the pivoting kernel on
// every system) and "rows" (LM_BATCHED_LU=rows or LM_BATCHED_LU_UNROLLED=1:
// the unrolled kernel, also the one that returns the LU factors).
static int batched_kernel_choice() {
    static const int choice = [] {
        const char *u = getenv("LM_BATCHED_LU_UNROLLED");
        if (u && u[0] == '1') return 2;
        const char *e = getenv("LM_BATCHED_LU");
        if (e && !strcmp(e, "rows")) return 2;
        if (e && !strcmp(e, "shift")) return 1;
        if (e && !strcmp(e, "wave")) return 3;
        return 0;
    }();
    return choice;
}

// diagnostics: the LM_4B_TRACE buffer (device pointer, 64 x 65536 int64), or null
static long long *lu4b_trace_buffer() {
    static long long *p = [] {
        long long *q = nullptr;
        if (getenv("LM_4B_TRACE") && cudaMalloc(&q, sizeof(long long) * 64 * 65536) != cudaSuccess) q = nullptr;
        return q;
    }();
    return p;
}
extern "C" void *lm_debug_lu4b_trace(void) { return lu4b_trace_buffer(); }

template <bool CLASSIFY>
static int launch_batched(int64_t n, int64_t batch, const double *A, double *X, double *LU, int64_t *d_piv,
                          int32_t *d_info, int32_t *d_cls, cudaStream_t s) {
    const int choice = batched_kernel_choice();
    if (LU == nullptr && n > 32 && (choice == 0 || choice == 3)) {
        // the fast path lists the systems it cannot prove; a small grid of
        // the pivoting kernel then solves exactly those
        Scratch redo;
        if (int rc = redo.alloc(sizeof(int) * (size_t)(batch + 1), s)) return rc;
        int *cnt = redo.as<int>(), *list = cnt + 1;
        LM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), s));
        if (choice == 3) {
            lu_batched_wave<CLASSIFY><<<(unsigned)batch, 64, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls, list, cnt);
            note_variant("wave64");
        } else {
            // six 64-thread systems per SM need ~200 KB of shared memory: ask
            // for the largest carveout (the default one fits fewer CTAs)
            if (int rc = func_attrs(lu_batched_nopiv<CLASSIFY>, 0, 100)) return rc;
            long long *trace = lu4b_trace_buffer();
            if (trace && batch <= 65536)
                lu_batched_nopiv<CLASSIFY, true>
                    <<<(unsigned)batch, 64, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls, list, cnt, trace);
            else
                lu_batched_nopiv<CLASSIFY><<<(unsigned)batch, 64, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls, list, cnt);
            note_variant("nopiv64");
        }
        static const bool noredo = getenv("LM_4B_NOREDO") != nullptr;  // diagnostics: leave info = -1 visible
        if (!noredo) {
            if (int rc = func_attrs(lu_batched_shift<64, 8, CLASSIFY>, 0, 100)) return rc;
            const int64_t g = batch < 6 * (int64_t)num_sms() ? batch : 6 * (int64_t)num_sms();
            lu_batched_shift<64, 8, CLASSIFY><<<(unsigned)g, 64, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls, list, cnt);
        }
        LM_LAUNCHED(2);
        return 0;
    }
    if (LU == nullptr && choice <= 1) {
        if (n <= 16)
            lu_batched_shift<16, 8, CLASSIFY><<<(unsigned)batch, 16, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls, nullptr, nullptr);
        else if (n <= 32)
            lu_batched_shift<32, 8, CLASSIFY><<<(unsigned)batch, 32, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls, nullptr, nullptr);
        else
            lu_batched_shift<64, 8, CLASSIFY><<<(unsigned)batch, 64, 0, s>>>(n, batch, A, X, d_piv, d_info, d_cls, nullptr, nullptr);
        note_variant(n > 32 ? "shift64" : "shift");
    } else {
        if (n <= 16)
            lu_batched_rows<16, CLASSIFY><<<(unsigned)batch, 16, 0, s>>>(n, batch, A, X, LU, d_piv, d_info, d_cls);
        else if (n <= 32)
            lu_batched_rows<32, CLASSIFY><<<(unsigned)batch, 32, 0, s>>>(n, batch, A, X, LU, d_piv, d_info, d_cls);
        else
            lu_batched_rows<64, CLASSIFY><<<(unsigned)batch, 64, 0, s>>>(n, batch, A, X, LU, d_piv, d_info, d_cls);
        note_variant("rows");
    }
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

extern "C" int lm_solve_batched_classified_from(int dtype, int64_t n, int64_t batch, const void *a, const void *b,
                                                void *x, int32_t *d_cls, int32_t *d_info, void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64, "solve_batched_classified_from: f64 only");
    LM_REQUIRE(n >= 1 && n <= 64, "solve_batched_classified_from: 1 <= n <= 64 (got %lld)", (long long)n);
    if (batch == 0) return 0;
    LM_REQUIRE(batch <= 0x7fffffff, "solve_batched_classified_from: batch too large");
    if (b != x)
        LM_CUDA(cudaMemcpyAsync(x, b, sizeof(double) * (size_t)(n * batch), cudaMemcpyDeviceToDevice,
                                as_stream(stream)));
    return launch_batched<true>(n, batch, (const double *)a, (double *)x, nullptr, nullptr, d_info, d_cls,
                                as_stream(stream));
}
