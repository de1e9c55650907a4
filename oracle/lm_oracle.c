/*
 * lm_oracle.c -- CPU restatement of the reference's compute loops.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product package
 * (paper_2502_03000_b200) never imports, links or calls anything here.
 *
 * Every function restates one numba loop nest of the reference
 * (/root/reference/pkg/src/lazymat/_loops.py) with the SAME per-element
 * operation order, one IEEE rounding per operation and no FMA
 * contraction (build with -ffp-contract=off; numba does not contract,
 * SURVEY.md finding 9).  It is therefore bit-identical to the reference
 * on every input -- pinned by tests/test_oracle_golden.py against golden
 * vectors produced by running the reference itself (tests/golden/).
 *
 * Operands are strided 2-D views: element (i,j) lives at
 * p[i*rs + j*cs] (column-major F-order is rs=1, cs=rows; a numpy .T view
 * swaps them).  1-D vectors are (p, n, stride).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double *p;
    int64_t rows, cols, rs, cs;
} lmo_view;

typedef struct {
    double *p;
    int64_t n, stride;
} lmo_vec;

#define AT(v, i, j) ((v).p[(int64_t)(i) * (v).rs + (int64_t)(j) * (v).cs])
#define VT(v, i) ((v).p[(int64_t)(i) * (v).stride])

/* _loops.py:15-34 (_analyze): one pass, j outer / i inner; bandwidths over
 * nonzeros, exact symmetry A[i,j]==A[j,i] for i<j when square. */
void lmo_analyze(lmo_view a, int square, int64_t *lbw, int64_t *ubw, int *sym)
{
    int64_t l = 0, u = 0;
    int s = 1;
    for (int64_t j = 0; j < a.cols; ++j) {
        for (int64_t i = 0; i < a.rows; ++i) {
            double v = AT(a, i, j);
            if (v != 0.0) {
                int64_t d = i - j;
                if (d > 0) {
                    if (d > l) l = d;
                } else if (-d > u) {
                    u = -d;
                }
            }
            if (square && i < j && v != AT(a, j, i)) s = 0;
        }
    }
    *lbw = l;
    *ubw = u;
    *sym = s;
}

/* _loops.py:37-84 (_fused1.._fused4, _fused_axpy): per element
 * acc = c0*s0; acc = acc + ck*sk for k = 1..n-1 (left to right). */
void lmo_fused(int n, const double *coeffs, const lmo_view *srcs, lmo_view out)
{
    for (int64_t j = 0; j < out.cols; ++j)
        for (int64_t i = 0; i < out.rows; ++i) {
            double acc = coeffs[0] * AT(srcs[0], i, j);
            for (int k = 1; k < n; ++k) acc = acc + coeffs[k] * AT(srcs[k], i, j);
            AT(out, i, j) = acc;
        }
}

/* Extension (no reference counterpart; SURVEY.md finding 4): postfix
 * element-wise program over sources, one IEEE rounding per node, the
 * semantics of naive_evaluate (expr.py:304-391) applied per element.
 * Encoding is shared with paper_2502_03000_b200/elementwise.py:
 *   op 0 LOAD k | 1 CONST idx | 2 ADD | 3 SUB | 4 MUL | 5 DIV | 6 ABS | 7 NEG */
int lmo_program(int nins, const int32_t *ops, const int32_t *args,
                const double *consts, const lmo_view *srcs, lmo_view out)
{
    double st[64];
    for (int64_t j = 0; j < out.cols; ++j)
        for (int64_t i = 0; i < out.rows; ++i) {
            int sp = 0;
            for (int q = 0; q < nins; ++q) {
                switch (ops[q]) {
                case 0: st[sp++] = AT(srcs[args[q]], i, j); break;
                case 1: st[sp++] = consts[args[q]]; break;
                case 2: sp--; st[sp - 1] = st[sp - 1] + st[sp]; break;
                case 3: sp--; st[sp - 1] = st[sp - 1] - st[sp]; break;
                case 4: sp--; st[sp - 1] = st[sp - 1] * st[sp]; break;
                case 5: sp--; st[sp - 1] = st[sp - 1] / st[sp]; break;
                case 6: st[sp - 1] = fabs(st[sp - 1]); break;
                case 7: st[sp - 1] = -st[sp - 1]; break;
                default: return -1;
                }
                if (sp <= 0 || sp > 63) return -2;
            }
            if (sp != 1) return -3;
            AT(out, i, j) = st[0];
        }
    return 0;
}

/* _loops.py:87-98 (_gemm): j-k-i; out zeroed, then out += A[i,k]*B[k,j]
 * with k ascending. */
void lmo_gemm(lmo_view a, lmo_view b, lmo_view out)
{
    int64_t p = a.rows, q = a.cols, r = b.cols;
    for (int64_t j = 0; j < r; ++j) {
        for (int64_t i = 0; i < p; ++i) AT(out, i, j) = 0.0;
        for (int64_t k = 0; k < q; ++k) {
            double bk = AT(b, k, j);
            for (int64_t i = 0; i < p; ++i) AT(out, i, j) = AT(out, i, j) + AT(a, i, k) * bk;
        }
    }
}

/* _loops.py:101-110 (_gemv) and :113-121 (_gemv_t). */
void lmo_gemv(lmo_view a, lmo_vec x, lmo_vec out, int trans)
{
    if (!trans) {
        for (int64_t i = 0; i < a.rows; ++i) VT(out, i) = 0.0;
        for (int64_t k = 0; k < a.cols; ++k) {
            double xk = VT(x, k);
            for (int64_t i = 0; i < a.rows; ++i) VT(out, i) = VT(out, i) + AT(a, i, k) * xk;
        }
    } else {
        for (int64_t j = 0; j < a.cols; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < a.rows; ++k) acc = acc + AT(a, k, j) * VT(x, k);
            VT(out, j) = acc;
        }
    }
}

/* _loops.py:124-141 (_syrk): upper triangle incl. diagonal with t
 * ascending, then bitwise mirror to the lower triangle. */
void lmo_syrk(lmo_view a, lmo_view out)
{
    int64_t n = a.rows, k = a.cols;
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i <= j; ++i) AT(out, i, j) = 0.0;
        for (int64_t t = 0; t < k; ++t) {
            double ajt = AT(a, j, t);
            for (int64_t i = 0; i <= j; ++i) AT(out, i, j) = AT(out, i, j) + AT(a, i, t) * ajt;
        }
    }
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = j + 1; i < n; ++i) AT(out, i, j) = AT(out, j, i);
}

/* _loops.py:144-158 (_diag_scale_left / _diag_scale_right). */
void lmo_diag_scale(lmo_vec d, lmo_view b, int right, lmo_view out)
{
    for (int64_t j = 0; j < b.cols; ++j) {
        double dj = right ? VT(d, j) : 0.0;
        for (int64_t i = 0; i < b.rows; ++i)
            AT(out, i, j) = right ? AT(b, i, j) * dj : VT(d, i) * AT(b, i, j);
    }
}

/* _loops.py:161-176 (_diag_of_product): out_d[i] = sum_k A[i,k]*B[k,i],
 * k ascending per element (the 8-row blocking does not change order). */
void lmo_diag_of_product(lmo_view a, lmo_view b, lmo_vec out)
{
    int64_t p = a.rows, q = a.cols;
    for (int64_t i0 = 0; i0 < p; i0 += 8) {
        int64_t ihi = i0 + 8 < p ? i0 + 8 : p;
        for (int64_t i = i0; i < ihi; ++i) VT(out, i) = 0.0;
        for (int64_t k = 0; k < q; ++k)
            for (int64_t i = i0; i < ihi; ++i) VT(out, i) = VT(out, i) + AT(a, i, k) * AT(b, k, i);
    }
}

/* _loops.py:179-188 (_trace_of_product): diag_of_product, then an
 * ascending-i sum starting from 0.0. */
double lmo_trace_of_product(lmo_view a, lmo_view b)
{
    int64_t p = a.rows;
    double *d = (double *)malloc(sizeof(double) * (size_t)(p > 0 ? p : 1));
    lmo_vec dv = {d, p, 1};
    lmo_diag_of_product(a, b, dv);
    double acc = 0.0;
    for (int64_t i = 0; i < p; ++i) acc = acc + d[i];
    free(d);
    return acc;
}

/* _loops.py:191-197 (_triple_diag_dot): acc += (a[i]*d[i])*c[i]. */
double lmo_triple_diag_dot(lmo_vec a, lmo_vec d, lmo_vec c)
{
    double acc = 0.0;
    for (int64_t i = 0; i < a.n; ++i) acc = acc + VT(a, i) * VT(d, i) * VT(c, i);
    return acc;
}

/* _loops.py:200-236 (_lu_factor): unblocked right-looking LU with
 * partial pivoting on an F-order n x n buffer (leading dim n).  Strict >
 * in the pivot search (lowest index wins ties); full-row swap; returns
 * failing column + 1 on an exactly-zero pivot. */
int lmo_lu_factor(double *lu, int64_t n, int64_t *piv)
{
    double *scratch = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
#define LU(i, j) lu[(int64_t)(i) + (int64_t)(j) * n]
    for (int64_t k = 0; k < n; ++k) {
        int64_t p = k;
        double best = fabs(LU(k, k));
        for (int64_t i = k + 1; i < n; ++i) {
            double v = fabs(LU(i, k));
            if (v > best) {
                best = v;
                p = i;
            }
        }
        piv[k] = p;
        if (LU(p, k) == 0.0) {
            free(scratch);
            return (int)(k + 1);
        }
        if (p != k)
            for (int64_t j = 0; j < n; ++j) {
                double t = LU(k, j);
                LU(k, j) = LU(p, j);
                LU(p, j) = t;
            }
        double pv = LU(k, k);
        for (int64_t i = k + 1; i < n; ++i) {
            double m = LU(i, k) / pv;
            LU(i, k) = m;
            scratch[i] = m;
        }
        for (int64_t j = k + 1; j < n; ++j) {
            double f = LU(k, j);
            for (int64_t i = k + 1; i < n; ++i) LU(i, j) = LU(i, j) - scratch[i] * f;
        }
    }
#undef LU
    free(scratch);
    return 0;
}

/* _loops.py:239-259 (_lu_solve_inplace): per RHS column: sequential
 * pivot swaps, unit-lower forward substitution, upper back substitution. */
void lmo_lu_solve(const double *lu, int64_t n, const int64_t *piv, double *x, int64_t ldx, int64_t m)
{
#define LU(i, j) lu[(int64_t)(i) + (int64_t)(j) * n]
#define X(i, c) x[(int64_t)(i) + (int64_t)(c) * ldx]
    for (int64_t c = 0; c < m; ++c) {
        for (int64_t i = 0; i < n; ++i) {
            int64_t p = piv[i];
            if (p != i) {
                double t = X(i, c);
                X(i, c) = X(p, c);
                X(p, c) = t;
            }
        }
        for (int64_t j = 0; j < n; ++j) {
            double yj = X(j, c);
            for (int64_t i = j + 1; i < n; ++i) X(i, c) = X(i, c) - LU(i, j) * yj;
        }
        for (int64_t j = n - 1; j >= 0; --j) {
            X(j, c) = X(j, c) / LU(j, j);
            double xj = X(j, c);
            for (int64_t i = 0; i < j; ++i) X(i, c) = X(i, c) - LU(i, j) * xj;
        }
    }
#undef LU
#undef X
}

/* _loops.py:262-283 (_pack_band): A(i,j) -> AB[kl+ku+i-j, j], with kl
 * zero fill rows on top; AB is F-order with leading dim ldab = 2kl+ku+1. */
void lmo_pack_band(lmo_view a, double *ab, int64_t ldab, int64_t kl, int64_t ku)
{
    int64_t n = a.rows, kv = kl + ku;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t r = 0; r < ldab; ++r) ab[r + j * ldab] = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        int64_t lo = j - ku < 0 ? 0 : j - ku;
        int64_t hi = j + kl > n - 1 ? n - 1 : j + kl;
        for (int64_t i = lo; i <= hi; ++i) ab[kv + i - j + j * ldab] = AT(a, i, j);
    }
}

/* _loops.py:286-330 (_band_factor): banded LU with partial pivoting. */
int lmo_band_factor(double *ab, int64_t ldab, int64_t n, int64_t *piv, int64_t kl, int64_t ku)
{
#define AB(r, c) ab[(int64_t)(r) + (int64_t)(c) * ldab]
    int64_t kv = kl + ku, ju = 0;
    for (int64_t j = 0; j < n; ++j) {
        int64_t km = kl < n - 1 - j ? kl : n - 1 - j;
        int64_t jp = 0;
        double best = fabs(AB(kv, j));
        for (int64_t t = 1; t <= km; ++t) {
            double v = fabs(AB(kv + t, j));
            if (v > best) {
                best = v;
                jp = t;
            }
        }
        piv[j] = j + jp;
        if (AB(kv + jp, j) == 0.0) return (int)(j + 1);
        int64_t cand = j + ku + jp;
        if (cand > ju) ju = cand;
        if (ju > n - 1) ju = n - 1;
        if (jp != 0)
            for (int64_t jj = j; jj <= ju; ++jj) {
                double t1 = AB(kv + j - jj, jj);
                AB(kv + j - jj, jj) = AB(kv + j + jp - jj, jj);
                AB(kv + j + jp - jj, jj) = t1;
            }
        if (km > 0) {
            double pv = AB(kv, j);
            for (int64_t t = 1; t <= km; ++t) AB(kv + t, j) = AB(kv + t, j) / pv;
            for (int64_t jj = j + 1; jj <= ju; ++jj) {
                double f = AB(kv + j - jj, jj);
                if (f != 0.0)
                    for (int64_t t = 1; t <= km; ++t)
                        AB(kv + j - jj + t, jj) = AB(kv + j - jj + t, jj) - AB(kv + t, j) * f;
            }
        }
    }
#undef AB
    return 0;
}

/* _loops.py:333-360 (_band_solve_inplace). */
void lmo_band_solve(const double *ab, int64_t ldab, int64_t n, const int64_t *piv, double *x, int64_t ldx,
                    int64_t m, int64_t kl, int64_t ku)
{
#define AB(r, c) ab[(int64_t)(r) + (int64_t)(c) * ldab]
#define X(i, c) x[(int64_t)(i) + (int64_t)(c) * ldx]
    int64_t kv = kl + ku;
    for (int64_t c = 0; c < m; ++c) {
        for (int64_t j = 0; j < n; ++j) {
            int64_t p = piv[j];
            if (p != j) {
                double t1 = X(j, c);
                X(j, c) = X(p, c);
                X(p, c) = t1;
            }
            int64_t km = kl < n - 1 - j ? kl : n - 1 - j;
            double xj = X(j, c);
            if (xj != 0.0)
                for (int64_t t = 1; t <= km; ++t) X(j + t, c) = X(j + t, c) - AB(kv + t, j) * xj;
        }
        for (int64_t j = n - 1; j >= 0; --j) {
            int64_t u = kv < n - 1 - j ? kv : n - 1 - j;
            double acc = X(j, c);
            for (int64_t t = 1; t <= u; ++t) acc = acc - AB(kv - t, j + t) * X(j + t, c);
            X(j, c) = acc / AB(kv, j);
        }
    }
#undef AB
#undef X
}

/* _loops.py:363-388 (_tri_solve_inplace): zero-diagonal check first,
 * then column-oriented back/forward substitution skipping zero x_j. */
int lmo_tri_solve(lmo_view a, double *x, int64_t ldx, int64_t m, int upper)
{
#define X(i, c) x[(int64_t)(i) + (int64_t)(c) * ldx]
    int64_t n = a.rows;
    for (int64_t j = 0; j < n; ++j)
        if (AT(a, j, j) == 0.0) return (int)(j + 1);
    for (int64_t c = 0; c < m; ++c) {
        if (upper) {
            for (int64_t j = n - 1; j >= 0; --j) {
                X(j, c) = X(j, c) / AT(a, j, j);
                double xj = X(j, c);
                if (xj != 0.0)
                    for (int64_t i = 0; i < j; ++i) X(i, c) = X(i, c) - AT(a, i, j) * xj;
            }
        } else {
            for (int64_t j = 0; j < n; ++j) {
                X(j, c) = X(j, c) / AT(a, j, j);
                double xj = X(j, c);
                if (xj != 0.0)
                    for (int64_t i = j + 1; i < n; ++i) X(i, c) = X(i, c) - AT(a, i, j) * xj;
            }
        }
    }
#undef X
    return 0;
}

/* _loops.py:391-396 (_transpose_copy). */
void lmo_transpose_copy(lmo_view a, lmo_view out)
{
    for (int64_t j = 0; j < a.rows; ++j)
        for (int64_t i = 0; i < a.cols; ++i) AT(out, i, j) = AT(a, j, i);
}

/* _loops.py:399-407 (_diag_materialise). */
void lmo_diag_materialise(lmo_vec d, lmo_view out)
{
    for (int64_t j = 0; j < out.cols; ++j)
        for (int64_t i = 0; i < out.rows; ++i) AT(out, i, j) = 0.0;
    for (int64_t i = 0; i < out.rows; ++i) AT(out, i, i) = VT(d, i);
}
