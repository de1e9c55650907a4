/*
 * lm_b200.h -- C ABI of the B200 (sm_100a) evaluation backend.
 *
 * This library replaces the reference's compute seam, the numba loop
 * module lazymat/_loops.py (/root/reference/pkg/src/lazymat/_loops.py:15-407),
 * one entry point per loop family.  The contract layer above it
 * (checks, trace events, flop counts, rc -> exception mapping;
 * lazymat/kernels.py) is mirrored in Python by
 * paper_2502_03000_b200/kernels.py and calls these functions through
 * ctypes (paper_2502_03000_b200/_native.py).
 *
 * Conventions:
 *  - All pointers are DEVICE pointers owned by the caller; the library
 *    never frees caller memory.  Internal scratch comes from the
 *    stream-ordered allocator (cudaMallocAsync) on the caller's stream.
 *  - Every call is asynchronous on `stream` (a cudaStream_t, NULL = the
 *    legacy default stream) and returns an int status:
 *        0   queued successfully
 *       <0   contract violation or CUDA error (lm_last_error() explains)
 *    Singular-matrix results are reported asynchronously through a
 *    device int32 `info` (0, or failing column + 1, exactly the
 *    reference's rc convention, _loops.py:200-205).
 *  - Matrices are strided views: element (i,j) is ptr[i*rs + j*cs]
 *    (in elements) -- numpy's strides divided by the item size.  F-order
 *    is rs=1, cs=rows; a transposed view swaps them; a diagonal vector
 *    of an F-order square has stride rows+1.
 *    Vectors are (ptr, n, stride).  No transpose flags: a view IS the
 *    transposition (the reference planner never sets trans flags,
 *    rewrite.py:628-629).
 *  - dtype: LM_F64 (the reference's only element type, matrix.py:97)
 *    or LM_F32 (extension, BASELINE configs 5).
 *  - Arithmetic that the reference does element by element with one
 *    rounding per operation (fused element-wise, diag scaling, LU
 *    factor/solve, batched small LU, triangular and band solves) is
 *    reproduced with the same operation order and NO FMA contraction, so
 *    results are bit-identical.  Reductions over many terms (GEMM, GEMV,
 *    SYRK, trace/diag of product) use parallel deterministic orders and
 *    are within the north-star tolerance (normwise 1e-12 f64).
 */
#ifndef LM_B200_H
#define LM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LM_ABI_VERSION 1

enum { LM_F64 = 0, LM_F32 = 1 };

typedef struct {
    void *ptr;
    int64_t rows, cols, rs, cs;
} lm_view;

typedef struct {
    void *ptr;
    int64_t n, stride;
} lm_vec;

/* ---- library ----------------------------------------------------------- */
int lm_abi_version(void);
/* Last error message of the calling thread ("" if none). */
const char *lm_last_error(void);
/* Number of kernels this library has launched since load (for the
 * bench's gpu_launches claim). */
int64_t lm_launch_count(void);
/* Name of the kernel variant the calling thread's last multi-variant call
 * launched (e.g. "stream_tma", "tc05p64"; "" if none): lets tests prove
 * that an environment switch selected the kernel it names. */
const char *lm_last_variant(void);

/* ---- element-wise family: _loops.py:37-84 (_fused1.._fused4, _fused_axpy) */
/* out = sum_k coeffs[k] * srcs[k], accumulated left to right per element,
 * one rounding per multiply and per add (kernels.py:32-62). */
int lm_fused_axpby(int dtype, int nterms, const double *coeffs, const lm_view *srcs, lm_view out,
                   void *stream);

/* Extension (Schur %, element /, abs, scalar +): postfix program over
 * sources, one rounding per node -- the per-element semantics of
 * naive_evaluate (expr.py:304-391) with R1 coefficient folding.
 * ops: 0 LOAD src | 1 CONST idx | 2 ADD | 3 SUB | 4 MUL | 5 DIV | 6 ABS | 7 NEG.
 * The program is JIT-compiled once per shape (NVRTC, sm_100a) into a
 * single fused streaming kernel; constants are runtime arguments. */
int lm_fused_program(int dtype, int nins, const int32_t *ops, const int32_t *args, int nconst,
                     const double *consts, int nsrc, const lm_view *srcs, lm_view out, void *stream);

/* The CUDA source generated for a program (inspection/tests).  Returns 0
 * and fills buf, or the needed buffer size if buflen is too small. */
int lm_program_source(int dtype, int flat, int nins, const int32_t *ops, const int32_t *args, int nconst,
                      int nsrc, char *buf, int64_t buflen);

/* dst = src (strided 2-D copy; the executor's RHS copy before solves,
 * rewrite.py:653, and the naive arm's view extraction). */
int lm_copy(int dtype, lm_view src, lm_view dst, void *stream);
/* *d_result = sum of the strided vector v (deterministic tree). */
int lm_vec_sum(int dtype, lm_vec v, void *d_result, void *stream);

/* ---- products: _loops.py:87-121 (_gemm, _gemv, _gemv_t), :124-141 (_syrk) */
/* out = a @ b (a p x q, b q x r).  r == 1 or p == 1 dispatch to the
 * split-K GEMV kernel; otherwise the FP64 DMMA tensor-core GEMM. */
int lm_gemm(int dtype, lm_view a, lm_view b, lm_view out, void *stream);
/* out = x @ (y @ z) and t = y @ z in ONE cooperative launch (the R6 plan of
 * a shape-skewed chain: two consecutive _gemm steps, _loops.py:87-98) when
 * t is at most 128 x 128 and dtype is f64: returns 1 (nothing launched) for
 * other shapes, so the caller runs the two lm_gemm calls instead. */
int lm_gemm_chain(int dtype, lm_view x, lm_view y, lm_view z, lm_view t, lm_view out, void *stream);
/* out = a @ x (trans=0) or a.T @ x (trans=1) (kernels.py:88-103). */
int lm_gemv(int dtype, lm_view a, lm_vec x, lm_vec out, int trans, void *stream);
/* out = a @ a.T, upper triangle computed, lower mirrored bitwise. */
int lm_syrk(int dtype, lm_view a, lm_view out, void *stream);

/* ---- diagonal / reduction family: _loops.py:144-197 ------------------- */
/* side 0: out[i,j] = d[i]*b[i,j];  side 1: out[i,j] = b[i,j]*d[j]. */
int lm_diag_scale(int dtype, lm_vec d, lm_view b, int side, lm_view out, void *stream);
/* out[i] = sum_k a[i,k]*b[k,i] (never forms a@b). */
int lm_diag_of_product(int dtype, lm_view a, lm_view b, lm_vec out, void *stream);
/* *d_result = sum_i sum_k a[i,k]*b[k,i]; d_result is one device element
 * of `dtype` (written asynchronously, deterministic reduction tree). */
int lm_trace_of_product(int dtype, lm_view a, lm_view b, void *d_result, void *stream);
/* *d_result = sum_i a[i]*d[i]*c[i]. */
int lm_triple_diag_dot(int dtype, lm_vec a, lm_vec d, lm_vec c, void *d_result, void *stream);

/* ---- structure scan: _loops.py:15-34 (_analyze) ------------------------- */
/* d_out[0] = lower bandwidth, d_out[1] = upper bandwidth, d_out[2] =
 * symmetric (0/1; only meaningful when square).  Exact comparisons. */
int lm_analyze(int dtype, lm_view a, int square, int64_t *d_out, void *stream);

/* ---- factorisation and solves: _loops.py:200-388 ----------------------- */
/* In-place LU with partial pivoting of the n x n F-order matrix `lu`
 * (cs == rows, rs == 1).  d_piv[k] = pivot row of column k (0-based,
 * sequential swap semantics), *d_info = 0 or failing column + 1. */
int lm_lu_factor(int dtype, lm_view lu, int64_t *d_piv, int32_t *d_info, void *stream);
/* Trailing-update arithmetic of the blocked LU: LM_LU_EXACT applies every
 * update in the reference's order with separately rounded multiply and
 * subtract (values and pivots bit-identical to _lu_factor); LM_LU_TENSOR runs
 * the trailing updates on the FP64 tensor cores (DMMA, FMA accumulation:
 * scaled residual <= 1e-10, pivots equal unless two candidates tie to
 * rounding); LM_LU_AUTO (what lm_lu_factor uses) is exact below n = 2048 and
 * tensor from there on, overridable with LM_LU_MODE=exact|tensor. */
enum { LM_LU_AUTO = 0, LM_LU_EXACT = 1, LM_LU_TENSOR = 2 };
int lm_lu_factor_mode(int dtype, lm_view lu, int64_t *d_piv, int32_t *d_info, int mode, void *stream);
/* Out-of-place form, the shape of _lu_factor itself (lazymat/_loops.py:200-236
 * copies its argument): src (F-order, left untouched) is copied into lu and
 * factored there.  The pivot-free path uses src as its restore point instead
 * of keeping a backup copy (n x n doubles of scratch and one more pass). */
int lm_lu_factor_from(int dtype, lm_view src, lm_view lu, int64_t *d_piv, int32_t *d_info, int mode, void *stream);
/* Solve with a factorisation from lm_lu_factor; x (n x m, F-order)
 * arrives holding B and is overwritten with X. */
int lm_lu_solve(int dtype, lm_view lu, const int64_t *d_piv, lm_view x, void *stream);
/* lm_lu_solve with the arithmetic chosen like lm_lu_factor_mode's: LM_LU_EXACT
 * is lm_lu_solve (_lu_solve_inplace's order, lazymat/_loops.py:239-259, bit
 * for bit); LM_LU_TENSOR (LM_LU_AUTO from n = 2048) runs both substitutions
 * as FP64 tensor-core products with the diagonal blocks' inverses (scaled
 * residual <= 1e-10, not bit-identical) when n is a multiple of 64 and the
 * right-hand sides a multiple of 32, and falls back to the exact order on
 * the device when a diagonal block is ill-conditioned. */
int lm_lu_solve_mode(int dtype, lm_view lu, const int64_t *d_piv, lm_view x, int mode, void *stream);
/* Banded solve (pack + factor + substitute) in place on x; kl/ku are
 * the detected bandwidths.  ab_work: (2kl+ku+1) x n device scratch. */
int lm_band_solve(int dtype, lm_view a, lm_view x, int64_t kl, int64_t ku, void *ab_work, int64_t *d_piv,
                  int32_t *d_info, void *stream);
/* Triangular solve in place (upper != 0: back substitution). */
int lm_tri_solve(int dtype, lm_view a, lm_view x, int upper, int32_t *d_info, void *stream);

/* ---- data movement: _loops.py:391-407 ------------------------------------ */
int lm_transpose_copy(int dtype, lm_view a, lm_view out, void *stream);
int lm_diag_materialise(int dtype, lm_vec d, lm_view out, void *stream);
/* out = I (n x n), used by explicit_inverse (kernels.py:282-299). */
int lm_set_identity(int dtype, lm_view out, void *stream);

/* ---- batched entry points (new; no reference counterpart) -------------- */
/* `batch` independent n x n systems A_b x_b = b_b (n <= 64), A stored
 * F-order contiguous per instance (stride n*n), one RHS column per
 * instance (stride n).  Exact reference op order (bit-identical to the
 * per-instance lazymat lu_factor + lu_solve).  x arrives holding b and is
 * overwritten with the solution; A is only read.  Optional outputs (NULL
 * to skip): lu_out (batch*n*n LU factors), d_piv (batch*n pivots).
 * d_info[b] = 0 or failing column + 1.  For 32 < n <= 64 without lu_out
 * this is two launches on `stream`: a pivot-free fast path that proves the
 * reference keeps every pivot on the diagonal (|multiplier| < 1) and
 * certifies its quotients, then the pivoting kernel on the systems it
 * could not prove (it marks them d_info = -1 in between; d_info is final
 * when the call's work completes). */
int lm_lu_solve_batched(int dtype, int64_t n, int64_t batch, const void *a, void *x, void *lu_out, int64_t *d_piv,
                        int32_t *d_info, void *stream);
/* lm_lu_solve_batched plus, in the same pass, each instance's R10 structure
 * class (rewrite.py:146-173 over _analyze): d_cls[b] = 0 general, 1 band
 * (lbw + ubw <= max(4, n/4)), 2 upper triangular, 3 lower triangular,
 * 4 symmetric.  Every instance is LU-solved; the caller re-solves the
 * band / triangular ones with their own kernels (their LU result and
 * d_info entry are not meaningful).  One pass (two launches for
 * 32 < n <= 64, as above), one host read. */
int lm_solve_batched_classified(int dtype, int64_t n, int64_t batch, const void *a, void *x, int32_t *d_cls,
                                int32_t *d_info, void *stream);
/* lm_solve_batched_classified with the right-hand sides read from b (dense,
 * batch*n contiguous doubles) and the solutions written to x (same layout;
 * b == x is the in-place call): the copy is one cudaMemcpyAsync on `stream`
 * inside the call instead of a separate framework copy. */
int lm_solve_batched_classified_from(int dtype, int64_t n, int64_t batch, const void *a, const void *b, void *x,
                                     int32_t *d_cls, int32_t *d_info, void *stream);
/* Batched structure classification of `batch` contiguous F-order n x n
 * matrices: d_out[3*b + {0,1,2}] = lbw, ubw, sym. */
int lm_analyze_batched(int dtype, int64_t n, int64_t batch, const void *a, int64_t *d_out, void *stream);
/* Grouped size-class kernel for E_b = A_b.T @ B_b + C_b % D_b and
 * s_b = trace(A_b @ B_b): all instances of one size n, contiguous per
 * instance.  Reads each operand once. */
int lm_expr_atb_schur_trace_batched(int dtype, int64_t n, int64_t batch, const void *a, const void *b,
                                    const void *c, const void *d, void *e, void *s, void *stream);

/* ---- the collective of the row-sharded configs ---- */
/* NCCL is resolved at run time: `path` (or NULL) names the library; the copy
 * already loaded in the process (torch's) is preferred.  One process per
 * GPU: rank 0 makes the 128-byte unique id, the host layer moves it to the
 * other ranks (any rendezvous), every rank calls lm_nccl_init_rank on its
 * device.  lm_nccl_init_all is the single-process, several-device form
 * (ncclCommInitAll; comms_out receives ndev communicators).  Returns -3 on an
 * NCCL error (lm_last_error() explains). */
#define LM_NCCL_ID_BYTES 128
int lm_nccl_load(const char *path, int *version_out);
int lm_nccl_unique_id(uint8_t *id_out);
int lm_nccl_init_rank(int nranks, int rank, const uint8_t *id, void **comm_out);
int lm_nccl_init_all(int ndev, const int *devs, void **comms_out);
/* In-place sum all-reduce of `count` elements on `stream` (asynchronous). */
int lm_allreduce_sum(void *comm, int dtype, void *d_buf, int64_t count, void *stream);
/* The 5b trace finish: one float64 (lazymat/kernels.py:157-164 per shard). */
int lm_allreduce_sum_f64(void *comm, double *d_val, void *stream);
int lm_nccl_destroy(void *comm);

/* ---- synthetic data (bench / tests only) ------------------------------- */
/* out(i,j) = U(lo,hi) from a counter-based hash of the GLOBAL index
 * (row0+i, col0+j) of a matrix with global_rows rows: any slice of a
 * distributed matrix can be generated consistently on any rank. */
int lm_fill_uniform(int dtype, lm_view out, uint64_t seed, int64_t row0, int64_t col0, int64_t global_rows,
                    double lo, double hi, void *stream);

/* numpy-identical seeded fill: element (b, i, j) of `batch` column-major
 * rows x cols matrices (element at out[b*bstride + i + j*ld]) is draw number
 * skip + b*bstream + i*rstream + j of np.random.default_rng(seed) (PCG64),
 * mapped as numpy's uniform(lo, hi) does (lo + (hi - lo) * next_double);
 * f32 output is that f64 value rounded to nearest.  (state, inc) is the
 * generator's 128-bit state right after seeding (bit_generator.state).
 * With bstream = rows*cols and rstream = cols this reproduces
 * np.asfortranarray(default_rng(seed).uniform(lo, hi, (batch, rows, cols)))
 * bit for bit -- the SURVEY.md 8(d) operand scheme, generated in HBM. */
int lm_fill_pcg64(int dtype, void *out, int64_t batch, int64_t rows, int64_t cols, int64_t ld, int64_t bstride,
                  int64_t bstream, int64_t rstream, uint64_t skip, uint64_t state_hi, uint64_t state_lo,
                  uint64_t inc_hi, uint64_t inc_lo, double lo, double hi, void *stream);

/* ---- diagnostics ---------------------------------------------------------- */
/* Factor one LU panel with the cluster kernel, recording clock64() per
 * column and phase (4 per column) into d_clock (tools/panel_probe.py). */
int lm_debug_lu_panel(lm_view a, int64_t j0, int nb, int64_t *d_piv, int32_t *d_info, long long *d_clock,
                      void *stream);
/* Diagnostics: c -= a b through the blocked LU's trailing-update GEMM (F-order
 * operands; tools/gemm_sub_probe.py times the kernel on config 4a's shapes). */
int lm_debug_gemm_sub(lm_view a, lm_view b, lm_view c, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* LM_B200_H */
