// lu_solve_tc.cu -- forward and back substitution on the FP64 tensor cores,
// the solve half of lm_lu_solve_mode's tensor mode (BASELINE config 4a:
// 8192 x 64 right-hand sides; lazymat/_loops.py:239-259 is the arithmetic it
// replaces, held to the north star's scaled residual <= 1e-10 instead of bit
// equality -- lm_lu_solve keeps the exact order).
//
// The exact wavefront (lu_solve.cu) spends ~15 us per 64-row block on its
// critical path: the last block's 64 x 64 x 32 contribution in separately
// rounded multiplies and subtracts, then a 64-step triangle.  Here both are
// DMMA products: the diagonal blocks' inverses L_II^-1 and U_II^-1 are formed
// first (one small kernel, all blocks in parallel), so block I's step is
//   X_I = T_II^-1 (X_I - sum_J T_IJ X_J)
// with every term a 64 x 64 x 32 mma.sync.m8n8k4.f64 product.  One
// cooperative launch, CTA (I, g) = rows [64 I, 64 I + 64) x right-hand sides
// [32 g, 32 g + 32), a release/acquire flag per (block, group); the T_IJ
// tiles do not depend on the flags and stream ahead through a 3-slot ring of
// half tiles (bulk copies on mbarriers), so the critical path per block is
// the flag, X_J's tile, two products and the store.
//
// Guard: the inversion kernel measures max|T_II^-1| max|T_II| per block; above
// 1e4 (or not finite: a zero pivot) it raises a device flag, this kernel
// returns at once and the exact wavefront, gated on the same flag, does the
// solve -- no host round trip.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {

// lu_solve.cu; only_if != null: run only when *only_if != 0
int lu_solve_wavefront(const double *LU, int64_t n, int64_t lda, double *X, int64_t ldx, int64_t m, cudaStream_t s,
                       const int *only_if);

namespace {

constexpr int TB = 64;    // rows per block
constexpr int TG = 32;    // right-hand sides per group
constexpr int TT = 256;   // 8 warps, 4 x 2; warp tile 16 rows x 16 columns
constexpr int TLA = 72;   // [k][i] tiles (T_IJ halves, the inverse): 72 = 8 (mod 16)
constexpr int TLB = 68;   // [c][k] tiles (X_J, Y): 68 = 4 (mod 8)
constexpr int TH = 32;    // K rows per half tile
constexpr int TSLOTS = 3;

struct TcArgs {
    const double *LU;
    int64_t lda, n;
    double *X;
    int64_t ldx;
    int nblk, ngrp;
    const double *inv;  // [2][nblk][64 x 64] F-order: L_II^-1 then U_II^-1
    int *flags;         // [2][nblk][ngrp], zeroed
    const int *bad;     // set by the inversion kernel: leave everything to the exact kernel
};

__device__ __forceinline__ unsigned saddr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_copy(double *smem, const double *gmem, unsigned bytes, unsigned long long *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     saddr(smem)),
                 "l"(gmem), "r"(bytes), "r"(saddr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            saddr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// acc (2 x 2 fragments of the warp) += A[k0.., rows] * B[cols, k0..] over nk K rows;
// pa / pb: the lane's element of fragment (0, 0) at k = 0
__device__ __forceinline__ void product(double (&acc)[2][2][2], const double *pa, const double *pb, int nk) {
#pragma unroll 4
    for (int k = 0; k < nk; k += 4) {
        const double a0 = pa[k * TLA], a1 = pa[k * TLA + 8];
        const double b0 = pb[k], b1 = pb[k + 8 * TLB];
        mma884(acc[0][0], a0, b0);
        mma884(acc[0][1], a0, b1);
        mma884(acc[1][0], a1, b0);
        mma884(acc[1][1], a1, b1);
    }
}

__global__ void __launch_bounds__(TT, 2) lu_solve_tc(TcArgs a) {
    if (*a.bad) return;  // (uniform over the grid: nobody reaches the grid barrier)
    extern __shared__ __align__(16) double tsm[];
    __shared__ unsigned long long full[TSLOTS], ibar;
    double *sRing = tsm;                       // [TSLOTS][TH][TLA]
    double *sInv = sRing + TSLOTS * TH * TLA;  // [TB][TLA]
    double *sB = sInv + TB * TLA;              // [TG][TLB]
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int I = blockIdx.x / a.ngrp, g = blockIdx.x - I * a.ngrp;
    const int64_t i0 = (int64_t)I * TB, c0 = (int64_t)g * TG;
    const int wr = warp >> 1, wc = warp & 1;
    const int fr = lane >> 2, fc = lane & 3;
    if (tid == 0) {
        for (int s = 0; s < TSLOTS; ++s) mbar_init(&full[s], TH);
        mbar_init(&ibar, TB);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // this CTA's rows, in the DMMA accumulator layout (rows 16 wr + 8 i + fr,
    // columns 16 wc + 8 j + 2 fc + h); they stay in registers over both sweeps
    double x[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                x[i][j][h] = __ldcg(a.X + i0 + 16 * wr + 8 * i + fr + (c0 + 16 * wc + 8 * j + 2 * fc + h) * a.ldx);
    const double *pa_ring = sRing + fc * TLA + 16 * wr + fr;
    const double *pa_inv = sInv + fc * TLA + 16 * wr + fr;
    const double *pb = sB + (16 * wc + fr) * TLB + fc;
    unsigned qi = 0, qc = 0;  // half tiles issued / consumed (running over both sweeps)
    for (int sweep = 0; sweep < 2; ++sweep) {
        const bool fwd = sweep == 0;
        int *flags = a.flags + (int64_t)sweep * a.nblk * a.ngrp;
        const int nJ = fwd ? I : a.nblk - 1 - I;
        // the inverse of this block's triangle (needed last)
        if (tid < TB)
            bulk_copy(sInv + tid * TLA, a.inv + ((int64_t)sweep * a.nblk + I) * TB * TB + tid * TB, TB * 8, &ibar);
        // half tile ql of the sweep -> ring (warp 0, one K row per lane)
        auto issue = [&](int ql) {
            if (ql < 2 * nJ) {
                if (warp == 0) {
                    const int t = ql >> 1, J = fwd ? t : a.nblk - 1 - t;
                    const int64_t col = (int64_t)J * TB + (ql & 1) * TH + lane;
                    const unsigned slot = qi % TSLOTS;
                    bulk_copy(sRing + (slot * TH + lane) * TLA, a.LU + i0 + col * a.lda, TB * 8, &full[slot]);
                }
                ++qi;
            }
        };
        issue(0);
        issue(1);
        issue(2);
        double acc[2][2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int t = 0; t < nJ; ++t) {
            const int J = fwd ? t : a.nblk - 1 - t;
            // X_J (final once its flag is up) -> sB [c][k]
            if (tid == 0) {
                const int *f = flags + (int64_t)J * a.ngrp + g;
                int v;
                do {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                } while (v == 0);
            }
            __syncthreads();
            for (int e = tid; e < TB * TG; e += TT) {
                const int k = e & (TB - 1), c = e >> 6;
                sB[c * TLB + k] = __ldcg(a.X + (int64_t)J * TB + k + (c0 + c) * a.ldx);
            }
            __syncthreads();
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
                const unsigned slot = qc % TSLOTS;
                mbar_wait(&full[slot], (qc / TSLOTS) & 1);
                product(acc, pa_ring + slot * TH * TLA, pb + half * TH, TH);
                ++qc;
                __syncthreads();  // the slot (and, after the second half, sB) is free
                issue(2 * t + half + 3);
            }
        }
        // Y = X_I - sum -> sB, then X_I = T_II^-1 Y
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    sB[(16 * wc + 8 * j + 2 * fc + h) * TLB + 16 * wr + 8 * i + fr] = x[i][j][h] - acc[i][j][h];
        mbar_wait(&ibar, sweep);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) x[i][j][0] = x[i][j][1] = 0.0;
        product(x, pa_inv, pb, TB);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    a.X[i0 + 16 * wr + 8 * i + fr + (c0 + 16 * wc + 8 * j + 2 * fc + h) * a.ldx] = x[i][j][h];
        __syncthreads();  // all rows stored (and sInv / sB read) before the flag and the next sweep's copies
        if (tid == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + (int64_t)I * a.ngrp + g), "r"(1) : "memory");
        }
        if (fwd) grid.sync();  // every row final before the back sweep reads any
    }
}

// Inverses of the diagonal blocks' triangles: blockIdx.y = 0 the unit lower
// one, 1 the upper one; thread c forms column c by substitution on e_c.
__global__ void __launch_bounds__(TB) tri_block_inverse(const double *LU, int64_t lda, int nblk, double *inv,
                                                        int *bad) {
    extern __shared__ __align__(16) double ism[];
    double(*T)[TB + 1] = reinterpret_cast<double(*)[TB + 1]>(ism);
    double(*V)[TB + 1] = T + TB;
    const int blk = blockIdx.x, upper = blockIdx.y, c = threadIdx.x;
    const double *src = LU + (int64_t)blk * TB * (lda + 1);
    for (int j = 0; j < TB; ++j) T[c][j] = src[c + j * lda];  // (row c: coalesced over the threads)
    for (int i = 0; i < TB; ++i) V[i][c] = i == c ? 1.0 : 0.0;
    __syncthreads();
    double tmax = 0.0, vmax = 0.0;
    if (!upper) {
        for (int j = c; j < TB; ++j) {
            const double xj = V[j][c];
            for (int i = j + 1; i < TB; ++i) V[i][c] = fma(-T[i][j], xj, V[i][c]);
        }
        tmax = 1.0;
    } else {
        for (int j = c; j >= 0; --j) {
            const double xj = V[j][c] / T[j][j];
            V[j][c] = xj;
            for (int i = 0; i < j; ++i) V[i][c] = fma(-T[i][j], xj, V[i][c]);
        }
        for (int i = 0; i <= c; ++i) tmax = fmax(tmax, fabs(T[i][c]));
    }
    double *dst = inv + ((int64_t)upper * nblk + blk) * TB * TB + (int64_t)c * TB;
    bool finite = true;
    for (int i = 0; i < TB; ++i) {
        const double v = V[i][c];
        dst[i] = v;
        vmax = fmax(vmax, fabs(v));
        finite = finite && (fabs(v) <= 1.7e308);
    }
    // block-level conditioning proxy max|T^-1| max|T| (reduced over the columns)
    __shared__ double rt[TB], rv[TB];
    __shared__ int rf;
    if (c == 0) rf = 1;
    rt[c] = tmax;
    rv[c] = vmax;
    __syncthreads();
    if (!finite) rf = 0;
    __syncthreads();
    if (c == 0) {
        double t = 0.0, v = 0.0;
        for (int i = 0; i < TB; ++i) {
            t = fmax(t, rt[i]);
            v = fmax(v, rv[i]);
        }
        if (!rf || !(t * v <= 1e4)) atomicExch(bad, 1);
    }
}

}  // namespace

// 0 = done; 1 = not applicable (the caller runs the exact solve)
int lu_solve_tensor(const double *LU, int64_t n, int64_t lda, double *X, int64_t ldx, int64_t m, cudaStream_t s) {
    static const bool off = getenv("LM_SOLVE_TC") && getenv("LM_SOLVE_TC")[0] == '0';
    if (off || n < 2 * TB || n % TB || m < TG || m % TG || (lda & 1) || (ldx & 1) || ((uintptr_t)LU & 15)) return 1;
    const int nblk = (int)(n / TB), ngrp = (int)(m / TG);
    const size_t smem = sizeof(double) * (TSLOTS * TH * TLA + TB * TLA + TG * TLB);
    if (int rc = func_attrs(lu_solve_tc, smem)) return rc;
    int per_sm = 0;
    LM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_solve_tc, TT, smem));
    if ((int64_t)per_sm * num_sms() < (int64_t)nblk * ngrp) return 1;  // all CTAs must be co-resident
    Scratch inv, state;
    if (int rc = inv.alloc(sizeof(double) * 2 * (size_t)nblk * TB * TB, s)) return rc;
    const size_t sb = sizeof(int) * (2 * (size_t)nblk * ngrp + 1);
    if (int rc = state.alloc(sb, s)) return rc;
    LM_CUDA(cudaMemsetAsync(state.p, 0, sb, s));
    int *bad = state.as<int>(), *flags = bad + 1;
    constexpr size_t ism = sizeof(double) * 2 * TB * (TB + 1);
    if (int rc = func_attrs(tri_block_inverse, ism)) return rc;
    tri_block_inverse<<<dim3((unsigned)nblk, 2), TB, ism, s>>>(LU, lda, nblk, inv.as<double>(), bad);
    LM_LAUNCHED(1);
    TcArgs args{LU, lda, n, X, ldx, nblk, ngrp, inv.as<double>(), flags, bad};
    void *kargs[] = {&args};
    LM_CUDA(cudaLaunchCooperativeKernel((const void *)lu_solve_tc, dim3((unsigned)(nblk * ngrp)), dim3(TT), kargs, smem,
                                        s));
    count_launch(1);
    note_variant("solve_tc");
    // ill-conditioned diagonal block somewhere: the exact wavefront does it all
    const int rc = lu_solve_wavefront(LU, n, lda, X, ldx, m, s, bad);
    LM_REQUIRE(rc != 1, "lu_solve: tensor-mode fallback needs the wavefront kernel");
    return rc;
}

}  // namespace lm
