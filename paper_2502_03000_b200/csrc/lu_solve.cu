// lu_solve.cu -- forward and back substitution for up to 64 right-hand
// sides (BASELINE config 4a: 8192 x 64) in the reference's exact order
// (lazymat/_loops.py:239-259: per column, x_i -= L[i,j] x_j for j
// ascending; then x_j /= U[j,j], x_i -= U[i,j] x_j for j descending; each
// product and difference rounded, no FMA).
//
// One cooperative launch, one CTA per 64-row block ("wavefront"): block I
// accumulates the contributions of the blocks J < I in ascending J as soon
// as each one is final (a release/acquire flag per block), then solves its
// own 64 x 64 triangle (one thread per right-hand side), publishes its rows
// and raises its flag.  A grid barrier separates the two sweeps; the back
// sweep runs in descending block order.  The critical path is one triangle
// per block instead of ~500 dependent kernel launches.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {

constexpr int WB = 64;        // rows per block
constexpr int WM = 64;        // max right-hand sides
constexpr int WT = 256;       // threads
constexpr int WLD = WB + 1;   // smem row stride (doubles)

struct WaveArgs {
    const double *LU;
    int64_t lda, n;
    double *X;
    int64_t ldx;
    int m, nblk;
    int *flags;  // [2][nblk], zeroed
    const int *only_if;  // null, or a device flag: do nothing unless it is set (lu_solve_tc.cu's fallback)
};

__device__ __forceinline__ void wait_flag(const int *f) {
    if (threadIdx.x == 0) {
        int v;
        do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        } while (v == 0);
    }
    __syncthreads();
}

__device__ __forceinline__ void raise_flag(int *f) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(f), "r"(1) : "memory");
    }
}

__global__ void __launch_bounds__(WT, 1) lu_solve_wave(WaveArgs a) {
    if (a.only_if && *a.only_if == 0) return;  // (uniform over the grid)
    extern __shared__ double sw[];
    double *sL = sw;              // [WB][WLD]: sL[i][j] = T[i0+i, j0+j]
    double *sX = sw + WB * WLD;   // [WB][WLD]: sX[j][c] = X[j0+j, c]
    double *sY = sX + WB * WLD;   // [WB][WLD]: this block's rows, sY[i][c]
    cg::grid_group grid = cg::this_grid();
    const int I = blockIdx.x, tid = threadIdx.x;
    const int64_t i0 = (int64_t)I * WB;
    const int rows = (int)((a.n - i0) < WB ? (a.n - i0) : WB);
    const int tr = tid % 16, tc = tid / 16;  // rows tr + 16a, columns tc + 16b
    const int m = a.m;

    for (int sweep = 0; sweep < 2; ++sweep) {
        const bool fwd = sweep == 0;
        int *flags = a.flags + sweep * a.nblk;
        // this block's current rows
        for (int e = tid; e < WB * m; e += WT) {
            const int i = e % WB, c = e / WB;
            sY[i * WLD + c] = i < rows ? a.X[(i0 + i) + (int64_t)c * a.ldx] : 0.0;
        }
        double acc[4][4];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int s = 0; s < 4; ++s) acc[r][s] = sY[(tr + 16 * r) * WLD + tc + 16 * s];
        // contributions of the other blocks, in the reference's order
        const int nJ = fwd ? I : a.nblk - 1 - I;
        for (int t = 0; t < nJ; ++t) {
            const int J = fwd ? t : a.nblk - 1 - t;
            const int64_t j0 = (int64_t)J * WB;
            const int cols = (int)((a.n - j0) < WB ? (a.n - j0) : WB);
            wait_flag(flags + J);
            for (int e = tid; e < WB * WB; e += WT) {
                const int i = e % WB, j = e / WB;
                sL[i * WLD + j] = (i < rows && j < cols) ? a.LU[(i0 + i) + (j0 + j) * a.lda] : 0.0;
            }
            for (int e = tid; e < WB * m; e += WT) {
                const int j = e % WB, c = e / WB;
                sX[j * WLD + c] = j < cols ? a.X[(j0 + j) + (int64_t)c * a.ldx] : 0.0;
            }
            __syncthreads();
            for (int q = 0; q < cols; ++q) {
                const int j = fwd ? q : cols - 1 - q;
                double l[4], x[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) l[r] = sL[(tr + 16 * r) * WLD + j];
#pragma unroll
                for (int s = 0; s < 4; ++s) x[s] = sX[j * WLD + tc + 16 * s];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int s = 0; s < 4; ++s) acc[r][s] = __dsub_rn(acc[r][s], __dmul_rn(l[r], x[s]));
            }
            __syncthreads();
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int s = 0; s < 4; ++s) sY[(tr + 16 * r) * WLD + tc + 16 * s] = acc[r][s];
        // the diagonal triangle
        for (int e = tid; e < WB * WB; e += WT) {
            const int i = e % WB, j = e / WB;
            sL[i * WLD + j] = (i < rows && j < rows) ? a.LU[(i0 + i) + (i0 + j) * a.lda] : 0.0;
        }
        __syncthreads();
        {
            // 4 lanes per right-hand side (consecutive lanes: one warp holds 8
            // columns), lane g owns rows g, g+4, ..., g+60 in registers; x_j is
            // broadcast from its owner with one shuffle per step
            const int c = tid / 4, g = tid % 4;
            const int base = (tid & 31) & ~3;  // lane of this column's g = 0
            double x[WB / 4];
#pragma unroll
            for (int r = 0; r < WB / 4; ++r) x[r] = (c < m) ? sY[(4 * r + g) * WLD + c] : 0.0;
            if (fwd) {
#pragma unroll
                for (int j = 0; j < WB; ++j) {
                    if (j >= rows) break;
                    const double xj = __shfl_sync(0xffffffffu, x[j / 4], base + (j % 4));
#pragma unroll
                    for (int r = 0; r < WB / 4; ++r) {
                        const int i = 4 * r + g;
                        if (i > j && i < rows) x[r] = __dsub_rn(x[r], __dmul_rn(sL[i * WLD + j], xj));
                    }
                }
            } else {
#pragma unroll
                for (int j = WB - 1; j >= 0; --j) {
                    if (j >= rows) continue;
                    if (g == j % 4) x[j / 4] = __ddiv_rn(x[j / 4], sL[j * WLD + j]);
                    const double xj = __shfl_sync(0xffffffffu, x[j / 4], base + (j % 4));
#pragma unroll
                    for (int r = 0; r < WB / 4; ++r) {
                        const int i = 4 * r + g;
                        if (i < j) x[r] = __dsub_rn(x[r], __dmul_rn(sL[i * WLD + j], xj));
                    }
                }
            }
            if (c < m)
#pragma unroll
                for (int r = 0; r < WB / 4; ++r) sY[(4 * r + g) * WLD + c] = x[r];
        }
        __syncthreads();
        for (int e = tid; e < WB * m; e += WT) {
            const int i = e % WB, c = e / WB;
            if (i < rows) a.X[(i0 + i) + (int64_t)c * a.ldx] = sY[i * WLD + c];
        }
        raise_flag(flags + I);
        if (fwd) grid.sync();  // every row final before the back sweep reads any
    }
}

// ---------------------------------------------------------------------------
// v2: right-hand sides split into groups of 32 -- the groups are independent
// solves, so CTA (I, g) handles rows [64I, 64I+64) x columns [32g, 32g+32)
// and waits only on the flags of its own group.  The wavefront's critical
// path per block (the last block's contribution + the triangle) shrinks by
// the group count: one contribution is 64x64x16 exact MACs instead of
// 64x64x64 on one SM, and the diagonal tile is staged once per sweep.
// Triangle: 8 lanes per right-hand side, lane g owns rows g, g+8, ...;
// x_j is broadcast with an 8-wide shuffle.
constexpr int G2 = 32;        // right-hand sides per group
constexpr int G2LD = G2 + 1;
constexpr int LPR = WT / G2;    // triangle: lanes per right-hand side (8)
constexpr int RPL = WB / LPR;   // rows per lane (8)
constexpr int APT = WB * G2 / WT;  // accumulation outputs per thread (8)

struct Wave2Args {
    const double *LU;
    int64_t lda, n;
    double *X;
    int64_t ldx;
    int m, nblk, ngrp;
    int *flags;  // [2][nblk][ngrp], zeroed
    unsigned long long *dbg;  // optional: [2][nblk] globaltimer at each flag raise (group 0)
    const int *only_if;       // as WaveArgs
};

__global__ void __launch_bounds__(WT, 2) lu_solve_wave2(Wave2Args a) {
    if (a.only_if && *a.only_if == 0) return;  // (uniform over the grid)
    extern __shared__ double sw2[];
    double *sL = sw2;              // [WB][WLD]: off-diagonal tile L[i0.., j0..]
    double *sD = sL + WB * WLD;    // [WB][WLD]: this block's diagonal tile (staged once per sweep)
    double *sX = sD + WB * WLD;    // [WB][G2LD]: sX[j][c]
    double *sY = sX + WB * G2LD;   // [WB][G2LD]: this block's rows
    cg::grid_group grid = cg::this_grid();
    const int I = blockIdx.x / a.ngrp, g = blockIdx.x - I * a.ngrp, tid = threadIdx.x;
    const int64_t i0 = (int64_t)I * WB;
    const int c0 = g * G2;
    const int mg = (a.m - c0) < G2 ? (a.m - c0) : G2;
    const int rows = (int)((a.n - i0) < WB ? (a.n - i0) : WB);
    const int cc = tid % G2, rr = tid / G2;  // accumulation: column cc, rows rr + (WT/G2) q
    constexpr int RS = WT / G2;              // row step of the accumulation (8)
    for (int sweep = 0; sweep < 2; ++sweep) {
        const bool fwd = sweep == 0;
        int *flags = a.flags + (int64_t)sweep * a.nblk * a.ngrp;
        // the diagonal tile never changes: off the critical path
        for (int e = tid; e < WB * WB; e += WT) {
            const int i = e % WB, j = e / WB;
            sD[i * WLD + j] = (i < rows && j < rows) ? a.LU[(i0 + i) + (i0 + j) * a.lda] : 0.0;
        }
        double acc[APT];
#pragma unroll
        for (int q = 0; q < APT; ++q) {
            const int i = rr + RS * q;
            acc[q] = (i < rows && cc < mg) ? a.X[(i0 + i) + (int64_t)(c0 + cc) * a.ldx] : 0.0;
        }
        const int nJ = fwd ? I : a.nblk - 1 - I;
        for (int t = 0; t < nJ; ++t) {
            const int J = fwd ? t : a.nblk - 1 - t;
            const int64_t j0 = (int64_t)J * WB;
            const int cols = (int)((a.n - j0) < WB ? (a.n - j0) : WB);
            for (int e = tid; e < WB * WB; e += WT) {
                const int i = e % WB, j = e / WB;
                sL[i * WLD + j] = (i < rows && j < cols) ? a.LU[(i0 + i) + (j0 + j) * a.lda] : 0.0;
            }
            wait_flag(flags + (int64_t)J * a.ngrp + g);
            for (int e = tid; e < WB * G2; e += WT) {
                const int j = e % WB, c = e / WB;
                sX[j * G2LD + c] = (j < cols && c < mg) ? a.X[(j0 + j) + (int64_t)(c0 + c) * a.ldx] : 0.0;
            }
            __syncthreads();
            if (cols == WB) {
#pragma unroll 8
                for (int q2 = 0; q2 < WB; ++q2) {
                    const int j = fwd ? q2 : WB - 1 - q2;
                    const double xv = sX[j * G2LD + cc];
#pragma unroll
                    for (int q = 0; q < APT; ++q)
                        acc[q] = __dsub_rn(acc[q], __dmul_rn(sL[(rr + RS * q) * WLD + j], xv));
                }
            } else {
                for (int q2 = 0; q2 < cols; ++q2) {
                    const int j = fwd ? q2 : cols - 1 - q2;
                    const double xv = sX[j * G2LD + cc];
#pragma unroll
                    for (int q = 0; q < APT; ++q)
                        acc[q] = __dsub_rn(acc[q], __dmul_rn(sL[(rr + RS * q) * WLD + j], xv));
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < APT; ++q) sY[(rr + RS * q) * G2LD + cc] = acc[q];
        __syncthreads();
        {
            // LPR lanes per right-hand side: c = tid / LPR, lane gl owns rows gl + LPR r
            const int c = tid / LPR, gl = tid % LPR;
            double x[RPL];
#pragma unroll
            for (int r = 0; r < RPL; ++r) x[r] = sY[(gl + LPR * r) * G2LD + c];
            if (fwd) {
#pragma unroll
                for (int j = 0; j < WB; ++j) {
                    if (j >= rows) break;
                    const double xj = __shfl_sync(0xffffffffu, x[j / LPR], j % LPR, LPR);
#pragma unroll
                    for (int r = 0; r < RPL; ++r) {
                        const int i = gl + LPR * r;
                        if (i > j && i < rows) x[r] = __dsub_rn(x[r], __dmul_rn(sD[i * WLD + j], xj));
                    }
                }
            } else {
#pragma unroll
                for (int j = WB - 1; j >= 0; --j) {
                    if (j >= rows) continue;
                    if (gl == j % LPR) x[j / LPR] = __ddiv_rn(x[j / LPR], sD[j * WLD + j]);
                    const double xj = __shfl_sync(0xffffffffu, x[j / LPR], j % LPR, LPR);
#pragma unroll
                    for (int r = 0; r < RPL; ++r) {
                        const int i = gl + LPR * r;
                        if (i < j) x[r] = __dsub_rn(x[r], __dmul_rn(sD[i * WLD + j], xj));
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < RPL; ++r) sY[(gl + LPR * r) * G2LD + c] = x[r];
        }
        __syncthreads();
        for (int e = tid; e < WB * G2; e += WT) {
            const int i = e % WB, c = e / WB;
            if (i < rows && c < mg) a.X[(i0 + i) + (int64_t)(c0 + c) * a.ldx] = sY[i * G2LD + c];
        }
        raise_flag(flags + (int64_t)I * a.ngrp + g);
        if (a.dbg && g == 0 && tid == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            a.dbg[sweep * a.nblk + I] = tt;
        }
        if (fwd) grid.sync();  // every row final before the back sweep reads any
    }
}

static int lu_solve_wavefront2(const double *LU, int64_t n, int64_t lda, double *X, int64_t ldx, int64_t m,
                               cudaStream_t s, const int *only_if) {
    const int nblk = (int)ceil_div(n, WB), ngrp = (int)ceil_div(m, G2);
    const size_t smem = sizeof(double) * (2 * WB * WLD + 2 * WB * G2LD);
    if (int rc = func_attrs(lu_solve_wave2, smem)) return rc;
    int per_sm = 0;
    LM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_solve_wave2, WT, smem));
    if ((int64_t)per_sm * num_sms() < (int64_t)nblk * ngrp) return 1;
    Scratch flags;
    const size_t fb = sizeof(int) * 2 * (size_t)nblk * ngrp;
    if (int rc = flags.alloc(fb, s)) return rc;
    LM_CUDA(cudaMemsetAsync(flags.p, 0, fb, s));
    static const bool want = getenv("LM_SOLVE_TRACE") != nullptr;
    static PerDevice<unsigned long long *> dbg_cache;
    unsigned long long *dbg = nullptr;
    if (want)
        if (int rc = dbg_cache.get(dbg, [](unsigned long long *&p) {
                LM_CUDA(cudaMalloc(&p, sizeof(unsigned long long) * 2 * 4096));
                return 0;
            }))
            return rc;
    Wave2Args args{LU, lda, n, X, ldx, (int)m, nblk, ngrp, flags.as<int>(), want && nblk <= 2048 ? dbg : nullptr,
                   only_if};
    void *kargs[] = {&args};
    LM_CUDA(cudaLaunchCooperativeKernel((const void *)lu_solve_wave2, dim3(nblk * ngrp), dim3(WT), kargs, smem, s));
    count_launch(1);
    if (args.dbg) {
        std::vector<unsigned long long> h(2 * nblk);
        cudaStreamSynchronize(s);
        cudaMemcpy(h.data(), dbg, sizeof(unsigned long long) * 2 * nblk, cudaMemcpyDeviceToHost);
        unsigned long long t0 = h[0];
        for (int i = 0; i < 2 * nblk; ++i) t0 = h[i] < t0 ? h[i] : t0;
        for (int sw = 0; sw < 2; ++sw)
            for (int i = 0; i < nblk; i += (nblk / 16 > 0 ? nblk / 16 : 1))
                fprintf(stderr, "SOLVETRACE sweep %d block %4d flag at %8.1f us\n", sw, i,
                        (h[sw * nblk + i] - t0) / 1e3);
    }
    return 0;
}

// 0 = done; 1 = not applicable (caller uses the launch-per-block path)
int lu_solve_wavefront(const double *LU, int64_t n, int64_t lda, double *X, int64_t ldx, int64_t m, cudaStream_t s,
                       const int *only_if) {
    if (m < 1 || n < 1) return 1;
    if (m > G2) {  // several right-hand-side groups: independent wavefronts
        const int rc = lu_solve_wavefront2(LU, n, lda, X, ldx, m, s, only_if);
        if (rc != 1) return rc;
    }
    if (m > WM) return 1;
    const int nblk = (int)ceil_div(n, WB);
    const size_t smem = sizeof(double) * 3 * WB * WLD;
    if (int rc = func_attrs(lu_solve_wave, smem)) return rc;
    int per_sm = 0;
    LM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_solve_wave, WT, smem));
    if ((int64_t)per_sm * num_sms() < nblk) return 1;  // all blocks must be co-resident
    Scratch flags;
    if (int rc = flags.alloc(sizeof(int) * 2 * nblk, s)) return rc;
    LM_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 2 * nblk, s));
    WaveArgs args{LU, lda, n, X, ldx, (int)m, nblk, flags.as<int>(), only_if};
    void *kargs[] = {&args};
    LM_CUDA(cudaLaunchCooperativeKernel((const void *)lu_solve_wave, dim3(nblk), dim3(WT), kargs, smem, s));
    count_launch(1);
    return 0;
}

}  // namespace lm
