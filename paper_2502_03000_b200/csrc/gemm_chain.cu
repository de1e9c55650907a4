// gemm_chain.cu -- out = X (Y Z) in ONE cooperative launch when the inner
// product T = Y Z is small (both dimensions <= 128).
//
// This is the plan R6 gives the shape-skewed chain of BASELINE config 3b,
// X (8000 x 100) * Y (100 x 8000) * Z (8000 x 100): gemm(Y, Z) -> T (100 x 100),
// then gemm(X, T) (lazymat/rewrite.py:317-328; the reference runs both
// through _gemm, lazymat/_loops.py:87-98).  320 MFLOP and 26 MB is ~9 us of
// B200 time, but as two library GEMMs it is three launches (split-K
// partials, their finish, the second GEMM), each a fraction of a wave
// (31 us in round 1).  Here every SM runs three phases of one kernel,
// separated by grid-wide barriers (cooperative launch, one CTA per SM):
//   1. a K slice of Y Z on DMMA (mma.sync.m8n8k4.f64; 16 warps over a
//      128 x 128 tile, 8 x 8 fragments outside T skipped) -> partial in HBM/L2;
//   2. T = sum of the per-SM partials in a fixed order (deterministic), a
//      slice of T per SM, written to the plan's T slot;
//   3. a slice of rows of X times T (T staged whole in shared memory) -> out.
// The executor fuses the two plan steps only when the plan would free
// nothing in between (rewrite.py _chain_fusable); the trace still records
// both gemm kernels.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {
namespace {

constexpr int CT = 512;        // 16 warps
// Shared-memory layouts follow the unit-stride direction of each F-order
// operand (so the 8-byte cp.async writes of a warp are consecutive), with
// row lengths = 4 (mod 16) doubles so the m8n8k4 fragment loads, served per
// half-warp, hit 16 distinct bank pairs.
constexpr int CK = 32;         // phase-1 K chunk (double-buffered)
constexpr int LDK = CK + 4;    // sZ [n][k]
constexpr int TMX = 128;       // largest p, q
constexpr int LDM = TMX + 4;   // sY [k][m]
constexpr int LDP = TMX + 4;   // sT [n][k]
constexpr int R3 = 64;         // largest phase-3 row tile
constexpr int LDX = R3 + 4;    // sX [k][m]
constexpr int kStage = CK * LDM + TMX * LDK;  // one phase-1 buffer (doubles)
constexpr int kSX = 2 * kStage > TMX * LDP ? 2 * kStage : TMX * LDP;  // sX after phase 1/3's other data
constexpr int kSmem = kSX + TMX * LDX;
constexpr int kMaxGroup = 32;  // phase 2: partials per thread (grids up to 8 * 32 CTAs)

// 8-byte asynchronous copy global -> shared; pred false writes zero (src-size 0):
// a CTA's whole slice is in flight at once instead of one load latency per loop trip
__device__ __forceinline__ void cpa8(double *smem, const double *gmem, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

struct ChainArgs {
    View<const double> x, y, z;
    View<double> t, out;
    double *part;  // [G][p*q] phase-1 partials
    int64_t kchunk;
    int rows3;     // phase-3 row tile (multiple of 8, <= R3)
    unsigned long long *dbg;  // LM_CHAIN_TRACE: %globaltimer of CTA 0 at the phase ends
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(CT, 1) gemm_chain_kernel(const __grid_constant__ ChainArgs g) {
    extern __shared__ __align__(16) double sm[];
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, fr = lane >> 2, fc = lane & 3;
    const int G = gridDim.x, b = blockIdx.x;
    const int p = (int)g.y.rows, q = (int)g.z.cols;
    const int64_t K = g.y.cols, M = g.x.rows;
    const bool mark = g.dbg && b == 0 && tid == 0;
    if (mark) g.dbg[0] = gtime();

    // X rows of this CTA's first phase-3 tile: independent of T, so their
    // copies are in flight from the start (own shared-memory region)
    double *sX = sm + kSX;  // (m, k) at k * LDX + m
    const int p4 = (p + 3) & ~3;
    const int R = g.rows3;
    const int64_t ntiles = (M + R - 1) / R;
    auto load_x = [&](int64_t tile) {
        const int64_t r0 = tile * R;
        const int rr = (int)(M - r0 < R ? M - r0 : R);
        for (int idx = tid; idx < rr * p4; idx += CT) {  // rows fastest: coalesced for F-order X
            const int m = idx % rr, k = idx / rr;
            cpa8(&sX[k * LDX + m], &g.x(r0 + m, k < p ? k : 0), k < p);
        }
    };
    if (b < ntiles) load_x(b);
    cpa_commit();

    // ---- phase 1: P_b = Y[:, kb:ke] Z[kb:ke, :], CK-deep chunks double-buffered
    {
        const int64_t kb = (int64_t)b * g.kchunk;
        const int64_t ke = kb + g.kchunk < K ? kb + g.kchunk : K;
        const int nch = ke > kb ? (int)((ke - kb + CK - 1) / CK) : 0;
        const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        auto sY = [&](int buf) { return sm + buf * kStage; };             // (m, k) at k * LDM + m
        auto sZ = [&](int buf) { return sm + buf * kStage + CK * LDM; };  // (n, k) at n * LDK + k
        auto issue = [&](int c) {
            const int64_t k0 = kb + (int64_t)c * CK;
            const int kc = (int)(ke - k0 < CK ? ke - k0 : CK), kc4 = (kc + 3) & ~3;  // k padding zero
            double *y = sY(c & 1), *z = sZ(c & 1);
            for (int idx = tid; idx < p * kc4; idx += CT) {  // m fastest: coalesced for F-order Y
                const int m = idx % p, k = idx / p;
                cpa8(&y[k * LDM + m], &g.y(m, k0 + (k < kc ? k : 0)), k < kc);
            }
            for (int idx = tid; idx < q * kc4; idx += CT) {  // k fastest: coalesced for F-order Z
                const int k = idx % kc4, n = idx / kc4;
                cpa8(&z[n * LDK + k], &g.z(k0 + (k < kc ? k : 0), n), k < kc);
            }
            cpa_commit();
        };
        if (nch > 0) issue(0);
        for (int c = 0; c < nch; ++c) {
            if (c + 1 < nch)
                issue(c + 1);
            else
                cpa_commit();  // empty group: the wait below stays "all but the newest"
            cpa_wait1();
            __syncthreads();
            const int64_t k0 = kb + (int64_t)c * CK;
            const int kc = (int)(ke - k0 < CK ? ke - k0 : CK), kc4 = (kc + 3) & ~3;
            const double *y = sY(c & 1), *z = sZ(c & 1);
            for (int kk = 0; kk < kc4; kk += 4) {
                double af[4], bf[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) af[i] = y[(kk + fc) * LDM + wm + 8 * i + fr];
#pragma unroll
                for (int j = 0; j < 4; ++j) bf[j] = z[(wn + 8 * j + fr) * LDK + kk + fc];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j)  // fragments outside T: warp-uniform skip
                        if (wm + 8 * i < p && wn + 8 * j < q) mma884(acc[i][j], af[i], bf[j]);
            }
            __syncthreads();  // buffer c & 1 is reloaded by issue(c + 2)
        }
        double *pb = g.part + (int64_t)b * p * q;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = wm + 8 * i + fr, n = wn + 8 * j + 2 * fc + h;
                    if (m < p && n < q) pb[m + (int64_t)n * p] = acc[i][j][h];
                }
    }
    if (mark) g.dbg[1] = gtime();
    grid.sync();
    if (mark) g.dbg[2] = gtime();

    // ---- phase 2: T = sum_b P_b, fixed order (8 groups of CTAs, then the groups)
    {
        const int E = p * q, per = (E + G - 1) / G;
        const int e0 = b * per, e1 = e0 + per < E ? e0 + per : E;
        double *red = sm;  // [8][64]
        const int le = tid & 63, grp = tid >> 6;
        const int b0 = grp * G / 8, b1 = (grp + 1) * G / 8;  // <= kMaxGroup partials per thread
        for (int base = e0; base < e1; base += 64) {
            const int e = base + le;
            double s = 0.0;
            if (e < e1) {
                // every load in flight first, then the fixed-order sum
                double v[kMaxGroup];
#pragma unroll
                for (int u = 0; u < kMaxGroup; ++u)
                    v[u] = b0 + u < b1 ? __ldcg(g.part + (int64_t)(b0 + u) * E + e) : 0.0;
#pragma unroll
                for (int u = 0; u < kMaxGroup; ++u) s += v[u];
            }
            red[grp * 64 + le] = s;
            __syncthreads();
            if (grp == 0 && e < e1) {
                double t = red[le];
#pragma unroll
                for (int h = 1; h < 8; ++h) t += red[h * 64 + le];
                g.t(e % p, e / p) = t;
            }
            __syncthreads();
        }
    }
    if (mark) g.dbg[3] = gtime();
    grid.sync();
    if (mark) g.dbg[4] = gtime();

    // ---- phase 3: out[r0:r0+R, :] = X[r0:r0+R, 0:p] T
    {
        double *sT = sm;  // (k, n) at n * LDP + k (over phase 1's buffers)
        for (int idx = tid; idx < q * p4; idx += CT) {
            const int k = idx % p4, n = idx / p4;
            sT[n * LDP + k] = k < p ? __ldcg(&g.t(k, n)) : 0.0;  // (written by other SMs: L2, not L1)
        }
        const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
        for (int64_t tile = b; tile < ntiles; tile += G) {
            const int64_t r0 = tile * R;
            const int rr = (int)(M - r0 < R ? M - r0 : R);
            if (tile != b) {  // later tiles (very tall X): load now
                __syncthreads();
                load_x(tile);
                cpa_commit();
            }
            cpa_wait0();
            __syncthreads();
            double acc[4][2][2];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            for (int kk = 0; kk < p4; kk += 4) {
                double af[4], bf[2];
#pragma unroll
                for (int i = 0; i < 4; ++i) af[i] = sX[(kk + fc) * LDX + wm + 8 * i + fr];
#pragma unroll
                for (int j = 0; j < 2; ++j) bf[j] = sT[(wn + 8 * j + fr) * LDP + kk + fc];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        if (wm + 8 * i < rr && wn + 8 * j < q) mma884(acc[i][j], af[i], bf[j]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int m = wm + 8 * i + fr, n = wn + 8 * j + 2 * fc + h;
                        if (m < rr && n < q) g.out(r0 + m, n) = acc[i][j][h];
                    }
        }
    }
    if (mark) g.dbg[5] = gtime();
}

}  // namespace
}  // namespace lm

using namespace lm;

// 0 = done; 1 = shapes not covered (caller runs the two GEMMs).
extern "C" int lm_gemm_chain(int dtype, lm_view x, lm_view y, lm_view z, lm_view t, lm_view out, void *stream) {
    clear_error();
    if (dtype != LM_F64) return 1;
    LM_REQUIRE(x.cols == y.rows && y.cols == z.rows, "gemm_chain: inner dimensions");
    LM_REQUIRE(t.rows == y.rows && t.cols == z.cols, "gemm_chain: T shape");
    LM_REQUIRE(out.rows == x.rows && out.cols == z.cols, "gemm_chain: out shape");
    const int64_t p = y.rows, q = z.cols, K = y.cols, M = x.rows;
    if (p < 1 || q < 1 || p > TMX || q > TMX || K < 1 || M < 1) return 1;
    cudaStream_t s = as_stream(stream);
    const size_t smem = sizeof(double) * (size_t)kSmem;
    if (int rc = func_attrs(gemm_chain_kernel, smem)) return rc;
    int per_sm = 0;
    LM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_chain_kernel, CT, smem));
    if (per_sm < 1) return 1;
    const int G = num_sms() < 8 * kMaxGroup ? num_sms() : 8 * kMaxGroup;
    Scratch part;
    if (int rc = part.alloc(sizeof(double) * (size_t)G * p * q, s)) return rc;
    ChainArgs g;
    g.x = View<const double>{(const double *)x.ptr, x.rows, x.cols, x.rs, x.cs};
    g.y = View<const double>{(const double *)y.ptr, y.rows, y.cols, y.rs, y.cs};
    g.z = View<const double>{(const double *)z.ptr, z.rows, z.cols, z.rs, z.cs};
    g.t = to_view<double>(t);
    g.out = to_view<double>(out);
    g.part = part.as<double>();
    g.kchunk = ceil_div(K, G);
    int rows3 = (int)((ceil_div(M, G) + 7) / 8 * 8);
    g.rows3 = rows3 < 8 ? 8 : rows3 > R3 ? R3 : rows3;
    static const bool trace = getenv("LM_CHAIN_TRACE") != nullptr;
    g.dbg = nullptr;
    unsigned long long *dbg = nullptr;
    if (trace) {
        LM_CUDA(cudaMalloc(&dbg, 8 * sizeof(unsigned long long)));
        g.dbg = dbg;
    }
    void *kargs[] = {&g};
    LM_CUDA(cudaLaunchCooperativeKernel((const void *)gemm_chain_kernel, dim3(G), dim3(CT), kargs, smem, s));
    count_launch(1);
    if (trace) {
        unsigned long long h[8];
        LM_CUDA(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, s));
        LM_CUDA(cudaStreamSynchronize(s));
        dbg = h;
        fprintf(stderr, "CHAINTRACE phase1 %.2f us, sync %.2f, phase2 %.2f, sync %.2f, phase3 %.2f (G=%d, M=%lld)\n",
                (dbg[1] - dbg[0]) * 1e-3, (dbg[2] - dbg[1]) * 1e-3, (dbg[3] - dbg[2]) * 1e-3,
                (dbg[4] - dbg[3]) * 1e-3, (dbg[5] - dbg[4]) * 1e-3, G, (long long)M);
        cudaFree(g.dbg);
    }
    return 0;
}
