// gemm_skinny.cu -- FP64 products with one or two short dimensions, the two
// shapes R6 makes of BASELINE config 3b's chain X (8000 x 100) * Y (100 x
// 8000) * Z (8000 x 100) -> X * (Y * Z) (lazymat/rewrite.py:317-328; both
// products run through _gemm, lazymat/_loops.py:87-98):
//
//   tall-K  (Y * Z: M, N <= 128, K large).  64 x 64 tiles cover a 100 x 100
//           output 1.6x over and need ~100 split-K partials plus a finish
//           launch.  Here ONE CTA per SM owns the whole (<= 128 x 128)
//           output over its own K slice (16 warps, 4 x 4, <= 4 x 4 DMMA
//           fragments each), the per-SM partials stay in L2, and after a
//           grid barrier every CTA sums a slice of the output over all
//           partials in a fixed order -- one launch, reproducible.
//   tall-M  (X * T: N, K <= 128, M large).  One CTA per band of <= 64 rows
//           (sized so that all bands are one wave), T whole in shared
//           memory, the band's K rows in eight copy groups (one mbarrier
//           each) so the DMMAs start after T and the first eighth.
//
// Fragment rows / columns are dealt to the warps round-robin (fragment f of
// a dimension belongs to warp coordinate f % 4), and warp w sits at
// (w / 4, (w + w / 4) % 4), so the four SM sub-partitions (warp % 4) get
// 43 / 42 / 42 / 42 of the 169 live fragments of a 100 x 100 output.
// Shared-memory rows: the outer-contiguous operand [k][m] with a row length
// = 8 (mod 16) doubles, the K-contiguous one [n][k] with a row length = 4
// (mod 8): both make an m8n8k4 fragment load two conflict-free wavefronts.
//
// Operands: A(m, k) unit-stride along m, B(k, n) unit-stride along k (what
// F-order matrices give), 16-byte aligned with even leading dimensions, M
// even and K a multiple of 4 (the tiles arrive as bulk copies of whole rows /
// column pieces); anything else stays on the tiled kernels (gemm.cu).  LM_GEMM_SKINNY=0
// disables both.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {
namespace {

constexpr int SKT = 512;  // 16 warps

struct SkinnyArgs {
    const double *a;
    int64_t a_sk;  // A(m,k) = a[m + k*a_sk]
    const double *b;
    int64_t b_sn;  // B(k,n) = b[k + n*b_sn]
    double *c;
    int64_t c_sm, c_sn;
    int64_t M, N, K;
    int64_t kchunk;  // tall-K: K range per CTA (multiple of 4, <= 64)
    double *part;    // tall-K: [gridDim.x][M*N] F-order partials
    int epb;         // tall-K: elements per reduction pass (multiple of 8, <= 512)
    int per;         // tall-K: output elements per CTA in the reduction
    int mb;          // tall-M: rows per CTA (multiple of 8, <= 64)
    int ldb;         // tall-M: smem row length of B (>= K, = 4 mod 8)
    int kg;          // tall-M: K rows per copy group (multiple of 4)
    int lda;         // tall-K: smem row length of A (M when the rows arrive in one piece per group)
    unsigned long long *dbg;  // LM_SKINNY_TRACE: phase timestamps of CTA 0 (globaltimer, ns)
};

__device__ __forceinline__ void stamp(const SkinnyArgs &g, int slot) {
    if (g.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g.dbg[slot] = t;
    }
}

__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}
// Bulk asynchronous copies (the TMA unit, no tensor map) completing on an
// mbarrier by transaction bytes.  Every issuing thread arrives on the
// stage's barrier itself -- expect_tx(bytes) before its copy, a plain arrive
// when it has nothing to copy -- so a phase completes only when all issuers
// have been there and all their bytes have landed.  (Per-lane 16-byte
// cp.async delivered ~10-25 GB/s per SM here: every group took ~2.5 us.)
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

// One k4 step of a warp's fragments: rows 8 (wr + 4 i), i < NI, columns
// 8 (wc + 4 j), j < NJ; pa / pb point at the lane's element of fragment
// (0, 0).  NI and NJ are compile-time (the warp's live fragment counts pick
// the instantiation once per kernel): the loop body is LDS.64 + DMMA only --
// with per-fragment run-time predicates the other instructions took as many
// issue slots as the DMMAs (11.6 instead of 7 us for config 3b's Y * Z).
template <int NI, int NJ, int FI, int FJ>
__device__ __forceinline__ void k4_step(double (&acc)[FI][FJ][2], const double *pa, const double *pb, int ldb) {
    double af[NI ? NI : 1], bf[NJ ? NJ : 1];
#pragma unroll
    for (int i = 0; i < NI; ++i) af[i] = pa[32 * i];
#pragma unroll
    for (int j = 0; j < NJ; ++j) bf[j] = pb[32 * j * ldb];
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) mma884(acc[i][j], af[i], bf[j]);
}
template <int V> using IC = std::integral_constant<int, V>;

// ---------------------------------------------------------------------------
// tall-K
// ---------------------------------------------------------------------------
// A CTA's whole K slice (<= 64 rows) is resident: B [n][68] arrives as one
// copy per column (the slice is contiguous in a column), A [k][lda] as one
// copy per group of 16 K rows when the rows are contiguous in HBM and M is a
// conflict-free row length, else one copy per row -- the TMA unit takes ~30
// cycles per copy whatever its size, so few large copies matter (one copy per
// column per 16-row stage: first stage ready after 5 us instead of 2).
constexpr int TK_SK = 16;                 // K rows per group (one mbarrier each)
constexpr int TK_NS = 4;                  // groups
constexpr int TK_KC = TK_SK * TK_NS;      // largest K slice
constexpr int TK_LDA = 136;               // [k][m] row length when A's rows are copied one by one
constexpr int TK_LDB = TK_KC + 4;         // [n][k], 68 = 4 (mod 8)
constexpr int TK_SMEM = (TK_KC * TK_LDA + 128 * TK_LDB) * 8;

__global__ void __launch_bounds__(SKT, 1) dgemm_tallk(SkinnyArgs g) {
    extern __shared__ __align__(16) double ksm[];
    __shared__ double red[SKT];
    __shared__ unsigned long long full[TK_NS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wr = warp >> 2, wc = ((warp & 3) + wr) & 3;
    const int fr = lane >> 2, fc = lane & 3;
    const int64_t M = g.M, N = g.N, MN = M * N;
    const int64_t kb = (int64_t)blockIdx.x * g.kchunk;
    const int64_t ke = kb + g.kchunk < g.K ? kb + g.kchunk : g.K;
    const int klen = ke > kb ? (int)(ke - kb) : 0;  // <= TK_KC, a multiple of 4
    const int nst = (klen + TK_SK - 1) / TK_SK;
    const int lda = g.lda;
    const bool a_rows = lda != M;  // A row by row
    double *sA = ksm, *sB = ksm + TK_KC * lda;
    const int nfr = (int)((M + 7) >> 3), nfc = (int)((N + 7) >> 3);
    unsigned live_i = 0, live_j = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (wr + 4 * i < nfr) live_i |= 1u << i;
        if (wc + 4 * i < nfc) live_j |= 1u << i;
    }
    if (tid == 0) {
#pragma unroll
        for (int st = 0; st < TK_NS; ++st) {
            const int rows = klen - st * TK_SK < TK_SK ? klen - st * TK_SK : TK_SK;
            const int cnt = (st == 0 ? (int)N : 0) + (rows <= 0 ? 0 : a_rows ? rows : 1);
            mbar_init(&full[st], cnt ? cnt : 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    stamp(g, 0);
    // issuers: thread n < N column n of B (group 0 needs all of B); thread
    // N + j row j of A, or A's group j in one piece
    if (klen > 0) {
        if (tid < N) {
            bulk_copy(sB + tid * TK_LDB, g.b + (int64_t)tid * g.b_sn + kb, (unsigned)(klen * 8), &full[0]);
        } else if (a_rows) {
            const int k = tid - (int)N;
            if (k < klen) bulk_copy(sA + k * lda, g.a + (kb + k) * g.a_sk, (unsigned)(M * 8), &full[k / TK_SK]);
        } else {
            const int st = tid - (int)N;
            if (st < nst) {
                const int rows = klen - st * TK_SK < TK_SK ? klen - st * TK_SK : TK_SK;
                bulk_copy(sA + st * TK_SK * lda, g.a + (kb + st * TK_SK) * g.a_sk, (unsigned)(rows * M * 8), &full[st]);
            }
        }
    }
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    auto main_loop = [&](auto ni, auto nj) {
        constexpr int NI = decltype(ni)::value, NJ = decltype(nj)::value;
        const double *pa = sA + fc * lda + 8 * wr + fr, *pb = sB + (8 * wc + fr) * TK_LDB + fc;
#pragma unroll 1
        for (int st = 0; st < nst; ++st) {
            mbar_wait(&full[st], 0);
            stamp(g, 8 + st);
            const int k0 = st * TK_SK;
            if (klen - k0 >= TK_SK) {
#pragma unroll
                for (int k = 0; k < TK_SK; k += 4) k4_step<NI, NJ>(acc, pa + (k0 + k) * lda, pb + k0 + k, TK_LDB);
            } else {
                for (int k = k0; k < klen; k += 4) k4_step<NI, NJ>(acc, pa + k * lda, pb + k, TK_LDB);
            }
        }
    };
    const int cnt_i = __popc(live_i), cnt_j = __popc(live_j);
    switch (cnt_i && cnt_j ? cnt_i * 5 + cnt_j : 0) {
#define LM_TK_CASE(I, J)              \
    case I * 5 + J:                   \
        main_loop(IC<I>{}, IC<J>{}); \
        break;
        LM_TK_CASE(1, 1) LM_TK_CASE(1, 2) LM_TK_CASE(1, 3) LM_TK_CASE(1, 4)
        LM_TK_CASE(2, 1) LM_TK_CASE(2, 2) LM_TK_CASE(2, 3) LM_TK_CASE(2, 4)
        LM_TK_CASE(3, 1) LM_TK_CASE(3, 2) LM_TK_CASE(3, 3) LM_TK_CASE(3, 4)
        LM_TK_CASE(4, 1) LM_TK_CASE(4, 2) LM_TK_CASE(4, 3) LM_TK_CASE(4, 4)
#undef LM_TK_CASE
        default:
            main_loop(IC<0>{}, IC<0>{});
    }
    stamp(g, 1);
    const bool direct = gridDim.x == 1;
    double *dst = direct ? g.c : g.part + (int64_t)blockIdx.x * MN;
    const int64_t d_sm = direct ? g.c_sm : 1, d_sn = direct ? g.c_sn : M;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t m = 8 * (wr + 4 * i) + fr, n = 8 * (wc + 4 * j) + 2 * fc + h;
                if (m < M && n < N) dst[m * d_sm + n * d_sn] = acc[i][j][h];
            }
    if (direct) return;
    stamp(g, 2);
    cg::this_grid().sync();
    pdl_trigger();  // the next kernel's launch may be processed while the slices are summed
    stamp(g, 3);
    // C slice = sum of the partials in a fixed order: thread (zg, el) sums the
    // partials z = zg (mod ZG) of element el of the pass, the ZG group sums are
    // added in group order
    const int epb = g.epb, ZG = SKT / epb, el = tid % epb, zg = tid / epb;
    const int64_t start = (int64_t)blockIdx.x * g.per;
    const int64_t end = start + g.per < MN ? start + g.per : MN;
    const int nz = (int)gridDim.x;
    for (int64_t e0 = start; e0 < end; e0 += epb) {
        const int64_t e = e0 + el;
        double s = 0.0;
        if (e < end && zg < ZG) {
            // batches of RB independent L2 loads (one round trip each), added in z order
            constexpr int RB = 24;
            const int64_t step = (int64_t)ZG * MN;
            const double *p = g.part + e + (int64_t)zg * MN;
            for (int z = zg; z < nz; z += RB * ZG, p += RB * step) {
                double v[RB];
#pragma unroll
                for (int i = 0; i < RB; ++i) v[i] = z + i * ZG < nz ? __ldcg(p + i * step) : 0.0;
#pragma unroll
                for (int i = 0; i < RB; ++i) s += v[i];
            }
        }
        red[tid] = s;
        __syncthreads();
        if (zg == 0 && e < end) {
            double v = red[el];
            for (int q = 1; q < ZG; ++q) v += red[q * epb + el];
            const int64_t n = e / M, m = e - n * M;
            g.c[m * g.c_sm + n * g.c_sn] = v;
        }
        __syncthreads();
    }
    stamp(g, 4);
}

// ---------------------------------------------------------------------------
// tall-M
// ---------------------------------------------------------------------------
constexpr int TM_LDA = 72;  // [k][m], 64 rows + 8: 72 = 8 (mod 16)
constexpr int TM_NG = 8;    // copy groups along K (one mbarrier each)

__global__ void __launch_bounds__(SKT, 1) dgemm_tallm(SkinnyArgs g) {
    pdl_wait();  // inputs may be the previous kernel's output (PDL)
    pdl_trigger();
    extern __shared__ __align__(16) double msm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wr = warp >> 2, wc = ((warp & 3) + wr) & 3;
    const int fr = lane >> 2, fc = lane & 3;
    const int64_t M = g.M, N = g.N, K = g.K;
    const int Kp = (int)((K + 3) & ~3ll), ldb = g.ldb, kg = g.kg;
    double *sA = msm, *sB = msm + Kp * TM_LDA;
    const int64_t m0 = (int64_t)blockIdx.x * g.mb;
    const int nfr = g.mb >> 3, nfc = (int)((N + 7) >> 3);
    unsigned live_i = 0, live_j = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (i < 2 && wr + 4 * i < nfr && m0 + 8 * (wr + 4 * i) < M) live_i |= 1u << i;
        if (wc + 4 * i < nfc) live_j |= 1u << i;
    }
    // issuers: thread k < K copies row k of the band (its rows of A's column
    // k) onto the barrier of k's group, thread Kp + n column n of B onto
    // group 0's
    __shared__ unsigned long long full[TM_NG];
    const bool b_one = g.b_sn == ldb;  // B contiguous with a conflict-free leading dimension: one copy
    if (tid == 0) {
#pragma unroll
        for (int grp = 0; grp < TM_NG; ++grp) {
            const int k0 = grp * kg;
            const int rows = k0 >= Kp ? 0 : Kp - k0 < kg ? Kp - k0 : kg;
            const int cnt = rows + (grp == 0 ? (b_one ? 1 : (int)N) : 0);
            mbar_init(&full[grp], cnt ? cnt : 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    stamp(g, 0);
    if (tid < Kp) {
        const int64_t rows = M - m0 < g.mb ? M - m0 : g.mb;
        bulk_copy(sA + tid * TM_LDA, g.a + m0 + (int64_t)tid * g.a_sk, (unsigned)(rows * 8), &full[tid / kg]);
    } else if (b_one) {
        if (tid == Kp) bulk_copy(sB, g.b, (unsigned)(N * ldb * 8), &full[0]);
    } else if (tid < Kp + N) {
        const int n = tid - Kp;
        bulk_copy(sB + n * ldb, g.b + (int64_t)n * g.b_sn, (unsigned)(K * 8), &full[0]);
    }
    double acc[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    auto main_loop = [&](auto ni, auto nj) {
        constexpr int NI = decltype(ni)::value, NJ = decltype(nj)::value;
        const double *pa = sA + fc * TM_LDA + 8 * wr + fr, *pb = sB + (8 * wc + fr) * ldb + fc;
        stamp(g, 1);
#pragma unroll 1
        for (int grp = 0; grp * kg < Kp; ++grp) {
            mbar_wait(&full[grp], 0);
            if (grp == 0) stamp(g, 2);
            const int k0 = grp * kg;
            const int k1 = k0 + kg < Kp ? k0 + kg : Kp;
            for (int k = k0; k < k1; k += 4) k4_step<NI, NJ>(acc, pa + k * TM_LDA, pb + k, ldb);
        }
        stamp(g, 3);
    };
    const int cnt_i = __popc(live_i), cnt_j = __popc(live_j);
    switch (cnt_i && cnt_j ? cnt_i * 5 + cnt_j : 0) {
#define LM_TM_CASE(I, J)              \
    case I * 5 + J:                   \
        main_loop(IC<I>{}, IC<J>{}); \
        break;
        LM_TM_CASE(1, 1) LM_TM_CASE(1, 2) LM_TM_CASE(1, 3) LM_TM_CASE(1, 4)
        LM_TM_CASE(2, 1) LM_TM_CASE(2, 2) LM_TM_CASE(2, 3) LM_TM_CASE(2, 4)
#undef LM_TM_CASE
        default:
            main_loop(IC<0>{}, IC<0>{});
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t m = m0 + 8 * (wr + 4 * i) + fr, n = 8 * (wc + 4 * j) + 2 * fc + h;
                if (((live_i >> i) & 1) && m < M && n < N) g.c[m * g.c_sm + n * g.c_sn] = acc[i][j][h];
            }
    stamp(g, 4);
}

// LM_SKINNY_TRACE=1: synchronous launches that print CTA 0's phase times
struct Trace {
    unsigned long long *dbg = nullptr;
    bool on() {
        static const bool t = getenv("LM_SKINNY_TRACE") && getenv("LM_SKINNY_TRACE")[0] == '1';
        return t;
    }
    void arm(SkinnyArgs &g) {
        if (on() && cudaMalloc(&dbg, 16 * sizeof(unsigned long long)) == cudaSuccess) {
            cudaMemset(dbg, 0, 16 * sizeof(unsigned long long));
            g.dbg = dbg;
        }
    }
    void report(const char *name, const char *const *phase, cudaStream_t s) {
        if (!dbg) return;
        unsigned long long h[16];
        cudaStreamSynchronize(s);
        cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
        fprintf(stderr, "SKINNYTRACE %s:", name);
        for (int i = 0; i < 4; ++i) fprintf(stderr, " %s %.2f us", phase[i], (double)(h[i + 1] - h[i]) * 1e-3);
        if (h[8]) {
            fprintf(stderr, " | stage ready at");
            for (int i = 8; i < 16 && h[i]; ++i) fprintf(stderr, " %.2f", (double)(h[i] - h[0]) * 1e-3);
        }
        fprintf(stderr, "\n");
        cudaFree(dbg);
        dbg = nullptr;
    }
};

bool skinny_enabled() {
    static const bool on = [] {
        const char *e = getenv("LM_GEMM_SKINNY");
        return !(e && e[0] == '0');
    }();
    return on;
}

int launch_tallk(SkinnyArgs &g, cudaStream_t s) {
    if (int rc = func_attrs(dgemm_tallk, TK_SMEM)) return rc;
    const int64_t sms = num_sms();
    g.kchunk = ceil_div(ceil_div(g.K, sms), 4) * 4;
    if (g.kchunk < 32) g.kchunk = 32;
    if (g.kchunk > TK_KC) return 1;  // K > 64 per SM: enough work per tile for the tiled kernels
    // rows of A contiguous in HBM and M a conflict-free row length (4 mod 8 or
    // 8 mod 16 doubles): 16 rows per copy, no padding
    g.lda = (g.a_sk == g.M && ((g.M & 7) == 4 || (g.M & 15) == 8)) ? (int)g.M : TK_LDA;
    const int64_t splits = ceil_div(g.K, g.kchunk);
    const int64_t MN = g.M * g.N;
    g.per = (int)(ceil_div(ceil_div(MN, splits), 8) * 8);
    g.epb = g.per < SKT ? g.per : SKT;
    Scratch part;
    if (splits > 1) {
        if (int rc = part.alloc(sizeof(double) * MN * splits, s)) return rc;
        g.part = part.as<double>();
    }
    Trace tr;
    tr.arm(g);
    void *kargs[] = {&g};
    LM_CUDA(cudaLaunchCooperativeKernel((const void *)dgemm_tallk, dim3((unsigned)splits), dim3(SKT), kargs, TK_SMEM,
                                        s));
    count_launch(1);
    static const char *const ph[] = {"main loop", "partial store", "grid barrier", "ordered sum"};
    tr.report("tall-K", ph, s);
    note_variant("gemm_tallk");
    return 0;
}

int launch_tallm(SkinnyArgs &g, cudaStream_t s) {
    const int64_t sms = num_sms();
    int64_t mb = ceil_div(ceil_div(g.M, sms), 8) * 8;
    g.mb = (int)(mb < 8 ? 8 : mb > 64 ? 64 : mb);
    const int Kp = (int)((g.K + 3) & ~3ll);
    g.ldb = (Kp & 7) == 4 ? Kp : Kp + 4;
    g.kg = (int)(ceil_div(ceil_div(Kp, TM_NG), 4) * 4);
    const int nrb = (int)ceil_div(g.N, 8) * 8;
    const size_t smem = sizeof(double) * ((size_t)Kp * TM_LDA + (size_t)nrb * g.ldb);
    if (int rc = func_attrs(dgemm_tallm, 128 * TM_LDA * 8 + 128 * 132 * 8)) return rc;
    Trace tr;
    tr.arm(g);
    LM_CUDA(launch_pdl(dgemm_tallm, dim3((unsigned)ceil_div(g.M, g.mb)), dim3(SKT), smem, s, g));
    LM_LAUNCHED(1);
    static const char *const ph[] = {"copy issue", "first group ready", "main loop", "store"};
    tr.report("tall-M", ph, s);
    note_variant("gemm_tallm");
    return 0;
}

}  // namespace

// 0: launched; 1: not a skinny product (or operands the kernels cannot take);
// < 0: error.
int try_dgemm_skinny(const double *a, int64_t a_sm, int64_t a_sk, const double *b, int64_t b_sk, int64_t b_sn,
                     double *c, int64_t c_sm, int64_t c_sn, int64_t M, int64_t N, int64_t K, cudaStream_t s) {
    if (!skinny_enabled() || a_sm != 1 || b_sk != 1 || N > 128 || N < 16) return 1;
    if (((uintptr_t)a & 15) || ((uintptr_t)b & 15) || (a_sk & 1) || (b_sn & 1) || a_sk < 0 || b_sn < 0) return 1;
    if ((K & 3) || (M & 1)) return 1;  // bulk copies: 16-byte row pieces, whole k4 steps
    const bool tallk = M <= 128 && M >= 16 && K >= 1024;
    const bool tallm = !tallk && K <= 128 && K >= 4 && M >= 1024;
    if (!tallk && !tallm) return 1;
    SkinnyArgs g{};
    g.a = a;
    g.a_sk = a_sk;
    g.b = b;
    g.b_sn = b_sn;
    g.c = c;
    g.c_sm = c_sm;
    g.c_sn = c_sn;
    g.M = M;
    g.N = N;
    g.K = K;
    return tallk ? launch_tallk(g, s) : launch_tallm(g, s);
}

}  // namespace lm
