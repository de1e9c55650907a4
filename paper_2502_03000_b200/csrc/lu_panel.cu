// lu_panel.cu -- the latency-critical piece of the exact LU (config 4a):
// factor a 32-column panel A[j0:n, j0:j0+32] in the reference's order
// (lazymat/_loops.py:200-236: first maximum of |A[i,k]|, full-row swap,
// multipliers by __ddiv_rn, rank-1 update with __dmul_rn/__dsub_rn).
//
// One thread-block CLUSTER (up to 16 CTAs of a GPC); thread t of CTA c owns
// panel rows c*rp + t (+ PT) in registers for the whole panel.  The kernel
// is issue-bound (every warp executes every column's code), so the design
// minimises per-warp instructions per column; rare actions (row swaps, row
// publication) sit behind warp-uniform branches.  Per column c:
//   1. each warp's first maximum (three redux.sync; |v| bits, then row) and
//      its candidate row -> local shared memory; one __syncthreads;
//   2. every warp forms the CTA candidate redundantly and PUSHES (key, row,
//      32 values) -- and row c if this CTA owns it -- to two target CTAs'
//      inboxes with st.async (remote stores that complete transaction bytes
//      on the receiver's mbarrier; no CTA reads remote shared memory, which
//      serialises on the owner SM's DSMEM port, and there is no cluster
//      barrier: a release barrier would also wait for outstanding global
//      stores -- pivots are kept in shared memory until the end);
//   3. the previous column's update of columns > c runs while the pushes
//      land; each CTA then waits on its own inbox mbarrier (expected bytes
//      posted by one thread; the parity alternates every other column);
//   4. every warp picks the winner among the cs inbox candidates and copies
//      the pivot row, applying the previous column's update to its columns
//      > c (the pusher published before applying it; same __dmul_rn /
//      __dsub_rn on the same operands -- bit-identical), swaps, computes
//      the multipliers and updates column c+1 first (look-ahead).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {

constexpr int PNB = 32;      // panel width
constexpr int PT = 256;      // threads per CTA
constexpr int PW = PT / 32;  // warps per CTA
constexpr int MAXCS = 16;    // largest cluster

struct ClusterPanelArgs {
    double *A;
    int64_t lda, n, j0;
    int nb, rp;  // panel width, rows per CTA
    int64_t *piv;
    int32_t *info;
    long long *dbg;  // optional per-column phase timestamps (CTA 0, thread 0)
    int64_t J0, J1;  // fused epilogue (J1 > J0): the panel's row swaps on the outer
                     // block's other columns [J0, j0) U [j0+nb, J1), then
                     // U12 = L11^-1 A12 on [j0+nb, J1) -- by CTA 0
};

// Fused epilogue of the panel (CTA 0): the panel's sequential swaps composed
// into one permutation of the touched rows (<= 2 nb), applied as a gather to
// the outer block's other columns in chunks of 32; then the unit-lower
// triangular solve of the nb rows of A12 (one thread per column, the
// reference's order: x_i -= L[i,j] x_j, j ascending, rounded mul and sub).
template <int R>
__device__ __forceinline__ void panel_epilogue(const double (&r)[R][PNB], const ClusterPanelArgs &a,
                                               const long long *lpiv) {
    __shared__ int tkey[2 * PNB], tsrc[2 * PNB];
    __shared__ int s_nt;
    __shared__ double gbuf[2 * PNB][33];
    __shared__ double sT[PNB][PNB + 1];
    const int tid = threadIdx.x, nb = a.nb;
    const int64_t j0 = a.j0, lda = a.lda;
    // compose the swaps (warp 0): lane k tracks the source row of top
    // position k; lane i tracks bottom position bkey (a row >= nb pivoted
    // up) and its source; ballot finds a bottom position in O(1)
    if (tid < 32) {
        const int lane = tid;
        int top_src = lane, bkey = -1, bsrc = 0, nbot = 0;
        for (int k = 0; k < nb; ++k) {
            const int p = (int)(a.piv[a.j0 + k] - a.j0);  // (written by this CTA's thread 0)
            if (p == k) continue;
            const int a_src = __shfl_sync(0xffffffffu, top_src, k);
            int b_src;
            if (p < nb) {
                b_src = __shfl_sync(0xffffffffu, top_src, p);
                if (lane == p) top_src = a_src;
            } else {
                const unsigned m = __ballot_sync(0xffffffffu, bkey == p);
                if (m) {
                    const int j = __ffs(m) - 1;
                    b_src = __shfl_sync(0xffffffffu, bsrc, j);
                    if (lane == j) bsrc = a_src;
                } else {
                    b_src = p;  // untouched so far: holds its own row
                    if (lane == nbot) {
                        bkey = p;
                        bsrc = a_src;
                    }
                    ++nbot;
                }
            }
            if (lane == k) top_src = b_src;
        }
        if (lane < nb) {
            tkey[lane] = lane;
            tsrc[lane] = top_src;
        }
        if (lane < nbot) {
            tkey[nb + lane] = bkey;
            tsrc[nb + lane] = bsrc;
        }
        if (lane == 0) s_nt = nb + nbot;
    }
    // L11 (unit lower) from the registers of rows 0..nb-1 (threads 0..nb-1, q = 0)
    if (tid < nb)
#pragma unroll
        for (int j = 0; j < PNB; ++j) sT[tid][j] = r[0][j];
    __syncthreads();
    const int nt = s_nt;
    const int64_t left = j0 - a.J0, right = a.J1 - (j0 + nb), ncol = left + right;
    auto colof = [&](int64_t c) { return c < left ? a.J0 + c : j0 + nb + (c - left); };
    for (int64_t cb = 0; cb < ncol && nt > 0; cb += 32) {
        const int w = (int)((ncol - cb) < 32 ? (ncol - cb) : 32);
        for (int e = tid; e < nt * w; e += PT) {
            const int i = e / w, cc = e - (e / w) * w;
            gbuf[i][cc] = a.A[(j0 + tsrc[i]) + colof(cb + cc) * lda];
        }
        __syncthreads();
        for (int e = tid; e < nt * w; e += PT) {
            const int i = e / w, cc = e - (e / w) * w;
            a.A[(j0 + tkey[i]) + colof(cb + cc) * lda] = gbuf[i][cc];
        }
        __syncthreads();
    }
    for (int64_t c = tid; c < right; c += PT) {
        double *col = a.A + j0 + (j0 + nb + c) * lda;
        double x[PNB];
#pragma unroll
        for (int i = 0; i < PNB; ++i) x[i] = i < nb ? col[i] : 0.0;
#pragma unroll
        for (int j = 0; j < PNB; ++j) {
            if (j >= nb) break;
            const double xj = x[j];
#pragma unroll
            for (int i = j + 1; i < PNB; ++i)
                if (i < nb) x[i] = __dsub_rn(x[i], __dmul_rn(sT[i][j], xj));
        }
#pragma unroll
        for (int i = 0; i < PNB; ++i)
            if (i < nb) col[i] = x[i];
    }
}

struct PanelSmem {
    double ival[2][MAXCS][PNB];         // inbox: each CTA's candidate row
    unsigned long long ikey[2][MAXCS];  // inbox: candidate keys ((|v| hi + 1) << 32 | lo), 0 = none
    long long irow[2][MAXCS];           // inbox: candidate rows
    double ik[2][PNB];                  // inbox: row c (pushed by its owner)
    unsigned long long bar[2];          // inbox mbarriers (transaction bytes of st.async pushes)
    double wv[2][PW][PNB];              // local: warp candidate rows
    unsigned long long wkey[2][PW];     // local: warp candidate keys
    int wrw[2][PW];                     // local: warp candidate rows
    double rk[2][PNB];                  // local: row c staged by its owner
    double U[PW][PNB];                  // per-warp copy of the current pivot row
    double K[PW][PNB];                  // per-warp copy of old row c (swap partner)
    long long piv[PNB];                 // pivots (CTA 0), written out at the end
    long long dclk[PNB * 8];            // debug clocks (CTA 0, thread 0)
};

__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned cluster_addr(unsigned local, unsigned rank) {
    unsigned r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// remote 8-byte store that completes `bytes` on the receiver's mbarrier
__device__ __forceinline__ void push_f64(unsigned raddr, double v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(v),
                 "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void push_b64(unsigned raddr, unsigned long long v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(v),
                 "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
}

// (value, row) "first maximum" over the lanes of a warp.  v >= 0 (|A| or
// +inf), valid = row participates.  Returns the winning row, and its value
// bits in (hi, lo) with hi = high word + 1 (0 = none).
__device__ __forceinline__ int warp_first_max(double v, bool valid, int row, unsigned &hi, unsigned &lo) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const unsigned h = valid ? (unsigned)(b >> 32) + 1u : 0u;
    hi = __reduce_max_sync(0xffffffffu, h);
    const unsigned l = (valid && h == hi) ? (unsigned)b : 0u;
    lo = __reduce_max_sync(0xffffffffu, l);
    const unsigned r = (valid && h == hi && (unsigned)b == lo) ? (unsigned)row : 0xffffffffu;
    const unsigned best = __reduce_min_sync(0xffffffffu, r);
    return hi == 0 ? -1 : (int)best;
}

// (key, row) first maximum over lanes: larger key, then smaller row.
__device__ __forceinline__ void key_first_max(unsigned long long key, int row, bool valid, unsigned &P,
                                              unsigned &who, unsigned &H, unsigned &L) {
    const unsigned h = valid ? (unsigned)(key >> 32) : 0u, l = valid ? (unsigned)key : 0u;
    H = __reduce_max_sync(0xffffffffu, h);
    L = __reduce_max_sync(0xffffffffu, h == H ? l : 0u);
    const bool top = valid && h == H && l == L && H != 0u;
    P = __reduce_min_sync(0xffffffffu, top ? (unsigned)row : 0xffffffffu);
    who = __ballot_sync(0xffffffffu, top && (unsigned)row == P);
}

// steps 1-3 for column c (all indices static after unrolling): candidates,
// pushes, arrive.
template <int R>
__device__ __forceinline__ void panel_push(const double (&r)[R][PNB], const double (&cv)[R], const int (&myrow)[R],
                                           const int c, PanelSmem &sm, cg::cluster_group &cl, int cs, int me,
                                           bool own_c, long long *dclk = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int par = c & 1;
    // this thread's best row (rows ascend with q: strict > keeps the first)
    double bv = 0.0;
    int bq = -1, brw = 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        if (myrow[q] < c) continue;  // rows above c and unused rows (-1)
        double v = fabs(cv[q]);
        if (v != v) {
            if (myrow[q] != c) continue;  // NaN never wins off the diagonal
            v = __longlong_as_double(0x7ff0000000000000LL);
        }
        if (bq < 0 || v > bv) {
            bv = v;
            bq = q;
            brw = myrow[q];
        }
    }
    unsigned whi, wlo;
    const int wrow = warp_first_max(bv, bq >= 0, brw, whi, wlo);
    // the warp's winning lane publishes its row (one lane per warp)
    if (whi != 0 && brw == wrow && bq >= 0) {
#pragma unroll
        for (int q = 0; q < R; ++q)
            if (q == bq) {
#pragma unroll
                for (int j = 0; j < PNB; ++j) sm.wv[par][wid][j] = r[q][j];
            }
    }
    // the owner of row c stages it (whole row: a swap moves the multipliers too)
    if (own_c) {
        bool mine = false;
#pragma unroll
        for (int q = 0; q < R; ++q) mine |= myrow[q] == c;
        if (__any_sync(0xffffffffu, mine) && mine) {
#pragma unroll
            for (int q = 0; q < R; ++q)
                if (myrow[q] == c) {
#pragma unroll
                    for (int j = 0; j < PNB; ++j) sm.rk[par][j] = r[q][j];
                }
        }
    }
    if (lane == 0) {
        sm.wkey[par][wid] = whi == 0 ? 0ull : (((unsigned long long)whi << 32) | wlo);
        sm.wrw[par][wid] = wrow;
    }
    if (dclk) dclk[4] = clock64();
    __syncthreads();
    if (dclk) dclk[5] = clock64();
    // the CTA candidate (every warp, redundantly) and the pushes
    unsigned P, who, H, L;
    {
        const bool ok = lane < PW;
        const unsigned long long k = ok ? sm.wkey[par][lane] : 0ull;
        const int rw = ok ? sm.wrw[par][lane] : 0;
        key_first_max(k, rw, ok && k != 0ull, P, who, H, L);
    }
    const int sw = who ? __ffs(who) - 1 : 0;
    const unsigned long long key = ((unsigned long long)H << 32) | L;
    const double myv = sm.wv[par][sw][lane];
    const double kvv = own_c ? sm.rk[par][lane] : 0.0;
    const unsigned a_val = smem_addr(&sm.ival[par][me][lane]), a_key = smem_addr(&sm.ikey[par][me]);
    const unsigned a_row = smem_addr(&sm.irow[par][me]), a_k = smem_addr(&sm.ik[par][lane]);
    const unsigned a_bar = smem_addr(&sm.bar[par]);
#pragma unroll
    for (int t0 = 0; t0 < MAXCS; t0 += PW) {
        const unsigned t = t0 + wid;
        if ((int)t < cs) {
            const unsigned rb = cluster_addr(a_bar, t);
            push_f64(cluster_addr(a_val, t), myv, rb);
            if (lane == 0) push_b64(cluster_addr(a_key, t), key, rb);
            if (lane == 1) push_b64(cluster_addr(a_row, t), (unsigned long long)P, rb);
            if (own_c) push_f64(cluster_addr(a_k, t), kvv, rb);
        }
    }
}

// Columns [K0, K0 + PKB) of the panel with a run-time column index kk: the
// body is emitted once per block of 8 columns (a fully unrolled 32-column
// kernel is ~21k instructions and stalls on instruction fetch: ncu
// no_instruction 12 of 20 stall cycles per issue).  Register indices stay
// static: the j loops start at the block's K0 and predicate on j vs kk.
constexpr int PKB = 4;

struct PanelLoop {
    int cs, me, rbeg, rend, nb;
    unsigned col_bytes;
    bool dbg_on;
    double u_prev;
    int info_col;
};

template <int R, int K0>
__device__ __forceinline__ void panel_cols(double (&r)[R][PNB], const int (&myrow)[R], PanelSmem &sm,
                                           cg::cluster_group &cl, PanelLoop &L) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int KE = K0 + PKB;
    const int kend = KE < L.nb ? KE : L.nb;
#pragma unroll 1
    for (int kk = K0; kk < kend; ++kk) {
        const int par = kk & 1;
        if (L.dbg_on) sm.dclk[kk * 8 + 0] = clock64();
        {
            const unsigned b = smem_addr(&sm.bar[par]);
            if (tid == 0) mbar_expect(b, L.col_bytes);
            mbar_wait(b, (unsigned)(kk >> 1) & 1u);  // column kk's inbox is complete
        }
        if (L.dbg_on) sm.dclk[kk * 8 + 1] = clock64();
        // the winner, this warp's copy of the pivot row (+ the missing update
        // of column kk-1 on its columns > kk)
        unsigned P, who, H, Lo;
        {
            const bool ok = lane < L.cs;
            const unsigned long long k = ok ? sm.ikey[par][lane] : 0ull;
            const int rw = ok ? sm.irow[par][lane] : 0;
            key_first_max(k, rw, ok && k != 0ull, P, who, H, Lo);
        }
        const int src = who ? __ffs(who) - 1 : 0;
        const int p = (int)P;
        {
            double u = sm.ival[par][src][lane];
            if (kk > 0) {
                const double mu = sm.ival[par][src][kk - 1];
                if (lane > kk) u = __dsub_rn(u, __dmul_rn(mu, L.u_prev));
            }
            sm.U[wid][lane] = u;
            bool mine_p = false;
#pragma unroll
            for (int q = 0; q < R; ++q) mine_p |= myrow[q] == p;
            if (p != kk && __any_sync(0xffffffffu, mine_p)) {
                double kv = sm.ik[par][lane];
                if (kk > 0) {
                    const double mk = sm.ik[par][kk - 1];
                    if (lane > kk) kv = __dsub_rn(kv, __dmul_rn(mk, L.u_prev));
                }
                sm.K[wid][lane] = kv;
            }
            L.u_prev = u;
            __syncwarp();
        }
        const double *U = sm.U[wid];
        const double ukk = U[kk];
        if (L.me == 0 && tid == 0) {
            sm.piv[kk] = p;
            if (ukk == 0.0 && L.info_col < 0) L.info_col = kk;
        }
        if (L.dbg_on) sm.dclk[kk * 8 + 2] = clock64();
        // full-row swap of rows kk and p (multipliers of columns < kk included)
        if (p != kk) {
            bool hit = false;
#pragma unroll
            for (int q = 0; q < R; ++q) hit |= myrow[q] == kk || myrow[q] == p;
            if (__any_sync(0xffffffffu, hit) && hit) {
                const double *Kr = sm.K[wid];
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    if (myrow[q] == kk) {
#pragma unroll
                        for (int j = 0; j < PNB; ++j) r[q][j] = U[j];
                    } else if (myrow[q] == p) {
#pragma unroll
                        for (int j = 0; j < PNB; ++j) r[q][j] = Kr[j];
                    }
                }
            }
        }
        // multipliers, then column kk+1 only
        double m[R], cn[R];
        bool below[R];
        const double u1 = kk + 1 < PNB ? U[kk + 1] : 0.0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            below[q] = myrow[q] > kk;
            double ck = r[q][K0];
#pragma unroll
            for (int j = K0 + 1; j < KE && j < PNB; ++j)
                if (kk == j) ck = r[q][j];
            m[q] = below[q] ? __ddiv_rn(ck, ukk) : 0.0;
            double c1 = r[q][K0 + 1 < PNB ? K0 + 1 : PNB - 1];
#pragma unroll
            for (int j = K0 + 2; j <= KE && j < PNB; ++j)
                if (kk + 1 == j) c1 = r[q][j];
            if (below[q]) c1 = __dsub_rn(c1, __dmul_rn(m[q], u1));
            cn[q] = c1;
#pragma unroll
            for (int j = K0; j < KE && j < PNB; ++j)
                if (below[q] && j == kk) r[q][j] = m[q];
#pragma unroll
            for (int j = K0 + 1; j <= KE && j < PNB; ++j)
                if (below[q] && j == kk + 1) r[q][j] = c1;
        }
        if (L.dbg_on) sm.dclk[kk * 8 + 3] = clock64();
        if (kk + 1 < L.nb) {
            const int c = kk + 1;
            panel_push<R>(r, cn, myrow, c, sm, cl, L.cs, L.me, c >= L.rbeg && c < L.rend,
                          L.dbg_on ? &sm.dclk[kk * 8] : nullptr);
        }
        if (L.dbg_on) sm.dclk[kk * 8 + 6] = clock64();
        // the rest of the update while the pushes land
#pragma unroll
        for (int q = 0; q < R; ++q)
            if (below[q]) {
#pragma unroll
                for (int j = K0 + 2; j <= KE && j < PNB; ++j)
                    if (j > kk + 1) r[q][j] = __dsub_rn(r[q][j], __dmul_rn(m[q], U[j]));
#pragma unroll
                for (int j = KE + 1; j < PNB; ++j) r[q][j] = __dsub_rn(r[q][j], __dmul_rn(m[q], U[j]));
            }
        if (L.dbg_on) sm.dclk[kk * 8 + 7] = clock64();
    }
}

template <int R>
__global__ void __launch_bounds__(PT, 1) lu_panel_cluster(ClusterPanelArgs a) {
    __shared__ PanelSmem sm;
    cg::cluster_group cl = cg::this_cluster();
    const int cs = (int)cl.num_blocks(), me = (int)cl.block_rank();
    const int tid = threadIdx.x;
    const int nb = a.nb;
    const int rbeg = me * a.rp;  // rows counted from j0
    const int h = (int)(a.n - a.j0);
    int rend = rbeg + a.rp;
    if (rend > h) rend = h;
    const long long t_start = clock64();
    double r[R][PNB];
    int myrow[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
        myrow[q] = rbeg + tid + q * PT;
        const bool own = myrow[q] < rend;
#pragma unroll
        for (int j = 0; j < PNB; ++j)
            r[q][j] = (own && j < nb) ? a.A[(a.j0 + myrow[q]) + (a.j0 + j) * a.lda] : 0.0;
        if (!own) myrow[q] = -1;
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&sm.bar[0])), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&sm.bar[1])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();  // barriers initialised and every CTA running before the first push
    const long long t_loaded = clock64();
    PanelLoop L;
    L.cs = cs;
    L.me = me;
    L.rbeg = rbeg;
    L.rend = rend;
    L.nb = nb;
    // bytes arriving per column: cs candidates (row + key + row index) + row c
    L.col_bytes = (unsigned)cs * (PNB * 8 + 16) + PNB * 8;
    L.dbg_on = a.dbg && me == 0 && tid == 0;
    L.u_prev = 0.0;
    L.info_col = -1;
    {
        double c0[R];
#pragma unroll
        for (int q = 0; q < R; ++q) c0[q] = r[q][0];
        panel_push<R>(r, c0, myrow, 0, sm, cl, cs, me, 0 >= rbeg && 0 < rend);
    }
    static_assert(PNB == 8 * PKB, "eight column blocks");
    panel_cols<R, 0>(r, myrow, sm, cl, L);
    if (nb > PKB) panel_cols<R, PKB>(r, myrow, sm, cl, L);
    if (nb > 2 * PKB) panel_cols<R, 2 * PKB>(r, myrow, sm, cl, L);
    if (nb > 3 * PKB) panel_cols<R, 3 * PKB>(r, myrow, sm, cl, L);
    if (nb > 4 * PKB) panel_cols<R, 4 * PKB>(r, myrow, sm, cl, L);
    if (nb > 5 * PKB) panel_cols<R, 5 * PKB>(r, myrow, sm, cl, L);
    if (nb > 6 * PKB) panel_cols<R, 6 * PKB>(r, myrow, sm, cl, L);
    if (nb > 7 * PKB) panel_cols<R, 7 * PKB>(r, myrow, sm, cl, L);
    cl.sync();  // no CTA may exit while others may still write its shared memory
    const long long t_loop = clock64();
    if (me == 0 && tid == 0) {
        for (int k = 0; k < nb; ++k) a.piv[a.j0 + k] = a.j0 + sm.piv[k];
        if (L.info_col >= 0 && *a.info == 0) *a.info = (int32_t)(a.j0 + L.info_col + 1);
        if (L.dbg_on) {
            for (int k = 0; k < 8 * nb; ++k) a.dbg[k] = sm.dclk[k];
            a.dbg[8 * nb + 0] = t_start;
            a.dbg[8 * nb + 1] = t_loaded;
            a.dbg[8 * nb + 2] = t_loop;
        }
    }
    // write-back through shared memory (the whole PanelSmem is dead now),
    // 4 columns per pass, so each warp stores whole column segments with
    // 16-byte lanes instead of 8-byte per-thread row stores
    {
        constexpr int WC = 4, LDW = R * PT + 2;
        static_assert(sizeof(PanelSmem) >= sizeof(double) * WC * LDW, "write-back staging fits");
        double *wb = reinterpret_cast<double *>(&sm);
        const int nrows = rend - rbeg;
        const bool vec = ((a.j0 + rbeg) % 2 == 0) && (a.lda % 2 == 0) && (((uintptr_t)a.A & 15) == 0);
        __syncthreads();  // all shared-memory traffic of the column loop is over
#pragma unroll
        for (int c0 = 0; c0 < PNB; c0 += WC) {
            if (c0 >= nb) break;
#pragma unroll
            for (int q = 0; q < R; ++q)
#pragma unroll
                for (int j = 0; j < WC; ++j) wb[j * LDW + tid + q * PT] = r[q][c0 + j];
            __syncthreads();
            for (int j = 0; j < WC && c0 + j < nb; ++j) {
                double *col = a.A + (a.j0 + rbeg) + (int64_t)(a.j0 + c0 + j) * a.lda;
                if (vec) {
                    for (int i = 2 * tid; i + 1 < nrows; i += 2 * PT)
                        *reinterpret_cast<double2 *>(col + i) = make_double2(wb[j * LDW + i], wb[j * LDW + i + 1]);
                    if ((nrows & 1) && tid == 0) col[nrows - 1] = wb[j * LDW + nrows - 1];
                } else {
                    for (int i = tid; i < nrows; i += PT) col[i] = wb[j * LDW + i];
                }
            }
            __syncthreads();
        }
    }
    if (a.J1 > a.J0 && me == 0) panel_epilogue<R>(r, a, nullptr);
    if (a.dbg && me == 0 && tid == 0) a.dbg[8 * nb + 3] = clock64();
}

static int max_cluster() {
    static PerDevice<int> cache;
    int mc = 8;
    cache.get(mc, [](int &mc) {
        mc = 8;
        if (cudaFuncSetAttribute(lu_panel_cluster<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess &&
            cudaFuncSetAttribute(lu_panel_cluster<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
            mc = 16;
        return 0;
    });
    return mc;
}

// smallest cluster whose CTAs hold <= R*PT rows each (R = 1 preferred)
bool panel_shape(int64_t h, int &cs, int &rp, int &R) {
    const int mc = max_cluster();
    for (R = 1; R <= 2; ++R)
        for (cs = 1; cs <= mc; cs *= 2) {
            rp = (int)ceil_div(h, cs);
            if (rp <= R * PT) return true;
        }
    return false;
}

int launch_panel_cluster(double *A, int64_t lda, int64_t n, int64_t j0, int nb, int64_t *piv, int32_t *info,
                         cudaStream_t s, long long *dbg, int64_t J0, int64_t J1) {
    int cs = 0, rp = 0, R = 0;
    LM_REQUIRE(panel_shape(n - j0, cs, rp, R), "lu: panel too tall for one cluster");
    LM_REQUIRE(J1 <= J0 || rp >= nb, "lu: fused panel epilogue needs the panel's top rows in CTA 0");
    ClusterPanelArgs args{A, lda, n, j0, nb, rp, piv, info, dbg, J0, J1};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(PT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (R == 1)
        LM_CUDA(cudaLaunchKernelEx(&cfg, lu_panel_cluster<1>, args));
    else
        LM_CUDA(cudaLaunchKernelEx(&cfg, lu_panel_cluster<2>, args));
    count_launch(1);
    return 0;
}

}  // namespace lm

// Diagnostics: factor ONE panel (rows j0.., columns j0..j0+nb) of the F-order
// n x n matrix with the cluster kernel, recording clock64() per column and
// phase (CTA 0, thread 0) into d_clock[8*nb].
extern "C" int lm_debug_lu_panel(lm_view a, int64_t j0, int nb, int64_t *d_piv, int32_t *d_info, long long *d_clock,
                                 void *stream) {
    lm::clear_error();
    LM_REQUIRE(a.rows == a.cols && a.rs == 1 && nb >= 1 && nb <= lm::PNB, "debug panel: bad arguments");
    return lm::launch_panel_cluster((double *)a.ptr, a.cs, a.rows, j0, nb, d_piv, d_info, lm::as_stream(stream),
                                    d_clock, 0, 0);
}
