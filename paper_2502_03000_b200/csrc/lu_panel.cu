// lu_panel.cu -- the latency-critical piece of the exact LU (config 4a):
// factor a 32-column panel A[j0:n, j0:j0+32] in the reference's order
// (lazymat/_loops.py:200-236: first maximum of |A[i,k]|, full-row swap,
// multipliers by __ddiv_rn, rank-1 update with __dmul_rn/__dsub_rn).
//
// One thread-block CLUSTER (up to 16 CTAs of a GPC); thread t of CTA c owns
// panel row c*rp + t in 32 registers for the whole panel.  Per column:
//   1. each warp finds its candidate with three redux.sync instructions
//      (max of the high word of |v|, max of the low word, min row) --
//      the exact "first maximum" order, no shuffles;
//   2. one __syncthreads; warp 0 forms the CTA candidate and PUSHES it
//      (value, row, the 32 row values) into the inbox of every CTA of the
//      cluster with remote DSMEM stores; the owner of row k pushes row k;
//   3. one cluster barrier (release/acquire) -- after it every CTA holds
//      all candidates locally: no remote round trip is on the critical
//      path (measured on the B200: barrier 0.25 us; a DSMEM round 0.2 us);
//   4. every warp reduces the cs candidates from local shared memory,
//      swaps (register copies), computes the multiplier and updates its
//      row from the winner's row in shared memory (broadcast reads).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {

constexpr int PNB = 32;      // panel width
constexpr int PT = 256;      // threads per CTA (8 warps: per-warp overheads are issue-bound)
constexpr int PW = PT / 32;  // warps per CTA
constexpr int MAXCS = 16;    // largest cluster
constexpr int SLOT = 2 + PNB;

struct ClusterPanelArgs {
    double *A;
    int64_t lda, n, j0;
    int nb, rp;  // panel width, rows per CTA
    int64_t *piv;
    int32_t *info;
    long long *dbg;  // optional per-column phase timestamps (CTA 0, thread 0)
};

struct PanelSmem {
    double inbox[2][MAXCS][SLOT];  // every CTA's candidate (parity double-buffered)
    double inboxk[2][PNB];         // row k, pushed by its owner
    double cand[PW][PNB];          // each warp's candidate row
    double rowk[PNB];              // row k, staged for the push
    unsigned whi[PW], wlo[PW];     // warp candidates: |v| bits (+1 on hi), row
    int wrow[PW];
    int s_p, s_src;                // the column's pivot row and its inbox slot
    double sU[PNB];                // the pivot row (fetched from its CTA)
    double rowk_in[PNB];           // old row k, for the CTA owning row p
};

// (value, row) "first maximum" over the lanes of a warp.  v >= 0 (|A| or
// +inf), valid = row participates.  Returns the winning row or -1, and its
// value bits in (hi, lo) with hi = high word + 1 (0 = none).
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

template <int R>
__global__ void __launch_bounds__(PT, 1) lu_panel_cluster(ClusterPanelArgs a) {
    __shared__ PanelSmem sm;
    cg::cluster_group cl = cg::this_cluster();
    const int cs = (int)cl.num_blocks(), me = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nb = a.nb;
    const int rbeg = me * a.rp;  // rows counted from j0
    const int h = (int)(a.n - a.j0);
    int rend = rbeg + a.rp;
    if (rend > h) rend = h;
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
    const bool dbg_on = a.dbg && me == 0 && tid == 0;

#pragma unroll
    for (int kk = 0; kk < PNB; ++kk) {
        if (kk >= nb) break;
        const int par = kk & 1;
        if (dbg_on) a.dbg[kk * 4 + 0] = clock64();
        // 1. this thread's best row, then the warp's
        double bv = 0.0;
        int bq = -1, brw = 0;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            if (myrow[q] < kk) continue;  // rows above k and unused rows (-1)
            double v = fabs(r[q][kk]);
            if (v != v) {
                if (myrow[q] != kk) continue;  // NaN never wins off the diagonal
                v = __longlong_as_double(0x7ff0000000000000LL);
            }
            if (bq < 0 || v > bv) {  // R <= 2 and rows ascend with q: strict >
                bv = v;
                bq = q;
                brw = myrow[q];
            }
        }
        unsigned whi, wlo;
        const int wrow = warp_first_max(bv, bq >= 0, brw, whi, wlo);
#pragma unroll
        for (int q = 0; q < R; ++q)  // static register indices only (no local memory)
            if (q == bq && myrow[q] == wrow) {
#pragma unroll
                for (int j = 0; j < PNB; ++j) sm.cand[wid][j] = r[q][j];
            }
#pragma unroll
        for (int q = 0; q < R; ++q)
            if (myrow[q] == kk) {
#pragma unroll
                for (int j = 0; j < PNB; ++j) sm.rowk[j] = r[q][j];
            }
        if (lane == 0) {
            sm.whi[wid] = whi;
            sm.wlo[wid] = wlo;
            sm.wrow[wid] = wrow;
        }
        __syncthreads();
        if (dbg_on) a.dbg[kk * 4 + 1] = clock64();
        // 2. CTA candidate -> every CTA's inbox; row k -> every inbox
        if (wid == 0) {
            const bool ok = lane < PW && sm.whi[lane] != 0;
            const unsigned h0 = ok ? sm.whi[lane] : 0u;
            const unsigned hi = __reduce_max_sync(0xffffffffu, h0);
            const unsigned l0 = (ok && h0 == hi) ? sm.wlo[lane] : 0u;
            const unsigned lo = __reduce_max_sync(0xffffffffu, l0);
            const unsigned r0 = (ok && h0 == hi && sm.wlo[lane] == lo) ? (unsigned)sm.wrow[lane] : 0xffffffffu;
            const unsigned row = __reduce_min_sync(0xffffffffu, r0);
            // the warp that owns the winning row
            const unsigned wmask = __ballot_sync(0xffffffffu, ok && (unsigned)sm.wrow[lane] == row);
            const int w = wmask ? __ffs(wmask) - 1 : 0;
            // the candidate's |value| itself (bits reassembled), -1 for none
            const double hv =
                hi == 0 ? -1.0 : __longlong_as_double((long long)(((unsigned long long)(hi - 1u) << 32) | lo));
            const double rowv = hi == 0 ? -1.0 : (double)row;
            // the row stays local (fetched by everyone after the barrier);
            // only (value, row) is pushed to every CTA -- 2 remote stores per lane
            sm.inbox[par][me][2 + lane] = sm.cand[w][lane];
            if (lane < cs) {
                double *dst = cl.map_shared_rank(&sm.inbox[par][me][0], lane);
                dst[0] = hv;
                dst[1] = rowv;
            }
        } else if (wid == 1 && kk >= rbeg && kk < rend) {
            sm.inboxk[par][lane] = sm.rowk[lane];
        }
        cl.sync();
        if (dbg_on) a.dbg[kk * 4 + 2] = clock64();
        // 3. the global winner from the local inbox (warp 0), broadcast in smem
        if (wid == 0) {
            double key = -1.0, rowd = -1.0;
            if (lane < cs) {
                key = sm.inbox[par][lane][0];
                rowd = sm.inbox[par][lane][1];
            }
            // larger |value| wins, then the lower row (the reference's strict-> scan)
            const bool ok = rowd >= 0.0;
            const unsigned long long kb = (unsigned long long)__double_as_longlong(key);
            const unsigned h0 = ok ? (unsigned)(kb >> 32) + 1u : 0u;
            const unsigned hi = __reduce_max_sync(0xffffffffu, h0);
            const unsigned l0 = (ok && h0 == hi) ? (unsigned)kb : 0u;
            const unsigned lo = __reduce_max_sync(0xffffffffu, l0);
            const unsigned r0 = (ok && h0 == hi && (unsigned)kb == lo) ? (unsigned)rowd : 0xffffffffu;
            const unsigned row = __reduce_min_sync(0xffffffffu, r0);
            const unsigned srcm = __ballot_sync(0xffffffffu, ok && (unsigned)rowd == row);
            const int src = __ffs(srcm) - 1;
            // one remote round trip: the pivot row (and old row k if we own p)
            sm.sU[lane] = cl.map_shared_rank(&sm.inbox[par][src][2], src)[lane];
            if ((int)row != kk && (int)row >= rbeg && (int)row < rend)
                sm.rowk_in[lane] = cl.map_shared_rank(&sm.inboxk[par][0], kk / a.rp)[lane];
            if (lane == 0) sm.s_p = (int)row;
        }
        __syncthreads();
        const int p = sm.s_p;
        const double *U = sm.sU;
        if (me == 0 && tid == 0) {
            a.piv[a.j0 + kk] = a.j0 + p;
            if (U[kk] == 0.0 && *a.info == 0) *a.info = (int32_t)(a.j0 + kk + 1);
        }
        if (dbg_on) a.dbg[kk * 4 + 3] = clock64();
        // 4. swap rows k and p (register copies), multipliers, rank-1 update
#pragma unroll
        for (int q = 0; q < R; ++q) {
            if (myrow[q] < 0) continue;
            if (p != kk) {
                if (myrow[q] == kk) {
#pragma unroll
                    for (int j = 0; j < PNB; ++j) r[q][j] = U[j];
                } else if (myrow[q] == p) {
#pragma unroll
                    for (int j = 0; j < PNB; ++j) r[q][j] = sm.rowk_in[j];
                }
            }
            if (myrow[q] > kk) {
                const double m = __ddiv_rn(r[q][kk], U[kk]);
                r[q][kk] = m;
#pragma unroll
                for (int j = kk + 1; j < PNB; ++j) r[q][j] = __dsub_rn(r[q][j], __dmul_rn(m, U[j]));
            }
        }
    }
    cl.sync();  // no CTA may exit while others may still write its inbox
#pragma unroll
    for (int q = 0; q < R; ++q)
        if (myrow[q] >= 0)
#pragma unroll
            for (int j = 0; j < PNB; ++j)
                if (j < nb) a.A[(a.j0 + myrow[q]) + (a.j0 + j) * a.lda] = r[q][j];
}

static int max_cluster() {
    static int mc = -1;
    if (mc < 0) {
        mc = 8;
        if (cudaFuncSetAttribute(lu_panel_cluster<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess &&
            cudaFuncSetAttribute(lu_panel_cluster<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
            mc = 16;
    }
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
                         cudaStream_t s, long long *dbg) {
    int cs = 0, rp = 0, R = 0;
    LM_REQUIRE(panel_shape(n - j0, cs, rp, R), "lu: panel too tall for one cluster");
    ClusterPanelArgs args{A, lda, n, j0, nb, rp, piv, info, dbg};
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
// phase (CTA 0, thread 0) into d_clock[4*nb].
extern "C" int lm_debug_lu_panel(lm_view a, int64_t j0, int nb, int64_t *d_piv, int32_t *d_info, long long *d_clock,
                                 void *stream) {
    lm::clear_error();
    LM_REQUIRE(a.rows == a.cols && a.rs == 1 && nb >= 1 && nb <= lm::PNB, "debug panel: bad arguments");
    return lm::launch_panel_cluster((double *)a.ptr, a.cs, a.rows, j0, nb, d_piv, d_info, lm::as_stream(stream),
                                    d_clock);
}
