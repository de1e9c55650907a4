// lu_fast.cu -- LU factorisation of large matrices (BASELINE config 4a)
// in the reference's exact operation order, two-level blocked.
//
// Reference: lazymat/_loops.py:200-236 (_lu_factor).  Every element
// A[i,j] receives A[i,j] = A[i,j] - L[i,k]*U[k,j] for k ascending, each
// product and difference rounded (__dmul_rn/__dsub_rn), multipliers
// L[i,k] = A[i,k] / pivot (__ddiv_rn), the pivot is the first maximum of
// |A[i,k]| over the current rows i >= k, full-row swaps.  Any blocking that
// keeps, per element, the update order k ascending performs exactly these
// operations, so values and pivots are bit-identical to the reference.
//
//   outer blocks of NB = 128 columns (trailing-update K = 128: the A22
//   read/write traffic is n^3/(3*128) * 16 B, 23 GB at n = 8192);
//   inside a block, panels of 32 columns factored by ONE thread-block
//   CLUSTER (16 CTAs, one per SM of a GPC): the panel rows live in the
//   cluster's shared memory, each column costs one cluster barrier -- the
//   candidates and the candidate rows are published in shared-memory
//   mailboxes before it and read over DSMEM after it;
//   row swaps of the other columns: one composed permutation per panel
//   (laswp_plan) applied as a gather (laswp_apply);
//   U12: 32-row triangular solves (one thread per column, the column in
//   registers, the triangle in shared memory) + order-preserving updates;
//   A22: order-preserving SIMT update, 128 x 128 tiles, 8 x 8 per thread.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace lm {

// ============================================================================
// order-preserving update  C -= A @ B  (k ascending, or descending if DESC)
// ============================================================================

constexpr int UT = 128, UK = 32, ULD = UT + 1;

template <bool DESC, bool SKIP_ZERO>
__global__ void __launch_bounds__(256) exact_update128(const double *__restrict__ A, int64_t lda,
                                                       const double *__restrict__ B, int64_t ldb, double *C,
                                                       int64_t ldc, int64_t M, int64_t N, int K) {
    extern __shared__ double su[];
    double *sA = su;             // [UK][ULD]: sA[kk][ii] = A[i0+ii, k]
    double *sB = su + UK * ULD;  // [UK][ULD]: sB[kk][cc] = B[k, c0+cc]
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = (int64_t)blockIdx.x * UT, c0 = (int64_t)blockIdx.y * UT;
    double acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int64_t i = i0 + tx + 16 * r, c = c0 + ty + 16 * s;
            acc[r][s] = (i < M && c < N) ? C[i + c * ldc] : 0.0;
        }
    const int nch = (K + UK - 1) / UK;
    for (int q = 0; q < nch; ++q) {
        const int ch = DESC ? (nch - 1 - q) : q;
        const int k0 = ch * UK;
        for (int e = threadIdx.x; e < UK * UT; e += 256) {
            const int ii = e % UT, kk = e / UT;
            const int64_t i = i0 + ii;
            const int k = k0 + kk;
            sA[kk * ULD + ii] = (i < M && k < K) ? A[i + (int64_t)k * lda] : 0.0;
        }
        for (int e = threadIdx.x; e < UK * UT; e += 256) {
            const int kk = e % UK, cc = e / UK;
            const int64_t c = c0 + cc;
            const int k = k0 + kk;
            sB[kk * ULD + cc] = (c < N && k < K) ? B[k + c * ldb] : 0.0;
        }
        __syncthreads();
        const int kend = (K - k0) < UK ? (K - k0) : UK;
        for (int t = 0; t < kend; ++t) {
            const int kk = DESC ? (kend - 1 - t) : t;
            double a[8], b[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) a[r] = sA[kk * ULD + tx + 16 * r];
#pragma unroll
            for (int s = 0; s < 8; ++s) b[s] = sB[kk * ULD + ty + 16 * s];
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int s = 0; s < 8; ++s)
                    if (!SKIP_ZERO || b[s] != 0.0) acc[r][s] = __dsub_rn(acc[r][s], __dmul_rn(a[r], b[s]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int64_t i = i0 + tx + 16 * r, c = c0 + ty + 16 * s;
            if (i < M && c < N) C[i + c * ldc] = acc[r][s];
        }
}

template <bool DESC, bool SKIP_ZERO>
int exact_update(const double *A, int64_t lda, const double *B, int64_t ldb, double *C, int64_t ldc, int64_t M,
                 int64_t N, int K, cudaStream_t s) {
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    const size_t smem = sizeof(double) * 2 * UK * ULD;
    static bool attr = false;
    if (!attr) {
        LM_CUDA(cudaFuncSetAttribute(exact_update128<DESC, SKIP_ZERO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        attr = true;
    }
    dim3 grid((unsigned)ceil_div(M, UT), (unsigned)ceil_div(N, UT));
    exact_update128<DESC, SKIP_ZERO><<<grid, 256, smem, s>>>(A, lda, B, ldb, C, ldc, M, N, K);
    LM_LAUNCHED(1);
    return 0;
}

// explicit instantiations used by lu.cu (solves)
template int exact_update<false, false>(const double *, int64_t, const double *, int64_t, double *, int64_t,
                                        int64_t, int64_t, int, cudaStream_t);
template int exact_update<true, false>(const double *, int64_t, const double *, int64_t, double *, int64_t,
                                       int64_t, int64_t, int, cudaStream_t);

// ============================================================================
// triangular solve on up to 32 rows, one thread per column of X
// ============================================================================

template <bool LOWER>
__global__ void __launch_bounds__(128) tri_cols(const double *__restrict__ T, int64_t ldt, double *X, int64_t ldx,
                                                int nb, int64_t ncols) {
    __shared__ double sT[32][33];  // sT[i][j] = T[i,j]
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
        const int i = e % nb, j = e / nb;
        sT[i][j] = T[i + (int64_t)j * ldt];
    }
    __syncthreads();
    const int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= ncols) return;
    double *xc = X + col * ldx;
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = i < nb ? xc[i] : 0.0;
    if (LOWER) {  // unit lower, forward: x_i -= T[i,j] x_j, j ascending
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j >= nb) break;
            const double xj = x[j];
#pragma unroll
            for (int i = j + 1; i < 32; ++i)
                if (i < nb) x[i] = __dsub_rn(x[i], __dmul_rn(sT[i][j], xj));
        }
    } else {  // upper, backward: x_j /= T[j,j]; x_i -= T[i,j] x_j, j descending
#pragma unroll
        for (int j = 31; j >= 0; --j) {
            if (j >= nb) continue;
            x[j] = __ddiv_rn(x[j], sT[j][j]);
            const double xj = x[j];
#pragma unroll
            for (int i = 0; i < j; ++i) x[i] = __dsub_rn(x[i], __dmul_rn(sT[i][j], xj));
        }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i)
        if (i < nb) xc[i] = x[i];
}

template <bool LOWER>
int tri32(const double *T, int64_t ldt, double *X, int64_t ldx, int nb, int64_t ncols, cudaStream_t s) {
    if (nb <= 0 || ncols <= 0) return 0;
    tri_cols<LOWER><<<(unsigned)ceil_div(ncols, 128), 128, 0, s>>>(T, ldt, X, ldx, nb, ncols);
    LM_LAUNCHED(1);
    return 0;
}
template int tri32<true>(const double *, int64_t, double *, int64_t, int, int64_t, cudaStream_t);
template int tri32<false>(const double *, int64_t, double *, int64_t, int, int64_t, cudaStream_t);

// ============================================================================
// row swaps of whole column ranges: compose, then gather
// ============================================================================

// list[0] = count, then (dst, src) pairs: final row dst takes old row src,
// for the sequential swaps piv[k0 .. k0+cnt) over rows [k0, n).
__global__ void __launch_bounds__(1024) laswp_plan(const int64_t *__restrict__ piv, int64_t k0, int cnt, int64_t n,
                                                   int32_t *list) {
    extern __shared__ int32_t content[];  // content[r - k0] = original row now at r
    __shared__ int count;
    const int64_t h = n - k0;
    for (int64_t r = threadIdx.x; r < h; r += blockDim.x) content[r] = (int32_t)(k0 + r);
    if (threadIdx.x == 0) count = 0;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int q = 0; q < cnt; ++q) {
            const int64_t k = k0 + q, p = piv[k];
            if (p != k) {
                const int32_t t = content[k - k0];
                content[k - k0] = content[p - k0];
                content[p - k0] = t;
            }
        }
    __syncthreads();
    for (int64_t r = threadIdx.x; r < h; r += blockDim.x)
        if (content[r] != (int32_t)(k0 + r)) {
            const int slot = atomicAdd(&count, 1);
            list[1 + 2 * slot] = (int32_t)(k0 + r);
            list[2 + 2 * slot] = content[r];
        }
    __syncthreads();
    if (threadIdx.x == 0) list[0] = count;
}

// one CTA per column; columns [a0, a1) then [b0, b1)
__global__ void __launch_bounds__(256) laswp_apply(double *A, int64_t lda, const int32_t *__restrict__ list, int64_t a0,
                                                   int64_t a1, int64_t b0) {
    __shared__ double v[512];
    const int64_t na = a1 - a0;
    const int64_t col = blockIdx.x < na ? a0 + blockIdx.x : b0 + (blockIdx.x - na);
    double *x = A + col * lda;
    const int cnt = list[0];
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) v[q] = x[list[2 + 2 * q]];
    __syncthreads();
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) x[list[1 + 2 * q]] = v[q];
}

// ============================================================================
// the panel: one cluster of CS CTAs holds rows [j0, n) x columns [j0, j0+nb)
// ============================================================================

constexpr int PNB = 32;      // panel width
constexpr int PT = 512;      // threads per CTA
constexpr int MB = 2 + PNB;  // mailbox slot: value, row, row values

struct ClusterPanelArgs {
    double *A;
    int64_t lda, n, j0;
    int nb, rp;  // panel width, rows per CTA
    int64_t *piv;
    int32_t *info;
};

__device__ __forceinline__ bool pbetter(double va, int64_t ia, double vb, int64_t ib) {
    if (ia < 0) return false;
    if (ib < 0) return true;
    return va > vb || (va == vb && ia < ib);
}

__global__ void __launch_bounds__(PT) lu_panel_cluster(ClusterPanelArgs a) {
    extern __shared__ double smp[];
    cg::cluster_group cl = cg::this_cluster();
    const int cs = (int)cl.num_blocks(), me = (int)cl.block_rank();
    const int ld = PNB + 1;
    double *sP = smp;                     // [rp][PNB+1]
    double *box = sP + (int64_t)a.rp * ld;  // [2][MB] candidate mailboxes
    double *boxk = box + 2 * MB;          // [2][PNB] row-k mailboxes
    double *sU = boxk + 2 * PNB;          // [PNB] pivot row
    __shared__ double wv[PT / 32];
    __shared__ int64_t wi[PT / 32];
    __shared__ int64_t s_p;
    __shared__ int s_w;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nb = a.nb;
    const int64_t rbeg = a.j0 + (int64_t)me * a.rp;
    int64_t rend = rbeg + a.rp;
    if (rend > a.n) rend = a.n;
    const int nrow = rend > rbeg ? (int)(rend - rbeg) : 0;

    for (int e = tid; e < nrow * nb; e += PT) {
        const int r = e % nrow, j = e / nrow;
        sP[r * ld + j] = a.A[(rbeg + r) + (a.j0 + j) * a.lda];
    }
    __syncthreads();

    for (int kk = 0; kk < nb; ++kk) {
        const int64_t k = a.j0 + kk;
        const int par = kk & 1;
        // 1. local candidate (first maximum of |A[i,k]| over owned rows i >= k)
        double bv = -1.0;
        int64_t bi = -1;
        for (int r = tid; r < nrow; r += PT) {
            const int64_t row = rbeg + r;
            if (row < k) continue;
            double v = fabs(sP[r * ld + kk]);
            if (v != v) {
                if (row != k) continue;
                v = __longlong_as_double(0x7ff0000000000000LL);
            }
            if (pbetter(v, row, bv, bi)) {
                bv = v;
                bi = row;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (pbetter(ov, oi, bv, bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            wv[wid] = bv;
            wi[wid] = bi;
        }
        __syncthreads();  // also: every row update of the previous column is done
        if (wid == 0) {
            double v = lane < PT / 32 ? wv[lane] : -1.0;
            int64_t i = lane < PT / 32 ? wi[lane] : -1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
                if (pbetter(ov, oi, v, i)) {
                    v = ov;
                    i = oi;
                }
            }
            // 2. publish: candidate value/row and the candidate's row values
            double *mb = box + par * MB;
            if (lane == 0) {
                mb[0] = v;
                mb[1] = (double)i;
            }
            if (i >= 0 && lane < nb) mb[2 + lane] = sP[(i - rbeg) * ld + lane];
        } else if (wid == 1 && k >= rbeg && k < rend && lane < nb) {
            boxk[par * PNB + lane] = sP[(k - rbeg) * ld + lane];
        }
        cl.sync();  // release the mailboxes / acquire everyone else's
        // 3. global winner (identical in every CTA)
        if (wid == 0) {
            double v = -1.0;
            int64_t i = -1;
            int w = -1;
            if (lane < cs) {
                const double *rb = cl.map_shared_rank(box + par * MB, lane);
                v = rb[0];
                i = (int64_t)rb[1];
                w = lane;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, o);
                const int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
                const int ow = __shfl_xor_sync(0xffffffffu, w, o);
                if (pbetter(ov, oi, v, i)) {
                    v = ov;
                    i = oi;
                    w = ow;
                }
            }
            if (lane < nb) sU[lane] = cl.map_shared_rank(box + par * MB, w)[2 + lane];
            if (lane == 0) {
                s_p = i;
                s_w = w;
            }
        }
        __syncthreads();
        const int64_t p = s_p;
        if (me == 0 && tid == 0) {
            a.piv[k] = p;
            if (sU[kk] == 0.0 && *a.info == 0) *a.info = (int32_t)(k + 1);
        }
        // 4. swap rows k and p inside the panel slice
        if (p != k) {
            if (p >= rbeg && p < rend && tid < nb) {
                const int owner = (int)((k - a.j0) / a.rp);
                sP[(p - rbeg) * ld + tid] = cl.map_shared_rank(boxk + par * PNB, owner)[tid];
            }
            if (k >= rbeg && k < rend && tid < nb) sP[(k - rbeg) * ld + tid] = sU[tid];
        }
        __syncthreads();
        // 5. multipliers and the rank-1 update of the panel rows below k
        const double pv = sU[kk];
        for (int r = tid; r < nrow; r += PT) {
            if (rbeg + r <= k) continue;
            double *row = sP + r * ld;
            const double m = __ddiv_rn(row[kk], pv);
            row[kk] = m;
            for (int j = kk + 1; j < nb; ++j) row[j] = __dsub_rn(row[j], __dmul_rn(m, sU[j]));
        }
    }
    cl.sync();  // nobody may exit while its mailboxes can still be read
    for (int e = tid; e < nrow * nb; e += PT) {
        const int r = e % nrow, j = e / nrow;
        a.A[(rbeg + r) + (a.j0 + j) * a.lda] = sP[r * ld + j];
    }
}

// cluster size and rows per CTA for a panel of height h; 0 if it does not fit
static int panel_cluster_size(int64_t h, int &rp) {
    static int max_cs = -1;
    if (max_cs < 0) {
        max_cs = 8;
        if (cudaFuncSetAttribute(lu_panel_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess)
            max_cs = 16;
    }
    for (int cs = 1; cs <= max_cs; cs *= 2) {
        rp = (int)ceil_div(h, cs);
        if (rp <= 4 * PT / 2 && sizeof(double) * ((size_t)rp * (PNB + 1) + 2 * MB + 3 * PNB) <= 200 * 1024 &&
            (rp <= PT || cs == max_cs))
            return cs;
    }
    return 0;
}

static int launch_panel_cluster(double *A, int64_t lda, int64_t n, int64_t j0, int nb, int64_t *piv, int32_t *info,
                                cudaStream_t s, bool &ok) {
    const int64_t h = n - j0;
    int rp = 0;
    const int cs = panel_cluster_size(h, rp);
    ok = cs > 0;
    if (!ok) return 0;
    const size_t smem = sizeof(double) * ((size_t)rp * (PNB + 1) + 2 * MB + 3 * PNB);
    LM_CUDA(cudaFuncSetAttribute(lu_panel_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ClusterPanelArgs args{A, lda, n, j0, nb, rp, piv, info};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(PT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, lu_panel_cluster, args);
    if (e != cudaSuccess) {
        cudaGetLastError();
        ok = false;  // cluster not schedulable: caller falls back
        return 0;
    }
    count_launch(1);
    return 0;
}

// rows [k0, k0+cnt) pivots applied to columns [a0, a1) U [b0, b1)
static int laswp(double *A, int64_t lda, int64_t n, const int64_t *piv, int64_t k0, int cnt, int64_t a0, int64_t a1,
                 int64_t b0, int64_t b1, int32_t *list, cudaStream_t s) {
    const int64_t ncols = (a1 - a0) + (b1 - b0);
    if (ncols <= 0 || cnt <= 0) return 0;
    const size_t sm = sizeof(int32_t) * (size_t)(n - k0);
    LM_REQUIRE(sm <= 200 * 1024, "laswp: n too large");
    static size_t attr = 0;
    if (sm > 48 * 1024 && sm > attr) {
        LM_CUDA(cudaFuncSetAttribute(laswp_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = sm;
    }
    laswp_plan<<<1, 1024, sm, s>>>(piv, k0, cnt, n, list);
    LM_LAUNCHED(1);
    laswp_apply<<<(unsigned)ncols, 256, 0, s>>>(A, lda, list, a0, a1, b0);
    LM_LAUNCHED(1);
    return 0;
}

constexpr int ONB = 128;  // outer block

// Returns 1 (and does nothing) when the cluster panel is not usable for
// this n, so the caller can take the cooperative-grid path.
int lu_factor_fast(double *A, int64_t n, int64_t lda, int64_t *piv, int32_t *info, cudaStream_t s) {
    int rp = 0;
    if (panel_cluster_size(n, rp) == 0) return 1;
    Scratch list;
    if (int rc = list.alloc(sizeof(int32_t) * (1 + 4 * ONB + 8), s)) return rc;
    int32_t *lp = list.as<int32_t>();
    for (int64_t J0 = 0; J0 < n; J0 += ONB) {
        const int NBJ = (int)((n - J0) < ONB ? (n - J0) : ONB);
        const int64_t J1 = J0 + NBJ;
        for (int64_t j0 = J0; j0 < J1; j0 += PNB) {
            const int nb = (int)((J1 - j0) < PNB ? (J1 - j0) : PNB);
            bool ok = false;
            if (int rc = launch_panel_cluster(A, lda, n, j0, nb, piv, info, s, ok)) return rc;
            LM_REQUIRE(ok, "lu: thread-block cluster for the panel could not be launched");
            // this panel's swaps on the rest of the outer block
            if (int rc = laswp(A, lda, n, piv, j0, nb, J0, j0, j0 + nb, J1, lp, s)) return rc;
            const int64_t rest = J1 - (j0 + nb);
            if (rest > 0) {
                if (int rc = tri32<true>(A + j0 + j0 * lda, lda, A + j0 + (j0 + nb) * lda, lda, nb, rest, s)) return rc;
                if (int rc = exact_update<false, false>(A + (j0 + nb) + j0 * lda, lda, A + j0 + (j0 + nb) * lda, lda,
                                                        A + (j0 + nb) + (j0 + nb) * lda, lda, n - (j0 + nb), rest, nb,
                                                        s))
                    return rc;
            }
        }
        // the outer block's swaps on everything left and right of it
        if (int rc = laswp(A, lda, n, piv, J0, NBJ, 0, J0, J1, n, lp, s)) return rc;
        if (J1 < n) {
            for (int64_t b0 = J0; b0 < J1; b0 += PNB) {
                const int nbb = (int)((J1 - b0) < PNB ? (J1 - b0) : PNB);
                if (int rc = tri32<true>(A + b0 + b0 * lda, lda, A + b0 + J1 * lda, lda, nbb, n - J1, s)) return rc;
                if (b0 + nbb < J1)
                    if (int rc = exact_update<false, false>(A + (b0 + nbb) + b0 * lda, lda, A + b0 + J1 * lda, lda,
                                                            A + (b0 + nbb) + J1 * lda, lda, J1 - (b0 + nbb), n - J1,
                                                            nbb, s))
                        return rc;
            }
            if (int rc = exact_update<false, false>(A + J1 + J0 * lda, lda, A + J0 + J1 * lda, lda, A + J1 + J1 * lda,
                                                    lda, n - J1, n - J1, NBJ, s))
                return rc;
        }
    }
    return 0;
}

}  // namespace lm
