// datagen.cu -- seeded synthetic operands generated on the device, drawn
// from exactly the stream numpy's np.random.default_rng(seed).uniform(lo, hi)
// produces (every BASELINE operand is a seeded numpy
// uniform fill, C-order draws stored column-major).
//
// numpy's default_rng is PCG64 (128-bit LCG, multiplier
// 0x2360ED051FC65DA44385DF649FCCF645, increment from the SeedSequence;
// XSL-RR 128->64 output applied to the state AFTER each step) and
// uniform(lo, hi) = lo + (hi - lo) * next_double, next_double =
// (next_uint64 >> 11) * 2^-53.  The host passes the generator's state
// right after seeding (bit_generator.state), so any seed scheme the
// caller likes (SeedSequence entropy lists included) maps to one call.
//
// Draw p of the stream (0-based) is out(state after p + 1 steps).  A thread
// jumps straight to its first draw with a table of the affine step map's
// powers (S -> A_k S + C_k = 2^k steps, computed once per call on the host)
// and then steps sequentially along one row of its matrix; the 32 lanes of
// a warp own 32 consecutive ROWS, so every store instruction of the warp
// writes 32 consecutive elements of one column-major column (coalesced).
// A 64 GB batch fills in tens of milliseconds instead of the minutes a host
// generator plus PCIe would take, and a host check of any element needs
// only bit_generator.advance(p).
#include "common.cuh"

namespace lm {
namespace {

struct U128 {
    uint64_t lo, hi;
};

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
#ifdef __CUDA_ARCH__
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
    r.hi = (uint64_t)(((unsigned __int128)a.lo * b.lo) >> 64) + a.lo * b.hi + a.hi * b.lo;
#endif
    return r;
}

__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
    return r;
}

constexpr U128 kMul = {0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull};

struct Pcg64Args {
    void *out;
    int64_t batch, rows, cols, ld, bstride;  // output layout (elements)
    int64_t bstream, rstream;                // stream positions per instance / per row
    uint64_t skip;                           // stream position of element (0, 0, 0)
    double lo, range;
    U128 state0, inc;
    int run;                                 // columns per thread
    int64_t rgroups, runs;                   // 32-row groups per instance, column runs per row
    U128 jumpA[64], jumpC[64];               // 2^k steps: S -> A_k S + C_k
};

__device__ __forceinline__ double pcg_double(U128 s) {
    const uint64_t x = s.hi ^ s.lo;
    const unsigned r = (unsigned)(s.hi >> 58);
    const uint64_t v = (x >> r) | (x << ((64u - r) & 63u));
    return (double)(v >> 11) * (1.0 / 9007199254740992.0);
}

template <class T>
__global__ void __launch_bounds__(256) fill_pcg64(const __grid_constant__ Pcg64Args a) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = (int)(t & 31);
    int64_t w = t >> 5;
    const int64_t jr = w % a.runs;
    w /= a.runs;
    const int64_t rg = w % a.rgroups;
    const int64_t b = w / a.rgroups;
    if (b >= a.batch) return;
    const int64_t i = rg * 32 + lane;
    if (i >= a.rows) return;
    const int64_t j0 = jr * a.run;
    const int64_t jn = (a.cols - j0) < a.run ? (a.cols - j0) : a.run;
    uint64_t p = a.skip + (uint64_t)(b * a.bstream + i * a.rstream + j0);
    U128 s = a.state0;
    for (int k = 0; p; ++k, p >>= 1)
        if (p & 1) s = add128(mul128(a.jumpA[k], s), a.jumpC[k]);
    T *out = reinterpret_cast<T *>(a.out) + b * a.bstride + i + j0 * a.ld;
    for (int64_t r = 0; r < jn; ++r) {
        s = add128(mul128(kMul, s), a.inc);
        const double v = __dadd_rn(a.lo, __dmul_rn(a.range, pcg_double(s)));
        out[r * a.ld] = (T)v;  // f32: round-to-nearest, as numpy's astype(float32)
    }
}

}  // namespace
}  // namespace lm

using namespace lm;

extern "C" int lm_fill_pcg64(int dtype, void *out, int64_t batch, int64_t rows, int64_t cols, int64_t ld,
                             int64_t bstride, int64_t bstream, int64_t rstream, uint64_t skip, uint64_t state_hi,
                             uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, double lo, double hi,
                             void *stream) {
    clear_error();
    LM_REQUIRE(dtype == LM_F64 || dtype == LM_F32, "fill_pcg64: bad dtype");
    LM_REQUIRE(batch >= 0 && rows >= 0 && cols >= 0, "fill_pcg64: negative extent");
    LM_REQUIRE(ld >= rows || cols <= 1, "fill_pcg64: ld < rows");
    if (batch == 0 || rows == 0 || cols == 0) return 0;
    LM_REQUIRE(out != nullptr, "fill_pcg64: null output");
    Pcg64Args a{};
    a.out = out;
    a.batch = batch;
    a.rows = rows;
    a.cols = cols;
    a.ld = ld;
    a.bstride = bstride;
    a.bstream = bstream;
    a.rstream = rstream;
    a.skip = skip;
    a.lo = lo;
    a.range = hi - lo;
    a.state0 = U128{state_lo, state_hi};
    a.inc = U128{inc_lo, inc_hi};
    a.run = (int)(cols < 256 ? cols : 256);
    a.rgroups = ceil_div(rows, 32);
    a.runs = ceil_div(cols, a.run);
    U128 A = kMul, C = a.inc;
    for (int k = 0; k < 64; ++k) {  // (A, C) applied twice: A^2 S + (A + 1) C
        a.jumpA[k] = A;
        a.jumpC[k] = C;
        C = mul128(C, add128(A, U128{1, 0}));
        A = mul128(A, A);
    }
    const int64_t threads = batch * a.rgroups * a.runs * 32;
    const int64_t blocks = ceil_div(threads, 256);
    LM_REQUIRE(blocks < (1ll << 31), "fill_pcg64: too many elements for one launch");
    cudaStream_t st = as_stream(stream);
    if (dtype == LM_F64)
        fill_pcg64<double><<<(unsigned)blocks, 256, 0, st>>>(a);
    else
        fill_pcg64<float><<<(unsigned)blocks, 256, 0, st>>>(a);
    LM_LAUNCHED(1);
    return 0;
}
