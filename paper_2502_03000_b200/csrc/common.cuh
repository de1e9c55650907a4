// common.cuh -- shared device/host helpers for the sm_100a backend.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <mutex>

#include "lm_b200.h"

namespace lm {

// ---- status / error plumbing ------------------------------------------------

void set_error(const char *fmt, ...);
void clear_error();
bool has_error();
void count_launch(int n = 1);
// Records which kernel variant a multi-variant entry point launched last
// (lm_last_variant(): tests prove the intended specialisation ran).
void note_variant(const char *name);
int num_sms();
void ensure_pool();
int current_device();  // cudaGetDevice, or -1

constexpr int kMaxDevices = 64;

// Lazily initialised launch state (grid sizes, stream handles) kept per
// device: init(value) runs once per device, thread-safe (std::call_once);
// every caller gets the value and init's status.  A process that drives
// several GPUs therefore sizes and configures each one separately.
template <class T> class PerDevice {
  public:
    template <class F> int get(T &out, F &&init) {
        const int dev = current_device();
        if (dev < 0 || dev >= kMaxDevices) {
            set_error("no current CUDA device (or device index >= %d)", kMaxDevices);
            return -2;
        }
        std::call_once(once_[dev], [&] { rc_[dev] = init(val_[dev]); });
        if (rc_[dev] && !has_error()) set_error("launch setup failed earlier on device %d", dev);
        out = val_[dev];
        return rc_[dev];
    }

  private:
    std::once_flag once_[kMaxDevices];
    T val_[kMaxDevices] = {};
    int rc_[kMaxDevices] = {};
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize >= bytes [, carveout])
// once per (kernel, device); thread-safe.  Kernel attributes are
// per-device state, so a second GPU in the same process needs its own call.
int ensure_func_attrs(const void *kernel, int smem_bytes, int carveout = -1);
template <class K> inline int func_attrs(K kernel, size_t smem_bytes, int carveout = -1) {
    return ensure_func_attrs(reinterpret_cast<const void *>(kernel), (int)smem_bytes, carveout);
}

#define LM_REQUIRE(cond, ...)                                                                 \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            ::lm::set_error(__VA_ARGS__);                                                     \
            return -1;                                                                        \
        }                                                                                     \
    } while (0)

#define LM_CUDA(call)                                                                         \
    do {                                                                                      \
        cudaError_t _e = (call);                                                              \
        if (_e != cudaSuccess) {                                                              \
            ::lm::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
            return -2;                                                                        \
        }                                                                                     \
    } while (0)

// After a <<<>>> launch.
#define LM_LAUNCHED(n)                                                                        \
    do {                                                                                      \
        cudaError_t _e = cudaGetLastError();                                                  \
        if (_e != cudaSuccess) {                                                              \
            ::lm::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e));  \
            return -2;                                                                        \
        }                                                                                     \
        ::lm::count_launch(n);                                                                \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- programmatic dependent launch (PDL) ------------------------------------
// A kernel launched with launch_pdl() may start while the previous kernel in
// the stream is still draining; it MUST call pdl_wait() before reading
// anything that kernel wrote (griddepcontrol.wait returns once the
// prerequisite grid has completed and its memory is visible).  A primary
// kernel calls pdl_trigger() once its remaining work no longer needs the
// SMs to itself, letting the dependent grid's CTAs launch early.  Chains of
// short dependent kernels (GEMV + ordered finish, x3 in config 3a) lose
// their launch gaps this way.  LM_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    if (!pdl_enabled()) {
        kern<<<grid, block, smem, s>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Stream-ordered scratch (cudaMallocAsync); freed on the same stream.
struct Scratch {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    Scratch() = default;
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    int alloc(size_t bytes, cudaStream_t st) {
        s = st;
        ensure_pool();
        if (bytes == 0) bytes = 16;
        cudaError_t e = cudaMallocAsync(&p, bytes, st);
        if (e != cudaSuccess) {
            set_error("cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
            p = nullptr;
            return -2;
        }
        return 0;
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

// ---- device-side strided views -----------------------------------------------

template <class T> struct View {
    T *p;
    int64_t rows, cols, rs, cs;
    __host__ __device__ T &operator()(int64_t i, int64_t j) const { return p[i * rs + j * cs]; }
};

template <class T> struct Vec {
    T *p;
    int64_t n, stride;
    __host__ __device__ T &operator[](int64_t i) const { return p[i * stride]; }
};

template <class T> inline View<T> to_view(const lm_view &v) {
    return View<T>{reinterpret_cast<T *>(v.ptr), v.rows, v.cols, v.rs, v.cs};
}
template <class T> inline Vec<T> to_vec(const lm_vec &v) {
    return Vec<T>{reinterpret_cast<T *>(v.ptr), v.n, v.stride};
}

inline bool f_contig(const lm_view &v) { return v.rs == 1 && (v.cs == v.rows || v.cols == 1); }

// ---- exactly rounded scalar ops (no FMA contraction, whatever the flags) ----

__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float rmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float radd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float rsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float rdiv(float a, float b) { return __fdiv_rn(a, b); }

// ---- streaming loads / stores ---------------------------------------------------

__device__ __forceinline__ double2 ld_stream(const double2 *p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ float4 ld_stream(const float4 *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(double2 *p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_stream(float4 *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

// 32-byte vectors (sm_100 LDG/STG.256): half the memory instructions of
// 16-byte vectors, which matters for kernels that are issue-limited at HBM
// rate (~5 instructions per 32 B moved per SM clock at 6.5 TB/s).
template <class T> struct alignas(32) Vec32 {
    static constexpr int N = 32 / sizeof(T);
    T v[N];
};
__device__ __forceinline__ Vec32<double> ld_stream32(const double *p) {
    Vec32<double> r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ Vec32<float> ld_stream32(const float *p) {
    Vec32<float> r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                   "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream32(double *p, const Vec32<double> &x) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(x.v[0]), "d"(x.v[1]), "d"(x.v[2]),
                 "d"(x.v[3])
                 : "memory");
}
__device__ __forceinline__ void st_stream32(float *p, const Vec32<float> &x) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(x.v[0]), "f"(x.v[1]),
                 "f"(x.v[2]), "f"(x.v[3]), "f"(x.v[4]), "f"(x.v[5]), "f"(x.v[6]), "f"(x.v[7])
                 : "memory");
}
inline bool aligned32(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 31) == 0; }

// Division by a run-time invariant 32-bit divisor: q = (umulhi(x, m) + x) >> s
// (exact for every 32-bit x; m, s computed on the host).
struct FastDiv {
    uint32_t d, m, s;
    FastDiv() = default;
    explicit FastDiv(uint32_t div) : d(div) {
        s = 0;
        while ((1ull << s) < div) ++s;
        m = (uint32_t)((((1ull << s) - div) << 32) / div + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t x) const {
        return (uint32_t)(((uint64_t)__umulhi(x, m) + x) >> s);
    }
};

template <class T> struct Vec16;  // 16-byte vector of T
template <> struct Vec16<double> {
    using type = double2;
    static constexpr int N = 2;
};
template <> struct Vec16<float> {
    using type = float4;
    static constexpr int N = 4;
};

// ---- warp / block reductions ------------------------------------------------------

template <class T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = radd(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block sum (fixed tree): every thread returns the total.
template <class T, int NT> __device__ T block_sum(T v, T *smem /* >= NT/32 */) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    T t = (threadIdx.x < NT / 32) ? smem[threadIdx.x] : T(0);
    if (wid == 0) {
#pragma unroll
        for (int o = NT / 64; o > 0; o >>= 1) t = radd(t, __shfl_xor_sync(0xffffffffu, t, o));
        if (lane == 0) smem[0] = t;
    }
    __syncthreads();
    return smem[0];
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Persistent-grid size: resident CTAs per SM (occupancy calculator) x SMs,
// so a grid-stride kernel runs as exactly one full wave (no tail wave).
template <class K> int resident_grid(K kernel, int threads, size_t smem = 0) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return per_sm * num_sms();
}

// shared launch helpers (elementwise.cu)
bool is_linear(const lm_view &v);  // enumerates its elements in F-order, unit step
int ew_grid(int64_t work_items);   // grid for 256-thread streaming kernels

}  // namespace lm
