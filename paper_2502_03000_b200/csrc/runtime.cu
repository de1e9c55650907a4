#include <cstdlib>
// runtime.cu -- library state: per-thread error text, launch counter,
// device properties cache.
#include <atomic>
#include <cstdarg>
#include <map>
#include <mutex>

#include "common.cuh"

namespace lm {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};
static thread_local const char *g_variant = "";

void note_variant(const char *name) { g_variant = name; }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void clear_error() { g_err[0] = 0; }

bool has_error() { return g_err[0] != 0; }

int current_device() {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    return dev;
}

int ensure_func_attrs(const void *kernel, int smem_bytes, int carveout) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, std::pair<int, int>> done;  // (kernel, dev) -> (smem, carveout)
    const int dev = current_device();
    if (dev < 0) {
        set_error("ensure_func_attrs: no current CUDA device");
        return -2;
    }
    std::lock_guard<std::mutex> lock(mu);
    auto it = done.find({kernel, dev});
    if (it != done.end() && it->second.first >= smem_bytes && (carveout < 0 || it->second.second == carveout))
        return 0;
    int have_smem = it != done.end() ? it->second.first : 0, have_co = it != done.end() ? it->second.second : -1;
    if (smem_bytes > have_smem) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
        if (e != cudaSuccess) {
            set_error("cudaFuncSetAttribute(smem %d): %s", smem_bytes, cudaGetErrorString(e));
            return -2;
        }
        have_smem = smem_bytes;
    }
    if (carveout >= 0 && carveout != have_co) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
        if (e != cudaSuccess) {
            set_error("cudaFuncSetAttribute(carveout %d): %s", carveout, cudaGetErrorString(e));
            return -2;
        }
        have_co = carveout;
    }
    done[{kernel, dev}] = {have_smem, have_co};
    return 0;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Keep freed stream-ordered allocations in the pool (the default release
// threshold of 0 returns memory to the OS at every synchronisation, and
// re-mapping it costs far more than the kernels that use the scratch).
void ensure_pool() {
    static PerDevice<int> once;
    int unused = 0;
    once.get(unused, [](int &) {
        const int dev = current_device();
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        return 0;
    });
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("LM_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int num_sms() {
    static PerDevice<int> cache;
    int n = 148;
    cache.get(n, [](int &v) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, current_device()) != cudaSuccess || v <= 0)
            v = 148;
        return 0;
    });
    return n;
}

}  // namespace lm

extern "C" {

int lm_abi_version(void) { return LM_ABI_VERSION; }

const char *lm_last_error(void) { return lm::g_err; }

int64_t lm_launch_count(void) { return lm::g_launches.load(std::memory_order_relaxed); }

const char *lm_last_variant(void) { return lm::g_variant; }

}  // extern "C"
