#include <cstdlib>
// runtime.cu -- library state: per-thread error text, launch counter,
// device properties cache.
#include <atomic>
#include <cstdarg>
#include <mutex>

#include "common.cuh"

namespace lm {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void clear_error() { g_err[0] = 0; }

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Keep freed stream-ordered allocations in the pool (the default release
// threshold of 0 returns memory to the OS at every synchronisation, and
// re-mapping it costs far more than the kernels that use the scratch).
void ensure_pool() {
    static bool done[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("LM_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

}  // namespace lm

extern "C" {

int lm_abi_version(void) { return LM_ABI_VERSION; }

const char *lm_last_error(void) { return lm::g_err; }

int64_t lm_launch_count(void) { return lm::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
