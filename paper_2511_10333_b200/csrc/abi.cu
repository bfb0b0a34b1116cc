// ABI plumbing: version, thread-local error text, device queries.
#include <atomic>
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace edgc {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
    static thread_local int cached = 0;
    if (!cached) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || cached <= 0)
            cached = 148;
    }
    return cached;
}

}  // namespace edgc

extern "C" int edgc_abi_version(void) { return EDGC_ABI_VERSION; }

extern "C" const char *edgc_last_error(void) { return edgc::g_err; }

extern "C" int64_t edgc_launch_count(void) { return (int64_t)edgc::g_launches.load(); }
