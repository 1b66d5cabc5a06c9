// hb_api.cu -- error reporting and library metadata for the C ABI.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "hb_common.cuh"

namespace hb {

static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

static std::atomic<long long> g_launches{0};

int check_launch(const char *what, int kernels) {
    g_launches.fetch_add(kernels, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(HB_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return HB_OK;
}

int device_sm_count() {
    static int cached = 0;
    if (cached == 0) {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
            cached = n;
        else
            cached = 148;
    }
    return cached;
}

}  // namespace hb

extern "C" {

int hb_abi_version(void) { return 1; }

const char *hb_last_error(void) { return hb::g_err; }

long long hb_launch_count(void) { return hb::g_launches.load(std::memory_order_relaxed); }

int hb_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

}  // extern "C"
