// Library-wide host helpers: version, last-error text, SM count.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace ap {

static thread_local char g_last_error[512] = "";

void set_last_error(const char* fmt, ...) {
    va_list ap_;
    va_start(ap_, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap_);
    va_end(ap_);
}

bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("ATTNPRED_PDL");
        v = !(e && e[0] == '0');
    }
    return v == 1;
}

int launch_status(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_last_error("%s: %s", what, cudaGetErrorString(e));
        return AP_ECUDA;
    }
    return AP_OK;
}

}  // namespace ap

extern "C" {

int ap_version(void) { return 10000; /* 1.0.0 */ }

const char* ap_last_error(void) { return ap::g_last_error; }

int ap_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return n;
}

static int g_sm_reserve = 0;

int ap_set_sm_reserve(int n) {
    const int sms = ap_device_sm_count();
    if (n < 0 || (sms > 0 && n >= sms)) {
        ap::set_last_error("ap_set_sm_reserve: %d SMs cannot be reserved (device has %d)", n, sms);
        return AP_EPARAM;
    }
    g_sm_reserve = n;
    return AP_OK;
}

int ap_sm_budget(void) {
    const int n = ap_device_sm_count() - g_sm_reserve;
    return n < 1 ? 1 : n;
}

}  // extern "C"
