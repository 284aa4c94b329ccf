// Library-level C ABI: version, error text, device info.
#include <stdarg.h>

#include "qs_common.cuh"

namespace qs {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    if (e == cudaErrorMemoryAllocation) return QS_ERR_OOM;
    return QS_ERR_CUDA;
}

}  // namespace qs

extern "C" {

const char* qs_version(void) { return "quakescan-b200 0.1.0 (sm_100a)"; }

const char* qs_last_error(void) { return qs::g_err; }

int qs_device_info(char* buf, size_t len) {
    int dev = 0;
    QS_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    cudaDeviceProp p;
    QS_CUDA(cudaGetDeviceProperties(&p, dev), "cudaGetDeviceProperties");
    snprintf(buf, len, "%s|%d.%d|%d|%zu", p.name, p.major, p.minor, p.multiProcessorCount,
             (size_t)p.totalGlobalMem);
    return QS_OK;
}

}  // extern "C"
