// bf_host.h — host-side helpers shared by the C-ABI translation units of libbf.so:
// thread-local error detail (bf_last_error), status helpers, device guard.
#pragma once
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: no-ops unless a profiler attaches

#include <cstdarg>
#include <cstdio>
#include <string>

#include "bf.h"

namespace bfh {

extern thread_local std::string g_last_error;

inline bf_status fail(bf_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

inline bf_status cuda_fail(cudaError_t e, const char *what) {
    return fail(BF_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// Plan facts for the other stages of the library (bf_ofdm_api.cu); defined in bf_api.cu.
bf_status plan_info(bf_plan_t p, int *n_ant, int *f, int *b, int *layout, int *device);

// Makes `dev` current for the scope of a call and restores the caller's device.
struct DeviceGuard {
    int prev = -1;
    bool changed = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) changed = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (changed) cudaSetDevice(prev);
    }
};

// NVTX range around one ABI call ("libbf" domain) so that nsys / ncu timelines show the
// host calls (route, apply, batch, host pipeline) above the kernels they enqueue.
struct NvtxRange {
    static nvtxDomainHandle_t domain() {
        static nvtxDomainHandle_t d = nvtxDomainCreateA("libbf");
        return d;
    }
    explicit NvtxRange(const char *name) {
        nvtxEventAttributes_t a{};
        a.version = NVTX_VERSION;
        a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        a.messageType = NVTX_MESSAGE_TYPE_ASCII;
        a.message.ascii = name;
        nvtxDomainRangePushEx(domain(), &a);
    }
    ~NvtxRange() { nvtxDomainRangePop(domain()); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

}  // namespace bfh

#define BF_CUDA(call)                                                \
    do {                                                             \
        cudaError_t e_ = (call);                                     \
        if (e_ != cudaSuccess) return bfh::cuda_fail(e_, #call);     \
    } while (0)
