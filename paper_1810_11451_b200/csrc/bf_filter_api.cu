// bf_filter_api.cu — host side of the filter stage (include/bf_filter.h):
// plan, twiddle table, H = DFT(h), launches of the fused filter kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "bf_filter.cuh"
#include "bf_filter_warp.cuh"
#include "bf_filter.h"
#include "bf_host.h"

using bfh::cuda_fail;
using bfh::DeviceGuard;
using bfh::fail;

struct bff_plan_s {
    int n = bff::kN, device = 0, num_sms = 0, ctas_per_sm = 0;
    // kernel: 3 (default) filter_warp_kernel<2, true> — one warp per signal, twiddle and H
    // tables in shared memory, 2 CTAs per SM, twiddles folded into the butterflies; 4 the same
    // without the folding; 0 filter_warp_kernel<3> (no tables, 3 CTAs per SM); 1 / 2 the
    // CTA-per-signal kernel filter_kernel<1 / 2> (kept for comparisons)
    int kind = 3;
    float2 *tw = nullptr, *H = nullptr;    // twiddles; DFT(h) / N
    float4 *tw3 = nullptr, *twp = nullptr; // pass-3 twiddle pairs; warp kernel's pass-2 bases
    bool have_taps = false;
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;
    int64_t launches = 0;
};

namespace {

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bf_status launch(bff_plan_t p, const float2 *s, float2 *y, int64_t n, int mode, cudaStream_t st) {
    bff::FParams fp{s, y, p->H, p->tw, p->tw3, p->twp, n, mode};
    const int64_t cap = (int64_t)p->num_sms * std::max(1, p->ctas_per_sm);
    const bool warpk = p->kind == 0 || p->kind >= 3;   // 4 signals (warps) per CTA
    const int64_t units = warpk ? (n + 3) / 4 : n;                 // warp kernel: 4 signals per CTA
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, cap));
    cudaEvent_t e1 = nullptr;
    if (p->profiling && mode == 0) {
        if (p->prof_used == p->prof_events.size()) {
            cudaEvent_t a, b;
            BF_CUDA(cudaEventCreate(&a));
            BF_CUDA(cudaEventCreate(&b));
            p->prof_events.emplace_back(a, b);
        }
        BF_CUDA(cudaEventRecord(p->prof_events[p->prof_used].first, st));
        e1 = p->prof_events[p->prof_used].second;
        ++p->prof_used;
    }
    if (p->kind == 0)
        bff::filter_warp_kernel<3><<<grid, bff::kThreads, bff::warp_smem_bytes(false), st>>>(fp);
    else if (p->kind == 3)
        bff::filter_warp_kernel<2, true><<<grid, bff::kThreads, bff::warp_smem_bytes(true), st>>>(fp);
    else if (p->kind == 4)
        bff::filter_warp_kernel<2><<<grid, bff::kThreads, bff::warp_smem_bytes(true), st>>>(fp);
    else if (p->kind == 1)
        bff::filter_kernel<1><<<grid, bff::kThreads, bff::smem_bytes(1), st>>>(fp);
    else
        bff::filter_kernel<2><<<grid, bff::kThreads, bff::smem_bytes(2), st>>>(fp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "filter_kernel launch");
    ++p->launches;
    if (e1) BF_CUDA(cudaEventRecord(e1, st));
    return BF_OK;
}

bf_status check_io(bff_plan_t p, const void *s, const void *y, int64_t n) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (n < 0) return fail(BF_ERR_INVALID_VALUE, "n_signals must be >= 0");
    if (n == 0) return BF_OK;
    if (!s || !y) return fail(BF_ERR_INVALID_VALUE, "NULL signal buffer");
    if (!aligned16(s) || !aligned16(y)) return fail(BF_ERR_MISALIGNED, "buffers must be 16-byte aligned");
    const uintptr_t s0 = reinterpret_cast<uintptr_t>(s), y0 = reinterpret_cast<uintptr_t>(y);
    const uintptr_t len = (uintptr_t)n * bff::kN * 8;
    if (s0 != y0 && s0 < y0 + len && y0 < s0 + len)
        return fail(BF_ERR_INVALID_VALUE, "y partially overlaps s (only exact aliasing is allowed)");
    return BF_OK;
}

}  // namespace

extern "C" {

bf_status bff_plan_create(int n, bff_plan_t *out) {
    if (!out) return fail(BF_ERR_INVALID_VALUE, "out is NULL");
    if (n < 1) return fail(BF_ERR_INVALID_VALUE, "n must be >= 1");
    if (n != bff::kN) return fail(BF_ERR_UNSUPPORTED, "filter length %d unsupported (2048 only)", n);
    int count = 0, dev = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(BF_ERR_NO_DEVICE, "no CUDA device: %s", cudaGetErrorString(e));
    }
    BF_CUDA(cudaGetDevice(&dev));
    bff_plan_t p = new (std::nothrow) bff_plan_s();
    if (!p) return fail(BF_ERR_OUT_OF_MEMORY, "host allocation of the plan failed");
    p->device = dev;
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaGetDeviceProperties"); }
    if (prop.major != 10) {
        delete p;
        return fail(BF_ERR_UNSUPPORTED, "libbf.so is built for sm_100a; device is sm_%d%d", prop.major,
                    prop.minor);
    }
    p->num_sms = prop.multiProcessorCount;
    // BFF_FILTER_KERNEL=warp_fold|warp_tab|warp|cta1|cta2 selects a kernel for comparison experiments
    if (const char *env = std::getenv("BFF_FILTER_KERNEL")) {
        const std::string k(env);
        p->kind = k == "warp" ? 0 : k == "cta1" ? 1 : k == "cta2" ? 2 : k == "warp_tab" ? 4 : 3;
    }
    const void *kern = p->kind == 0   ? (const void *)bff::filter_warp_kernel<3>
                       : p->kind == 3 ? (const void *)bff::filter_warp_kernel<2, true>
                       : p->kind == 4 ? (const void *)bff::filter_warp_kernel<2>
                       : p->kind == 1 ? (const void *)bff::filter_kernel<1> : (const void *)bff::filter_kernel<2>;
    const int smem = p->kind == 0 ? bff::warp_smem_bytes(false)
                     : p->kind >= 3 ? bff::warp_smem_bytes(true) : bff::smem_bytes(p->kind);
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaFuncSetAttribute (filter)"); }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->ctas_per_sm, kern, bff::kThreads, smem);
    if (e != cudaSuccess) { delete p; return cuda_fail(e, "occupancy query"); }
    if (cudaMalloc(&p->tw, bff::kTwN * sizeof(float2)) != cudaSuccess ||
        cudaMalloc(&p->tw3, bff::kTw3N * sizeof(float4)) != cudaSuccess ||
        cudaMalloc(&p->twp, bff::kTwpN * sizeof(float4)) != cudaSuccess ||
        cudaMalloc(&p->H, bff::kN * sizeof(float2)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p->tw);
        cudaFree(p->tw3);
        cudaFree(p->twp);
        cudaFree(p->H);
        delete p;
        return fail(BF_ERR_OUT_OF_MEMORY, "cudaMalloc of the filter plan tables failed");
    }
    bff::twiddle_kernel<<<(bff::kTwN + 255) / 256, 256>>>(p->tw);
    bff::twiddle3_kernel<<<(bff::kTw3N + 255) / 256, 256>>>(p->tw3);
    bff::twiddle_warp_kernel<<<(bff::kTwpN + 255) / 256, 256>>>(p->twp);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(p->tw);
        cudaFree(p->tw3);
        cudaFree(p->twp);
        cudaFree(p->H);
        delete p;
        return cuda_fail(e, "twiddle table");
    }
    p->launches += 3;
    *out = p;
    return BF_OK;
}

bf_status bff_set_taps(bff_plan_t p, const void *h_dev, void *stream) {
    bfh::NvtxRange nvtx_("bff_set_taps");
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (!h_dev) return fail(BF_ERR_INVALID_VALUE, "h_dev is NULL");
    if (!aligned16(h_dev)) return fail(BF_ERR_MISALIGNED, "h_dev must be 16-byte aligned");
    DeviceGuard g(p->device);
    // the plan keeps DFT(h) / N (mode 2): the filter's inverse-transform scale, folded in
    bf_status s = launch(p, static_cast<const float2 *>(h_dev), p->H, 1, 2,
                         static_cast<cudaStream_t>(stream));
    if (s == BF_OK) p->have_taps = true;
    return s;
}

bf_status bff_apply(bff_plan_t p, const void *s_dev, void *y_dev, int64_t n_signals, void *stream) {
    bfh::NvtxRange nvtx_("bff_apply");
    bf_status s = check_io(p, s_dev, y_dev, n_signals);
    if (s != BF_OK || n_signals == 0) return s;
    if (!p->have_taps) return fail(BF_ERR_NO_PRECODERS, "bff_set_taps was not called");
    DeviceGuard g(p->device);
    return launch(p, static_cast<const float2 *>(s_dev), static_cast<float2 *>(y_dev), n_signals, 0,
                  static_cast<cudaStream_t>(stream));
}

bf_status bff_fft(bff_plan_t p, const void *x_dev, void *X_dev, int64_t n_signals, void *stream) {
    bfh::NvtxRange nvtx_("bff_fft");
    bf_status s = check_io(p, x_dev, X_dev, n_signals);
    if (s != BF_OK || n_signals == 0) return s;
    DeviceGuard g(p->device);
    return launch(p, static_cast<const float2 *>(x_dev), static_cast<float2 *>(X_dev), n_signals, 1,
                  static_cast<cudaStream_t>(stream));
}

bf_status bff_destroy(bff_plan_t p) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    {
        DeviceGuard g(p->device);
        cudaFree(p->tw);
        cudaFree(p->tw3);
        cudaFree(p->twp);
        cudaFree(p->H);
        for (auto &ev : p->prof_events) {
            cudaEventDestroy(ev.first);
            cudaEventDestroy(ev.second);
        }
    }
    delete p;
    return BF_OK;
}

bf_status bff_plan_set_profiling(bff_plan_t p, int enable) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    p->profiling = enable != 0;
    return BF_OK;
}

bf_status bff_plan_kernel_time(bff_plan_t p, double *total_ms, int64_t *n_launches) {
    if (!p || !total_ms || !n_launches) return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    DeviceGuard g(p->device);
    double sum = 0.0;
    for (size_t i = 0; i < p->prof_used; ++i) {
        BF_CUDA(cudaEventSynchronize(p->prof_events[i].second));
        float ms = 0.f;
        BF_CUDA(cudaEventElapsedTime(&ms, p->prof_events[i].first, p->prof_events[i].second));
        sum += ms;
    }
    *total_ms = sum;
    *n_launches = (int64_t)p->prof_used;
    p->prof_used = 0;
    return BF_OK;
}

bf_status bff_plan_launch_count(bff_plan_t p, int64_t *count) {
    if (!p || !count) return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    *count = p->launches;
    return BF_OK;
}

}  // extern "C"
