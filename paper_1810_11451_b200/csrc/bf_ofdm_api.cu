// bf_ofdm_api.cu — host side of the OFDM output stage (include/bf_ofdm.h): plan, R workspace,
// chunked bf_apply -> IFFT-kernel launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "bf_filter.cuh"
#include "bf_host.h"
#include "bf_ofdm.cuh"
#include "bf_ofdm.h"

using bfh::cuda_fail;
using bfh::DeviceGuard;
using bfh::fail;

namespace {
constexpr int64_t kDefaultChunk = 4096;   // symbols per bf_apply + IFFT pair
// nb = 26 (1560 subcarriers, e.g. 50 MHz at 30 kHz): the IFFT kernel specialised for this
// half band skips the all-zero rows of bins at compile time
constexpr int kHalf26 = 26 * 60 / 2;
}

struct bf_ofdm_plan_s {
    bf_plan_t bf = nullptr;
    int n = bfofdm::kN, cp = 0, nb = 0, A = 64, B = 60, f = 0, device = 0;
    float scale = 1.0f;
    int num_sms = 0, ctas_per_sm = 0;
    // IFFT kernel (BFO_OFDM_KERNEL): 1 sb ofdm_ifft_kernel<1, 4> (bulk-copy fetch), 2 db
    // <2, 6>, 3 cpa <1, 4, true> (cp.async fetch; the default: of1 0.855 of copy BW vs 0.84 sb,
    // 0.83 db, 0.72 cpa_db — profiles/r02_of1_kernels.jsonl), 4 cpa_db <2, 6, true>
    int kind = 3;
    bool spec = true;           // use the nb = 26 specialisation when it applies (BFO_OFDM_SPEC=0: off)
    bool out16 = false;         // bf_ofdm_plan_set_output: int16 samples x 2^out_exp
    int out_exp = 12;
    int64_t chunk = kDefaultChunk;
    float2 *tw = nullptr;
    float2 *R = nullptr;        // workspace [chunk nb][A][B]
    int64_t R_cap = 0;          // symbols
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;
    int64_t launches = 0;
};

namespace {

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool overlap(const void *a, size_t na, const void *b, size_t nb) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
    return a && b && na && nb && a0 < b0 + nb && b0 < a0 + na;
}

size_t y_bytes(bf_ofdm_plan_t p, int64_t n_sym) {
    return (size_t)n_sym * p->A * (p->cp + p->n) * (p->out16 ? 4 : 8);
}
size_t r_bytes(bf_ofdm_plan_t p, int64_t n_sym) { return (size_t)n_sym * p->nb * p->A * p->B * 8; }

bf_status launch_ifft(bf_ofdm_plan_t p, const float2 *R, int64_t n_sym, float2 *y, cudaStream_t st) {
    bfofdm::OParams op{R, y, p->tw, n_sym * p->A, p->A, p->nb, p->B, p->nb * p->B / 2, p->cp,
                       p->out16 ? ldexpf(p->scale, p->out_exp) : p->scale};
    const int64_t cap = (int64_t)p->num_sms * std::max(1, p->ctas_per_sm);
    const int nwarps = (p->kind == 2 || p->kind == 4) ? 6 : 4;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((op.n_sig + nwarps - 1) / nwarps, cap));
    cudaEvent_t e1 = nullptr;
    if (p->profiling) {
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
    if (p->kind == 2)
        bfofdm::ofdm_ifft_kernel<2, 6><<<grid, 6 * 32, bfofdm::smem_bytes(2, 6), st>>>(op);
    else if (p->kind == 3 && op.half == kHalf26 && p->A == 64 && p->B == 60 && p->spec)
        (p->out16 ? bfofdm::ofdm_ifft_kernel<1, 4, true, true, kHalf26>
                  : bfofdm::ofdm_ifft_kernel<1, 4, true, false, kHalf26>)
            <<<grid, 4 * 32, bfofdm::smem_bytes(1, 4), st>>>(op);
    else if (p->kind == 3 && p->out16)
        bfofdm::ofdm_ifft_kernel<1, 4, true, true><<<grid, 4 * 32, bfofdm::smem_bytes(1, 4), st>>>(op);
    else if (p->kind == 3)
        bfofdm::ofdm_ifft_kernel<1, 4, true><<<grid, 4 * 32, bfofdm::smem_bytes(1, 4), st>>>(op);
    else if (p->kind == 4)
        bfofdm::ofdm_ifft_kernel<2, 6, true><<<grid, 6 * 32, bfofdm::smem_bytes(2, 6), st>>>(op);
    else
        bfofdm::ofdm_ifft_kernel<1, 4><<<grid, 4 * 32, bfofdm::smem_bytes(1, 4), st>>>(op);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "ofdm_ifft_kernel launch");
    ++p->launches;
    if (e1) BF_CUDA(cudaEventRecord(e1, st));
    return BF_OK;
}

bf_status check_y(bf_ofdm_plan_t p, const void *y, int64_t n_sym) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (n_sym < 0) return fail(BF_ERR_INVALID_VALUE, "n_sym must be >= 0");
    if (n_sym > 0 && !y) return fail(BF_ERR_INVALID_VALUE, "y_dev is NULL");
    if (y && !aligned16(y)) return fail(BF_ERR_MISALIGNED, "y_dev must be 16-byte aligned");
    if ((int64_t)n_sym * p->nb >= ((int64_t)1 << 31))
        return fail(BF_ERR_UNSUPPORTED, "n_sym * nb must be < 2^31 blocks");
    return BF_OK;
}

}  // namespace

extern "C" {

bf_status bf_ofdm_plan_create(bf_plan_t bf, int n, int cp, int nb, float scale, bf_ofdm_plan_t *out) {
    if (!out) return fail(BF_ERR_INVALID_VALUE, "out is NULL");
    if (!bf) return fail(BF_ERR_INVALID_VALUE, "bf plan is NULL");
    int A = 0, f = 0, B = 0, layout = 0, dev = 0;
    bf_status s = bfh::plan_info(bf, &A, &f, &B, &layout, &dev);
    if (s != BF_OK) return s;
    if (layout != BF_LAYOUT_INTERLEAVED)
        return fail(BF_ERR_UNSUPPORTED, "the OFDM stage takes an interleaved fp32 bf plan (layout %d)", layout);
    if (n != bfofdm::kN) return fail(BF_ERR_UNSUPPORTED, "IFFT size %d unsupported (2048 only)", n);
    if (cp < 0 || cp >= n) return fail(BF_ERR_INVALID_VALUE, "cp must be in [0, n)");
    if (nb < 1 || (int64_t)nb * B > n)
        return fail(BF_ERR_INVALID_VALUE, "nb must be >= 1 with nb * %d <= n", B);
    if (!(scale == scale) || scale - scale != 0.0f) return fail(BF_ERR_INVALID_VALUE, "scale must be finite");
    DeviceGuard g(dev);
    bf_ofdm_plan_t p = new (std::nothrow) bf_ofdm_plan_s();
    if (!p) return fail(BF_ERR_OUT_OF_MEMORY, "host allocation of the plan failed");
    p->bf = bf;
    p->n = n;
    p->cp = cp;
    p->nb = nb;
    p->A = A;
    p->B = B;
    p->f = f;
    p->device = dev;
    p->scale = scale;
    cudaError_t e0_ = cudaSuccess;
    // BFO_OFDM_KERNEL=sb|db selects the IFFT kernel for comparison experiments (default below)
    if (const char *env = std::getenv("BFO_OFDM_KERNEL")) {
        const std::string k(env);
        p->kind = k == "db" ? 2 : k == "sb" ? 1 : k == "cpa_db" ? 4 : 3;
    }
    const bool db = p->kind == 2 || p->kind == 4;
    e0_ = cudaFuncSetAttribute(bfofdm::ofdm_ifft_kernel<1, 4, true, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, bfofdm::smem_bytes(1, 4));
    for (const void *k : {(const void *)bfofdm::ofdm_ifft_kernel<1, 4, true, false, kHalf26>,
                          (const void *)bfofdm::ofdm_ifft_kernel<1, 4, true, true, kHalf26>})
        if (e0_ == cudaSuccess)
            e0_ = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bfofdm::smem_bytes(1, 4));
    if (const char *env = std::getenv("BFO_OFDM_SPEC")) p->spec = std::atoi(env) != 0;
    const void *kern = p->kind == 2   ? (const void *)bfofdm::ofdm_ifft_kernel<2, 6>
                       : p->kind == 3 ? (const void *)bfofdm::ofdm_ifft_kernel<1, 4, true>
                       : p->kind == 4 ? (const void *)bfofdm::ofdm_ifft_kernel<2, 6, true>
                                      : (const void *)bfofdm::ofdm_ifft_kernel<1, 4>;
    const int smem = db ? bfofdm::smem_bytes(2, 6) : bfofdm::smem_bytes(1, 4);
    const int threads = db ? 6 * 32 : 4 * 32;
    cudaError_t e = e0_;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->ctas_per_sm, kern, threads, smem);
    if (e == cudaSuccess) e = cudaMalloc(&p->tw, bff::kTwN * sizeof(float2));
    if (e == cudaSuccess) {
        bff::twiddle_kernel<<<(bff::kTwN + 255) / 256, 256>>>(p->tw);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p->tw);
        delete p;
        return cuda_fail(e, "OFDM plan setup");
    }
    p->launches = 1;
    *out = p;
    return BF_OK;
}

bf_status bf_ofdm_ifft(bf_ofdm_plan_t p, const void *R_dev, int64_t n_sym, void *y_dev, void *stream) {
    bfh::NvtxRange nvtx_("bf_ofdm_ifft");
    bf_status s = check_y(p, y_dev, n_sym);
    if (s != BF_OK || n_sym == 0) return s;
    if (!R_dev) return fail(BF_ERR_INVALID_VALUE, "R_dev is NULL");
    if (!aligned16(R_dev)) return fail(BF_ERR_MISALIGNED, "R_dev must be 16-byte aligned");
    if (overlap(R_dev, r_bytes(p, n_sym), y_dev, y_bytes(p, n_sym)))
        return fail(BF_ERR_INVALID_VALUE, "y overlaps R");
    DeviceGuard g(p->device);
    return launch_ifft(p, static_cast<const float2 *>(R_dev), n_sym, static_cast<float2 *>(y_dev),
                       static_cast<cudaStream_t>(stream));
}

bf_status bf_ofdm_apply(bf_ofdm_plan_t p, const void *S_dev, const int32_t *tags_dev, int64_t n_sym,
                        void *y_dev, void *stream) {
    bfh::NvtxRange nvtx_("bf_ofdm_apply");
    bf_status s = check_y(p, y_dev, n_sym);
    if (s != BF_OK || n_sym == 0) return s;
    const size_t sb = (size_t)n_sym * p->nb * p->f * p->B * 8;
    if (overlap(S_dev, sb, y_dev, y_bytes(p, n_sym)) ||
        overlap(tags_dev, (size_t)n_sym * p->nb * 4, y_dev, y_bytes(p, n_sym)))
        return fail(BF_ERR_INVALID_VALUE, "y overlaps S or the tags");
    DeviceGuard g(p->device);
    const int64_t chunk = std::min(n_sym, p->chunk);
    if (chunk > p->R_cap) {
        cudaFree(p->R);
        p->R = nullptr;
        p->R_cap = 0;
        cudaError_t e = cudaMalloc(&p->R, r_bytes(p, chunk));
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(BF_ERR_OUT_OF_MEMORY, "R workspace of %lld symbols", (long long)chunk);
        }
        p->R_cap = chunk;
    }
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t s_sym = (int64_t)p->nb * p->f * p->B * 2;   // floats of S per symbol
    for (int64_t m0 = 0; m0 < n_sym; m0 += chunk) {
        const int64_t c = std::min(chunk, n_sym - m0);
        const float *S = static_cast<const float *>(S_dev);
        s = bf_apply(p->bf, S ? S + m0 * s_sym : nullptr, tags_dev ? tags_dev + m0 * p->nb : nullptr,
                     p->R, c * p->nb, stream);
        if (s != BF_OK) return s;
        s = launch_ifft(p, p->R, c,
                        reinterpret_cast<float2 *>(static_cast<char *>(y_dev) +
                                                   y_bytes(p, m0)), st);
        if (s != BF_OK) return s;
    }
    return BF_OK;
}

bf_status bf_ofdm_plan_set_output(bf_ofdm_plan_t p, int format, int exponent) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (format != BF_OFDM_OUT_F32 && format != BF_OFDM_OUT_I16)
        return fail(BF_ERR_INVALID_VALUE, "unknown output format %d", format);
    if (exponent < -126 || exponent > 127) return fail(BF_ERR_INVALID_VALUE, "exponent out of range");
    if (format == BF_OFDM_OUT_I16 && p->kind != 3)
        return fail(BF_ERR_UNSUPPORTED, "int16 output is built for the default IFFT kernel only");
    p->out16 = format == BF_OFDM_OUT_I16;
    p->out_exp = exponent;
    return BF_OK;
}

bf_status bf_ofdm_plan_set_chunk(bf_ofdm_plan_t p, int64_t symbols) {
    if (!p || symbols < 0) return fail(BF_ERR_INVALID_VALUE, "invalid chunk");
    p->chunk = symbols == 0 ? kDefaultChunk : symbols;
    return BF_OK;
}

bf_status bf_ofdm_destroy(bf_ofdm_plan_t p) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    {
        DeviceGuard g(p->device);
        cudaFree(p->tw);
        cudaFree(p->R);
        for (auto &ev : p->prof_events) {
            cudaEventDestroy(ev.first);
            cudaEventDestroy(ev.second);
        }
    }
    delete p;
    return BF_OK;
}

bf_status bf_ofdm_plan_set_profiling(bf_ofdm_plan_t p, int enable) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    p->profiling = enable != 0;
    return BF_OK;
}

bf_status bf_ofdm_plan_kernel_time(bf_ofdm_plan_t p, double *total_ms, int64_t *n_launches) {
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

bf_status bf_ofdm_plan_launch_count(bf_ofdm_plan_t p, int64_t *count) {
    if (!p || !count) return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    *count = p->launches;
    return BF_OK;
}

}  // extern "C"
