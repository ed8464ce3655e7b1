// probes.cu — micro-benchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry (no FP32 peak there).
// Bench infrastructure only; not on the beamforming path.
//
// bfp_ffma_peak: every SM runs CTAs whose threads execute an 8 x 8 register
// outer product of 3-register FFMAs (the same operand pattern as the
// beamforming kernel's complex MAC), timed with CUDA events.
#include <cuda_runtime.h>
#include <cstdint>

namespace {

__global__ void __launch_bounds__(256) ffma_outer(float *out, int iters, float seed) {
    float a[8], b[8], c[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = seed + threadIdx.x * 1e-7f + i * 1e-3f;
        b[i] = seed - i * 2e-3f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) c[i][j] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) c[i][j] = fmaf(a[i], b[j], c[i][j]);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += c[i][j];
    if (s == 1.2345f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;   // keep the work alive
}

}  // namespace

extern "C" {

// Returns 0 on success.  *tflops = FP32 FLOP/s (2 per FFMA) / 1e12 achieved.
int bfp_ffma_peak(int iters, int ctas_per_sm, double *tflops, double *ms_out, int *sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return 1;
    *sms = prop.multiProcessorCount;
    const int grid = prop.multiProcessorCount * ctas_per_sm;
    float *out = nullptr;
    if (cudaMalloc(&out, (size_t)grid * 256 * sizeof(float)) != cudaSuccess) return 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ffma_outer<<<grid, 256>>>(out, iters / 10 + 1, 1.0f);   // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        ffma_outer<<<grid, 256>>>(out, iters, 1.0f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return 3;
    const double flops = 2.0 * 64.0 * (double)iters * 256.0 * grid;
    *tflops = flops / (best * 1e-3) / 1e12;
    *ms_out = best;
    return 0;
}

}  // extern "C"
