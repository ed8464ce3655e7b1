// Throughput of packed fp32x2 (FFMA2 / FADD2) against scalar FFMA / FADD on sm_100a:
// independent chains, every SM, CUDA events.  Not part of the product library.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

template <int MODE>
__global__ void __launch_bounds__(256) probe(float *out, int iters, float x) {
    constexpr int N = 8;
    if (MODE == 0 || MODE == 2) {          // scalar FFMA / FADD: 2 N independent chains
        float a[2 * N];
        for (int i = 0; i < 2 * N; ++i) a[i] = x * (threadIdx.x + i);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 2 * N; ++i) {
                if (MODE == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(x), "f"(0.5f));
                else asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(x));
            }
        }
        float s = 0;
        for (int i = 0; i < 2 * N; ++i) s += a[i];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else {                               // packed: N independent 2-wide chains (same flops)
        uint64_t a[N];
        float2 xx = make_float2(x, x), hh = make_float2(0.5f, 0.5f);
        const uint64_t X = *reinterpret_cast<uint64_t *>(&xx), H = *reinterpret_cast<uint64_t *>(&hh);
        for (int i = 0; i < N; ++i) {
            float2 v = make_float2(x * (threadIdx.x + 2 * i), x * (threadIdx.x + 2 * i + 1));
            a[i] = *reinterpret_cast<uint64_t *>(&v);
        }
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < N; ++i) a[i] = MODE == 1 ? ffma2(a[i], X, H) : fadd2(a[i], X);
        }
        float s = 0;
        for (int i = 0; i < N; ++i) { float2 v = *reinterpret_cast<float2 *>(&a[i]); s += v.x + v.y; }
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    }
}

// dependent-chain latency: one warp, one chain, clock64 around 4096 dependent ops
template <int MODE>
__global__ void lat(float *out, long long *cyc, float x) {
    float a = x * threadIdx.x;
    uint64_t b;
    float2 v = make_float2(a, a + 1.f), xx = make_float2(x, x);
    b = *reinterpret_cast<uint64_t *>(&v);
    const uint64_t X = *reinterpret_cast<uint64_t *>(&xx);
    const long long t0 = clock64();
    for (int i = 0; i < 4096; ++i) {
        if (MODE == 0) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(a) : "f"(x));
        else if (MODE == 1) b = ffma2(b, X, X);
        else if (MODE == 2) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a) : "f"(x));
        else b = fadd2(b, X);
    }
    const long long t1 = clock64();
    float2 r = *reinterpret_cast<float2 *>(&b);
    out[threadIdx.x] = a + r.x + r.y;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
    const int iters = 1 << 14, grid = sms * 8;
    const char *names[4] = {"FFMA (scalar)", "FFMA2 (fp32x2)", "FADD (scalar)", "FADD2 (fp32x2)"};
    for (int rep = 0; rep < 2; ++rep)
        for (int mode = 0; mode < 4; ++mode) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            auto launch = [&]() {
                if (mode == 0) probe<0><<<grid, 256>>>(out, iters, 1.0001f);
                if (mode == 1) probe<1><<<grid, 256>>>(out, iters, 1.0001f);
                if (mode == 2) probe<2><<<grid, 256>>>(out, iters, 1.0001f);
                if (mode == 3) probe<3><<<grid, 256>>>(out, iters, 1.0001f);
            };
            launch();
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double lane_ops = (double)grid * 256 * iters * 16;   // fp32 results
            const double flops = lane_ops * (mode < 2 ? 2.0 : 1.0);
            if (rep == 1)
                printf("{\"op\": \"%s\", \"ms\": %.3f, \"Gresults_per_s\": %.1f, \"TFLOPs\": %.2f}\n",
                       names[mode], ms, lane_ops / ms / 1e6, flops / ms / 1e9);
        }
    long long *cyc;
    cudaMalloc(&cyc, 8);
    const char *ln[4] = {"FFMA", "FFMA2", "FADD", "FADD2"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) lat<0><<<1, 32>>>(out, cyc, 1.0001f);
            if (mode == 1) lat<1><<<1, 32>>>(out, cyc, 1.0001f);
            if (mode == 2) lat<2><<<1, 32>>>(out, cyc, 1.0001f);
            if (mode == 3) lat<3><<<1, 32>>>(out, cyc, 1.0001f);
        }
        long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("{\"op\": \"%s\", \"dependent_latency_cycles\": %.2f}\n", ln[mode], c / 4096.0);
    }
    return 0;
}
