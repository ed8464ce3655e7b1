// Energy per tcgen05.mma by kind (not part of the product): every SM issues a long
// stream of M = N = 128 MMAs with A in TMEM and B in shared memory, operands filled
// with random bits of the given format, so that power / rate = energy per MMA.
//   mode 0: kind::tf32, K = 8     (random tf32 values, 11-bit significands)
//   mode 1: kind::f16 bf16, K = 16 (random bf16)
//   mode 2: kind::f16 fp16, K = 16 (random fp16 in [-1, 1])
//   mode 3: kind::tf32, K = 8, zero A (toggle floor)
// mmp_run(mode, iters, reps, &ms) -> 0; ms = average per launch.
#include <cstdio>
#include <cstdint>
#include "../../paper_1810_11451_b200/csrc/bf_ffma.cuh"
#include "../../paper_1810_11451_b200/csrc/tc_ptx.cuh"

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

// random value of the format, packed into 32 bits (one tf32 or two 16-bit values)
__device__ __forceinline__ uint32_t rnd_word(int mode, uint32_t seed) {
    const uint32_t h = hash32(seed);
    if (mode == 0 || mode == 3) {
        // sign | exponent in [2^-4, 2) | 10 random mantissa bits, low 13 bits zero
        const uint32_t e = 123u + (h >> 28) % 5u;
        return (h & 0x80000000u) | (e << 23) | (h & 0x007FE000u);
    }
    if (mode == 1) {
        auto bf = [](uint32_t r) { return (uint32_t)((r & 0x8000u) | ((120u + (r >> 12) % 7u) << 7) | (r & 0x7Fu)); };
        return bf(h & 0xFFFFu) | (bf(h >> 16) << 16);
    }
    auto hf = [](uint32_t r) { return (uint32_t)((r & 0x8000u) | ((10u + (r >> 11) % 5u) << 10) | (r & 0x3FFu)); };
    return hf(h & 0xFFFFu) | (hf(h >> 16) << 16);
}

constexpr int KB_PER_GROUP = 9;   // 9 MMAs per accumulation chain (f = 36: KP = 72)

__global__ void __launch_bounds__(128, 1) mma_power(int mode, int iters) {
    extern __shared__ __align__(1024) uint32_t Bs[];       // 9 x 2 core-matrix chunks x 128 rows x 16 B
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    if (tid == 0) { bfk::mbar_init(&bar, 1); bfk::mbar_fence_init(); }
    const int words = KB_PER_GROUP * 2 * 128 * 4;
    for (int i = tid; i < words; i += 128) Bs[i] = rnd_word(mode == 3 ? 0 : mode, 0x9E3779B9u * (i + 1) + blockIdx.x);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before_sync(); __syncthreads(); tc::fence_after_sync();
    const uint32_t base = tmem_base, lane_base = (uint32_t)(32 * warp) << 16;
    for (int c0 = 0; c0 < 128; c0 += 8) {   // A: columns [0, 128)
        uint32_t v[8];
        for (int i = 0; i < 8; ++i)
            v[i] = mode == 3 ? 0u : rnd_word(mode, 0x85EBCA6Bu * (tid * 128 + c0 + i + 1) + 77u * blockIdx.x);
        tc::tmem_st8(base + lane_base + c0, v);
    }
    tc::tmem_st_wait(); tc::fence_before_sync(); __syncthreads(); tc::fence_after_sync();
    if (tid == 0) {
        const uint32_t idesc = (mode == 0 || mode == 3) ? tc::idesc_tf32(128, 128)
                             : (mode == 1 ? tc::idesc_bf16(128, 128) : idesc_f16(128, 128));
        const uint32_t b0 = tc::smem_u32(Bs);
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = base + 256 + 128 * (it & 1);
#pragma unroll
            for (int kb = 0; kb < KB_PER_GROUP; ++kb) {
                const uint64_t desc = tc::smem_desc(b0 + (uint32_t)(2 * kb * 16 * 128), 16 * 128, 128);
                if (mode == 0 || mode == 3)
                    tc::mma_tf32_ts(d, base + kb * 8, desc, idesc, kb != 0);
                else
                    tc::mma_bf16_ts(d, base + kb * 8, desc, idesc, kb != 0);
            }
        }
        tc::mma_commit(&bar);
    }
    bfk::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    tc::fence_before_sync(); __syncthreads();
    if (warp == 0) tc::tmem_free<512>(base);
}

extern "C" int mmp_run(int mode, int iters, int reps, float *ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = KB_PER_GROUP * 2 * 128 * 16;
    cudaFuncSetAttribute(mma_power, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_power<<<sms, 128, smem>>>(mode, iters);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) mma_power<<<sms, 128, smem>>>(mode, iters);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) {
        printf("mmp: %s\n", cudaGetErrorString(e));
        return (int)e;
    }
    *ms_out = ms / reps;
    return 0;
}
