// Energy per tcgen05.mma with cta_group::2 (2-SM MMA, M = 256) vs cta_group::1
// (not part of the product; companion of mma_power.cu).  Clusters of 2 CTAs: the
// leader CTA's thread 0 issues M = 256 (128 rows from each CTA's TMEM), N = 128,
// K = 8 tf32 (or K = 16 bf16) MMAs with A in TMEM and B split across the two
// CTAs' shared memory (each holds N/2 = 64 rows at the same offset).
// mmp2_run(kind, iters, reps, &ms): kind 0 tf32, 1 bf16.
#include <cstdio>
#include <cstdint>
#include "../../paper_1810_11451_b200/csrc/bf_ffma.cuh"
#include "../../paper_1810_11451_b200/csrc/tc_ptx.cuh"

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t rnd_word(int kind, uint32_t seed) {
    const uint32_t h = hash32(seed);
    if (kind == 0) {
        const uint32_t e = 123u + (h >> 28) % 5u;
        return (h & 0x80000000u) | (e << 23) | (h & 0x007FE000u);
    }
    auto bf = [](uint32_t r) { return (uint32_t)((r & 0x8000u) | ((120u + (r >> 12) % 7u) << 7) | (r & 0x7Fu)); };
    return bf(h & 0xFFFFu) | (bf(h >> 16) << 16);
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int KB = 9;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_power2(int kind, int iters) {
    extern __shared__ __align__(1024) uint32_t Bs[];   // this CTA's 64 rows of B: KB x 2 chunks x 64 rows x 16 B
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = cluster_rank();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;"
                     ::"r"(tc::smem_u32(&tmem_base)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    if (tid == 0) { bfk::mbar_init(&bar, 1); bfk::mbar_fence_init(); }
    const int words = KB * 2 * 64 * 4;
    for (int i = tid; i < words; i += 128) Bs[i] = rnd_word(kind, 0x9E3779B9u * (i + 1) + 31u * rank);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before_sync(); __syncthreads(); tc::fence_after_sync();
    const uint32_t base = tmem_base, lane_base = (uint32_t)(32 * warp) << 16;
    for (int c0 = 0; c0 < 128; c0 += 8) {
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) v[i] = rnd_word(kind, 0x85EBCA6Bu * (tid * 128 + c0 + i + 1) + 77u * rank + 13u * blockIdx.x);
        tc::tmem_st8(base + lane_base + c0, v);
    }
    tc::tmem_st_wait();
    tc::fence_before_sync();
    cluster_sync();
    tc::fence_after_sync();
    if (rank == 0 && tid == 0) {
        // M = 256, N = 128: instruction descriptor M >> 4 = 16, N >> 3 = 16
        const uint32_t idesc = kind == 0 ? tc::idesc_tf32(256, 128) : tc::idesc_bf16(256, 128);
        const uint32_t b0 = tc::smem_u32(Bs);
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = base + 256 + 128 * (it & 1);
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
                const uint64_t desc = tc::smem_desc(b0 + (uint32_t)(2 * kb * 16 * 64), 16 * 64, 128);
                const uint32_t a = base + kb * 8, acc = kb != 0;
                if (kind == 0)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(d), "r"(a), "l"(desc), "r"(idesc), "r"(acc) : "memory");
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(d), "r"(a), "l"(desc), "r"(idesc), "r"(acc) : "memory");
            }
        }
        // arrive on both CTAs' barrier (same smem offset) once every MMA completed
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(tc::smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    }
    bfk::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    tc::fence_before_sync();
    cluster_sync();
    if (warp == 0) {
        tc::fence_after_sync();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
    }
}

extern "C" int mmp2_run(int kind, int iters, int reps, float *ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 2 * KB * 2 * 64 * 16;   // 2x: headroom if the unit reads more rows than assumed
    cudaFuncSetAttribute(mma_power2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms / 2 * 2;
    mma_power2<<<grid, 128, smem>>>(kind, iters);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) mma_power2<<<grid, 128, smem>>>(kind, iters);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) {
        printf("mmp2: %s\n", cudaGetErrorString(e));
        return (int)e;
    }
    *ms_out = ms / reps;
    return 0;
}
