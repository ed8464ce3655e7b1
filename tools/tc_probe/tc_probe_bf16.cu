// Probe: kind::f16 (bf16 inputs, fp32 accumulate) MMA with A in TMEM (two bf16 per
// 32-bit column) and B in shared memory (no-swizzle K-major core matrices of
// 8 rows x 16 bytes = 8 bf16), M = N = 128, K = 16 per instruction.
#include <cstdio>
#include <cuda_bf16.h>
#include "../../paper_1810_11451_b200/csrc/bf_ffma.cuh"
#include "../../paper_1810_11451_b200/csrc/tc_ptx.cuh"

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

// A: [128][K] bf16 (row-major), B: [128 (n)][K] bf16; D = A B^T fp32 [128][128]
__global__ void __launch_bounds__(128, 1) probe(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *D, int K) {
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    extern __shared__ __align__(1024) __nv_bfloat16 Bs[];
    const int tid = threadIdx.x, warp = tid / 32;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    if (tid == 0) { bfk::mbar_init(&bar, 1); bfk::mbar_fence_init(); }
    // B core matrices: K chunk kc of 8 elements (16 B), N group ng of 8 rows
    for (int idx = tid; idx < 128 * K; idx += 128) {
        const int n = idx / K, k = idx % K;
        const int kc = k / 8, ng = n / 8, r = n % 8, e = k % 8;
        Bs[((kc * 16 + ng) * 8 + r) * 8 + e] = B[n * K + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before_sync(); __syncthreads(); tc::fence_after_sync();
    const uint32_t base = tmem_base, lane_base = (uint32_t)(32 * warp) << 16;
    for (int c0 = 0; c0 < K / 2; c0 += 8) {
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) {
            const int k = 2 * (c0 + i);
            const uint16_t lo = __bfloat16_as_ushort(A[tid * K + k]);
            const uint16_t hi = __bfloat16_as_ushort(A[tid * K + k + 1]);
            v[i] = (uint32_t)lo | ((uint32_t)hi << 16);
        }
        tc::tmem_st8(base + lane_base + 256 + c0, v);
    }
    tc::tmem_st_wait(); tc::fence_before_sync(); __syncthreads(); tc::fence_after_sync();
    if (tid == 0) {
        for (int kb = 0; kb < K / 16; ++kb) {
            // one MMA covers 2 K chunks (2 x 16 B): LBO = next K chunk, SBO = next 8-row group
            const uint64_t desc = tc::smem_desc(tc::smem_u32(Bs) + kb * 2 * 16 * 128, 16 * 128, 128);
            mma_f16_ts(base, base + 256 + kb * 8, desc, idesc_bf16(128, 128), kb > 0);
        }
        tc::mma_commit(&bar);
    }
    bfk::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    for (int c0 = 0; c0 < 128; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(base + lane_base + c0, v);
        tc::tmem_ld_wait();
        for (int i = 0; i < 16; ++i) D[tid * 128 + c0 + i] = __uint_as_float(v[i]);
    }
    tc::fence_before_sync(); __syncthreads();
    if (warp == 0) tc::tmem_free<512>(base);
}

extern "C" int tcp_bf16(const void *A, const void *B, float *D, int K) {
    void *dA, *dB; float *dD;
    cudaMalloc(&dA, 128 * K * 2); cudaMalloc(&dB, 128 * K * 2); cudaMalloc(&dD, 128 * 128 * 4);
    cudaMemcpy(dA, A, 128 * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, 128 * K * 2, cudaMemcpyHostToDevice);
    const int smem = 128 * K * 2;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>((const __nv_bfloat16 *)dA, (const __nv_bfloat16 *)dB, dD, K);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("probe: %s\n", cudaGetErrorString(e)); return (int)e; }
    cudaMemcpy(D, dD, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
    return 0;
}
