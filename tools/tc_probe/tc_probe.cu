// Development probe for the tcgen05 building blocks used by the tensor-core
// beamforming path: TMEM alloc, tcgen05.st of A rows, kind::tf32 MMA with A in
// TMEM and B in shared memory (no-swizzle K-major core matrices), commit to an
// mbarrier and tcgen05.ld of D.  One CTA of 128 threads; D = A[128 x K] * B^T
// with B given as [N=128][K].  Not part of the product library.
#include <cstdio>
#include "../../paper_1810_11451_b200/csrc/bf_ffma.cuh"
#include "../../paper_1810_11451_b200/csrc/tc_ptx.cuh"

__global__ void __launch_bounds__(128, 1) tc_probe(const float *A, const float *B, float *D, int K) {
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    extern __shared__ __align__(1024) float Bs[];
    const int tid = threadIdx.x, warp = tid / 32;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    if (tid == 0) { bfk::mbar_init(&bar, 1); bfk::mbar_fence_init(); }
    for (int idx = tid; idx < 128 * K; idx += 128) {
        const int n = idx / K, k = idx % K;
        const int kc = k / 4, ng = n / 8, r = n % 8, e = k % 4;
        Bs[((kc * 16 + ng) * 8 + r) * 4 + e] = B[n * K + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t base = tmem_base;
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    for (int c0 = 0; c0 < K; c0 += 8) {
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(A[tid * K + c0 + i]);
        tc::tmem_st8(base + lane_base + 256 + c0, v);
    }
    tc::tmem_st_wait();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_tf32(128, 128);
        for (int kb = 0; kb < K / 8; ++kb) {
            const uint64_t desc = tc::smem_desc(tc::smem_u32(Bs) + kb * 2 * 16 * 128, 16 * 128, 128);
            tc::mma_tf32_ts(base, base + 256 + kb * 8, desc, idesc, kb > 0);
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
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(base);
}

extern "C" int tcp_run(const float *A, const float *B, float *D, int K) {
    float *dA, *dB, *dD;
    cudaMalloc(&dA, 128 * K * 4); cudaMalloc(&dB, 128 * K * 4); cudaMalloc(&dD, 128 * 128 * 4);
    cudaMemcpy(dA, A, 128 * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, 128 * K * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xFF, 128 * 128 * 4);
    const int smem = 128 * K * 4;
    cudaFuncSetAttribute(tc_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tc_probe<<<1, 128, smem>>>(dA, dB, dD, K);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("tc_probe: %s\n", cudaGetErrorString(e)); return (int)e; }
    cudaMemcpy(D, dD, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
    return 0;
}
