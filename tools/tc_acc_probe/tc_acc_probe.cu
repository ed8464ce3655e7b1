// Accumulation-error probe for tcgen05.mma kind::tf32 and kind::f16 (fp16 inputs; fp32
// accumulate in TMEM).
//
// DESIGN.md §7 bounds the tensor path's error with a model of how one MMA adds
// its K = 8 exact products to the accumulator.  This probe measures that model:
// every CTA runs one independent problem
//     D = C + sum_{m < nmma} A_m x B_m^T        (A_m, B_m: 128 x 8, C, D: 128 x 128)
// with C written into TMEM by tcgen05.st (any fp32 value, so the accumulator can
// be large, tiny or of opposite sign), the A_m in TMEM and the B_m in shared memory
// (the product kernel's operand placement), one MMA per m with accumulate = 1
// (or accumulate = 0 for the first one when c_mode == 0), and D read back with
// tcgen05.ld.  tools/tc_acc_probe/run.py generates adversarial inputs and compares
// D with the exact sums.  Not part of the product library.
#include <cstdio>
#include "../../paper_1810_11451_b200/csrc/bf_ffma.cuh"
#include "../../paper_1810_11451_b200/csrc/tc_ptx.cuh"

constexpr int kMaxMma = 32;

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// KIND 0: kind::tf32, K = 8 per MMA; KIND 1: kind::f16 with fp16 A/B, K = 16 per MMA (the
// host passes fp16-exact values as fp32; two per 32-bit word, even K element low).
template <int KIND>
__global__ void __launch_bounds__(128, 1)
acc_probe(const float *A, const float *B, const float *C, float *D, int nmma, int c_mode) {
    constexpr int KK = KIND ? 16 : 8;
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    extern __shared__ __align__(1024) float Bs[];   // nmma x [2 K-chunks][16][8][4]
    const int tid = threadIdx.x, warp = tid / 32;
    const int64_t p = blockIdx.x;
    const float *Ap = A + p * nmma * 128 * KK, *Bp = B + p * nmma * 128 * KK;
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    if (tid == 0) { bfk::mbar_init(&bar, 1); bfk::mbar_fence_init(); }
    for (int idx = tid; idx < nmma * 128 * 8; idx += 128) {   // one 32-bit word each
        const int m = idx / 1024, rem = idx % 1024, n = rem / 8, w = rem % 8;
        const int kc = w / 4, ng = n / 8, r = n % 8, e = w % 4;
        const float *src = Bp + (m * 128 + n) * KK;
        Bs[m * 1024 + ((kc * 16 + ng) * 8 + r) * 4 + e] =
            KIND ? __uint_as_float(pack_f16x2(src[2 * w], src[2 * w + 1])) : src[w];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t base = tmem_base;
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    // C -> D columns [0, 128) of this thread's lane (row tid)
    for (int c0 = 0; c0 < 128; c0 += 8) {
        uint32_t v[8];
        for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(C[p * 128 * 128 + tid * 128 + c0 + i]);
        tc::tmem_st8(base + lane_base + c0, v);
    }
    // A_m -> columns [256 + 8 m, 256 + 8 m + 8)
    for (int m = 0; m < nmma; ++m) {
        uint32_t v[8];
        const float *src = Ap + (m * 128 + tid) * KK;
        for (int i = 0; i < 8; ++i)
            v[i] = KIND ? pack_f16x2(src[2 * i], src[2 * i + 1]) : __float_as_uint(src[i]);
        tc::tmem_st8(base + lane_base + 256 + 8 * m, v);
    }
    tc::tmem_st_wait();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (tid == 0) {
        const uint32_t idesc = KIND ? (tc::idesc_bf16(128, 128) & ~((7u << 7) | (7u << 10)))
                                    : tc::idesc_tf32(128, 128);
        for (int m = 0; m < nmma; ++m) {
            const uint64_t desc = tc::smem_desc(tc::smem_u32(Bs + m * 1024), 16 * 128, 128);
            if (KIND)
                tc::mma_bf16_ts(base, base + 256 + 8 * m, desc, idesc, (c_mode != 0 || m > 0) ? 1u : 0u);
            else
                tc::mma_tf32_ts(base, base + 256 + 8 * m, desc, idesc, (c_mode != 0 || m > 0) ? 1u : 0u);
        }
        tc::mma_commit(&bar);
    }
    bfk::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    for (int c0 = 0; c0 < 128; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(base + lane_base + c0, v);
        tc::tmem_ld_wait();
        for (int i = 0; i < 16; ++i) D[p * 128 * 128 + tid * 128 + c0 + i] = __uint_as_float(v[i]);
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(base);
}

// A, B: [np][nmma][128][K] fp32 (tf32 or fp16-exact values; K = 8 or 16 by kind);
// C, D: [np][128][128].
extern "C" int acc_run_kind(const float *A, const float *B, const float *C, float *D, int np,
                            int nmma, int c_mode, int kind) {
    if (nmma < 1 || nmma > kMaxMma || np < 1) return -1;
    const int KK = kind ? 16 : 8;
    const size_t ab = (size_t)np * nmma * 128 * KK * 4, cd = (size_t)np * 128 * 128 * 4;
    float *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, ab); cudaMalloc(&dB, ab); cudaMalloc(&dC, cd); cudaMalloc(&dD, cd);
    cudaMemcpy(dA, A, ab, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, ab, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C, cd, cudaMemcpyHostToDevice);
    const int smem = nmma * 1024 * 4;
    if (kind) {
        cudaFuncSetAttribute(acc_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        acc_probe<1><<<np, 128, smem>>>(dA, dB, dC, dD, nmma, c_mode);
    } else {
        cudaFuncSetAttribute(acc_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        acc_probe<0><<<np, 128, smem>>>(dA, dB, dC, dD, nmma, c_mode);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("acc_probe: %s\n", cudaGetErrorString(e)); return (int)e; }
    cudaMemcpy(D, dD, cd, cudaMemcpyDeviceToHost);
    cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dD);
    return 0;
}

extern "C" int acc_run(const float *A, const float *B, const float *C, float *D, int np, int nmma,
                       int c_mode) {
    return acc_run_kind(A, B, C, D, np, nmma, c_mode, 0);
}
