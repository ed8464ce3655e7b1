// Write-bandwidth micro-benchmarks for the R stream (30,720-byte blocks):
// mode 0: warp STG.64 of 256 B rows (the tc epilogue pattern)
// mode 1: STG.128 (each warp writes 512 contiguous bytes per instruction)
// mode 2: TMA bulk store (cp.async.bulk.global.shared) of whole 30,720-B blocks
//         from a double-buffered shared staging area
// mode 3: cudaMemsetAsync
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(128) w_stg64(float2 *R, long long nblk) {
    const long long per = (nblk + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
    const int m = threadIdx.x;
    const int bsel = m >= 60, j = m - 60 * bsel;
    for (long long blk = b0; blk + 1 < b1; blk += 2) {
        if (m < 120) {
            float2 *Rb = R + (blk + bsel) * 3840;
#pragma unroll 8
            for (int a = 0; a < 64; ++a) __stcs(Rb + a * 60 + j, make_float2(a, j));
        }
    }
}

// 8 warps: two per RE quarter, each writing half of the antennas (STG.64)
__global__ void __launch_bounds__(256) w_stg64x2(float2 *R, long long nblk) {
    const long long per = (nblk + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
    const int m = threadIdx.x & 127, half = threadIdx.x >> 7;
    const int bsel = m >= 60, j = m - 60 * bsel;
    for (long long blk = b0; blk + 1 < b1; blk += 2) {
        if (m < 120) {
            float2 *Rb = R + (blk + bsel) * 3840;
#pragma unroll 8
            for (int a = half * 32; a < half * 32 + 32; ++a) __stcs(Rb + a * 60 + j, make_float2(a, j));
        }
    }
}

// 4 warps, lane pairs exchange so each lane stores 16 B (2 REs of one antenna)
__global__ void __launch_bounds__(128) w_stg128x(float4 *R, long long nblk) {
    const long long per = (nblk + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
    const int m = threadIdx.x;
    const int bsel = m >= 60, j = m - 60 * bsel;
    const int odd = j & 1;
    for (long long blk = b0; blk + 1 < b1; blk += 2) {
        float4 *Rb = R + (blk + bsel) * 1920;
#pragma unroll 4
        for (int a = 0; a < 64; a += 2) {
            float re0 = a + j, im0 = j, re1 = a + 1 + j, im1 = -j;
            float send_re = odd ? re0 : re1, send_im = odd ? im0 : im1;
            float got_re = __shfl_xor_sync(0xffffffffu, send_re, 1);
            float got_im = __shfl_xor_sync(0xffffffffu, send_im, 1);
            float4 v = odd ? make_float4(got_re, got_im, re1, im1) : make_float4(re0, im0, got_re, got_im);
            const int ant = a + odd, jj = j - odd;
            if (m < 120) __stcs(Rb + (ant * 60 + jj) / 2, v);
        }
    }
}

__global__ void __launch_bounds__(128) w_stg128(float4 *R, long long nblk) {
    const long long per = (nblk + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
    for (long long blk = b0; blk < b1; ++blk) {
        float4 *Rb = R + blk * 1920;
        for (int i = threadIdx.x; i < 1920; i += 128) __stcs(Rb + i, make_float4(i, 1, 2, 3));
    }
}

__global__ void __launch_bounds__(128) w_bulk(float *R, long long nblk) {
    extern __shared__ __align__(128) float st[];   // 2 x 7680 floats
    const long long per = (nblk + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
    int buf = 0;
    for (long long blk = b0; blk < b1; ++blk) {
        float *S = st + buf * 7680;
        if (threadIdx.x == 0 && blk - b0 >= 2)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        for (int i = threadIdx.x; i < 7680; i += 128) S[i] = (float)i;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(R + blk * 7680), "r"((uint32_t)__cvta_generic_to_shared(S)), "r"(30720) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        buf ^= 1;
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// NW warps per CTA, each lane storing VEC floats (4: STG.128, 8: STG.256) per instruction,
// consecutive lanes consecutive addresses: the widest-store ceiling of the R stream.
// order 0: contiguous block range per CTA; 1: grid-stride; 2: pseudo-random block order
template <int VEC>
__global__ void w_vec(float *R, long long nblk, int order) {
    const long long per = (nblk + gridDim.x - 1) / gridDim.x;
    const long long b0 = blockIdx.x * per, b1 = min(nblk, b0 + per);
    for (long long it = b0; it < b1; ++it) {
        long long blk = it;
        if (order == 1) blk = (it - b0) * gridDim.x + blockIdx.x;
        if (order == 2) blk = (it * 2654435761LL + 12345) % nblk;   // nblk a power of two: bijective
        if (blk >= nblk) continue;
        float *Rb = R + blk * 7680;
        for (int i = threadIdx.x * VEC; i < 7680; i += blockDim.x * VEC) {
            const float x = (float)i;
            if (VEC == 8)
                asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};"
                             :: "l"(Rb + i), "f"(x) : "memory");
            else
                __stcs(reinterpret_cast<float4 *>(Rb + i), make_float4(x, x, x, x));
        }
    }
}

extern "C" int wbw_vec(int vec, int warps, int order, void *R, long long nblk, int reps, float *ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = -1; rep < reps; ++rep) {
        if (rep == 0) cudaEventRecord(a);
        if (vec == 8) w_vec<8><<<sms, 32 * warps>>>((float *)R, nblk, order);
        else w_vec<4><<<sms, 32 * warps>>>((float *)R, nblk, order);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms / reps;
    return (int)cudaGetLastError();
}

extern "C" int wbw_run(int mode, void *R, long long nblk, int ctas_per_sm, int reps, float *ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * ctas_per_sm;
    cudaFuncSetAttribute(w_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 30720);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = -1; rep < reps; ++rep) {
        if (rep == 0) cudaEventRecord(a);
        if (mode == 0) w_stg64<<<grid, 128>>>((float2 *)R, nblk);
        else if (mode == 1) w_stg128<<<grid, 128>>>((float4 *)R, nblk);
        else if (mode == 2) w_bulk<<<grid, 128, 2 * 30720>>>((float *)R, nblk);
        else if (mode == 4) w_stg64x2<<<grid, 256>>>((float2 *)R, nblk);
        else if (mode == 5) w_stg128x<<<grid, 128>>>((float4 *)R, nblk);
        else if (mode == 3) cudaMemsetAsync(R, 0, (size_t)nblk * 30720);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    *ms_out = ms / reps;
    return (int)cudaGetLastError();
}
