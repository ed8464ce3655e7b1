// bf_ffma.cuh — sm_100a CUDA-core beamforming kernel (hot path a4 + a5 + a7).
//
// Computes, for a stream of blocks, R[n] = W[g(n)] x S[n] with W 64 x F and
// S F x 60 complex fp32 (§III).
//
// Design:
//  * Persistent CTAs of 96 threads (3 warps), ~4 resident per SM, each owning
//    a contiguous range of the (group-sorted) block list, so W changes at most
//    a few times per CTA.
//  * W of the current group lives in shared memory, pre-laid-out by
//    bf_set_precoders as Wp[k][j][ag] float4 = (re w[8ag+2j][k], re w[8ag+2j+1][k],
//    im w[8ag+2j][k], im w[8ag+2j+1][k]), 512*F bytes, loaded with one
//    cp.async.bulk (TMA bulk copy) per group change.
//  * S blocks (480*F contiguous bytes, either layout) stream HBM -> shared
//    through a 2-stage ring filled by cp.async.bulk with mbarrier completion,
//    two blocks ahead of compute.
//  * Each thread owns an 8-antenna x 5-RE register tile (80 fp32 accumulators):
//    antennas 8ag..8ag+7, REs rg, rg+12, .., rg+48 (ag = t/12, rg = t%12).  Per
//    k it reads 4 LDS.128 of W (conflict-free, broadcast across rg) and 5 S
//    values, and issues 160 FFMA: re = fma(wr,sr,re); im = fma(wi,sr,im) for all
//    8 antennas per S value, then re = fma(-wi,si,re); im = fma(wr,si,im).  The
//    order keeps one S operand in the reuse cache for runs of 16 FFMAs, so only
//    W and the accumulator are read from the register file (register-bank
//    conflicts were the top issue stall, see profiles/).  The paper's three fixes carry
//    over: no extra FLOPs, every product fused, no permutes (re/im sit in
//    separate registers).  Accumulators start at +0.0f (bit-exact identity).
//  * Results: for F <= 12 (where this kernel is AUTO's choice and R is 95-99 % of the
//    bytes) the block's R is staged in shared memory in its global layout and written
//    by one 30 720 B bulk store; for larger F straight from registers to HBM with
//    streaming 32-bit stores.  Both use 32-bit stores of re and im separately, so no
//    even/odd pairing constrains the accumulators.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace bfk {

constexpr int kAnt = 64;          // antennas (rows of W)
constexpr int kB = 60;            // resource elements (cols of S)
constexpr int kMaxF = 36;         // flows
constexpr int kThreads = 96;      // 8 antenna groups x 12 RE groups
constexpr int kTA = 8;            // antennas per thread
constexpr int kTR = 5;            // REs per thread
constexpr int kRG = 12;           // RE groups
constexpr int kAG = 8;            // antenna groups
constexpr int kRBlockFloats = 2 * kAnt * kB;   // 7680 floats = 30,720 B per block

// I/O formats (the kernels' LAYOUT parameter; include/bf.h bf_layout):
//   0 interleaved complex fp32 S/W/R;  1 planar complex fp32 S/W/R;
//   2 interleaved fp32 S/W, R as interleaved fp16 (re, im) pairs (SURVEY.md §8(f)
//     row 4: halves the dominant R stream; R rounded once, RN, from fp32);
//   3 interleaved fp32 S/W, R as interleaved int16 (re, im) fronthaul samples:
//     round-to-nearest-even of R x 2^e, saturated to [-32768, 32767] (NaN -> 0).
__host__ __device__ constexpr bool r_is_16bit(int layout) { return layout == 2 || layout == 3; }
__host__ __device__ constexpr int r_block_bytes(int layout) { return r_is_16bit(layout) ? 15360 : 30720; }
__device__ __forceinline__ uint32_t pack_half2(float re, float im) {
    const __half2 h = __floats2half2_rn(re, im);
    return *reinterpret_cast<const uint32_t *>(&h);
}
// (sat_rne_s16(re * scale), sat_rne_s16(im * scale)), re in the low half; NaN -> 0.
// (A clamp + 1.5 x 2^23 magic-add version measured slower in the tensor epilogue.)
__device__ __forceinline__ uint32_t pack_i16x2(float re, float im, float scale) {
    short a, b;
    asm("cvt.rni.sat.s16.f32 %0, %1;" : "=h"(a) : "f"(re * scale));
    asm("cvt.rni.sat.s16.f32 %0, %1;" : "=h"(b) : "f"(im * scale));
    return (uint32_t)(uint16_t)a | ((uint32_t)(uint16_t)b << 16);
}

struct KParams {
    const float4 *Wp;         // [n_groups][F][32] float4 (plan-owned relayout)
    const float *S;           // [n_blocks] x 2*F*60 floats
    const int32_t *perm;      // [n_items] block ids (group-sorted) or NULL = identity
    const int32_t *offsets;   // [n_groups + 2] group starts of the sorted order, or NULL = group 0
    float *R;                 // [n_blocks] x 7680 floats (16-bit layouts: x 3840 words)
    int64_t n_items;
    int n_groups;
    float out_scale;          // layout 3: 2^e applied before the int16 rounding
};

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    // (a suspend-time hint on try_wait measured no different: tools/sustained_exp.py)
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(smem_addr(bar)), "r"(parity) : "memory");
    } while (!done);
}
// TMA bulk copy global -> shared (no tensor map), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
// Bulk store shared -> global (bulk-group completion), and the waits for its source
// reads / full completion.
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes, uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 ::"l"(dst), "r"(smem_addr(src)), "r"(bytes), "l"(policy) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <int F>
struct Smem {
    static constexpr int kWBytes = 512 * F;            // F x 64 complex
    static constexpr int kSBytes = 480 * F;            // F x 60 complex
    static constexpr int kSFloats = 120 * F;
    static constexpr int kStages = 2;
    static constexpr int kOffS = kWBytes;
    static constexpr int kOffBar = kOffS + kStages * kSBytes;     // multiple of 16
    static constexpr int kOffMeta = kOffBar + 4 * 8;
    // Small f (the AUTO region of this kernel): the block's R is staged in shared
    // memory in its global layout and leaves as ONE bulk store (30 720 B, full lines),
    // instead of 80 scattered 32-bit stores per thread; 4 CTAs per SM still fit.
    static constexpr bool kStageR = F <= 12;
    static constexpr int kOffR = (kOffMeta + 4 * 8 + 127) / 128 * 128;
    static constexpr int kBytes = kStageR ? kOffR + kRBlockFloats * 4 : kOffMeta + 4 * 8;
};

template <int F, int LAYOUT>
__global__ void __launch_bounds__(kThreads, 4) bf_ffma_kernel(const KParams p) {
    using L = Smem<F>;
    extern __shared__ __align__(128) unsigned char smem[];
    const float4 *Ws = reinterpret_cast<const float4 *>(smem);
    float *Ss = reinterpret_cast<float *>(smem + L::kOffS);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::kOffBar);   // full[0..1], w
    int64_t *meta_blk = reinterpret_cast<int64_t *>(smem + L::kOffMeta);  // [2]
    int32_t *meta_grp = reinterpret_cast<int32_t *>(smem + L::kOffMeta + 16);  // [2]

    const int t = threadIdx.x;
    const int ag = t / kRG;
    const int rg = t - ag * kRG;
    const int64_t n = p.n_items;
    const int64_t begin = n * blockIdx.x / gridDim.x;
    const int64_t end = n * (blockIdx.x + 1) / gridDim.x;
    if (begin >= end) return;

    uint64_t pol_stream = 0, pol_keep = 0;
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], 1);
        mbar_fence_init();
        pol_stream = policy_evict_first();
        pol_keep = policy_evict_last();
    }
    __syncthreads();

    // group of an item: walk the routing offsets (items are visited in increasing
    // order, so the walk is amortised O(1)); items past offsets[G] are invalid.
    // The walk starts at begin's group, found by binary search (first g with
    // offsets[g + 1] > begin), so a CTA late in the list does not chase G
    // dependent global loads before its first block.
    int gi = 0;
    if (p.offsets && t == 0) {
        int lo = 0, hi = p.n_groups;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(p.offsets + mid + 1) > begin) hi = mid; else lo = mid + 1;
        }
        gi = lo;
    }
    auto group_of = [&](int64_t item) -> int32_t {
        if (!p.offsets) return 0;
        while (gi < p.n_groups && item >= __ldg(p.offsets + gi + 1)) ++gi;
        return gi;   // == n_groups for invalid tags
    };
    auto issue = [&](int stage, int64_t item) {   // thread 0 only
        const int64_t blk = p.perm ? (int64_t)__ldg(p.perm + item) : item;
        const int32_t g = group_of(item);
        meta_blk[stage] = blk;
        meta_grp[stage] = g;
        mbar_arrive_expect_tx(&bars[stage], L::kSBytes);
        bulk_g2s(Ss + stage * L::kSFloats, p.S + blk * L::kSFloats, L::kSBytes, &bars[stage],
                 pol_stream);
    };
    if (t == 0) {
        issue(0, begin);
        if (begin + 1 < end) issue(1, begin + 1);
    }

    int cur_g = -1;
    uint32_t wphase = 0;
    for (int64_t item = begin, it = 0; item < end; ++item, ++it) {
        const int stage = static_cast<int>(it & 1);
        mbar_wait(&bars[stage], static_cast<uint32_t>((it >> 1) & 1));
        const int64_t blk = meta_blk[stage];
        const int g = meta_grp[stage];
        const bool valid = (unsigned)g < (unsigned)p.n_groups;
        if (valid && g != cur_g) {            // CTA-uniform: reload W of the new group
            if (t == 0) {
                mbar_arrive_expect_tx(&bars[2], L::kWBytes);
                bulk_g2s(const_cast<float4 *>(Ws), p.Wp + (int64_t)g * F * 32, L::kWBytes,
                         &bars[2], pol_keep);
            }
            mbar_wait(&bars[2], wphase);
            wphase ^= 1u;
            cur_g = g;
        }

        float are[kTA][kTR], aim[kTA][kTR];
#pragma unroll
        for (int a = 0; a < kTA; ++a)
#pragma unroll
            for (int r = 0; r < kTR; ++r) { are[a][r] = +0.0f; aim[a][r] = +0.0f; }

        const float *S = Ss + stage * L::kSFloats;
        if (valid) {
#pragma unroll 2
            for (int k = 0; k < F; ++k) {
                float4 w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) w[j] = Ws[k * 32 + j * 8 + ag];
                float sr[kTR], si[kTR];
#pragma unroll
                for (int r = 0; r < kTR; ++r) {
                    if (LAYOUT != 1) {
                        const float2 v =
                            reinterpret_cast<const float2 *>(S)[k * kB + rg + kRG * r];
                        sr[r] = v.x;
                        si[r] = v.y;
                    } else {
                        sr[r] = S[k * kB + rg + kRG * r];
                        si[r] = S[F * kB + k * kB + rg + kRG * r];
                    }
                }
                // w[j] = (wr[2j], wr[2j+1], wi[2j], wi[2j+1]): wr[a] and wi[a] land in
                // registers of the same parity, so with the S operand held in the
                // reuse cache across a run of 16 FFMAs the two uncached operands
                // (W and the accumulator) can sit in different register banks.
                float wr[kTA], wi[kTA];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    wr[2 * j] = w[j].x; wr[2 * j + 1] = w[j].y;
                    wi[2 * j] = w[j].z; wi[2 * j + 1] = w[j].w;
                }
#pragma unroll
                for (int r = 0; r < kTR; ++r)
#pragma unroll
                    for (int a = 0; a < kTA; ++a) {
                        are[a][r] = fmaf(wr[a], sr[r], are[a][r]);
                        aim[a][r] = fmaf(wi[a], sr[r], aim[a][r]);
                    }
#pragma unroll
                for (int r = 0; r < kTR; ++r)
#pragma unroll
                    for (int a = 0; a < kTA; ++a) {
                        are[a][r] = fmaf(-wi[a], si[r], are[a][r]);
                        aim[a][r] = fmaf(wr[a], si[r], aim[a][r]);
                    }
            }
        }
        // staged R: the previous block's bulk store must have read the staging buffer
        if (L::kStageR && t == 0) bulk_wait_read();
        __syncthreads();                       // stage `stage` and meta are free again
        if (t == 0 && item + 2 < end) issue(stage, item + 2);

        if (valid) {
            float *Rb = p.R + blk * (r_block_bytes(LAYOUT) / 4);
            float *Rd = L::kStageR ? reinterpret_cast<float *>(smem + L::kOffR) : Rb;
            // staged: plain shared-memory stores; direct: streaming global stores
            auto st32 = [&](float *a, uint32_t v) {
                if (L::kStageR) *reinterpret_cast<uint32_t *>(a) = v;
                else __stcs(reinterpret_cast<unsigned int *>(a), v);
            };
#pragma unroll
            for (int a = 0; a < kTA; ++a) {
                const int i = ag * kTA + a;
#pragma unroll
                for (int r = 0; r < kTR; ++r) {
                    const int j = rg + kRG * r;
                    if (LAYOUT == 0) {
                        // two 32-bit stores instead of one float2: a 64-bit store would
                        // pin (re, im) to an even/odd register pair for the whole k loop,
                        // which forces register-bank conflicts in half of the FFMAs.
                        st32(Rd + 2 * (i * kB + j), __float_as_uint(are[a][r]));
                        st32(Rd + 2 * (i * kB + j) + 1, __float_as_uint(aim[a][r]));
                    } else if (LAYOUT == 2) {
                        st32(Rd + i * kB + j, pack_half2(are[a][r], aim[a][r]));
                    } else if (LAYOUT == 3) {
                        st32(Rd + i * kB + j, pack_i16x2(are[a][r], aim[a][r], p.out_scale));
                    } else {
                        st32(Rd + i * kB + j, __float_as_uint(are[a][r]));
                        st32(Rd + kAnt * kB + i * kB + j, __float_as_uint(aim[a][r]));
                    }
                }
            }
            if (L::kStageR) {
                fence_proxy_async_smem();      // this thread's writes -> the bulk copy
                __syncthreads();
                if (t == 0) bulk_s2g(Rb, Rd, (uint32_t)r_block_bytes(LAYOUT), pol_stream);
            }
        }
    }
    if (L::kStageR && t == 0) bulk_wait_all();
}

}  // namespace bfk
