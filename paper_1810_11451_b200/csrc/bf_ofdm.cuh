// bf_ofdm.cuh — OFDM output stage of the beamformer: per (symbol, antenna) the unnormalised
// inverse DFT of the beamformed subcarriers, n = 2048, plus the cyclic prefix (SURVEY.md §8(f)
// row 4, "fuse the per-antenna OFDM IFFT"; the pipeline stages of PAPER.md:41, 49 (§II) and
// the IFFT of PAPER.md:67-71 (§III); readings O1-O5 in DESIGN.md §2).
//
// Input: R of the beamforming stage, interleaved complex fp32 [blk][A][B] (bf.h layout 0);
// symbol m is the nb blocks m nb .. m nb + nb - 1, its Nsc = nb B subcarriers q = 0 .. Nsc - 1
// are (block q / B, element q % B), subcarrier q sits in IDFT bin (q - Nsc/2) mod n (O2).
// Output: y [n_sym][A][cp + n], x[t] = scale sum_bin X[bin] e^{+2 pi i bin t / n} (O3),
// y[t'] = x[n - cp + t'] for t' < cp, y[cp + t] = x[t] (O4).
//
// One warp per signal (symbol, antenna), the filter's warp transform (bf_filter_warp.cuh:
// radix 64 then radix 32 with one warp-local exchange, packed fp32x2, twiddles folded into
// the butterflies): the inverse as conj(FFT(conj(X))).  The nb runs of B subcarriers of a
// signal (480 contiguous bytes each in R) arrive in the warp's buffer in subcarrier order by
// nb bulk copies on the warp's mbarrier, issued for the NEXT signal as soon as the current
// transform's last pass has read the buffer; the bin mapping (zeros between the two halves)
// is applied when the lanes load their 64 points.  Outputs stream from registers, the last
// cp samples stored twice (prefix and body).  HBM bytes per signal: 8 Nsc read + 8 (cp + n)
// written (DESIGN.md §10 row 4).
#pragma once
#include "bf_filter_warp.cuh"

namespace bfofdm {

using bff::c2;
using bff::kN;
using bff::kWarpPad;

struct OParams {
    const float2 *R;      // [n_sym nb][A][B] complex fp32
    float2 *y;            // [n_sym][A][cp + n]
    const float2 *tw;     // tw[m] = w^m, w = e^{-2 pi i / n} (bff::twiddle_kernel)
    int64_t n_sig;        // n_sym A
    int A, nb, B, half;   // half = nb B / 2
    int cp;
    float scale;
};

constexpr int kThreads = 128;   // 4 warps, one signal each at a time
// exchange buffers, their mbarriers, the CTA's copy of the pass-2 twiddles (folded order)
__host__ __device__ constexpr int smem_bytes() { return 4 * kWarpPad * 8 + 4 * 8 + kN * 8; }

// the nb runs of signal sig -> buf[0, nb B) (subcarrier order), completion on bar.  Called by
// every lane of the warp after the buffer's last generic reads (__syncwarp before).
__device__ __forceinline__ void fetch_symbol(c2 *buf, const OParams &p, int64_t sig, uint64_t *bar,
                                             int l) {
    const int64_t m = sig / p.A;
    const int a = (int)(sig - m * p.A);
    const uint32_t rb = (uint32_t)p.B * 8;
    if (l == 0) bfk::mbar_arrive_expect_tx(bar, rb * (uint32_t)p.nb);
    __syncwarp();
    const float2 *src = p.R + ((m * p.nb) * (int64_t)p.A + a) * p.B;
    const int64_t blk_stride = (int64_t)p.A * p.B;
    const uint64_t pol = bfk::policy_evict_first();     // R's last use
    for (int i = l; i < p.nb; i += 32) {
        bfk::fence_proxy_async_smem();                   // generic reads before the async write
        bfk::bulk_g2s(buf + i * p.B, src + i * blk_stride, rb, bar, pol);
    }
}

__device__ __forceinline__ c2 conj_xor(float2 v) {
    uint32_t im;   // sign flip on the integer pipe (the transforms keep the FMA pipe busy)
    asm("xor.b32 %0, %1, 0x80000000;" : "=r"(im) : "r"(__float_as_uint(v.y)));
    return bff::pk(v.x, __uint_as_float(im));
}

__global__ void __launch_bounds__(kThreads, 2) ofdm_ifft_kernel(const OParams p) {
    extern __shared__ __align__(128) unsigned char osm[];
    const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    c2 *buf = reinterpret_cast<c2 *>(osm) + warp * kWarpPad;
    uint64_t *bar = reinterpret_cast<uint64_t *>(osm + 4 * kWarpPad * 8) + warp;
    float2 *tws = reinterpret_cast<float2 *>(osm + 4 * kWarpPad * 8 + 4 * 8);   // folded order
    for (int i = threadIdx.x; i < kN; i += kThreads)
        tws[i] = p.tw[(bff::tws_fold_r(i) * bff::tws_fold_j(i)) & (kN - 1)];   // w^(r j)
    const int64_t gw = (int64_t)blockIdx.x * 4 + warp, nw = (int64_t)gridDim.x * 4;
    if (l == 0) {
        bfk::mbar_init(bar, 1);
        bfk::mbar_fence_init();
    }
    __syncwarp();
    if (gw < p.n_sig) fetch_symbol(buf, p, gw, bar, l);
    __syncthreads();                                    // the twiddle table
    const int half = p.half, nh = kN - p.half, L = p.cp + kN, tcp = kN - p.cp;
    const c2 osc = bff::pk(p.scale, -p.scale);          // output conj and scale in one FMUL2
    uint32_t phase = 0;
    for (int64_t sig = gw; sig < p.n_sig; sig += nw) {
        c2 a[64];
        bfk::mbar_wait(bar, phase);
        phase ^= 1u;
        // bin l + 32 s: subcarrier bin + Nsc/2 (bins 0 .. half - 1), bin - (n - half) (the
        // negative half), zero between (O2); conj for the inverse
#pragma unroll
        for (int s = 0; s < 64; ++s) {
            const int bin = l + 32 * s;
            const int q = bin < half ? bin + half : bin - nh;
            c2 x = 0ull;
            if (bin < half || bin >= nh) x = conj_xor(bff::up(buf[q]));   // predicated load
            a[s] = x;
        }
        const int64_t nxt = sig + nw;
        bff::fft2048_warp_x<true, true>(a, buf, nullptr, tws, l, [&] {
            if (nxt < p.n_sig) {
                __syncwarp();
                fetch_symbol(buf, p, nxt, bar, l);
            }
        });
        float2 *dst = p.y + sig * L;
#pragma unroll
        for (int s = 0; s < 64; ++s) {
            const int t = l + 32 * s;
            const float2 v = bff::up(bff::mul2(a[s], osc));
            __stcs(dst + p.cp + t, v);
            if (t >= tcp) __stcs(dst + (t - tcp), v);     // cyclic prefix (O4)
        }
    }
}

}  // namespace bfofdm
