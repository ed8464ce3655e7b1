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
// the butterflies), the inverse as a forward transform read back in reversed time order.
// The nb runs of B subcarriers of a signal (480 contiguous bytes each in R) arrive in the
// warp's buffer in BIN order by bulk copies on the warp's mbarrier (the zero bins written
// by the lanes), issued for the NEXT signal as soon as the current transform's last pass
// has read the buffer.  Outputs stream from registers, the last cp samples stored twice
// (prefix and body).  HBM bytes per signal: 8 Nsc read + 8 (cp + n)
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

// One bulk copy of a signal's fetch: a run of subcarriers of one block -> its bins (O2).
// The runs of blocks at or above the middle go to bins 0, 1, ..., those below to bins
// n - half, ...; a block straddling the middle (nb odd) is two copies (30 REs = 240 B each).
// Plan-constant per copy index c < n_copies; a lane keeps the descriptors of copies l and
// l + 32 in registers, so a fetch is one 64-bit add and one copy per lane.
struct CopyDesc {
    int64_t src_off;    // float2 offset from the signal's first run
    uint32_t dst;       // bin of the first element
    uint32_t bytes;     // 0: no copy
};
__device__ __forceinline__ CopyDesc copy_desc(const OParams &p, int c) {
    const int half = p.half, B = p.B;
    const int straddle = (half % B) ? half / B : -1;
    const int n_copies = p.nb + (straddle >= 0 ? 1 : 0);
    CopyDesc d{0, 0, 0};
    if (c >= n_copies) return d;
    const int i = (straddle >= 0 && c > straddle) ? c - 1 : c;
    const int part = (straddle >= 0 && c == straddle + 1) ? 1 : 0;
    const int q0 = i * B, q1 = q0 + B;
    d.src_off = (int64_t)i * p.A * B;
    if (q1 <= half) {
        d.dst = q0 + kN - half;
        d.bytes = B * 8;
    } else if (q0 >= half) {
        d.dst = q0 - half;
        d.bytes = B * 8;
    } else if (part == 0) {
        d.dst = q0 + kN - half;
        d.bytes = (half - q0) * 8;
    } else {
        d.dst = 0;
        d.src_off += half - q0;
        d.bytes = (q1 - half) * 8;
    }
    return d;
}

// the subcarriers of signal sig -> buf in bin order, completion on bar; the zero bins
// [half, n - half) written with generic stores.  Called by every lane after the buffer's
// last generic reads (__syncwarp before).
__device__ __forceinline__ void fetch_symbol(c2 *buf, const OParams &p, int64_t sig, uint64_t *bar,
                                             int l, const CopyDesc &d0, const CopyDesc &d1) {
    const int half = p.half;
    float4 *z = reinterpret_cast<float4 *>(buf + half);
    const int nz = (kN - 2 * half) / 2;
    for (int i = l; i < nz; i += 32) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t m = sig / p.A;
    const int a = (int)(sig - m * p.A);
    const float2 *src = p.R + ((m * p.nb) * (int64_t)p.A + a) * p.B;
    if (l == 0) bfk::mbar_arrive_expect_tx(bar, (uint32_t)(2 * half) * 8u);
    __syncwarp();
    const uint64_t pol = bfk::policy_evict_first();                     // R's last use
    if (d0.bytes) {
        bfk::fence_proxy_async_smem();                                  // generic reads first
        bfk::bulk_g2s(buf + d0.dst, src + d0.src_off, d0.bytes, bar, pol);
    }
    if (d1.bytes) bfk::bulk_g2s(buf + d1.dst, src + d1.src_off, d1.bytes, bar, pol);
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
    const CopyDesc d0 = copy_desc(p, l), d1 = copy_desc(p, l + 32);
    if (gw < p.n_sig) fetch_symbol(buf, p, gw, bar, l, d0, d1);
    __syncthreads();                                    // the twiddle table
    const int L = p.cp + kN, cp = p.cp;
    const c2 osc = bff::pk(p.scale, p.scale);
    uint32_t phase = 0;
    for (int64_t sig = gw; sig < p.n_sig; sig += nw) {
        c2 a[64];
        bfk::mbar_wait(bar, phase);
        phase ^= 1u;
        __syncwarp();                                   // the other lanes' zero-bin stores
#pragma unroll
        for (int s = 0; s < 64; ++s) a[s] = buf[l + 32 * s];              // X[bin], bin = l + 32 s
        const int64_t nxt = sig + nw;
        // x[t] = scale sum_bin X[bin] e^{+2 pi i bin t / n} = scale F[(n - t) mod n], F the
        // forward DFT of X: the inverse without conjugations, the time reversal in the stores
        bff::fft2048_warp_x<true, true>(a, buf, nullptr, tws, l, [&] {
            if (nxt < p.n_sig) {
                __syncwarp();
                fetch_symbol(buf, p, nxt, bar, l, d0, d1);
            }
        });
        float2 *dst = p.y + sig * L;
        float2 *body = dst + cp + kN - l;               // F[k], k = l + 32 s -> t = n - k
#pragma unroll
        for (int s = 0; s < 64; ++s) {
            const float2 v = bff::up(bff::mul2(a[s], osc));
            if (s == 0) __stcs(l == 0 ? dst + cp : body, v);             // k = 0 -> t = 0
            else __stcs(body - 32 * s, v);
        }
        // cyclic prefix (O4): y[t'] = x[n - cp + t'] — t = n - k >= n - cp, i.e. 1 <= k <= cp
#pragma unroll
        for (int s = 0; s < 64; ++s) {
            if (32 * s > cp) break;                     // warp-uniform
            const int k = l + 32 * s;
            if (k >= 1 && k <= cp) __stcs(dst + (cp - k), bff::up(bff::mul2(a[s], osc)));
        }
    }
}

}  // namespace bfofdm
