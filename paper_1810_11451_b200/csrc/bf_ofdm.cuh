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

#ifndef BFO_CPA_UNROLL
#define BFO_CPA_UNROLL 4
#endif
constexpr int kCpaUnroll = BFO_CPA_UNROLL;   // the cp.async fetch loop: 4 batches the table loads (0.846 -> 0.860, profiles/r02_of1_unroll.jsonl)

struct OParams {
    const float2 *R;      // [n_sym nb][A][B] complex fp32
    float2 *y;            // [n_sym][A][cp + n] complex fp32 (or int16 pairs, OUT16)
    const float2 *tw;     // tw[m] = w^m, w = e^{-2 pi i / n} (bff::twiddle_kernel)
    int64_t n_sig;        // n_sym A
    int A, nb, B, half;   // half = nb B / 2
    int cp;
    float scale;          // OUT16: scale 2^e
};

// per CTA: NW warps x NBUF (exchange / input buffer + its mbarrier), the CTA's copy of the
// pass-2 twiddles (folded order)
// mbarrier region rounded up to 16 B: the twiddle table and the run table after it are read
// with 16-byte loads
__host__ __device__ constexpr int bar_bytes(int nbuf, int nw) { return (nw * nbuf * 8 + 15) / 16 * 16; }
__host__ __device__ constexpr int smem_bytes(int nbuf, int nw) {
    return nw * nbuf * kWarpPad * 8 + bar_bytes(nbuf, nw) + kN * 8 + 64 * 16;   // + run table
}

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

// NBUF buffers per warp, NW warps per CTA.  NBUF = 1 (4 warps, 2 CTAs per SM): the next
// signal's runs can be fetched only once the current transform's pass 2 has read the
// buffer (the exchange reuses it).  NBUF = 2 (6 warps, 1 CTA per SM, 216 KB of shared
// memory): signal j's input and exchange live in buffer j % 2, and signal j + 1's fetch is
// issued as soon as signal j's input is in registers — a whole signal of lead time, for 6
// warps per SM instead of 8.
// The same fetch with per-lane 16-byte cp.async (LDGSTS) instead of bulk copies: the bulk
// copies of 480 B are served one at a time per SM (~60 cycles each, i.e. 26 per signal
// about as long as the signal's whole compute: ncu shows the warps waiting on the fetch
// even with a second buffer and a whole signal of lead time).  Lane l moves chunk l of
// every run (30 chunks per 480-B run); the plan-constant run table (tab) is in shared
// memory and read as broadcasts; each lane's copies arrive on the warp's mbarrier
// (count 32) through cp.async.mbarrier.arrive.noinc.
// HALF > 0: the kernel is specialised for half = HALF (the loads skip the rows of 32 bins
// that are zero as a whole, so only the two partial rows at the band edges are zero-filled)
// CT (with HALF): the run table at compile time — measured faster for the int16 output
// (0.68 -> 0.81 of copy BW) and slower for fp32 output (0.86 -> 0.825,
// profiles/r02_of1_spec2.jsonl), so the kernel takes it for OUT16 only
template <int HALF = 0, bool CT = false>
__device__ __forceinline__ void fetch_symbol_cpa(c2 *buf, const OParams &p, int64_t sig, uint64_t *bar,
                                                 int l, const CopyDesc *tab, int n_copies) {
    const int half = HALF > 0 ? HALF : p.half;
    if (HALF > 0) {
        constexpr int e0 = (HALF + 31) / 32 * 32, b1 = (kN - HALF) / 32 * 32;   // partial rows
        constexpr int n0 = (e0 - HALF) / 2, n1 = (kN - HALF - b1) / 2;        // float4 counts
        if (l < n0) reinterpret_cast<float4 *>(buf + HALF)[l] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (l < n1) reinterpret_cast<float4 *>(buf + b1)[l] = make_float4(0.f, 0.f, 0.f, 0.f);
        static_assert(n0 <= 32 && n1 <= 32, "partial rows");
    } else {
        float4 *z = reinterpret_cast<float4 *>(buf + half);
        const int nz = (kN - 2 * half) / 2;
        for (int i = l; i < nz; i += 32) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const int64_t m = sig / p.A;
    const int a = (int)(sig - m * p.A);
    const float2 *src = p.R + ((m * p.nb) * (int64_t)p.A + a) * p.B + 2 * l;   // chunk l: 2 points
    const uint32_t dst0 = bfk::smem_addr(buf) + 16u * l;
    if (CT && HALF > 0) {
        // the run table at compile time (n_ant 64, b 60, nb = 2 HALF / 60 blocks, none
        // straddling the middle): one cp.async per run and lane, immediate offsets
        static_assert(HALF % 60 == 0, "specialisation for whole blocks per half");
        if (l < 30) {
#pragma unroll
            for (int c = 0; c < 2 * HALF / 60; ++c) {
                constexpr int kB = 60, kRun = 64 * 60;     // points per run, per block of R
                const int bin = c * kB >= HALF ? c * kB - HALF : c * kB + kN - HALF;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             ::"r"(dst0 + 8u * bin), "l"(src + (int64_t)c * kRun) : "memory");
            }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bfk::smem_addr(bar))
                     : "memory");
        return;
    }
#pragma unroll(kCpaUnroll)
    for (int c = 0; c < n_copies; ++c) {
        const CopyDesc d = tab[c];
        if (16u * l < d.bytes)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                         ::"r"(dst0 + 8u * d.dst), "l"(src + d.src_off) : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bfk::smem_addr(bar))
                 : "memory");
}

// the time samples of one output position: complex fp32, or (OUT16) int16 (re, im)
// fronthaul samples sat(rne(y 2^e)) — 2^e is folded into the scale (exact), cvt.rni.sat
// maps NaN to 0
template <bool OUT16>
__device__ __forceinline__ void store_sample(float2 *y, int64_t i, float2 v) {
    if (OUT16) {
        short a, b;
        asm("cvt.rni.sat.s16.f32 %0, %1;" : "=h"(a) : "f"(v.x));
        asm("cvt.rni.sat.s16.f32 %0, %1;" : "=h"(b) : "f"(v.y));
        __stcs(reinterpret_cast<unsigned int *>(y) + i, (uint32_t)(uint16_t)a | ((uint32_t)(uint16_t)b << 16));
    } else {
        __stcs(y + i, v);
    }
}

template <int NBUF, int NW, bool CPA = false, bool OUT16 = false, int HALF = 0>
__global__ void __launch_bounds__(NW * 32, NBUF == 1 ? 2 : 1) ofdm_ifft_kernel(const OParams p) {
    extern __shared__ __align__(128) unsigned char osm[];
    const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    c2 *bufs = reinterpret_cast<c2 *>(osm) + warp * NBUF * kWarpPad;
    uint64_t *bars = reinterpret_cast<uint64_t *>(osm + NW * NBUF * kWarpPad * 8) + warp * NBUF;
    float2 *tws = reinterpret_cast<float2 *>(osm + NW * NBUF * kWarpPad * 8 + bar_bytes(NBUF, NW));
    for (int i = threadIdx.x; i < kN; i += NW * 32)
        tws[i] = p.tw[(bff::tws_fold_r(i) * bff::tws_fold_j(i)) & (kN - 1)];   // w^(r j), folded order
    const int64_t gw = (int64_t)blockIdx.x * NW + warp, nw = (int64_t)gridDim.x * NW;
    if (l == 0) {
        for (int b = 0; b < NBUF; ++b) bfk::mbar_init(bars + b, CPA ? 32 : 1);
        bfk::mbar_fence_init();
    }
    __syncwarp();
    const CopyDesc d0 = copy_desc(p, l), d1 = copy_desc(p, l + 32);
    CopyDesc *tab = reinterpret_cast<CopyDesc *>(osm + NW * NBUF * kWarpPad * 8 + bar_bytes(NBUF, NW) + kN * 8);
    const int n_copies = p.nb + ((p.half % p.B) ? 1 : 0);
    if (CPA) {
        for (int c = threadIdx.x; c < 64; c += NW * 32) tab[c] = copy_desc(p, c);
        __syncthreads();
    }
    auto fetch = [&](c2 *b, int64_t sg, uint64_t *br) {
        if (CPA) fetch_symbol_cpa<HALF, OUT16>(b, p, sg, br, l, tab, n_copies);
        else fetch_symbol(b, p, sg, br, l, d0, d1);
    };
    if (gw < p.n_sig) fetch(bufs, gw, bars);
    __syncthreads();                                    // the twiddle table
    const int L = p.cp + kN, cp = p.cp;
    const c2 osc = bff::pk(p.scale, p.scale);
    uint32_t j = 0;                                     // this warp's signal counter
    for (int64_t sig = gw; sig < p.n_sig; sig += nw, ++j) {
        const int cur = NBUF == 1 ? 0 : (int)(j & 1);
        c2 *buf = bufs + cur * kWarpPad;
        c2 a[64];
        bfk::mbar_wait(bars + cur, NBUF == 1 ? (j & 1) : ((j >> 1) & 1));
        __syncwarp();                                   // the other lanes' zero-bin stores
#pragma unroll
        for (int s = 0; s < 64; ++s) {                  // X[bin], bin = l + 32 s
            if (HALF > 0 && 32 * s >= HALF && 32 * s + 31 < kN - HALF) a[s] = 0ull;   // zero row
            else a[s] = buf[l + 32 * s];
        }
        const int64_t nxt = sig + nw;
        if (NBUF == 2 && nxt < p.n_sig) {               // the other buffer: free since signal j - 1
            c2 *nbuf = bufs + (cur ^ 1) * kWarpPad;
            fetch(nbuf, nxt, bars + (cur ^ 1));
        }
        // x[t] = scale sum_bin X[bin] e^{+2 pi i bin t / n} = scale F[(n - t) mod n], F the
        // forward DFT of X: the inverse without conjugations, the time reversal in the stores
        bff::fft2048_warp_x<true, true>(a, buf, nullptr, tws, l, [&] {
            if (NBUF == 1 && nxt < p.n_sig) {
                __syncwarp();
                fetch(buf, nxt, bars);
            }
        });
        const int64_t dst = sig * L;                    // sample index of the signal's start
        const int64_t body = dst + cp + kN - l;         // F[k], k = l + 32 s -> t = n - k
#pragma unroll
        for (int s = 0; s < 64; ++s) {
            const float2 v = bff::up(bff::mul2(a[s], osc));
            if (s == 0) store_sample<OUT16>(p.y, l == 0 ? dst + cp : body, v);   // k = 0 -> t = 0
            else store_sample<OUT16>(p.y, body - 32 * s, v);
        }
        // cyclic prefix (O4): y[t'] = x[n - cp + t'] — t = n - k >= n - cp, i.e. 1 <= k <= cp
#pragma unroll
        for (int s = 0; s < 64; ++s) {
            if (32 * s > cp) break;                     // warp-uniform
            const int k = l + 32 * s;
            if (k >= 1 && k <= cp) store_sample<OUT16>(p.y, dst + (cp - k), bff::up(bff::mul2(a[s], osc)));
        }
    }
}

}  // namespace bfofdm
