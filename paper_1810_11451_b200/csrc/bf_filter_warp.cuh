// bf_filter_warp.cuh — warp-per-signal variant of the fused filter y = IFFT(H . FFT(s)),
// n = 2048 (§III), packed fp32x2 arithmetic.
//
// The CTA kernel (bf_filter.cuh) spends its time moving data through shared memory: two
// cross-warp exchanges per transform (16 KB written and read each) plus the input stage,
// about 144 KB of shared traffic per signal against 32 KB of HBM traffic.  Here one warp
// owns one signal and every lane 64 of its points, so a transform is two passes with ONE
// exchange (warp-local: __syncwarp, no CTA barrier):
//   pass 1: radix 64 — lane l transforms x[l + 32 r], r < 64 (8 x 8, constant twiddles)
//           and writes y[64 l + r'] to the warp's shared buffer;
//   pass 2: radix 32 — lane l transforms the columns j = l and l + 32: y[j + 64 r], r < 32,
//           times w^(r j), giving X[j + 64 r'] — i.e. lane l ends holding X[l + 32 s] for
//           s < 64, exactly the input order of pass 1, so MULT by H and the inverse
//           transform (conj(FFT(conj(.))) / N) continue from registers.
// A signal's input arrives in the warp's buffer by a TMA bulk copy issued as soon as the
// previous signal's last pass has read the buffer (it overlaps that pass's arithmetic and
// stores); outputs go straight to HBM (64 coalesced 8-byte stores per lane).  Shared
// traffic: 80 KB per signal (16 KB input + one 16 KB exchange written and read per
// transform), against 144 KB in the CTA kernel.
// 128 threads per CTA (4 independent warps).  Default variant (MINC = 2): 255 registers,
// 2 CTAs per SM, and room in shared memory for the CTA's copies of the pass-2 twiddles
// w^(r j) and of H — no twiddle products, no L1 table loads (fl1: 0.79 of HBM vs 0.69
// for the 3-CTA variant that forms twiddles from binary powers and reads H through L1).
#pragma once
#include "bf_filter.cuh"

namespace bff {

// per-warp exchange slots: one pad per 64 (pass 1's row stores and pass 2's column reads
// both conflict-free).  Pairing the row stores as STS.128 (two pads per 64) measured 0.6 %
// slower (profiles/r02_filter_fold.txt).
constexpr int kWarpPad = kN + kN / 64;
__device__ __forceinline__ int wpad(int i) { return i + (i >> 6); }
// 4 warps per CTA: exchange buffers, their mbarriers, and (TAB variant) the CTA's copies
// of the pass-2 twiddles w^(r j) (r < 32, j < 64) and of H
__host__ __device__ constexpr int warp_smem_bytes(bool tab) {
    return 4 * kWarpPad * 8 + 4 * 8 + (tab ? 2 * kN * 8 : 0);
}

// W64^m = cos(2 pi m / 64) - i sin(2 pi m / 64), fp32 (rounded once from fp64)
__device__ constexpr float2 kW64[64] = {
    {1.0f, -0.0f}, {0.9951847195625305f, -0.0980171412229538f}, {0.9807852506637573f, -0.19509032368659973f}, {0.9569403529167175f, -0.290284663438797f},
    {0.9238795042037964f, -0.3826834261417389f}, {0.8819212913513184f, -0.4713967442512512f}, {0.8314695954322815f, -0.5555702447891235f}, {0.7730104327201843f, -0.6343932747840881f},
    {0.7071067690849304f, -0.7071067690849304f}, {0.6343932747840881f, -0.7730104327201843f}, {0.5555702447891235f, -0.8314695954322815f}, {0.4713967442512512f, -0.8819212913513184f},
    {0.3826834261417389f, -0.9238795042037964f}, {0.290284663438797f, -0.9569403529167175f}, {0.19509032368659973f, -0.9807852506637573f}, {0.0980171412229538f, -0.9951847195625305f},
    {6.123234262925839e-17f, -1.0f}, {-0.0980171412229538f, -0.9951847195625305f}, {-0.19509032368659973f, -0.9807852506637573f}, {-0.290284663438797f, -0.9569403529167175f},
    {-0.3826834261417389f, -0.9238795042037964f}, {-0.4713967442512512f, -0.8819212913513184f}, {-0.5555702447891235f, -0.8314695954322815f}, {-0.6343932747840881f, -0.7730104327201843f},
    {-0.7071067690849304f, -0.7071067690849304f}, {-0.7730104327201843f, -0.6343932747840881f}, {-0.8314695954322815f, -0.5555702447891235f}, {-0.8819212913513184f, -0.4713967442512512f},
    {-0.9238795042037964f, -0.3826834261417389f}, {-0.9569403529167175f, -0.290284663438797f}, {-0.9807852506637573f, -0.19509032368659973f}, {-0.9951847195625305f, -0.0980171412229538f},
    {-1.0f, -1.2246468525851679e-16f}, {-0.9951847195625305f, 0.0980171412229538f}, {-0.9807852506637573f, 0.19509032368659973f}, {-0.9569403529167175f, 0.290284663438797f},
    {-0.9238795042037964f, 0.3826834261417389f}, {-0.8819212913513184f, 0.4713967442512512f}, {-0.8314695954322815f, 0.5555702447891235f}, {-0.7730104327201843f, 0.6343932747840881f},
    {-0.7071067690849304f, 0.7071067690849304f}, {-0.6343932747840881f, 0.7730104327201843f}, {-0.5555702447891235f, 0.8314695954322815f}, {-0.4713967442512512f, 0.8819212913513184f},
    {-0.3826834261417389f, 0.9238795042037964f}, {-0.290284663438797f, 0.9569403529167175f}, {-0.19509032368659973f, 0.9807852506637573f}, {-0.0980171412229538f, 0.9951847195625305f},
    {-1.8369701465288538e-16f, 1.0f}, {0.0980171412229538f, 0.9951847195625305f}, {0.19509032368659973f, 0.9807852506637573f}, {0.290284663438797f, 0.9569403529167175f},
    {0.3826834261417389f, 0.9238795042037964f}, {0.4713967442512512f, 0.8819212913513184f}, {0.5555702447891235f, 0.8314695954322815f}, {0.6343932747840881f, 0.7730104327201843f},
    {0.7071067690849304f, 0.7071067690849304f}, {0.7730104327201843f, 0.6343932747840881f}, {0.8314695954322815f, 0.5555702447891235f}, {0.8819212913513184f, 0.4713967442512512f},
    {0.9238795042037964f, 0.3826834261417389f}, {0.9569403529167175f, 0.290284663438797f}, {0.9807852506637573f, 0.19509032368659973f}, {0.9951847195625305f, 0.0980171412229538f},
};

// in-place DFT64 of a[0..63] (natural input order) as 8 x 8: r = r0 + 8 r1, k = k1 + 8 k2;
// output X[k1 + 8 k2] is left in a[8 k1 + k2] (tr64).
__host__ __device__ constexpr int tr64(int k) { return ((k & 7) << 3) | (k >> 3); }
__device__ __forceinline__ void dft64(c2 (&a)[64]) {
#pragma unroll
    for (int r0 = 0; r0 < 8; ++r0) dft8<8>(a + r0);          // over r1: a[r0 + 8 k1]
#pragma unroll
    for (int r0 = 1; r0 < 8; ++r0)
#pragma unroll
        for (int k1 = 1; k1 < 8; ++k1) {
            const int m = (r0 * k1) & 63;
            if (m == 16) a[r0 + 8 * k1] = mul2(swp(a[r0 + 8 * k1]), pk(1.0f, -1.0f));   // -i
            else a[r0 + 8 * k1] = cmul(a[r0 + 8 * k1], kW64[m]);
        }
    // outer DFT8 over r0 for each k1: element (r0, k1) is at a[r0 + 8 k1], so the 8 inputs
    // of k1 are a[8 k1 .. 8 k1 + 7]; output k2 lands in a[8 k1 + k2] = X[k1 + 8 k2]
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) dft8<1>(a + 8 * k1);
}

// in-place DFT32 of the stride-2 subset a[h], a[h + 2], ..., a[h + 62] as 8 x 4:
// r = r0 + 4 r1 (r0 < 4, r1 < 8), k = k1 + 8 k2 (k1 < 8, k2 < 4); output X[k1 + 8 k2] in
// a[h + 2 (4 k1 + k2)] (tr32).
__host__ __device__ constexpr int tr32(int k) { return ((k & 7) << 2) | (k >> 3); }
template <int H>
__device__ __forceinline__ void dft32s2(c2 (&a)[64]) {
    // element r of the subset is a[H + 2 r]; r = r0 + 4 r1
#pragma unroll
    for (int r0 = 0; r0 < 4; ++r0) dft8<8>(a + H + 2 * r0);   // over r1: stride 8 in a
    // twiddle (r0, k1) by W32^(r0 k1) = W64^(2 r0 k1); element (r0, k1) at a[H + 2 (r0 + 4 k1)]
#pragma unroll
    for (int r0 = 1; r0 < 4; ++r0)
#pragma unroll
        for (int k1 = 1; k1 < 8; ++k1) {
            const int m = (2 * r0 * k1) & 63;
            c2 &x = a[H + 2 * (r0 + 4 * k1)];
            if (m == 16) x = mul2(swp(x), pk(1.0f, -1.0f));
            else x = cmul(x, kW64[m]);
        }
    // outer DFT4 over r0 for each k1: elements a[H + 2 (4 k1 + r0)], r0 < 4 (stride 2)
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
        c2 *b = a + H + 8 * k1;
        dft4(b[0], b[2], b[4], b[6]);
    }
}

// ---- twiddle-folded butterflies (FOLD variant) -------------------------------------------
// A twiddled radix-2 butterfly (x + w b, x - w b) costs four packed instructions as
// multiply-then-add (FMUL2 + FFMA2 for w b, FADD2, FADD2); as p = x + w b (two FFMA2,
// broadcast operands) and x - w b = 2 x - p (one FFMA2, ptxas folds the negation) it
// costs three.  Twiddle kinds, compile-time after unrolling: 0 = 1, 1 = -i, 2 = general.
__device__ __forceinline__ c2 neg2(c2 a) { const float2 v = up(a); return pk(-v.x, -v.y); }
__device__ __forceinline__ c2 twb(int k, c2 x, float2 w) {
    return k == 0 ? x : k == 1 ? mul2(swp(x), pk(1.0f, -1.0f)) : cmul(x, w);
}
__device__ __forceinline__ void bfly(int k, c2 &x, c2 &b, float2 w) {
    if (k == 0) {
        const c2 t = add2(x, b);
        b = sub2(x, b);
        x = t;
    } else if (k == 1) {
        const c2 t = add_mi(x, b);
        b = sub_mi(x, b);
        x = t;
    } else {
        const c2 p = fma2(swp(b), pk(-w.y, w.y), fma2(b, pk(w.x, w.x), x));
        b = fma2(x, pk(2.0f, 2.0f), neg2(p));
        x = p;
    }
}
// forward DFT4 of (x0 w0, x1 w1, x2 w2, x3 w3) in place, kinds k0..k3
__device__ __forceinline__ void dft4k(c2 &x0, c2 &x1, c2 &x2, c2 &x3, int k0, int k1, int k2,
                                      int k3, float2 w0, float2 w1, float2 w2, float2 w3) {
    x0 = twb(k0, x0, w0);
    bfly(k2, x0, x2, w2);                // x0 = t0 = x0 + x2, x2 = t1 = x0 - x2
    x1 = twb(k1, x1, w1);
    bfly(k3, x1, x3, w3);                // x1 = t2, x3 = d
    const c2 X0 = add2(x0, x1), X2 = sub2(x0, x1), X1 = add_mi(x2, x3), X3 = sub_mi(x2, x3);
    x0 = X0; x1 = X1; x2 = X2; x3 = X3;
}
// kind of the twiddle W64^m
__host__ __device__ constexpr int kind64(int m) { return (m & 63) == 0 ? 0 : (m & 63) == 16 ? 1 : 2; }
// forward DFT8 of (v[r S] w[r]), r < 8, in place; kinds k[r].  W8 and W8^3 folded too:
// e + W8 o = e + kH (o.x + o.y, o.y - o.x) — one FFMA2 for the bracket, one per output.
template <int S>
__device__ __forceinline__ void dft8k(c2 *v, const int (&k)[8], const float2 (&w)[8]) {
    c2 e0 = v[0], e1 = v[2 * S], e2 = v[4 * S], e3 = v[6 * S];
    c2 o0 = v[S], o1 = v[3 * S], o2 = v[5 * S], o3 = v[7 * S];
    dft4k(e0, e1, e2, e3, k[0], k[2], k[4], k[6], w[0], w[2], w[4], w[6]);
    dft4k(o0, o1, o2, o3, k[1], k[3], k[5], k[7], w[1], w[3], w[5], w[7]);
    const c2 u1 = fma2(swp(o1), pk(1.0f, -1.0f), o1);           // sqrt2 W8 o1
    const c2 u3 = fma2(swp(o3), pk(1.0f, -1.0f), neg2(o3));     // sqrt2 W8^3 o3
    v[0] = add2(e0, o0); v[4 * S] = sub2(e0, o0);
    v[S] = fma2(u1, pk(kH, kH), e1); v[5 * S] = fma2(u1, pk(-kH, -kH), e1);
    v[2 * S] = add_mi(e2, o2); v[6 * S] = sub_mi(e2, o2);
    v[3 * S] = fma2(u3, pk(kH, kH), e3); v[7 * S] = fma2(u3, pk(-kH, -kH), e3);
}
template <int S>
__device__ __forceinline__ void dft8k0(c2 *v) {
    constexpr int k[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const float2 w[8] = {};
    dft8k<S>(v, k, w);
}
// dft64 with the inter-stage twiddles W64^(r0 k1) folded into the outer DFT8s
__device__ __forceinline__ void dft64f(c2 (&a)[64]) {
#pragma unroll
    for (int r0 = 0; r0 < 8; ++r0) dft8k0<8>(a + r0);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
        int k[8];
        float2 w[8];
#pragma unroll
        for (int r0 = 0; r0 < 8; ++r0) {
            k[r0] = kind64(r0 * k1);
            w[r0] = kW64[(r0 * k1) & 63];
        }
        dft8k<1>(a + 8 * k1, k, w);
    }
}
// the folded kernel's twiddle table: float2 slot i holds w^(r j) for j = (i / 2) % 64,
// r = r0 + 4 (2 q + i % 2), (r0, q) = ((i / 128) / 4, (i / 128) % 4): the two twiddles a
// lane needs for r1 = 2q, 2q + 1 of one DFT8 are one 16-byte load
__host__ __device__ constexpr int tws_fold_r(int i) { return (i >> 9) + 4 * (2 * ((i >> 7) & 3) + (i & 1)); }
__host__ __device__ constexpr int tws_fold_j(int i) { return (i >> 1) & 63; }
// dft32s2 with the pass-2 table twiddles w^(r j) (tws) folded into the DFT8s over r1 and
// the inner twiddles W32^(r0 k1) into the DFT4s over r0
template <int H>
__device__ __forceinline__ void dft32s2f(c2 (&a)[64], const float2 *tws, int l) {
#pragma unroll
    for (int r0 = 0; r0 < 4; ++r0) {
        int k[8];
        float2 w[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {        // r1 = 2q, 2q + 1: one LDS.128 (tws_fold_index)
            const float4 v = reinterpret_cast<const float4 *>(tws)[(r0 * 4 + q) * 64 + l + 32 * H];
            w[2 * q] = make_float2(v.x, v.y);
            w[2 * q + 1] = make_float2(v.z, v.w);
            k[2 * q] = r0 + 8 * q == 0 ? 0 : 2;
            k[2 * q + 1] = 2;
        }
        dft8k<8>(a + H + 2 * r0, k, w);
    }
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) {
        c2 *b = a + H + 8 * k1;
        dft4k(b[0], b[2], b[4], b[6], 0, kind64(2 * k1), kind64(4 * k1), kind64(6 * k1),
              make_float2(1.0f, 0.0f), kW64[(2 * k1) & 63], kW64[(4 * k1) & 63], kW64[(6 * k1) & 63]);
    }
}

// One transform (forward, natural order in and out) of the signal a lane holds as
// a[s] = x[l + 32 s]; buf: the warp's exchange slots.  On return a[s] = X[l + 32 s].
// next: the input of the warp's next signal, fetched into buf once the last pass has read
// it (nullptr: not this transform, or no next signal); bar: the warp's fetch mbarrier.
__device__ __forceinline__ void fetch_signal(c2 *buf, const float2 *src, uint64_t *bar) {
    bfk::mbar_arrive_expect_tx(bar, (uint32_t)(kN * 8));
    bfk::bulk_g2s(buf, src, kN * 8, bar, bfk::policy_evict_first());
}
// FOLD: twiddles folded into the butterflies (needs TAB).  fetch(): called by every lane
// once pass 2 has read the exchange buffer (it may refill buf with the next input)
template <bool TAB, bool FOLD, class Fetch>
__device__ __forceinline__ void fft2048_warp_x(c2 (&a)[64], c2 *buf, const float4 *__restrict__ twp,
                                               const float2 *tws, int l, Fetch &&fetch) {
    // pass 1: radix 64, inputs a[r] = x[l + 32 r]; output y[64 l + k] = X1[k] (a[tr64(k)])
    if (FOLD) dft64f(a);
    else dft64(a);
    __syncwarp();                       // every lane's reads of buf (input / last pass) are done
#pragma unroll
    for (int k = 0; k < 64; ++k) sts64(buf + wpad(64 * l + k), a[tr64(k)]);
    __syncwarp();
    // pass 2: radix 32, columns j = l + 32 h: inputs y[j + 64 r] = buf[j + 65 r], r < 32
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int r = 0; r < 32; ++r) a[h + 2 * r] = buf[wpad(l + 32 * h + 64 * r)];
    fetch();
    // twiddles w^(r j): TAB — from the CTA's shared table tws[r][j] (rounded once);
    // otherwise r = 8 b + c from T1[c] = w^(c j), c < 8 and T2[b] = w^(8 b j), b < 4, with
    // twp[e][j] = (w^(2^e j)) for e < 5 (float2 pairs of j and j + 32 in one float4)
    if (FOLD) {
        static_assert(!FOLD || TAB, "the folded pass 2 reads the shared twiddle table");
        dft32s2f<0>(a, tws, l);
        dft32s2f<1>(a, tws, l);
    } else if (TAB) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int r = 1; r < 32; ++r) a[h + 2 * r] = cmul(a[h + 2 * r], tws[r * 64 + l + 32 * h]);
    } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        float2 t1[8], t2[4];
#pragma unroll
        for (int e = 0; e < 5; ++e) {
            const float4 w = __ldg(twp + e * 32 + l);
            const float2 wj = h == 0 ? make_float2(w.x, w.y) : make_float2(w.z, w.w);
            if (e < 3) t1[1 << e] = wj;
            else t2[1 << (e - 3)] = wj;                     // w^(8 j), w^(16 j)
        }
        t1[3] = tmul(t1[1], t1[2]);
        t1[5] = tmul(t1[4], t1[1]);
        t1[6] = tmul(t1[4], t1[2]);
        t1[7] = tmul(t1[4], t1[3]);
        t2[3] = tmul(t2[1], t2[2]);
#pragma unroll
        for (int r = 1; r < 32; ++r) {
            const int b = r >> 3, c = r & 7;
            const float2 w = b == 0 ? t1[c] : (c == 0 ? t2[b] : tmul(t2[b], t1[c]));
            a[h + 2 * r] = cmul(a[h + 2 * r], w);
        }
    }
    }
    if (!FOLD) {
        dft32s2<0>(a);
        dft32s2<1>(a);
    }
    // X[j + 64 k] is in a[h + 2 tr32(k)]: rename to a[h + 2 k] (compile-time permutation)
    c2 t[64];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < 32; ++k) t[h + 2 * k] = a[h + 2 * tr32(k)];
#pragma unroll
    for (int s = 0; s < 64; ++s) a[s] = t[s];
}
template <bool TAB, bool FOLD = false>
__device__ __forceinline__ void fft2048_warp(c2 (&a)[64], c2 *buf, const float4 *__restrict__ twp,
                                             const float2 *tws, int l, const float2 *next,
                                             uint64_t *bar) {
    fft2048_warp_x<TAB, FOLD>(a, buf, twp, tws, l, [&] {
        if (next) {                // last transform of the signal: the buffer is free now
            __syncwarp();
            if (l == 0) {
                bfk::fence_proxy_async_smem();         // generic reads before the async write
                fetch_signal(buf, next, bar);
            }
        }
    });
}

// MINC: CTAs per SM the register budget is sized for (3: 168 registers, 12 warps per SM;
// 2: 255 registers, 8 warps)
template <int MINC, bool FOLD = false>
__global__ void __launch_bounds__(kThreads, MINC) filter_warp_kernel(const FParams p) {
    // with 255 registers (2 CTAs per SM) shared memory has room for the twiddle and H tables
    constexpr bool TAB = MINC == 2;
    extern __shared__ __align__(128) unsigned char fsm[];
    const int warp = threadIdx.x >> 5, l = threadIdx.x & 31;
    c2 *buf = reinterpret_cast<c2 *>(fsm) + warp * kWarpPad;
    uint64_t *bar = reinterpret_cast<uint64_t *>(fsm + 4 * kWarpPad * 8) + warp;
    float2 *tws = reinterpret_cast<float2 *>(fsm + 4 * kWarpPad * 8 + 4 * 8);   // [32][64]
    float2 *Hs = tws + kN;                                                      // [2048]
    if (TAB) {
        for (int i = threadIdx.x; i < kN; i += kThreads) {
            tws[i] = FOLD ? p.tw[(tws_fold_r(i) * tws_fold_j(i)) & (kN - 1)]       // w^(r j)
                          : p.tw[((i >> 6) * (i & 63)) & (kN - 1)];
            // H in lane pairs: float4 (H[l + 32 s], H[l + 32 (s + 1)]) at [s / 2][l], s even,
            // so the MULT reads two values per LDS.128
            if (p.mode == 0) {
                const int pr = i >> 1, e = (pr & 31) + 32 * (2 * (pr >> 5) + (i & 1));
                Hs[i] = p.H[e];
            }
        }
        __syncthreads();
    }
    const int64_t gw = (int64_t)blockIdx.x * 4 + warp, nw = (int64_t)gridDim.x * 4;
    constexpr float inv_n = 1.0f / kN;
    const c2 oscale = p.mode == 0 ? pk(1.0f, -1.0f) : (p.mode == 2 ? pk(inv_n, inv_n) : pk(1.0f, 1.0f));
    const int trips = p.mode == 0 ? 2 : 1;
    // the input of a signal -> buf[0, 2048) (natural order), completion on the warp's bar
    if (l == 0) {
        bfk::mbar_init(bar, 1);
        bfk::mbar_fence_init();
        if (gw < p.n_sig) fetch_signal(buf, p.s + gw * kN, bar);
    }
    __syncwarp();
    uint32_t phase = 0;
    for (int64_t sig = gw; sig < p.n_sig; sig += nw) {
        c2 a[64];
        bfk::mbar_wait(bar, phase);
        phase ^= 1u;
#pragma unroll
        for (int s = 0; s < 64; ++s) a[s] = buf[l + 32 * s];
#pragma unroll 1
        for (int trip = 0; trip < trips; ++trip) {
            const bool last = trip == trips - 1 && sig + nw < p.n_sig;
            const float2 *nx = last ? p.s + (sig + nw) * kN : nullptr;
            fft2048_warp<TAB, FOLD>(a, buf, p.twp, tws, l, nx, bar);
            if (trip == 0 && trips == 2) {
#pragma unroll
                for (int s = 0; s < 64; s += 2) {
                    if (TAB) {
                        const float4 h = reinterpret_cast<const float4 *>(Hs)[(s >> 1) * 32 + l];
                        a[s] = cmul_conj(a[s], make_float2(h.x, h.y));
                        a[s + 1] = cmul_conj(a[s + 1], make_float2(h.z, h.w));
                    } else {
                        a[s] = cmul_conj(a[s], __ldg(p.H + l + 32 * s));
                        a[s + 1] = cmul_conj(a[s + 1], __ldg(p.H + l + 32 * (s + 1)));
                    }
                }
            }
        }
        float2 *dst = p.y + sig * kN;
        if (p.mode == 0) {
            // the conj of the conj trick as a sign flip on the integer pipe (LOP3), not an
            // FMUL2 on the FMA pipe the transforms keep ~2/3 busy
#pragma unroll
            for (int s = 0; s < 64; ++s) {
                const float2 v = up(a[s]);
                uint32_t im;   // inline PTX: a C-level XOR becomes neg.f32 -> FADD on the FMA pipe
                asm("xor.b32 %0, %1, 0x80000000;" : "=r"(im) : "r"(__float_as_uint(v.y)));
                __stcs(dst + l + 32 * s, make_float2(v.x, __uint_as_float(im)));
            }
        } else {
#pragma unroll
            for (int s = 0; s < 64; ++s) __stcs(dst + l + 32 * s, up(mul2(a[s], oscale)));
        }
    }
}

// pass-2 base twiddles of the warp kernel: twp[e 32 + l] = (w^(2^e l), w^(2^e (l + 32))),
// e < 5, fp64-evaluated, rounded once.
constexpr int kTwpN = 5 * 32;
static __global__ void twiddle_warp_kernel(float4 *twp) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= kTwpN) return;
    const int e = i / 32, l = i % 32;
    double s0, c0, s1, c1;
    sincospi(-2.0 * (double)(((l) << e) % kN) / kN, &s0, &c0);
    sincospi(-2.0 * (double)(((l + 32) << e) % kN) / kN, &s1, &c1);
    twp[i] = make_float4((float)c0, (float)s0, (float)c1, (float)s1);
}

}  // namespace bff
