// bf_filter.cuh — fused filter stage y = IFFT(H . FFT(s)) for n = 2048
// (§III: "The filter algorithm computes IFFT(MULT(FFT(s))) where
// MULT is the pointwise multiplication by the FFT of the filter sequence and
// FFT sizes are all 2048").
//
// One CTA of 128 threads per signal (grid-stride over signals).  The forward
// FFT, the pointwise product with H and the inverse FFT run in one kernel, so
// each signal is read from HBM once and written once (32 KB per signal) — the
// paper replaced its hand FFT by a vendor library; here the three steps are
// fused, which a library call sequence cannot do.
//
// Arithmetic in packed fp32x2 (FADD2 / FMUL2 / FFMA2, one instruction per complex add,
// two per complex multiply).  FFT: Stockham autosort, passes radix 16, 16, 8 (2048 = 16 * 16 * 8).  A pass with
// stride Ns and radix R: butterfly j loads x[j + r N/R] (r < R), multiplies by
// w^(r k N/(Ns R)) with k = j mod Ns and w = e^{-2 pi i / N} (fp32 table built in
// fp64), does a DFT_R, and writes y[(j / Ns) Ns R + k + r Ns].  Thread t owns
// butterfly t (and t + 128 in the radix-8 pass), so the first pass reads
// x[t + 128 r] straight from HBM (coalesced) and the last pass leaves
// X[t + 128 q] (natural order) in registers: MULT by H, and the inverse
// transform (conj(FFT(conj(.))) / N) starts from registers again.  Between
// passes values go through shared memory (two exchanges per transform) with the padded
// index i + i/16 (conflict-free for every pattern of the three passes).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "bf_ffma.cuh"   // mbarrier / bulk-copy helpers

namespace bff {

constexpr int kN = 2048;
constexpr int kThreads = 128;
// signals per CTA iteration (instruction streams interleaved in every thread): template
// parameter NS of the kernel, 1 or 2; min_ctas(NS) CTAs of 128 threads per SM
__host__ __device__ constexpr int min_ctas(int ns) { return ns == 1 ? 4 : 3; }
// Exchange buffers (one per signal of the iteration), float2 slots with one padding slot
// per 16: every access pattern of the three passes is then conflict-free (two
// wavefronts per 64-bit warp access).  Values enter and leave them as 64-bit register
// pairs (sts64 below): a 128-bit slot holding two values would cost register moves to
// assemble each store's aligned quad.
constexpr int kPad = kN + kN / 16;
__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
// Twiddles of the two twiddled passes: each thread loads the binary powers of its base
// twiddle and forms the others with at most three products (relative error <= ~4 2^-24,
// far inside the filter's 1e-5 normwise contract): 4 instead of 15 shared loads in pass 2
// and 3 instead of 7 L1 loads in pass 3 — shared / L1 bandwidth, not the FMA pipe, bounds
// this kernel once its arithmetic is packed.
// Pass-2 table in shared memory: [k][e] = w^(8 k 2^e), k < 16, e < 4.
constexpr int kTw2 = 16 * 4;
// Pass-3 table (plan-owned global, read through L1): [e][t] = (w^(2^e t), w^(2^e (t + 128))),
// e < 3, t < 128.
constexpr int kTw3N = 3 * 128;
constexpr int kTwN = kN;                     // plan twiddle table tw[m] = w^m (float2)

// ---- packed complex arithmetic (fp32x2: FADD2 / FMUL2 / FFMA2) ---------------------------
// A complex value is one 64-bit register pair (re, im).  Blackwell's packed fp32x2
// instructions do both halves in one issue slot at the FFMA rate (tools/fp32x2_probe:
// 74 TFLOP/s for FFMA2 and FFMA alike), and ptxas folds half swaps, per-half negation and
// scalar broadcasts into their operands, so a complex add is one instruction and a
// complex multiply two — half the instructions of the scalar form.  Each half is an IEEE
// fp32 operation rounded to nearest.
typedef unsigned long long c2;
__device__ __forceinline__ c2 pk(float x, float y) {
    const float2 v = make_float2(x, y);
    return *reinterpret_cast<const c2 *>(&v);
}
__device__ __forceinline__ c2 pk(float2 v) { return *reinterpret_cast<const c2 *>(&v); }
__device__ __forceinline__ float2 up(c2 a) { return *reinterpret_cast<const float2 *>(&a); }
__device__ __forceinline__ c2 swp(c2 a) { const float2 v = up(a); return pk(v.y, v.x); }
__device__ __forceinline__ c2 add2(c2 a, c2 b) {
    c2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ c2 sub2(c2 a, c2 b) {
    c2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ c2 mul2(c2 a, c2 b) {
    c2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ c2 fma2(c2 a, c2 b, c2 c) {
    c2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// a * w, w = (c, s) = c + i s:  (a.x c - a.y s, a.y c + a.x s) = swap(a) (-s, s) + a (c, c).
// ptxas takes (c, c) and (-s, s) straight from w's register pair (broadcast operand, per-
// half negation): FMUL2 + FFMA2, no extra registers.
__device__ __forceinline__ c2 cmul(c2 a, float2 w) { return fma2(swp(a), pk(-w.y, w.y), mul2(a, pk(w.x, w.x))); }
// conj(a * h) = (a.x hx - a.y hy, -a.y hx - a.x hy) = swap(a) (-hy, -hy) + a (hx, -hx)
__device__ __forceinline__ c2 cmul_conj(c2 a, float2 h) {
    const float2 v = up(a);
    return fma2(pk(-v.y, -v.x), pk(h.y, h.y), mul2(pk(v.x, -v.y), pk(h.x, h.x)));
}
// complex product of two twiddles (float2 in, float2 out)
__device__ __forceinline__ float2 tmul(float2 a, float2 b) { return up(cmul(pk(a), b)); }
// p[r] = w^r for r = 1..R-1 (R = 8 or 16) from p[1], p[2], p[4] (and p[8]) loaded
template <int R>
__device__ __forceinline__ void tw_powers(float2 (&p)[16]) {
    p[3] = tmul(p[1], p[2]);
    p[5] = tmul(p[4], p[1]);
    p[6] = tmul(p[4], p[2]);
    p[7] = tmul(p[4], p[3]);
    if (R == 16) {
#pragma unroll
        for (int r = 1; r < 8; ++r) p[8 + r] = tmul(p[8], p[r]);
    }
}
// a * (c + i s) for compile-time constants
__device__ __forceinline__ c2 cmulc(c2 a, float c, float s) { return cmul(a, make_float2(c, s)); }
// 64-bit shared store of a register pair (inline PTX: the compiler may not merge two of
// them into a 128-bit store, which would need register moves)
__device__ __forceinline__ void sts64(c2 *dst, c2 v) {
    const float2 f = up(v);   // two 32-bit operands: a .b64 operand costs a register-pair copy
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "f"(f.x), "f"(f.y) : "memory");
}
// x + (-i) y = (x.x + y.y, x.y - y.x) and x - (-i) y, in one FFMA2 each
__device__ __forceinline__ c2 add_mi(c2 x, c2 y) { return fma2(swp(y), pk(1.0f, -1.0f), x); }
__device__ __forceinline__ c2 sub_mi(c2 x, c2 y) { return fma2(swp(y), pk(-1.0f, 1.0f), x); }

constexpr float kC1 = 0.92387953251128675613f, kS1 = 0.38268343236508977173f;   // cos, sin(pi/8)
constexpr float kH = 0.70710678118654752440f;

// forward DFT4 (w = -i) in place; MI2: x2 arrives still to be multiplied by -i (folded)
template <bool MI2 = false>
__device__ __forceinline__ void dft4(c2 &x0, c2 &x1, c2 &x2, c2 &x3) {
    const c2 t0 = MI2 ? add_mi(x0, x2) : add2(x0, x2);
    const c2 t1 = MI2 ? sub_mi(x0, x2) : sub2(x0, x2);
    const c2 t2 = add2(x1, x3), d = sub2(x1, x3);
    x0 = add2(t0, t2);
    x2 = sub2(t0, t2);
    x1 = add_mi(t1, d);                       // t1 + (-i) d
    x3 = sub_mi(t1, d);
}

// forward DFT8 in place (v[k] <- sum_r v[r] e^{-2 pi i r k / 8}) on v[0], v[S], ..., v[7 S]
template <int S>
__device__ __forceinline__ void dft8(c2 *v) {
    c2 e0 = v[0], e1 = v[2 * S], e2 = v[4 * S], e3 = v[6 * S];
    c2 o0 = v[S], o1 = v[3 * S], o2 = v[5 * S], o3 = v[7 * S];
    dft4(e0, e1, e2, e3);
    dft4(o0, o1, o2, o3);
    o1 = cmulc(o1, kH, -kH);                  // W8   = (1 - i) / sqrt2
    o3 = cmulc(o3, -kH, -kH);                 // W8^3 = (-1 - i) / sqrt2
    v[0] = add2(e0, o0); v[4 * S] = sub2(e0, o0);
    v[S] = add2(e1, o1); v[5 * S] = sub2(e1, o1);
    v[2 * S] = add_mi(e2, o2); v[6 * S] = sub_mi(e2, o2);   // W8^2 = -i, folded
    v[3 * S] = add2(e3, o3); v[7 * S] = sub2(e3, o3);
}

// forward DFT16, 4 x 4: n = n2 + 4 n1, k = k1 + 4 k2,
// X[k1 + 4 k2] = sum_n2 W4^(n2 k2) W16^(n2 k1) sum_n1 v[n2 + 4 n1] W4^(n1 k1).
// The result is left TRANSPOSED in place: X[k1 + 4 k2] is in v[4 k1 + k2] (tr16).
__host__ __device__ constexpr int tr16(int k) { return ((k & 3) << 2) | (k >> 2); }
__device__ __forceinline__ void dft16(c2 (&v)[16]) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[n2 + 4], v[n2 + 8], v[n2 + 12]);
    // twiddle u[n2][k1] = v[n2 + 4 k1] by W16^(n2 k1), W16^m = cos(pi m / 8) - i sin(pi m / 8);
    // W16^4 = -i on v[10] is folded into the outer DFT4 of k1 = 2
    v[5] = cmulc(v[5], kC1, -kS1);            // W^1
    v[9] = cmulc(v[9], kH, -kH);              // W^2
    v[13] = cmulc(v[13], kS1, -kC1);          // W^3
    v[6] = cmulc(v[6], kH, -kH);              // W^2
    v[14] = cmulc(v[14], -kH, -kH);           // W^6
    v[7] = cmulc(v[7], kS1, -kC1);            // W^3
    v[11] = cmulc(v[11], -kH, -kH);           // W^6
    v[15] = cmulc(v[15], -kC1, kS1);          // W^9
    // outer DFT4 over n2 for each k1: inputs v[4 k1 + n2] -> X[k1 + 4 k2] in v[4 k1 + k2]
    dft4(v[0], v[1], v[2], v[3]);
    dft4(v[4], v[5], v[6], v[7]);
    dft4<true>(v[8], v[9], v[10], v[11]);
    dft4(v[12], v[13], v[14], v[15]);
}

// The kNS forward FFTs of the iteration's signals (radix 16, 16, 8 Stockham), instruction
// streams interleaved (independent chains for the schedulers) and sharing each pass's
// barriers.  In: v[s][q] = x_s[t + 128 q].  Out: v[s][q] = X_s[t + 128 q].  sm holds kNS
// exchange buffers of kPad slots.
template <int kNS>
__device__ __forceinline__ void fft2048(c2 (&v)[kNS][16], c2 *sm, const float2 *tw2,
                                        const float4 *__restrict__ tw3, int t) {
    // pass 1: Ns = 1, R = 16 (no twiddles); y[16 j + r]
#pragma unroll
    for (int s = 0; s < kNS; ++s) {
        dft16(v[s]);
#pragma unroll
        for (int r = 0; r < 16; ++r) sts64(sm + s * kPad + pad(16 * t + r), v[s][tr16(r)]);
    }
    __syncthreads();
    // pass 2: Ns = 16, R = 16; twiddles w^(8 r k), k = j mod 16; y[(j/16) 256 + k + 16 r]
    const int k = t & 15;
#pragma unroll
    for (int s = 0; s < kNS; ++s)
#pragma unroll
        for (int r = 0; r < 16; ++r) v[s][r] = sm[s * kPad + pad(t + 128 * r)];
    {
        float2 p[16];
        p[1] = tw2[k * 4];
        p[2] = tw2[k * 4 + 1];
        p[4] = tw2[k * 4 + 2];
        p[8] = tw2[k * 4 + 3];
        tw_powers<16>(p);
#pragma unroll
        for (int r = 1; r < 16; ++r)
#pragma unroll
            for (int s = 0; s < kNS; ++s) v[s][r] = cmul(v[s][r], p[r]);
    }
#pragma unroll
    for (int s = 0; s < kNS; ++s) dft16(v[s]);
    __syncthreads();
    const int base = (t >> 4) * 256 + k;
#pragma unroll
    for (int s = 0; s < kNS; ++s)
#pragma unroll
        for (int r = 0; r < 16; ++r) sts64(sm + s * kPad + pad(base + 16 * r), v[s][tr16(r)]);
    __syncthreads();
    // pass 3: Ns = 256, R = 8, butterflies j = t and t + 128; twiddles w^(r j); y[j + 256 r]
#pragma unroll
    for (int s = 0; s < kNS; ++s)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            v[s][2 * r] = sm[s * kPad + pad(t + 256 * r)];
            v[s][2 * r + 1] = sm[s * kPad + pad(t + 128 + 256 * r)];
        }
    {
        float2 p[16], q[16];                  // w^(r t), w^(r (t + 128))
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            const float4 w = __ldg(tw3 + e * 128 + t);
            p[1 << e] = make_float2(w.x, w.y);
            q[1 << e] = make_float2(w.z, w.w);
        }
        tw_powers<8>(p);
        tw_powers<8>(q);
#pragma unroll
        for (int r = 1; r < 8; ++r)
#pragma unroll
            for (int s = 0; s < kNS; ++s) {
                v[s][2 * r] = cmul(v[s][2 * r], p[r]);
                v[s][2 * r + 1] = cmul(v[s][2 * r + 1], q[r]);
            }
    }
#pragma unroll
    for (int s = 0; s < kNS; ++s) {
        dft8<2>(v[s]);        // butterfly t:       v[0], v[2], ..., v[14]
        dft8<2>(v[s] + 1);    // butterfly t + 128: v[1], v[3], ..., v[15]
    }
    __syncthreads();          // shared memory free for the next transform
    // X[t + 256 r] = v[2 r], X[t + 128 + 256 r] = v[2 r + 1]  ->  v[q] = X[t + 128 q]
}

__host__ __device__ constexpr int smem_bytes(int ns) {   // dynamic shared memory
    return ns * kN * 8 + ns * kPad * 8 + kTw2 * 8 + 8;
}

struct FParams {
    const float2 *s;     // [n_sig][2048]
    float2 *y;           // [n_sig][2048] (may alias s exactly: a signal is read, into
                         // the prefetch stage, before the CTA writes it)
    const float2 *H;     // [2048] DFT(h) / N (plan-owned)
    const float2 *tw;    // [2048] twiddle table w^m (plan-owned)
    const float4 *tw3;   // [3][128] pass-3 base twiddle pairs (plan-owned)
    const float4 *twp;   // [5][32] pass-2 base twiddle pairs of the warp kernel (plan-owned)
    int64_t n_sig;
    int mode;            // 0: filter; 1: forward FFT only;
                         // 2: forward FFT scaled by 1/N (builds the plan's H from h)
};

template <int kNS>
__global__ void __launch_bounds__(kThreads, min_ctas(kNS)) filter_kernel(const FParams p) {
    // stage: the CTA's next kNS signals, prefetched with TMA bulk copies (16 KB each)
    // while the current ones are transformed; sm: the exchange slots.  H and the pass-3
    // twiddles are read through L1 (shared by the CTAs of an SM).
    extern __shared__ __align__(128) unsigned char fsm[];
    float2 *stage = reinterpret_cast<float2 *>(fsm);                         // kNS x kN
    c2 *sm = reinterpret_cast<c2 *>(fsm + kNS * kN * 8);                     // kNS x kPad
    float2 *tw2 = reinterpret_cast<float2 *>(sm + kNS * kPad);               // kTw2
    uint64_t *barp = reinterpret_cast<uint64_t *>(tw2 + kTw2);
    uint64_t &bar = *barp;
    const int t = threadIdx.x;
    for (int i = t; i < kTw2; i += kThreads) {   // pass 2: [k][e] = w^(8 k 2^e)
        const int k = i / 4, e = i % 4;
        tw2[i] = p.tw[(8 * k << e) & (kN - 1)];
    }
    if (t == 0) {
        bfk::mbar_init(&bar, 1);
        bfk::mbar_fence_init();
    }
    __syncthreads();
    const uint64_t pol = bfk::policy_evict_first();
    const int64_t G = gridDim.x;
    // signals of iteration base: base + s G, s < kNS
    auto prefetch = [&](int64_t base) {
        int cnt = 0;
        for (int s = 0; s < kNS; ++s) cnt += base + s * G < p.n_sig;
        if (cnt == 0) return;
        bfk::mbar_arrive_expect_tx(&bar, (uint32_t)(cnt * kN * 8));
        for (int s = 0; s < kNS; ++s)
            if (base + s * G < p.n_sig)
                bfk::bulk_g2s(stage + s * kN, p.s + (base + s * G) * kN, kN * 8, &bar, pol);
    };
    if (t == 0) prefetch(blockIdx.x);
    constexpr float inv_n = 1.0f / kN;
    uint32_t phase = 0;
    for (int64_t base = blockIdx.x; base < p.n_sig; base += kNS * G) {
        c2 v[kNS][16];
        bfk::mbar_wait(&bar, phase);
        phase ^= 1u;
#pragma unroll
        for (int s = 0; s < kNS; ++s) {
            const bool ok = base + s * G < p.n_sig;
#pragma unroll
            for (int q = 0; q < 16; ++q) v[s][q] = ok ? pk(stage[s * kN + t + 128 * q]) : 0ull;
        }
        __syncthreads();                                  // stage consumed by every thread
        if (t == 0) prefetch(base + kNS * G);
        // forward FFT, MULT by H, inverse FFT as conj(FFT(conj(.))) / N — one copy of
        // the transform code in a two-trip loop keeps register pressure at one FFT's.
        // conj(X H) is one packed complex multiply with the plan's H operands, and the
        // plan stores H / N (exact: N = 2^11), so neither the conj nor the 1/N costs here.
        const int trips = p.mode == 0 ? 2 : 1;
#pragma unroll 1
        for (int trip = 0; trip < trips; ++trip) {
            fft2048<kNS>(v, sm, tw2, p.tw3, t);
            if (trip == 0 && trips == 2) {
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const float2 h = __ldg(p.H + t + 128 * q);
#pragma unroll
                    for (int s = 0; s < kNS; ++s) v[s][q] = cmul_conj(v[s][q], h);
                }
            }
        }
        // output: conj (mode 0), 1/N (mode 2) or as is; the mode test outside the loops
        const c2 oscale = p.mode == 0 ? pk(1.0f, -1.0f) : (p.mode == 2 ? pk(inv_n, inv_n) : pk(1.0f, 1.0f));
#pragma unroll
        for (int s = 0; s < kNS; ++s) {
            const int64_t sig = base + s * G;
            if (sig >= p.n_sig) break;
            float2 *dst = p.y + sig * kN;
#pragma unroll
            for (int q = 0; q < 16; ++q) __stcs(dst + t + 128 * q, up(mul2(v[s][q], oscale)));
        }
    }
}

// tw[m] = e^{-2 pi i m / N}, evaluated in fp64 and rounded once.
static __global__ void twiddle_kernel(float2 *tw) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= kTwN) return;
    double s, c;
    sincospi(-2.0 * (double)m / kN, &s, &c);
    tw[m] = make_float2((float)c, (float)s);
}

// tw3[e 128 + t] = (w^(r t), w^(r (t + 128))) with r = 2^e, fp64-evaluated, rounded once.
static __global__ void twiddle3_kernel(float4 *tw3) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= kTw3N) return;
    const int r = 1 << (i / 128), t = i % 128;
    double s0, c0, s1, c1;
    sincospi(-2.0 * (double)((r * t) % kN) / kN, &s0, &c0);
    sincospi(-2.0 * (double)((r * (t + 128)) % kN) / kN, &s1, &c1);
    tw3[i] = make_float4((float)c0, (float)s0, (float)c1, (float)s1);
}

}  // namespace bff
