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
// FFT: Stockham autosort, passes radix 16, 16, 8 (2048 = 16 * 16 * 8).  A pass with
// stride Ns and radix R: butterfly j loads x[j + r N/R] (r < R), multiplies by
// w^(r k N/(Ns R)) with k = j mod Ns and w = e^{-2 pi i / N} (fp32 table built in
// fp64), does a DFT_R, and writes y[(j / Ns) Ns R + k + r Ns].  Thread t owns
// butterfly t (and t + 128 in the radix-8 pass), so the first pass reads
// x[t + 128 r] straight from HBM (coalesced) and the last pass leaves
// X[t + 128 q] (natural order) in registers: MULT by H, and the inverse
// transform (conj(FFT(conj(.))) / N) starts from registers again.  Between
// passes values go through shared memory (two exchanges per transform) with
// the padded index i + i/16 (conflict-free for the stride-16 writes of pass 1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "bf_ffma.cuh"   // mbarrier / bulk-copy helpers

namespace bff {

constexpr int kN = 2048;
constexpr int kThreads = 128;
constexpr int kPad = kN + kN / 8;            // padded shared-memory slots (float2): 2 per 16
// Twiddle table tw[m] = w^m = e^{-2 pi i m / N} (fp64-evaluated, rounded once), read
// through L1.  A pass needs w^(c r k) for r < R: the kernel loads the binary powers
// w^(c k 2^e) from the table and forms the others with at most 3 complex products
// (relative error <= 4 * 2^-24), which keeps 4 instead of R - 1 twiddles live.
constexpr int kTwN = kN;
// Per-pass tables in shared memory, laid out so that a thread reads two twiddles
// per 128-bit load: pass 2 [k][r - 1] (k < 16, rows of 18 slots: 15 twiddles
// w^(8 r k), r = 1..15, padded so 8 lanes of an LDS.128 hit distinct banks),
// pass 3 [r - 1][t] = (w^(r t), w^(r (t + 128))) for r = 1..7, t < 128 (a plan-owned
// global table read through L1 — shared by the 5 CTAs of an SM, and keeping the
// shared memory per CTA small enough for 5 resident CTAs).
constexpr int kTw2Row = 18;
constexpr int kTw2 = 0, kTwS = kTw2 + 16 * kTw2Row;
constexpr int kTw3N = 7 * 128;                  // float4 entries of the pass-3 table



// exchange-buffer index: 2 padding slots per 16 keep every access pattern below
// conflict-free and make a pass-1 thread's 16 outputs 16-byte aligned (STS.128)
__device__ __forceinline__ int pad(int i) { return i + 2 * (i >> 4); }

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }   // a * (-i)
__device__ __forceinline__ float2 conj2(float2 a) { return make_float2(a.x, -a.y); }

// w^(m r) for r in [1, 16) from b[e] = w^(m 2^e), e < 4 (r is a compile-time constant).
__device__ __forceinline__ float2 tw_pow(const float2 (&b)[4], int r) {
    float2 acc = make_float2(1.0f, 0.0f);
    bool first = true;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (r & (1 << e)) {
            acc = first ? b[e] : cmul(acc, b[e]);
            first = false;
        }
    }
    return acc;
}

// forward DFT4 (w = -i) in place
__device__ __forceinline__ void dft4(float2 &x0, float2 &x1, float2 &x2, float2 &x3) {
    const float2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = mul_mi(csub(x1, x3));
    x0 = cadd(t0, t2);
    x2 = csub(t0, t2);
    x1 = cadd(t1, t3);
    x3 = csub(t1, t3);
}

// forward DFT8 in place (v[k] <- sum_r v[r] e^{-2 pi i r k / 8})
template <int S>
__device__ __forceinline__ void dft8(float2 *v) {   // elements v[0], v[S], ..., v[7 S]
    float2 e0 = v[0], e1 = v[2 * S], e2 = v[4 * S], e3 = v[6 * S];
    float2 o0 = v[S], o1 = v[3 * S], o2 = v[5 * S], o3 = v[7 * S];
    dft4(e0, e1, e2, e3);
    dft4(o0, o1, o2, o3);
    const float h = 0.70710678118654752440f;
    // o_k *= W8^k: W8 = (1 - i)/sqrt2, W8^2 = -i, W8^3 = (-1 - i)/sqrt2
    o1 = make_float2((o1.x + o1.y) * h, (o1.y - o1.x) * h);
    o2 = mul_mi(o2);
    o3 = make_float2((o3.y - o3.x) * h, -(o3.x + o3.y) * h);
    v[0] = cadd(e0, o0); v[4 * S] = csub(e0, o0);
    v[S] = cadd(e1, o1); v[5 * S] = csub(e1, o1);
    v[2 * S] = cadd(e2, o2); v[6 * S] = csub(e2, o2);
    v[3 * S] = cadd(e3, o3); v[7 * S] = csub(e3, o3);
}

// forward DFT16, 4 x 4: n = n2 + 4 n1, k = k1 + 4 k2,
// X[k1 + 4 k2] = sum_n2 W4^(n2 k2) W16^(n2 k1) sum_n1 v[n2 + 4 n1] W4^(n1 k1).
// The result is left TRANSPOSED in place: X[k1 + 4 k2] is in v[4 k1 + k2]
// (tr16(k) below), which saves a 16-value copy; callers index with tr16.
__host__ __device__ constexpr int tr16(int k) { return ((k & 3) << 2) | (k >> 2); }
__device__ __forceinline__ void dft16(float2 (&v)[16]) {
    const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;   // cos, sin(pi/8)
    const float h = 0.70710678118654752440f;
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4(v[n2], v[n2 + 4], v[n2 + 8], v[n2 + 12]);
    // u[n2][k1] = v[n2 + 4 k1] after the inner DFT4s; twiddle by W16^(n2 k1)
    // W16^1 = c1 - i s1, W16^2 = h - i h, W16^3 = s1 - i c1, W16^4 = -i, W16^6 = -h - i h,
    // W16^9 = -c1 + i s1... only n2 k1 in {1, 2, 3, 2, 4, 6, 3, 6, 9} occur.
    v[5] = make_float2(v[5].x * c1 + v[5].y * s1, v[5].y * c1 - v[5].x * s1);        // W^1
    v[9] = make_float2((v[9].x + v[9].y) * h, (v[9].y - v[9].x) * h);               // W^2
    v[13] = make_float2(v[13].x * s1 + v[13].y * c1, v[13].y * s1 - v[13].x * c1);  // W^3
    v[6] = make_float2((v[6].x + v[6].y) * h, (v[6].y - v[6].x) * h);               // W^2
    v[10] = mul_mi(v[10]);                                                         // W^4
    v[14] = make_float2((v[14].y - v[14].x) * h, -(v[14].x + v[14].y) * h);         // W^6
    v[7] = make_float2(v[7].x * s1 + v[7].y * c1, v[7].y * s1 - v[7].x * c1);       // W^3
    v[11] = make_float2((v[11].y - v[11].x) * h, -(v[11].x + v[11].y) * h);        // W^6
    v[15] = make_float2(-v[15].x * c1 - v[15].y * s1, v[15].x * s1 - v[15].y * c1); // W^9
    // outer DFT4 over n2 for each k1: inputs v[4 k1 + n2] -> X[k1 + 4 k2] in v[4 k1 + k2]
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
}

// NS forward FFTs of the CTA's NS signals at once (radix 16, 16, 8 Stockham): the
// signals' instruction streams interleave (independent chains for the schedulers)
// and share each pass's barriers.  In: v[s][q] = x_s[t + 128 q].  Out: v[s][q] =
// X_s[t + 128 q].  sm holds NS exchange buffers of kPad slots.
template <int NS>
__device__ __forceinline__ void fft2048(float2 (&v)[NS][16], float2 *sm, const float2 *tw,
                                        const float4 *__restrict__ tw3, int t) {
    // pass 1: Ns = 1, R = 16 (no twiddles); y[16 j + r]
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        dft16(v[s]);
#pragma unroll
        for (int r = 0; r < 16; r += 2) {
            const float2 a = v[s][tr16(r)], b = v[s][tr16(r + 1)];
            *reinterpret_cast<float4 *>(sm + s * kPad + pad(16 * t + r)) = make_float4(a.x, a.y, b.x, b.y);
        }
    }
    __syncthreads();
    // pass 2: Ns = 16, R = 16; twiddles w^(8 r k), k = j mod 16; y[(j/16) 256 + k + 16 r]
    const int k = t & 15;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
#pragma unroll
        for (int r = 0; r < 16; ++r) v[s][r] = sm[s * kPad + pad(t + 128 * r)];
    }
#pragma unroll
    for (int r = 1; r < 16; r += 2) {
        const float4 w = *reinterpret_cast<const float4 *>(tw + kTw2 + k * kTw2Row + (r - 1));
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            v[s][r] = cmul(v[s][r], make_float2(w.x, w.y));
            if (r + 1 < 16) v[s][r + 1] = cmul(v[s][r + 1], make_float2(w.z, w.w));
        }
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) dft16(v[s]);
    __syncthreads();
    const int base = (t >> 4) * 256 + k;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
#pragma unroll
        for (int r = 0; r < 16; ++r) sm[s * kPad + pad(base + 16 * r)] = v[s][tr16(r)];
    }
    __syncthreads();
    // pass 3: Ns = 256, R = 8, butterflies j = t and t + 128; twiddles w^(r j); y[j + 256 r]
#pragma unroll
    for (int s = 0; s < NS; ++s) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            v[s][2 * r] = sm[s * kPad + pad(t + 256 * r)];
            v[s][2 * r + 1] = sm[s * kPad + pad(t + 128 + 256 * r)];
        }
    }
#pragma unroll
    for (int r = 1; r < 8; ++r) {
        const float4 w = __ldg(tw3 + (r - 1) * 128 + t);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            v[s][2 * r] = cmul(v[s][2 * r], make_float2(w.x, w.y));
            v[s][2 * r + 1] = cmul(v[s][2 * r + 1], make_float2(w.z, w.w));
        }
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        dft8<2>(v[s]);        // butterfly t:       v[0], v[2], ..., v[14]
        dft8<2>(v[s] + 1);    // butterfly t + 128: v[1], v[3], ..., v[15]
    }
    __syncthreads();          // shared memory free for the next transform
    // X[t + 256 r] = v[2 r], X[t + 128 + 256 r] = v[2 r + 1]  ->  v[q] = X[t + 128 q]
}

constexpr int kNS = 2;        // signals per CTA iteration
constexpr int kSmemBytes = (kNS * kN + kNS * kPad + kTwS) * 8 + 8;   // dynamic shared memory

struct FParams {
    const float2 *s;     // [n_sig][2048]
    float2 *y;           // [n_sig][2048] (may alias s exactly: a signal is read, into
                         // the prefetch stage, before the CTA writes it)
    const float2 *H;     // [2048] FFT of the filter sequence (plan-owned)
    const float2 *tw;    // [2048] twiddle table (plan-owned)
    const float4 *tw3;   // [7][128] pass-3 twiddle pairs (plan-owned)
    int64_t n_sig;
    int mode;            // 0: filter (H holds DFT(h) / N); 1: forward FFT only;
                         // 2: forward FFT scaled by 1/N (builds the plan's H from h)
};

__global__ void __launch_bounds__(kThreads, 3) filter_kernel(const FParams p) {
    // stage: the CTA's next kNS signals, prefetched with TMA bulk copies (16 KB each)
    // while the current ones are transformed; sm: kNS exchange buffers.  H and the
    // pass-3 twiddles are read through L1 (shared by the CTAs of an SM).
    extern __shared__ __align__(128) unsigned char fsm[];
    float2 *stage = reinterpret_cast<float2 *>(fsm);                 // kNS x kN
    float2 *sm = stage + kNS * kN;                                     // kNS x kPad
    float2 *tws = sm + kNS * kPad;                                     // kTwS
    uint64_t *barp = reinterpret_cast<uint64_t *>(tws + kTwS);
    uint64_t &bar = *barp;
    const int t = threadIdx.x;
    for (int i = t; i < kTwS; i += kThreads) {   // pass 2: [k][r - 1], rows of kTw2Row slots
        const int k = i / kTw2Row, rr = i % kTw2Row;
        tws[i] = p.tw[(rr < 15 ? 8 * (rr + 1) * k : 0) & (kN - 1)];
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
        float2 v[kNS][16];
        bfk::mbar_wait(&bar, phase);
        phase ^= 1u;
#pragma unroll
        for (int s = 0; s < kNS; ++s) {
            const bool ok = base + s * G < p.n_sig;
#pragma unroll
            for (int q = 0; q < 16; ++q) v[s][q] = ok ? stage[s * kN + t + 128 * q] : make_float2(0.f, 0.f);
        }
        __syncthreads();                                  // stage consumed by every thread
        if (t == 0) prefetch(base + kNS * G);
        // forward FFT, MULT by H, inverse FFT as conj(FFT(conj(.))) / N — one copy of
        // the transform code in a two-trip loop keeps register pressure at one FFT's.
        // The plan stores H / N (exact: N = 2^11), so the 1/N costs nothing here.
        const int trips = p.mode == 0 ? 2 : 1;
#pragma unroll 1
        for (int trip = 0; trip < trips; ++trip) {
            fft2048<kNS>(v, sm, tws, p.tw3, t);
            if (trip == 0 && trips == 2) {
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const float2 h = __ldg(p.H + t + 128 * q);
#pragma unroll
                    for (int s = 0; s < kNS; ++s) v[s][q] = conj2(cmul(v[s][q], h));
                }
            }
        }
#pragma unroll
        for (int s = 0; s < kNS; ++s) {
            const int64_t sig = base + s * G;
            if (sig >= p.n_sig) break;
            float2 *dst = p.y + sig * kN;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                float2 o = v[s][q];
                if (p.mode == 0) o = conj2(o);
                else if (p.mode == 2) o = make_float2(o.x * inv_n, o.y * inv_n);
                __stcs(dst + t + 128 * q, o);
            }
        }
    }
}

// tw[m] = e^{-2 pi i m / N}, evaluated in fp64 and rounded once.
__global__ void twiddle_kernel(float2 *tw) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= kTwN) return;
    double s, c;
    sincospi(-2.0 * (double)m / kN, &s, &c);
    tw[m] = make_float2((float)c, (float)s);
}

// tw3[(r - 1) 128 + t] = (w^(r t), w^(r (t + 128))), fp64-evaluated, rounded once.
__global__ void twiddle3_kernel(float4 *tw3) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= kTw3N) return;
    const int r = i / 128 + 1, t = i % 128;
    double s0, c0, s1, c1;
    sincospi(-2.0 * (double)((r * t) % kN) / kN, &s0, &c0);
    sincospi(-2.0 * (double)((r * (t + 128)) % kN) / kN, &s1, &c1);
    tw3[i] = make_float4((float)c0, (float)s0, (float)c1, (float)s1);
}

}  // namespace bff
