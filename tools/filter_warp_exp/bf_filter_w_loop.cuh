// bf_filter_w.cuh — the filter stage y = IFFT(H . FFT(s)), n = 2048, one WARP per signal
// (§III: "The filter algorithm computes IFFT(MULT(FFT(s))) where MULT is
// the pointwise multiplication by the FFT of the filter sequence and FFT sizes are all
// 2048").
//
// Each lane holds 64 of the signal's 2048 points in registers, so a transform is two
// in-register passes (DFT-32 x 2 and DFT-64 per lane) with ONE exchange through the warp's
// own shared-memory buffer in between — no CTA barriers, one exchange instead of the two
// of a 16-points-per-thread radix-16/16/8 design, and the exchanges move 128-bit pairs.
//
// Two factorisations of N = 2048 (w = e^{-2 pi i / N}, W_m = e^{-2 pi i / m}):
//   A  n = n1 + 64 n2 (n1 < 64, n2 < 32), k = k2 + 32 k1:
//        Y[n1][k2] = sum_n2 x[n1 + 64 n2] W32^(n2 k2)          (lane l: n1 = 2l, 2l + 1)
//        X[k2 + 32 k1] = sum_n1 w^(n1 k2) Y[n1][k2] W64^(n1 k1)  (lane l: k2 = l)
//      input: lane l owns the residues 2l, 2l + 1 mod 64 (128-bit loads);
//      output: lane l owns X[l + 32 m], m < 64.
//   B  n = n1 + 32 n2 (n1 < 32, n2 < 64), k = k2 + 64 k1:
//        Y[n1][k2] = sum_n2 x[n1 + 32 n2] W64^(n2 k2)            (lane l: n1 = l)
//        X[k2 + 64 k1] = sum_n1 w^(n1 k2) Y[n1][k2] W32^(n1 k1)  (lane l: k2 = 2l, 2l + 1)
//      input: lane l owns x[l + 32 m] (A's output ownership); output: residues 2l, 2l + 1
//      mod 64 (A's input ownership, 128-bit stores).
// The filter runs A forward, multiplies by H/N and conjugates in registers, runs B (the
// inverse as conj(DFT(conj(.))) / N; the plan stores H / N, exact for N = 2^11) and
// stores conj of the result: the signal is read once and written once (32 KB).
//
// The inter-pass twiddles w^(n1 k2) come from two fp64-evaluated tables (16 KB each, the
// layouts below) copied into shared memory once per CTA; the in-pass twiddles W32, W64
// are compile-time constants.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "bf_filter.cuh"   // dft4 / dft8 / cmul / mbarrier and bulk-copy helpers

namespace bffw {

constexpr int kN = 2048;
constexpr int kWarps = 12;                     // warps (signals in flight) per CTA, 1 CTA per SM
constexpr int kThreads = 32 * kWarps;
constexpr int kXBuf = kN;                     // float2 per warp buffer (16 KB: one signal)
constexpr int kTab = 32 * 32;                  // float4: twiddle table [k2][l]
constexpr int kSmemBytes = kTab * 16 + kN * 8 + kWarps * kXBuf * 8;   // table, H / N, buffers: 224 KB

// cos(2 pi m / 64), m = 0..16 (fp32-rounded; C[16] = 0 exactly)
__device__ constexpr float kC16[17] = {
    1.0f, 0.9951847195625305f, 0.9807852506637573f, 0.9569403529167175f, 0.9238795042037964f,
    0.8819212913513184f, 0.8314695954322815f, 0.7730104327201843f, 0.7071067690849304f,
    0.6343932747840881f, 0.5555702447891235f, 0.4713967442512512f, 0.3826834261417389f,
    0.290284663438797f, 0.19509032368659973f, 0.0980171412229538f, 0.0f};

// a * W64^M: W64^M = (-i)^q W64^r with M mod 64 = 16 q + r; W64^r = cos(2 pi r / 64) -
// i sin(2 pi r / 64) = C[r] - i C[16 - r].  M is a constant after unrolling at every call
// site, so the branches and the table reads fold into immediates (checked in the SASS).
__device__ __forceinline__ float2 tw64(float2 a, int M) {
    const int m = M & 63, q = m >> 4, r = m & 15;
    if (r != 0) {
        const float c = kC16[r], s = kC16[16 - r];     // W = c - i s
        a = make_float2(fmaf(a.x, c, a.y * s), fmaf(a.y, c, -(a.x * s)));
    }
    if (q == 1) a = make_float2(a.y, -a.x);                  // * (-i)
    else if (q == 2) a = make_float2(-a.x, -a.y);            // * (-1)
    else if (q == 3) a = make_float2(-a.y, a.x);             // * (+i)
    return a;
}

// DFT-32 of v[B + n], n < 32 (natural order in), n = p + 8 q, k = kq + 4 kp:
// X[k] = sum_p W8^(p kp) W32^(p kq) sum_q v[B + p + 8 q] W4^(q kq); X[k] lands in
// v[B + pos32(k)], pos32(kq + 4 kp) = kp + 8 kq.
__host__ __device__ constexpr int pos32(int k) { return (k >> 2) + 8 * (k & 3); }
template <int B>
__device__ __forceinline__ void dft32(float2 (&v)[64]) {
#pragma unroll
    for (int p = 0; p < 8; ++p) bff::dft4(v[B + p], v[B + p + 8], v[B + p + 16], v[B + p + 24]);
#pragma unroll
    for (int p = 1; p < 8; ++p) {
        v[B + p + 8] = tw64(v[B + p + 8], 2 * p);
        v[B + p + 16] = tw64(v[B + p + 16], 4 * p);
        v[B + p + 24] = tw64(v[B + p + 24], 6 * p);
    }
#pragma unroll
    for (int kq = 0; kq < 4; ++kq) bff::dft8<1>(&v[B + 8 * kq]);
}

// DFT-64 of v (natural order in), n = p + 8 q, k = kq + 8 kp: X[k] in v[pos64(k)],
// pos64(kq + 8 kp) = kp + 8 kq.
__host__ __device__ constexpr int pos64(int k) { return (k >> 3) + 8 * (k & 7); }
__device__ __forceinline__ void dft64(float2 (&v)[64]) {
#pragma unroll
    for (int p = 0; p < 8; ++p) bff::dft8<8>(&v[p]);
#pragma unroll
    for (int p = 1; p < 8; ++p) {
#pragma unroll
        for (int kq = 1; kq < 8; ++kq) v[p + 8 * kq] = tw64(v[p + 8 * kq], p * kq);
    }
#pragma unroll
    for (int kq = 0; kq < 8; ++kq) bff::dft8<1>(&v[8 * kq]);
}

// DFT-64 with TRANSPOSED input (x[n] in v[pos64(n)], i.e. x[p + 8 q] in v[q + 8 p], as
// dft64 leaves its output) and natural-order output (X[k] in v[k]).
__device__ __forceinline__ void dft64t(float2 (&v)[64]) {
#pragma unroll
    for (int p = 0; p < 8; ++p) bff::dft8<1>(&v[8 * p]);     // over q: v[8 p + kq]
#pragma unroll
    for (int p = 1; p < 8; ++p) {
#pragma unroll
        for (int kq = 1; kq < 8; ++kq) v[8 * p + kq] = tw64(v[8 * p + kq], p * kq);
    }
#pragma unroll
    for (int kq = 0; kq < 8; ++kq) bff::dft8<8>(&v[kq]);     // over p: X[kq + 8 kp] in v[kq + 8 kp]
}

// L2 prefetch of `bytes` (multiple of 16) at a 16-byte-aligned global address
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// bulk store shared -> global (bulk-group completion) and its read-completion wait
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes, uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 ::"l"(dst), "r"(bfk::smem_addr(src)), "r"(bytes), "l"(policy) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Exchange buffer: 32 rows of 32 16-byte chunks (a complex pair each), chunk c of row r at
// r * 32 + (c ^ (r & 7)): a warp access that walks the chunks of one row, or one chunk of
// 8 consecutive rows, touches 8 distinct 16-byte bank groups per quarter-warp (conflict-free
// 128-bit accesses) without padding, so 12 warps' buffers and the tables fit in 224 KB.
__device__ __forceinline__ int sw(int r, int c) { return r * 32 + (c ^ (r & 7)); }
__device__ __forceinline__ float4 ldq(const float4 *b, int i) { return b[i]; }
__device__ __forceinline__ void stq(float4 *b, int i, float2 a, float2 c) {
    b[i] = make_float4(a.x, a.y, c.x, c.y);
}

struct WParams {
    const float2 *s;     // [n_sig][2048]
    float2 *y;           // [n_sig][2048]; may alias s exactly (a warp reads its whole
                         // signal before it writes any of it)
    const float2 *H;     // [2048] H / N (mode 0)
    const float4 *tab;   // [kTab] inter-pass twiddles (plan-owned)
    int64_t n_sig;
    int mode;            // 0: filter; 1: forward FFT; 2: forward FFT scaled by 1/N
};

__global__ void __launch_bounds__(kThreads, 1) filter_warp_kernel(const WParams p) {
    extern __shared__ __align__(128) unsigned char fsm[];
    float4 *tabA = reinterpret_cast<float4 *>(fsm);
    float2 *Hs = reinterpret_cast<float2 *>(tabA + kTab);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float2 *buf = Hs + kN + warp * kXBuf;
    float4 *bq = reinterpret_cast<float4 *>(buf);
    for (int i = threadIdx.x; i < kTab; i += kThreads) tabA[i] = p.tab[i];
    if (p.mode == 0)
        for (int i = threadIdx.x; i < kN; i += kThreads) Hs[i] = p.H[i];
    __syncthreads();
    const uint64_t pol = bfk::policy_evict_first();
    const int64_t nw = (int64_t)gridDim.x * kWarps;
    const int trips = p.mode == 0 ? 2 : 1;
    for (int64_t sig = (int64_t)blockIdx.x * kWarps + warp; sig < p.n_sig; sig += nw) {
        float2 v[64];
        // the warp's next signal goes to L2 now, ~one signal's compute ahead of its loads
        if (lane == 0 && sig + nw < p.n_sig) prefetch_l2(p.s + (sig + nw) * kN, kN * 8);
        // lane owns x[2l + 64 n2], x[2l + 1 + 64 n2] -> v[n2], v[32 + n2]
        const float4 *src = reinterpret_cast<const float4 *>(p.s + sig * kN) + lane;
#pragma unroll
        for (int n2 = 0; n2 < 32; ++n2) {
            const float4 q = __ldcs(src + 32 * n2);
            v[n2] = make_float2(q.x, q.y);
            v[32 + n2] = make_float2(q.z, q.w);
        }
        // trip 0: X = DFT(s); trip 1 (filter): DFT(conj(X . H / N)) — one copy of the
        // transform code (the instruction cache holds one transform, not two)
#pragma unroll 1
        for (int trip = 0; trip < trips; ++trip) {
            dft32<0>(v);
            dft32<32>(v);
            // the previous signal's staged output must have left the buffer
            if (lane == 0) bulk_wait_read();
            __syncwarp();
            // Y[2l + j][k2] in v[32 j + pos32(k2)]: twiddle by w^((2l + j) k2), write the
            // pair to row k2 of the exchange buffer (layout [k2][n1])
#pragma unroll
            for (int k2 = 0; k2 < 32; ++k2) {
                float2 a = v[pos32(k2)], b = v[32 + pos32(k2)];
                if (k2 > 0) {
                    const float4 t = tabA[k2 * 32 + lane];
                    a = bff::cmul(a, make_float2(t.x, t.y));
                    b = bff::cmul(b, make_float2(t.z, t.w));
                }
                stq(bq, sw(k2, lane), a, b);
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 32; ++i) {             // row l: Y[2i][l], Y[2i + 1][l]
                const float4 q = ldq(bq, sw(lane, i));
                v[2 * i] = make_float2(q.x, q.y);
                v[2 * i + 1] = make_float2(q.z, q.w);
            }
            __syncwarp();                              // buffer free again
            dft64(v);                                  // X[l + 32 m] in v[pos64(m)]
            if (trip + 1 < trips) {
                // MULT: conj(X . H / N), back to the residue ownership through the buffer
#pragma unroll
                for (int m = 0; m < 64; ++m)
                    buf[lane + 32 * m] = bff::conj2(bff::cmul(v[pos64(m)], Hs[lane + 32 * m]));
                __syncwarp();
#pragma unroll
                for (int n2 = 0; n2 < 32; ++n2) {
                    const float4 q = bq[lane + 32 * n2];
                    v[n2] = make_float2(q.x, q.y);
                    v[32 + n2] = make_float2(q.z, q.w);
                }
                __syncwarp();
            }
        }
        // stage the result in natural order (X[l + 32 m]), one 16 KB bulk store:
        // filter conj(.) (the inverse's outer conjugation), mode 2 scaled by 1/N
        const float sc = p.mode == 2 ? 1.0f / kN : 1.0f, sg = p.mode == 0 ? -sc : sc;
#pragma unroll
        for (int m = 0; m < 64; ++m) {
            const float2 o = v[pos64(m)];
            buf[lane + 32 * m] = make_float2(o.x * sc, o.y * sg);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) bulk_s2g(p.y + sig * kN, buf, kN * 8, pol);
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Inter-pass twiddles, fp64-evaluated and rounded once:
//   [k2][l] = (w^(2l k2), w^((2l + 1) k2)),      k2 < 32, l < 32
__global__ void table_kernel(float4 *tab) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= kTab) return;
    const int k2 = i / 32, l = i % 32;
    const int m0 = (2 * l * k2) % kN, m1 = ((2 * l + 1) * k2) % kN;
    double s0, c0, s1, c1;
    sincospi(-2.0 * (double)m0 / kN, &s0, &c0);
    sincospi(-2.0 * (double)m1 / kN, &s1, &c1);
    tab[i] = make_float4((float)c0, (float)s0, (float)c1, (float)s1);
}

}  // namespace bffw
