// bf_api.cu — host side of libbf.so: the C ABI declared in include/bf.h.
//
// Plan object, argument validation, W relayout, block ->
// group routing (a3, stable counting sort), dispatch to the per-f kernel
// instantiation (a4+a5+a7), the f = 0 path (a8), and the host-buffer pipeline
// used for end-to-end measurement.  PAPER.md:84-86 defines the operation.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "bf.h"
#include "bf_dispatch.h"
#include "bf_host.h"
#include "bf_ffma.cuh"
#include "bf_tc.cuh"

namespace bfh {
thread_local std::string g_last_error;
}

namespace {

using bfh::fail;
using bfh::cuda_fail;
using bfh::DeviceGuard;

constexpr int kMaxGroups = 1024;
constexpr int kRouteThreads = 256;         // 8 warps
constexpr int kRouteMinTile = 512;          // small batches still spread over several CTAs
constexpr int kRouteMaxTable = 65536;      // tiles x (groups + 1) entries
constexpr int64_t kDefaultHostChunk = 2048;
constexpr int kDefaultOutExp = 12;          // int16 output: |R| < 8 fits, 2^-12 resolution
constexpr int kHostSlots = 3;
constexpr size_t kMaxProfEvents = 1 << 16;  // timed launches kept between kernel_time() calls
// AUTO variant table, per layout (measured with
// tools/sweep_f.py on c3's recipe, 100 000 blocks per f, both variants, f <= 12, every
// layout: profiles/r01_sweep_auto_v5.jsonl — both kernels with their staged bulk-store
// epilogues): the smallest f from which the tensor-core kernel is faster.  Below it
// both kernels are store-bound and within a few percent: interleaved f = 1 (equal),
// planar f <= 6 (within +-4 %), fp16 output f <= 3 (FFMA 5-16 % ahead), int16 output
// f <= 3 (FFMA 0.32 vs 0.43 ms at f = 1; profiles/r01_sweep_auto_v7.jsonl, 18-warp tensor
// kernel).  From there on
// the tensor kernel wins, by 2.2-2.6x at f = 36.  Round 2 (fp16-term tensor kernel,
// profiles/r02_sweep_auto_f16.txt): interleaved f = 1 FFMA 0.553 vs 0.560 ms, planar
// within +-3 % up to f = 6, fp16 and int16 output FFMA ahead up to f = 4 (0.36 vs 0.37,
// 0.45 vs 0.47 ms), the tensor kernel from f = 5; with two R stages for fp16 output the
// tensor kernel leads there from f = 3 (0.307 vs 0.322 ms), and with the staged two-stage
// int16 epilogue from f = 4 (0.429 vs 0.445 ms; profiles/r02_rstage_ring.txt); after the
// round-2 kernel work the tensor kernel also leads interleaved from f = 1 (0.548 vs 0.554 ms)
// and planar from f = 2 (0.563 vs 0.571; f = 1 and 6 within 0.2 %; profiles/
// r02_sweep_auto_final.txt).
constexpr int kAutoTensorMinF[4] = {1, 2, 3, 4};   // [layout]
// bf_apply_batch: 1 = one contiguous cost range of all the launch's jobs per CTA, 0 = every
// job split over all CTAs
constexpr int kBatchSplit = 1;

BfKernelTable g_table;      // FFMA kernels [f][layout]
BfKernelTable g_table_tc;   // tcgen05 split-TF32 kernels [f][layout]
BfKernelEntry g_server[4];  // slot-server kernels [layout]
std::once_flag g_table_once;

void init_table() {
    std::memset(&g_table, 0, sizeof(g_table));
    std::memset(&g_table_tc, 0, sizeof(g_table_tc));
    bf_register_f01_06(g_table, g_table_tc);
    bf_register_f07_12(g_table, g_table_tc);
    bf_register_f13_18(g_table, g_table_tc);
    bf_register_f19_24(g_table, g_table_tc);
    bf_register_f25_30(g_table, g_table_tc);
    bf_register_f31_36(g_table, g_table_tc);
    bf_register_batch(g_table_tc);
    bf_register_server(g_server);
}

// ---------------------------------------------------------------------------
// Device helpers: W relayout (a2) and routing (a3)
// ---------------------------------------------------------------------------

// Wp[g][k][j][ag] = float4(re w[8ag+2j][k], re w[8ag+2j+1][k], im w[8ag+2j][k],
// im w[8ag+2j+1][k]) — the layout bf_ffma_kernel reads with one conflict-free
// LDS.128 per (k, j); re and im of one antenna land in same-parity registers.
__global__ void bf_relayout_w(const float *__restrict__ W, int n_groups, int F, int layout,
                              float4 *__restrict__ Wp) {
    const int64_t total = (int64_t)n_groups * F * 32;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = idx / (F * 32);
        const int rem = (int)(idx - g * F * 32);
        const int k = rem / 32, j = (rem % 32) / 8, ag = rem % 8;
        const int i0 = ag * 8 + 2 * j, i1 = i0 + 1;
        float4 v;
        if (layout != BF_LAYOUT_PLANAR) {
            const float *Wg = W + g * 64 * F * 2;
            v = make_float4(Wg[(i0 * F + k) * 2], Wg[(i1 * F + k) * 2],
                            Wg[(i0 * F + k) * 2 + 1], Wg[(i1 * F + k) * 2 + 1]);
        } else {
            const float *Wr = W + g * 2 * 64 * F, *Wi = Wr + 64 * F;
            v = make_float4(Wr[i0 * F + k], Wr[i1 * F + k], Wi[i0 * F + k], Wi[i1 * F + k]);
        }
        Wp[idx] = v;
    }
}

// Builds the pre-split B image of one or more groups (bf_set_precoders):
// img[g][t][kc][ng][r][e] = term t of B'[n = 8 ng + r][kk = 4 kc + e], t = 0: W1, 1: W2.
__global__ void bf_tc_build_wimg(const float *__restrict__ W, int F, int layout,
                                 uint32_t *__restrict__ img, int32_t *__restrict__ wflags) {
    // One CTA per group.  Image: [W1 fp16 core matrices: KP/8 K-chunks x 16 row groups x
    // 8 rows x 8 halves] then [W2, the same layout], with B'[n][kk] the real embedding
    // (n = 2i + c_out, kk = 2k + c_in) of W scaled by 2^tau, tau placing the group's largest
    // component in [2^14, 2^15); W1 = tf32(B'), W2 = tf32(B' - W1) (round to nearest, ties
    // away), each rounded to fp16 (exact in fp16's normal range; B' = W1 + W2 + W3 with
    // |W3| <= 2^-22 |B'|).  Flags: bit 0 = the group is exact in one fp16
    // term (W2 == 0 and W1 exact: identity, selection, small integers — the kernel then
    // multiplies S3 instead of W2); bit 1 = outside the tensor domain (an entry not 0 and
    // not in [2^-40, 2^40), NaN, Inf, or a nonzero element, max(|re|, |im|), more than
    // kRelRange binades below the largest component); bits 8-15 = tau + 128.
    const int g = blockIdx.x;
    const int KP = bftc::kp_of(F);
    __shared__ int s_emax;
    if (threadIdx.x == 0) s_emax = 0;
    __syncthreads();
    const uint32_t *wg = reinterpret_cast<const uint32_t *>(W) + (int64_t)g * 128 * F;
    auto comp = [&](int i, int k, int c) -> uint32_t {   // bits of Wr (c = 0) / Wi (c = 1)
        return layout != BF_LAYOUT_PLANAR ? wg[(i * F + k) * 2 + c] : wg[c * 64 * F + i * F + k];
    };
    int emax = 0, bad = 0;
    for (int e = threadIdx.x; e < 64 * F; e += blockDim.x) {
        const uint32_t ur = comp(e / F, e % F, 0) & 0x7FFFFFFFu, ui = comp(e / F, e % F, 1) & 0x7FFFFFFFu;
        bad |= !(ur == 0u || (ur >= bftc::kDomLo && ur < bftc::kDomHi));
        bad |= !(ui == 0u || (ui >= bftc::kDomLo && ui < bftc::kDomHi));
        emax = max(emax, (int)(max(ur, ui) >> 23));
    }
    atomicMax(&s_emax, emax);
    __syncthreads();
    emax = s_emax;
    const uint32_t lo = (uint32_t)(emax - bftc::kRelRange) << 23;
    for (int e = threadIdx.x; e < 64 * F; e += blockDim.x) {
        const uint32_t ur = comp(e / F, e % F, 0) & 0x7FFFFFFFu, ui = comp(e / F, e % F, 1) & 0x7FFFFFFFu;
        bad |= emax != 0 && max(ur, ui) - 1u < lo - 1u;
    }
    bad = __syncthreads_or(bad);
    const int tau = emax != 0 && !bad ? 141 - emax : 0;
    const float sc = __uint_as_float((uint32_t)(127 + tau) << 23);
    const int half_words = KP * 64;                       // 32-bit words per part
    uint32_t *out = img + (int64_t)g * 2 * half_words;
    int inexact = 0;
    for (int w = threadIdx.x; w < half_words; w += blockDim.x) {
        const int kc = w / 512, r2 = w % 512;
        const int ng = r2 / 32, r = (r2 / 4) % 8, e2 = r2 % 4;
        const int n = ng * 8 + r, i = n >> 1, cout = n & 1;
        float t1[2], t2[2];
        for (int h = 0; h < 2; ++h) {
            const int kk = kc * 8 + 2 * e2 + h, k = kk >> 1, cin = kk & 1;
            float v = 0.0f;
            if (k < F && !bad) {
                const float wr = __uint_as_float(comp(i, k, 0)), wi = __uint_as_float(comp(i, k, 1));
                // B'[2i][2k] = wr, B'[2i][2k+1] = -wi, B'[2i+1][2k] = wi, B'[2i+1][2k+1] = wr
                v = (cout == 0 ? (cin == 0 ? wr : -wi) : (cin == 0 ? wi : wr)) * sc;
            }
            t1[h] = tc::to_tf32(v);
            t2[h] = tc::to_tf32(v - t1[h]);
            inexact |= t2[h] != 0.0f || __half2float(__float2half_rn(t1[h])) != t1[h];
        }
        out[w] = tc::pack_f16x2(t1[0], t1[1]);
        out[half_words + w] = tc::pack_f16x2(t2[0], t2[1]);
    }
    inexact = __syncthreads_or(inexact);
    if (threadIdx.x == 0) wflags[g] = (inexact ? 0 : 1) | (bad ? 2 : 0) | ((tau + 128) << 8);
}

// a8 with tags (f = 0): +0.0 for every block whose tag is in [0, G); blocks with other
// tags are left unwritten, as bf.h states, and flagged for BF_CHECK=1.
__global__ void bf_zero_tagged(const int32_t *__restrict__ gidx, int64_t n, int G,
                               int vec_per_block, uint4 *__restrict__ R, int32_t *__restrict__ err) {
    const int64_t total = n * vec_per_block;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t blk = idx / vec_per_block;
        const int32_t g = __ldg(gidx + blk);
        if ((unsigned)g < (unsigned)G) R[idx] = make_uint4(0u, 0u, 0u, 0u);
        else if (idx == blk * vec_per_block) atomicOr(err, 1);
    }
}

__device__ __forceinline__ int route_bin(int32_t g, int G) {
    return (unsigned)g < (unsigned)G ? g : G;   // invalid tags -> bin G (sorted last)
}

// Pass 1: per-tile histogram -> table[tile][bin], bins 0..G (G = invalid).
__global__ void bf_route_hist(const int32_t *__restrict__ gidx, int64_t n, int G, int tile,
                              int32_t *__restrict__ table, int32_t *__restrict__ err) {
    extern __shared__ int32_t hist[];
    for (int b = threadIdx.x; b <= G; b += blockDim.x) hist[b] = 0;
    __syncthreads();
    const int64_t ts = (int64_t)blockIdx.x * tile;
    const int64_t te = min(n, ts + tile);
    int bad = 0;
    for (int64_t i = ts + threadIdx.x; i < te; i += blockDim.x) {
        const int b = route_bin(__ldg(gidx + i), G);
        bad |= (b == G);
        atomicAdd(&hist[b], 1);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1);
    for (int b = threadIdx.x; b <= G; b += blockDim.x)
        table[(int64_t)blockIdx.x * (G + 1) + b] = hist[b];
}

// Pass 2 (one CTA of 1024 threads per bin): table[tile][bin] <- start of the tile's
// items within the bin (exclusive scan of the bin's column over the tiles, 1024 tiles
// per step, every load in flight at once); bin_tot[bin] <- the bin's total.
__global__ void __launch_bounds__(1024) bf_route_colscan(int32_t *__restrict__ table, int P, int G,
                                                         int32_t *__restrict__ bin_tot) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t btot;
    const int b = blockIdx.x, nb = G + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t carry = 0;
    for (int t0 = 0; t0 < P; t0 += 1024) {
        const int t = t0 + threadIdx.x;
        const int32_t v = t < P ? table[(int64_t)t * nb + b] : 0;
        int32_t inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += u;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {                          // exclusive prefix of the 32 warp totals
            const int32_t w = wsum[lane];
            int32_t wi = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int32_t u = __shfl_up_sync(0xffffffffu, wi, d);
                if (lane >= d) wi += u;
            }
            wsum[lane] = wi - w;
            if (lane == 31) btot = wi;
        }
        __syncthreads();
        if (t < P) table[(int64_t)t * nb + b] = carry + wsum[warp] + inc - v;
        carry += btot;
        __syncthreads();                          // wsum / btot are reused by the next step
    }
    if (threadIdx.x == 0) bin_tot[b] = carry;
}

// Exclusive scan of the G + 1 bin totals into start[] (shared), by warp 0.
__device__ __forceinline__ void bin_starts(const int32_t *__restrict__ bin_tot, int nb,
                                           int32_t *start) {
    const int lane = threadIdx.x & 31;
    if ((threadIdx.x >> 5) == 0) {
        int32_t carry = 0;
        for (int b0 = 0; b0 < nb; b0 += 32) {
            const int b = b0 + lane;
            const int32_t v = b < nb ? bin_tot[b] : 0;
            int32_t inc = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int32_t u = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += u;
            }
            if (b < nb) start[b] = carry + inc - v;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
}

// Pass 3: stable scatter.  Each warp owns a contiguous sub-tile; ranks come
// from __match_any_sync so the output order is (bin, block id) exactly.
__global__ void bf_route_scatter(const int32_t *__restrict__ gidx, int64_t n, int G, int tile,
                                 const int32_t *__restrict__ table,
                                 const int32_t *__restrict__ bin_tot, int32_t *__restrict__ perm,
                                 int32_t *__restrict__ offsets) {
    extern __shared__ int32_t cnt[];   // [8][G + 1], then start[G + 1]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nb = G + 1;
    int32_t *start = cnt + 8 * nb;
    for (int e = threadIdx.x; e < 8 * nb; e += blockDim.x) cnt[e] = 0;
    bin_starts(bin_tot, nb, start);
    __syncthreads();
    if (blockIdx.x == 0) {                // offsets[0..G] = bin starts, offsets[G + 1] = n
        for (int b = threadIdx.x; b < nb; b += blockDim.x) offsets[b] = start[b];
        if (threadIdx.x == 0) offsets[nb] = (int32_t)n;
    }
    const int64_t ts = (int64_t)blockIdx.x * tile;
    const int per_warp = tile / 8;
    const int64_t ws = ts + (int64_t)warp * per_warp;
    const int64_t we = min(n, ws + per_warp);
    int32_t *mycnt = cnt + warp * nb;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t base = ws; base < we; base += 32) {
        const int64_t i = base + lane;
        const int b = i < we ? route_bin(__ldg(gidx + i), G) : -1;
        const unsigned m = __match_any_sync(0xffffffffu, b);
        if (b >= 0 && (m & lt) == 0) mycnt[b] += __popc(m);
        __syncwarp();
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        int32_t run = start[b] + table[(int64_t)blockIdx.x * nb + b];
        for (int w = 0; w < 8; ++w) {
            const int32_t c = cnt[w * nb + b];
            cnt[w * nb + b] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int64_t base = ws; base < we; base += 32) {
        const int64_t i = base + lane;
        const int b = i < we ? route_bin(__ldg(gidx + i), G) : -1;
        const unsigned m = __match_any_sync(0xffffffffu, b);
        if (b >= 0) {
            const int32_t pos = mycnt[b] + __popc(m & lt);
            perm[pos] = (int32_t)i;
        }
        __syncwarp();
        if (b >= 0 && (m & lt) == 0) mycnt[b] += __popc(m);
        __syncwarp();
    }
}

// Small batches (n <= kRouteSmallN, G <= kRouteSmallG): the whole stable counting
// sort in ONE CTA of 32 warps — per-warp histograms (match_any), a bin-major
// prefix, then the stable scatter — one launch instead of three (streaming
// chunks of a few thousand blocks are latency-bound, bench --config c5).
constexpr int kRouteSmallN = 16384;
constexpr int kRouteSmallG = 256;

__global__ void __launch_bounds__(1024) bf_route_small(const int32_t *__restrict__ gidx, int n, int G,
                                                       int32_t *__restrict__ perm,
                                                       int32_t *__restrict__ offsets,
                                                       int32_t *__restrict__ err) {
    extern __shared__ int32_t cnt[];   // [32][G + 1], then tot[G + 1]
    constexpr int kPer = kRouteSmallN / 1024;          // tags per lane, kept in registers
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nb = G + 1;
    int32_t *tot = cnt + 32 * nb;
    // every tag is loaded once, all loads in flight together (no dependent chain)
    const int per = ((n + 31) / 32 + 31) / 32 * 32;    // items per warp, multiple of 32
    const int ws = warp * per, we = min(n, ws + per);
    int bins[kPer];
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        const int i = ws + 32 * r + lane;
        bins[r] = (32 * r < per && i < we) ? route_bin(__ldg(gidx + i), G) : -1;
    }
    for (int e = threadIdx.x; e < 33 * nb; e += blockDim.x) cnt[e] = 0;
    __syncthreads();
    int32_t *mycnt = cnt + warp * nb;
    const unsigned lt = (1u << lane) - 1u;
    int bad = 0;
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        if (32 * r >= per) break;
        const int b = bins[r];
        bad |= (b == G);
        const unsigned m = __match_any_sync(0xffffffffu, b);
        if (b >= 0 && (m & lt) == 0) mycnt[b] += __popc(m);
        __syncwarp();
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) *err = 1;
    // per bin, exclusive prefix over the 32 warps: one warp per bin, lane = warp index
    for (int b = warp; b < nb; b += 32) {
        const int32_t c = cnt[lane * nb + b];
        int32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += u;
        }
        cnt[lane * nb + b] = inc - c;
        if (lane == 31) tot[b] = inc;
    }
    __syncthreads();
    if (warp == 0) {                                          // exclusive scan over bins
        int32_t carry = 0;
        for (int b0 = 0; b0 < nb; b0 += 32) {
            const int b = b0 + lane;
            const int32_t v = b < nb ? tot[b] : 0;
            int32_t inc = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int32_t u = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += u;
            }
            if (b < nb) tot[b] = carry + inc - v;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x) offsets[b] = tot[b];
    if (threadIdx.x == 0) offsets[nb] = n;
    for (int e = threadIdx.x; e < 32 * nb; e += blockDim.x) cnt[e] += tot[e % nb];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
        if (32 * r >= per) break;
        const int b = bins[r];
        const unsigned m = __match_any_sync(0xffffffffu, b);
        if (b >= 0) perm[mycnt[b] + __popc(m & lt)] = ws + 32 * r + lane;
        __syncwarp();
        if (b >= 0 && (m & lt) == 0) mycnt[b] += __popc(m);
        __syncwarp();
    }
}

template <typename T>
bf_status grow(T **ptr, int64_t *cap, int64_t need, const char *what) {
    if (*cap >= need) return BF_OK;
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    *cap = 0;
    const int64_t n = std::max<int64_t>(need, 1);
    if (cudaMalloc(reinterpret_cast<void **>(ptr), n * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        return fail(BF_ERR_OUT_OF_MEMORY, "cudaMalloc of %s (%lld bytes) failed", what,
                    (long long)(n * sizeof(T)));
    }
    *cap = n;
    return BF_OK;
}

bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

}  // namespace

struct bf_plan_s {
    int n_ant = 64, f = 0, b = 60, layout = 0, device = 0, num_sms = 0;
    int n_groups = 0;
    BfKernelEntry kern{};       // FFMA kernel of this (f, layout)
    BfKernelEntry kern_tc{};    // tensor-core kernel of this (f, layout)
    int ctas_per_sm = 0;
    int sm_share = 0;           // bf_plan_set_sm_share (0 = every SM)
    int out_exp = kDefaultOutExp;   // int16 output: R x 2^out_exp before the rounding
    int variant = BF_VARIANT_AUTO;
    float4 *Wp = nullptr;       // FFMA precoder image
    int64_t Wp_cap = 0;
    float *Wimg = nullptr;      // tensor-core (pre-split B) precoder image
    int64_t Wimg_cap = 0;
    int32_t *wexact = nullptr;  // per group: bit 0 W exactly tf32, bit 1 outside the tensor domain
    int64_t wexact_cap = 0;
    bool w_in_domain = true;    // every group inside the tensor domain (AUTO may pick tensor)
    // routing workspace
    int32_t *perm = nullptr, *table = nullptr, *offsets = nullptr, *err = nullptr;
    int64_t perm_cap = 0, table_cap = 0, offsets_cap = 0, err_cap = 0;
    // host pipeline
    int64_t host_chunk = kDefaultHostChunk, slot_cap = 0;
    float *hS[kHostSlots] = {}, *hR[kHostSlots] = {};
    int32_t *hG[kHostSlots] = {};
    int64_t hS_cap[kHostSlots] = {}, hR_cap[kHostSlots] = {}, hG_cap[kHostSlots] = {};
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d[kHostSlots] = {}, ev_comp[kHostSlots] = {}, ev_d2h[kHostSlots] = {},
                ev_start = nullptr;
    // instrumentation
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;
    int64_t launches = 0;
};

namespace {

bf_status launched(bf_plan_t p, const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, what);
    ++p->launches;
    return BF_OK;
}

// Stable counting sort of blocks by tag into perm (+offsets).
bf_status route(bf_plan_t p, const int32_t *gidx, int64_t n, int32_t *perm, int32_t *offsets,
                cudaStream_t st) {
    const int G = p->n_groups;
    bf_status s;
    if (n <= kRouteSmallN && G <= kRouteSmallG) {
        if ((s = grow(&p->err, &p->err_cap, 1, "routing flag")) != BF_OK) return s;
        BF_CUDA(cudaMemsetAsync(p->err, 0, sizeof(int32_t), st));
        const size_t smem = 33 * (G + 1) * sizeof(int32_t);
        bf_route_small<<<1, 1024, smem, st>>>(gidx, (int)n, G, perm, offsets, p->err);
        return launched(p, "bf_route_small launch");
    }
    int64_t tile = kRouteMinTile;
    const int64_t max_tiles = std::max<int64_t>(1, kRouteMaxTable / (G + 1));
    if ((n + tile - 1) / tile > max_tiles) tile = (n + max_tiles - 1) / max_tiles;
    tile = (tile + kRouteThreads - 1) / kRouteThreads * kRouteThreads;
    const int64_t P = (n + tile - 1) / tile;
    // table [P][G + 1] of per-tile bin counts, then the G + 1 bin totals
    if ((s = grow(&p->table, &p->table_cap, (P + 1) * (G + 1), "routing table")) != BF_OK) return s;
    int32_t *bin_tot = p->table + P * (G + 1);
    if ((s = grow(&p->err, &p->err_cap, 1, "routing flag")) != BF_OK) return s;
    BF_CUDA(cudaMemsetAsync(p->err, 0, sizeof(int32_t), st));
    const size_t hist_smem = (G + 1) * sizeof(int32_t);
    bf_route_hist<<<(unsigned)P, kRouteThreads, hist_smem, st>>>(gidx, n, G, (int)tile,
                                                                  p->table, p->err);
    if ((s = launched(p, "bf_route_hist launch")) != BF_OK) return s;
    bf_route_colscan<<<(unsigned)(G + 1), 1024, 0, st>>>(p->table, (int)P, G, bin_tot);
    if ((s = launched(p, "bf_route_colscan launch")) != BF_OK) return s;
    const size_t sc_smem = 9 * (G + 1) * sizeof(int32_t);
    bf_route_scatter<<<(unsigned)P, kRouteThreads, sc_smem, st>>>(gidx, n, G, (int)tile,
                                                                    p->table, bin_tot, perm,
                                                                    offsets);
    if ((s = launched(p, "bf_route_scatter launch")) != BF_OK) return s;
    return BF_OK;
}

bf_status check_tags_if_requested(bf_plan_t p, cudaStream_t st) {
    const char *env = std::getenv("BF_CHECK");
    if (!env || std::strcmp(env, "1") != 0) return BF_OK;
    int32_t h = 0;
    BF_CUDA(cudaMemcpyAsync(&h, p->err, sizeof(h), cudaMemcpyDeviceToHost, st));
    BF_CUDA(cudaStreamSynchronize(st));
    if (h) return fail(BF_ERR_INVALID_VALUE, "group_idx has entries outside [0, %d)", p->n_groups);
    return BF_OK;
}

// Per-f variant table: which kernel BF_VARIANT_AUTO runs.
// Precoders outside the tensor domain send AUTO to the FFMA kernel; an
// explicit BF_VARIANT_TENSOR still runs the tensor kernel, whose fix-up then recomputes
// those groups' blocks with FFMA arithmetic.
bool use_tensor(bf_plan_t p) {
    if (p->variant == BF_VARIANT_TENSOR) return true;
    if (p->variant == BF_VARIANT_FFMA) return false;
    return p->w_in_domain && p->f >= kAutoTensorMinF[p->layout];
}

int sms_used(bf_plan_t p) {
    return p->sm_share > 0 ? std::min(p->sm_share, p->num_sms) : p->num_sms;
}

// Grid of the beamforming kernel for n_items blocks: persistent CTAs, one per SM
// (tensor) or ctas_per_sm per SM (FFMA), over the plan's SM share.
int grid_for(bf_plan_t p, int64_t n_items, bool tensor) {
    const int64_t cap = (int64_t)sms_used(p) * (tensor ? 1 : std::max(1, p->ctas_per_sm));
    return (int)std::max<int64_t>(1, std::min<int64_t>(n_items, cap));
}

// CUDA events around a plan's beamforming kernel when profiling is on (bench.py).
bf_status prof_begin(bf_plan_t p, cudaStream_t st, cudaEvent_t *e1) {
    *e1 = nullptr;
    if (!p->profiling || p->prof_used >= kMaxProfEvents) return BF_OK;
    if (p->prof_used == p->prof_events.size()) {
        cudaEvent_t a, b;
        BF_CUDA(cudaEventCreate(&a));
        BF_CUDA(cudaEventCreate(&b));
        p->prof_events.emplace_back(a, b);
    }
    BF_CUDA(cudaEventRecord(p->prof_events[p->prof_used].first, st));
    *e1 = p->prof_events[p->prof_used].second;
    ++p->prof_used;
    return BF_OK;
}

bftc::TcJob tc_job(bf_plan_t p, const void *S, const int32_t *perm, const int32_t *offsets,
                   void *R, int64_t n) {
    bftc::TcJob j{};
    j.Wimg = p->Wimg;
    j.Wp = p->Wp;
    j.S = static_cast<const float *>(S);
    j.perm = perm;
    j.offsets = offsets;
    j.wexact = p->wexact;
    j.R = static_cast<float *>(R);
    j.n_items = n;
    j.n_groups = p->n_groups;
    j.f = p->f;
    j.out_scale = ldexpf(1.0f, p->out_exp);
    return j;
}

// Device-resident apply of routed blocks (validated arguments): perm / offsets
// from route(), or both NULL for untagged blocks (all group 0).
bf_status apply_routed(bf_plan_t p, const void *S, const int32_t *perm, const int32_t *offsets,
                       void *R, int64_t n, cudaStream_t st) {
    if (n == 0) return BF_OK;
    const size_t r_bytes = (size_t)n * bfk::r_block_bytes(p->layout);
    if (p->f == 0) {   // a8: the empty sum, +0.0f everywhere
        BF_CUDA(cudaMemsetAsync(R, 0, r_bytes, st));
        return BF_OK;
    }
    bf_status s;
    bfk::KParams kp{};
    kp.Wp = p->Wp;
    kp.S = static_cast<const float *>(S);
    kp.R = static_cast<float *>(R);
    kp.n_items = n;
    kp.n_groups = p->n_groups;
    kp.perm = perm;
    kp.offsets = offsets;
    kp.out_scale = ldexpf(1.0f, p->out_exp);
    const bool tensor = use_tensor(p);
    const int grid = grid_for(p, n, tensor);
    const BfKernelEntry &kern = tensor ? p->kern_tc : p->kern;
    bftc::TcParams tp{};
    tp.job[0] = tc_job(p, S, perm, offsets, R, n);
    tp.n_jobs = 1;
    cudaEvent_t e1;
    if ((s = prof_begin(p, st, &e1)) != BF_OK) return s;
    void *args_ffma[] = {&kp};
    void *args_tc[] = {&tp};
    cudaError_t e = cudaLaunchKernel(kern.fn, dim3(grid),
                                     dim3(tensor ? bftc::kThreads : bfk::kThreads),
                                     tensor ? args_tc : args_ffma, (size_t)kern.smem_bytes, st);
    if (e != cudaSuccess) return cuda_fail(e, "beamforming kernel launch");
    if ((s = launched(p, "beamforming kernel launch")) != BF_OK) return s;
    if (e1) BF_CUDA(cudaEventRecord(e1, st));
    return BF_OK;
}

// One launch of the runtime-f tensor kernel over up to kMaxJobs validated jobs of
// tensor-variant plans (same device and layout); profiling / launch count on the
// first job's plan.
bf_status launch_batch(const bf_batch_job *jobs, int n, cudaStream_t st) {
    bf_plan_t p0 = jobs[0].plan;
    const BfKernelEntry &kern = g_table_tc[0][p0->layout];   // smem attribute set at plan create
    bftc::TcParams tp{};
    int64_t tiles = 0;
    for (int i = 0; i < n; ++i) {
        tp.job[i] = tc_job(jobs[i].plan, jobs[i].S_dev, jobs[i].perm_dev, jobs[i].offsets_dev,
                           jobs[i].R_dev, jobs[i].n_blocks);
        tiles += (jobs[i].n_blocks + 1) / 2;
    }
    tp.n_jobs = n;
    // how the jobs are split over the CTAs (TcParams.split): BF_BATCH_SPLIT=0|1 for experiments
    static const int split = [] {
        const char *e = std::getenv("BF_BATCH_SPLIT");
        return e ? (std::atoi(e) != 0 ? 1 : 0) : kBatchSplit;
    }();
    tp.split = split;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, sms_used(p0)));
    bf_status s;
    cudaEvent_t e1;
    if ((s = prof_begin(p0, st, &e1)) != BF_OK) return s;
    void *args[] = {&tp};
    cudaError_t e = cudaLaunchKernel(kern.fn, dim3(grid), dim3(bftc::kThreads), args,
                                     (size_t)kern.smem_bytes, st);
    if (e != cudaSuccess) return cuda_fail(e, "batched beamforming kernel launch");
    if ((s = launched(p0, "batched beamforming kernel launch")) != BF_OK) return s;
    if (e1) BF_CUDA(cudaEventRecord(e1, st));
    return BF_OK;
}

// Device-resident apply (validated arguments): routes tagged blocks into the
// plan's workspace, then applies.
bf_status apply_device(bf_plan_t p, const void *S, const int32_t *gidx, void *R, int64_t n,
                       cudaStream_t st) {
    if (n == 0) return BF_OK;
    if (p->f == 0 && gidx) {   // a8 with tags: zero the validly tagged blocks only
        bf_status s;
        if ((s = grow(&p->err, &p->err_cap, 1, "routing flag")) != BF_OK) return s;
        BF_CUDA(cudaMemsetAsync(p->err, 0, sizeof(int32_t), st));
        const int vpb = bfk::r_block_bytes(p->layout) / 16;
        const int64_t total = n * vpb;
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)p->num_sms * 8);
        bf_zero_tagged<<<blocks, 256, 0, st>>>(gidx, n, p->n_groups, vpb, static_cast<uint4 *>(R),
                                                p->err);
        if ((s = launched(p, "bf_zero_tagged launch")) != BF_OK) return s;
        return check_tags_if_requested(p, st);
    }
    // tagged blocks are always routed — also with one group, so that tags outside
    // [0, n_groups) leave their blocks unwritten as bf.h states (a caller with one W
    // and no tags passes group_idx = NULL and skips the routing)
    if (p->f > 0 && gidx) {
        bf_status s;
        if ((s = grow(&p->perm, &p->perm_cap, n, "perm")) != BF_OK) return s;
        if ((s = grow(&p->offsets, &p->offsets_cap, p->n_groups + 2, "offsets")) != BF_OK) return s;
        if ((s = route(p, gidx, n, p->perm, p->offsets, st)) != BF_OK) return s;
        if ((s = check_tags_if_requested(p, st)) != BF_OK) return s;
        return apply_routed(p, S, p->perm, p->offsets, R, n, st);
    }
    return apply_routed(p, S, nullptr, nullptr, R, n, st);
}

bf_status ensure_host_pipeline(bf_plan_t p, bool tagged) {
    bf_status s;
    const int64_t C = p->host_chunk;
    for (int i = 0; i < kHostSlots; ++i) {
        if (p->f > 0 &&
            (s = grow(&p->hS[i], &p->hS_cap[i], C * 120 * p->f, "host-pipeline S slot")) != BF_OK)
            return s;
        if ((s = grow(&p->hR[i], &p->hR_cap[i], C * (bfk::r_block_bytes(p->layout) / 4),
                      "host-pipeline R slot")) !=
            BF_OK)
            return s;
        if (tagged && (s = grow(&p->hG[i], &p->hG_cap[i], C, "host-pipeline tag slot")) != BF_OK)
            return s;
    }
    if (!p->s_h2d) {
        BF_CUDA(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
        BF_CUDA(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking));
        BF_CUDA(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming));
        for (int i = 0; i < kHostSlots; ++i) {
            BF_CUDA(cudaEventCreateWithFlags(&p->ev_h2d[i], cudaEventDisableTiming));
            BF_CUDA(cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming));
            BF_CUDA(cudaEventCreateWithFlags(&p->ev_d2h[i], cudaEventDisableTiming));
            BF_CUDA(cudaEventRecord(p->ev_d2h[i], p->s_d2h));
        }
    }
    return BF_OK;
}

bf_status validate_layout_and_dims(int n_ant, int f, int b, int layout) {
    if (n_ant < 1 || f < 0 || b < 1)
        return fail(BF_ERR_INVALID_VALUE, "dimensions must satisfy n_ant >= 1, f >= 0, b >= 1 "
                                          "(got n_ant=%d f=%d b=%d)", n_ant, f, b);
    if (layout != BF_LAYOUT_INTERLEAVED && layout != BF_LAYOUT_PLANAR &&
        layout != BF_LAYOUT_INTERLEAVED_F16OUT && layout != BF_LAYOUT_INTERLEAVED_I16OUT)
        return fail(BF_ERR_INVALID_VALUE, "unknown layout %d", layout);
    if (n_ant != bfk::kAnt || b != bfk::kB || f > bfk::kMaxF)
        return fail(BF_ERR_UNSUPPORTED, "compiled domain is n_ant=64, b=60, 0<=f<=36 "
                                        "(got n_ant=%d f=%d b=%d)", n_ant, f, b);
    return BF_OK;
}

}  // namespace

extern "C" {

int bf_version(void) { return BF_VERSION; }

const char *bf_status_string(bf_status s) {
    switch (s) {
        case BF_OK: return "BF_OK";
        case BF_ERR_INVALID_VALUE: return "BF_ERR_INVALID_VALUE";
        case BF_ERR_UNSUPPORTED: return "BF_ERR_UNSUPPORTED";
        case BF_ERR_NO_PRECODERS: return "BF_ERR_NO_PRECODERS";
        case BF_ERR_MISALIGNED: return "BF_ERR_MISALIGNED";
        case BF_ERR_OUT_OF_MEMORY: return "BF_ERR_OUT_OF_MEMORY";
        case BF_ERR_CUDA: return "BF_ERR_CUDA";
        case BF_ERR_NO_DEVICE: return "BF_ERR_NO_DEVICE";
    }
    return "BF_ERR_UNKNOWN";
}

const char *bf_last_error(void) { return bfh::g_last_error.c_str(); }

bf_status bf_plan_create(int n_ant, int f, int b, int layout, bf_plan_t *out) {
    if (!out) return fail(BF_ERR_INVALID_VALUE, "out is NULL");
    bf_status s = validate_layout_and_dims(n_ant, f, b, layout);
    if (s != BF_OK) return s;
    int dev = 0, count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(BF_ERR_NO_DEVICE, "no CUDA device: %s", cudaGetErrorString(e));
    }
    BF_CUDA(cudaGetDevice(&dev));
    std::call_once(g_table_once, init_table);
    bf_plan_t p = new (std::nothrow) bf_plan_s();
    if (!p) return fail(BF_ERR_OUT_OF_MEMORY, "host allocation of the plan failed");
    p->n_ant = n_ant;
    p->f = f;
    p->b = b;
    p->layout = layout;
    p->device = dev;
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaGetDeviceProperties"); }
    if (prop.major != 10) {
        delete p;
        return fail(BF_ERR_UNSUPPORTED, "libbf.so is built for sm_100a; device %d is sm_%d%d",
                    dev, prop.major, prop.minor);
    }
    p->num_sms = prop.multiProcessorCount;
    if (f > 0) {
        p->kern = g_table[f][layout];
        e = cudaFuncSetAttribute(p->kern.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 p->kern.smem_bytes);
        if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaFuncSetAttribute"); }
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p->ctas_per_sm, p->kern.fn,
                                                          bfk::kThreads, p->kern.smem_bytes);
        if (e != cudaSuccess) { delete p; return cuda_fail(e, "occupancy query"); }
        if (p->ctas_per_sm < 1) {
            delete p;
            return fail(BF_ERR_UNSUPPORTED, "kernel for f=%d cannot be resident", f);
        }
        p->kern_tc = g_table_tc[f][layout];
        e = cudaFuncSetAttribute(p->kern_tc.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 p->kern_tc.smem_bytes);
        if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaFuncSetAttribute (tc)"); }
        // the runtime-f kernel of bf_apply_batch for this layout (idempotent per device)
        const BfKernelEntry &kb = g_table_tc[0][layout];
        e = cudaFuncSetAttribute(kb.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kb.smem_bytes);
        if (e != cudaSuccess) { delete p; return cuda_fail(e, "cudaFuncSetAttribute (batch)"); }
    }
    *out = p;
    return BF_OK;
}

bf_status bf_set_precoders(bf_plan_t p, const void *W_dev, int n_groups, void *stream) {
    bfh::NvtxRange nvtx_("bf_set_precoders");
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (n_groups < 1) return fail(BF_ERR_INVALID_VALUE, "n_groups must be >= 1");
    if (n_groups > kMaxGroups)
        return fail(BF_ERR_UNSUPPORTED, "n_groups=%d exceeds %d", n_groups, kMaxGroups);
    DeviceGuard guard(p->device);
    if (p->f > 0) {
        if (!W_dev) return fail(BF_ERR_INVALID_VALUE, "W_dev is NULL");
        if (!aligned(W_dev, 16)) return fail(BF_ERR_MISALIGNED, "W_dev is not 16-byte aligned");
        bf_status s = grow(&p->Wp, &p->Wp_cap, (int64_t)n_groups * p->f * 32, "precoders");
        if (s != BF_OK) return s;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int64_t total = (int64_t)n_groups * p->f * 32;
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
        bf_relayout_w<<<blocks, 256, 0, st>>>(static_cast<const float *>(W_dev), n_groups, p->f,
                                              p->layout, p->Wp);
        if ((s = launched(p, "bf_relayout_w launch")) != BF_OK) return s;
        const int64_t img = (int64_t)n_groups * bftc::kp_of(p->f) * 128;   // 32-bit words
        if ((s = grow(&p->Wimg, &p->Wimg_cap, img, "tensor-core precoders")) != BF_OK) return s;
        if ((s = grow(&p->wexact, &p->wexact_cap, n_groups, "precoder flags")) != BF_OK) return s;
        bf_tc_build_wimg<<<n_groups, 256, 0, st>>>(static_cast<const float *>(W_dev), p->f, p->layout,
                                                  reinterpret_cast<uint32_t *>(p->Wimg), p->wexact);
        if ((s = launched(p, "bf_tc_build_wimg launch")) != BF_OK) return s;
        // the one synchronisation of the call: AUTO's kernel choice depends on whether
        // every group lies inside the tensor domain
        std::vector<int32_t> flags(n_groups);
        BF_CUDA(cudaMemcpyAsync(flags.data(), p->wexact, n_groups * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, st));
        BF_CUDA(cudaStreamSynchronize(st));
        p->w_in_domain = std::none_of(flags.begin(), flags.end(), [](int32_t v) { return (v & 2) != 0; });
    }
    p->n_groups = n_groups;
    return BF_OK;
}

static bf_status validate_apply(bf_plan_t p, const void *S, const int32_t *gidx, const void *R,
                                int64_t n, bool device) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (n < 0) return fail(BF_ERR_INVALID_VALUE, "n_blocks must be >= 0");
    if (n >= (int64_t(1) << 31)) return fail(BF_ERR_UNSUPPORTED, "n_blocks must be < 2^31");
    if (n == 0) return BF_OK;
    if (!R) return fail(BF_ERR_INVALID_VALUE, "R is NULL");
    if (p->f > 0) {
        if (!S) return fail(BF_ERR_INVALID_VALUE, "S is NULL");
        if (p->n_groups < 1) return fail(BF_ERR_NO_PRECODERS, "bf_set_precoders was not called");
    }
    if (device) {
        if (!aligned(R, 16) || (S && !aligned(S, 16)))
            return fail(BF_ERR_MISALIGNED, "S and R must be 16-byte aligned");
        if (gidx && !aligned(gidx, 4)) return fail(BF_ERR_MISALIGNED, "group_idx misaligned");
    }
    if (p->f > 0) {
        const uintptr_t s0 = reinterpret_cast<uintptr_t>(S), s1 = s0 + (uintptr_t)n * 480 * p->f;
        const uintptr_t r0 = reinterpret_cast<uintptr_t>(R),
                        r1 = r0 + (uintptr_t)n * bfk::r_block_bytes(p->layout);
        if (s0 < r1 && r0 < s1) return fail(BF_ERR_INVALID_VALUE, "R overlaps S");
    }
    return BF_OK;
}

bf_status bf_apply(bf_plan_t p, const void *S_dev, const int32_t *group_idx_dev, void *R_dev,
                   int64_t n_blocks, void *stream) {
    bfh::NvtxRange nvtx_("bf_apply");
    bf_status s = validate_apply(p, S_dev, group_idx_dev, R_dev, n_blocks, true);
    if (s != BF_OK || n_blocks == 0) return s;
    DeviceGuard guard(p->device);
    return apply_device(p, S_dev, group_idx_dev, R_dev, n_blocks,
                        static_cast<cudaStream_t>(stream));
}

bf_status bf_route(bf_plan_t p, const int32_t *group_idx_dev, int64_t n_blocks, int32_t *perm_dev,
                   int32_t *offsets_dev, void *stream) {
    bfh::NvtxRange nvtx_("bf_route");
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (p->n_groups < 1) return fail(BF_ERR_NO_PRECODERS, "bf_set_precoders was not called");
    if (n_blocks < 0 || n_blocks >= (int64_t(1) << 31))
        return fail(BF_ERR_INVALID_VALUE, "n_blocks out of range");
    if (!offsets_dev || (n_blocks > 0 && (!group_idx_dev || !perm_dev)))
        return fail(BF_ERR_INVALID_VALUE, "NULL buffer");
    DeviceGuard guard(p->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n_blocks == 0) {
        BF_CUDA(cudaMemsetAsync(offsets_dev, 0, (p->n_groups + 2) * sizeof(int32_t), st));
        return BF_OK;
    }
    return route(p, group_idx_dev, n_blocks, perm_dev, offsets_dev, st);
}

bf_status bf_apply_routed(bf_plan_t p, const void *S_dev, const int32_t *perm_dev,
                          const int32_t *offsets_dev, void *R_dev, int64_t n_blocks, void *stream) {
    bfh::NvtxRange nvtx_("bf_apply_routed");
    bf_status s = validate_apply(p, S_dev, perm_dev, R_dev, n_blocks, true);
    if (s != BF_OK || n_blocks == 0) return s;
    if ((perm_dev == nullptr) != (offsets_dev == nullptr))
        return fail(BF_ERR_INVALID_VALUE, "perm and offsets must be given together");
    if (offsets_dev && !aligned(offsets_dev, 4)) return fail(BF_ERR_MISALIGNED, "offsets misaligned");
    DeviceGuard guard(p->device);
    return apply_routed(p, S_dev, perm_dev, offsets_dev, R_dev, n_blocks,
                        static_cast<cudaStream_t>(stream));
}

bf_status bf_apply_batch(const bf_batch_job *jobs, int n_jobs, void *stream) {
    bfh::NvtxRange nvtx_("bf_apply_batch");
    if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return fail(BF_ERR_INVALID_VALUE, "bad job list");
    if (n_jobs == 0) return BF_OK;
    const bf_plan_t p0 = jobs[0].plan;
    if (!p0) return fail(BF_ERR_INVALID_VALUE, "job 0: plan is NULL");
    for (int i = 0; i < n_jobs; ++i) {   // every argument check before anything is enqueued
        const bf_batch_job &jb = jobs[i];
        bf_status s = validate_apply(jb.plan, jb.S_dev, jb.perm_dev, jb.R_dev, jb.n_blocks, true);
        if (s != BF_OK) {
            const std::string why = bfh::g_last_error;
            return fail(s, "job %d: %s", i, why.c_str());
        }
        if (jb.plan->device != p0->device || jb.plan->layout != p0->layout)
            return fail(BF_ERR_INVALID_VALUE, "job %d: every plan must share the device and layout "
                                              "of job 0", i);
        if ((jb.perm_dev == nullptr) != (jb.offsets_dev == nullptr))
            return fail(BF_ERR_INVALID_VALUE, "job %d: perm and offsets must be given together", i);
        if (jb.offsets_dev && !aligned(jb.offsets_dev, 4))
            return fail(BF_ERR_MISALIGNED, "job %d: offsets misaligned", i);
        if (jb.offsets_dev && jb.plan->n_groups + 2 > bftc::kOffsSlots)
            return fail(BF_ERR_UNSUPPORTED, "job %d: n_groups=%d exceeds the batched kernel's %d",
                        i, jb.plan->n_groups, bftc::kOffsSlots - 2);
    }
    DeviceGuard guard(p0->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // f == 0 and FFMA-variant jobs run as their own applies, in order; the others are
    // packed into launches of at most kMaxJobs jobs and kOffsSlots group offsets.
    bf_batch_job pack[bftc::kMaxJobs];
    int np = 0, slots = 0;
    bf_status s;
    for (int i = 0; i <= n_jobs; ++i) {
        const bool end = i == n_jobs;
        const bf_batch_job *jb = end ? nullptr : &jobs[i];
        // AUTO plans join the pack (one launch for the window beats the small-f
        // per-kernel edge of the FFMA kernel) unless their precoders lie outside the
        // tensor domain; plans set to FFMA run on their own
        const bool tc = !end && jb->n_blocks > 0 && jb->plan->f > 0 &&
                        jb->plan->variant != BF_VARIANT_FFMA &&
                        (jb->plan->variant == BF_VARIANT_TENSOR || jb->plan->w_in_domain);
        const int need = tc && jb->offsets_dev ? jb->plan->n_groups + 2 : 0;
        if (np > 0 && (end || !tc || np == bftc::kMaxJobs || slots + need > bftc::kOffsSlots)) {
            if ((s = launch_batch(pack, np, st)) != BF_OK) return s;
            np = 0;
            slots = 0;
        }
        if (end) break;
        if (tc) {
            pack[np++] = *jb;
            slots += need;
        } else if (jb->n_blocks > 0) {
            if ((s = apply_routed(jb->plan, jb->S_dev, jb->perm_dev, jb->offsets_dev, jb->R_dev,
                                  jb->n_blocks, st)) != BF_OK)
                return s;
        }
    }
    return BF_OK;
}

bf_status bf_apply_host(bf_plan_t p, const void *S_host, const int32_t *group_idx_host,
                        void *R_host, int64_t n_blocks, void *stream) {
    bfh::NvtxRange nvtx_("bf_apply_host");
    bf_status s = validate_apply(p, S_host, group_idx_host, R_host, n_blocks, false);
    if (s != BF_OK || n_blocks == 0) return s;
    DeviceGuard guard(p->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool tagged = group_idx_host != nullptr;
    if ((s = ensure_host_pipeline(p, tagged)) != BF_OK) return s;
    const int64_t C = p->host_chunk;
    const size_t s_blk = (size_t)480 * p->f, r_blk = (size_t)bfk::r_block_bytes(p->layout);
    BF_CUDA(cudaEventRecord(p->ev_start, st));
    BF_CUDA(cudaStreamWaitEvent(p->s_h2d, p->ev_start, 0));
    BF_CUDA(cudaStreamWaitEvent(p->s_d2h, p->ev_start, 0));
    int last = 0;
    for (int64_t c0 = 0, c = 0; c0 < n_blocks; c0 += C, ++c) {
        const int slot = (int)(c % kHostSlots);
        const int64_t nc = std::min(C, n_blocks - c0);
        // slot is free once its previous device->host copy has drained
        BF_CUDA(cudaStreamWaitEvent(p->s_h2d, p->ev_d2h[slot], 0));
        if (p->f > 0)
            BF_CUDA(cudaMemcpyAsync(p->hS[slot], static_cast<const char *>(S_host) + c0 * s_blk,
                                    nc * s_blk, cudaMemcpyHostToDevice, p->s_h2d));
        if (tagged)
            BF_CUDA(cudaMemcpyAsync(p->hG[slot], group_idx_host + c0, nc * sizeof(int32_t),
                                    cudaMemcpyHostToDevice, p->s_h2d));
        BF_CUDA(cudaEventRecord(p->ev_h2d[slot], p->s_h2d));
        BF_CUDA(cudaStreamWaitEvent(st, p->ev_h2d[slot], 0));
        if ((s = apply_device(p, p->hS[slot], tagged ? p->hG[slot] : nullptr, p->hR[slot], nc,
                              st)) != BF_OK)
            return s;
        BF_CUDA(cudaEventRecord(p->ev_comp[slot], st));
        BF_CUDA(cudaStreamWaitEvent(p->s_d2h, p->ev_comp[slot], 0));
        BF_CUDA(cudaMemcpyAsync(static_cast<char *>(R_host) + c0 * r_blk, p->hR[slot], nc * r_blk,
                                cudaMemcpyDeviceToHost, p->s_d2h));
        BF_CUDA(cudaEventRecord(p->ev_d2h[slot], p->s_d2h));
        last = slot;
    }
    BF_CUDA(cudaStreamWaitEvent(st, p->ev_d2h[last], 0));
    return BF_OK;
}

bf_status bf_destroy(bf_plan_t p) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    {
        DeviceGuard guard(p->device);
        cudaFree(p->Wp);
        cudaFree(p->Wimg);
        cudaFree(p->wexact);
        cudaFree(p->perm);
        cudaFree(p->table);
        cudaFree(p->offsets);
        cudaFree(p->err);
        for (int i = 0; i < kHostSlots; ++i) {
            cudaFree(p->hS[i]);
            cudaFree(p->hR[i]);
            cudaFree(p->hG[i]);
            if (p->ev_h2d[i]) cudaEventDestroy(p->ev_h2d[i]);
            if (p->ev_comp[i]) cudaEventDestroy(p->ev_comp[i]);
            if (p->ev_d2h[i]) cudaEventDestroy(p->ev_d2h[i]);
        }
        if (p->ev_start) cudaEventDestroy(p->ev_start);
        if (p->s_h2d) cudaStreamDestroy(p->s_h2d);
        if (p->s_d2h) cudaStreamDestroy(p->s_d2h);
        for (auto &ev : p->prof_events) {
            cudaEventDestroy(ev.first);
            cudaEventDestroy(ev.second);
        }
    }
    delete p;
    return BF_OK;
}

bf_status bf_plan_set_profiling(bf_plan_t p, int enable) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    p->profiling = enable != 0;
    return BF_OK;
}

bf_status bf_plan_kernel_time(bf_plan_t p, double *total_ms, int64_t *n_launches) {
    if (!p || !total_ms || !n_launches) return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    DeviceGuard guard(p->device);
    double sum = 0.0;
    for (size_t i = 0; i < p->prof_used; ++i) {
        BF_CUDA(cudaEventSynchronize(p->prof_events[i].second));
        float ms = 0.f;
        BF_CUDA(cudaEventElapsedTime(&ms, p->prof_events[i].first, p->prof_events[i].second));
        sum += ms;
    }
    *total_ms = sum;
    *n_launches = (int64_t)p->prof_used;
    p->prof_used = 0;
    return BF_OK;
}

bf_status bf_plan_launch_count(bf_plan_t p, int64_t *count) {
    if (!p || !count) return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    *count = p->launches;
    return BF_OK;
}

bf_status bf_plan_set_variant(bf_plan_t p, int variant) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (variant != BF_VARIANT_AUTO && variant != BF_VARIANT_FFMA && variant != BF_VARIANT_TENSOR)
        return fail(BF_ERR_INVALID_VALUE, "unknown variant %d", variant);
    p->variant = variant;
    return BF_OK;
}

}  // extern "C"

bf_status bfh::plan_info(bf_plan_t p, int *n_ant, int *f, int *b, int *layout, int *device) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    *n_ant = p->n_ant;
    *f = p->f;
    *b = p->b;
    *layout = p->layout;
    *device = p->device;
    return BF_OK;
}

extern "C" {

bf_status bf_plan_get_variant(bf_plan_t p, int *resolved) {
    if (!p || !resolved) return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    *resolved = p->f == 0 ? BF_VARIANT_AUTO : (use_tensor(p) ? BF_VARIANT_TENSOR : BF_VARIANT_FFMA);
    return BF_OK;
}

bf_status bf_plan_set_host_chunk(bf_plan_t p, int64_t blocks) {
    if (!p || blocks < 0) return fail(BF_ERR_INVALID_VALUE, "invalid chunk");
    p->host_chunk = blocks == 0 ? kDefaultHostChunk : blocks;
    return BF_OK;
}

bf_status bf_plan_set_output_exponent(bf_plan_t p, int e) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (e < -64 || e > 64) return fail(BF_ERR_INVALID_VALUE, "output exponent %d outside [-64, 64]", e);
    p->out_exp = e;
    return BF_OK;
}

bf_status bf_plan_set_sm_share(bf_plan_t p, int sms) {
    if (!p) return fail(BF_ERR_INVALID_VALUE, "plan is NULL");
    if (sms < 0) return fail(BF_ERR_INVALID_VALUE, "sms must be >= 0 (got %d)", sms);
    p->sm_share = sms;
    return BF_OK;
}

// ---------------------------------------------------------------------------
// slot server (include/bf.h bf_server_*)
// ---------------------------------------------------------------------------
}  // extern "C"

struct bf_server_s {
    bf_plan_t plan = nullptr;
    bftc::SrvMailbox *mb = nullptr;        // mapped pinned host memory
    bftc::SrvMailbox *mb_dev = nullptr;    // its device address
    bftc::SrvDev *dev = nullptr;
    cudaStream_t stream = nullptr;
    bool running = false;
    unsigned long long next = 0;           // last submitted slot
};

namespace {
volatile bftc::SrvMailbox *vmb(bf_server_t s) { return s->mb; }
bf_status server_post(bf_server_t s, const void *S, void *R, int64_t n, int stop, uint64_t *ticket) {
    const unsigned long long k = s->next + 1;
    // at most kSrvRing slots in flight: the descriptor entry of slot k - ring must be consumed
    if (k > (unsigned long long)bftc::kSrvRing) {
        const unsigned long long need = k - bftc::kSrvRing;
        while (vmb(s)->done < need) {
            const cudaError_t q = cudaStreamQuery(s->stream);
            if (q != cudaErrorNotReady)
                return q == cudaSuccess ? fail(BF_ERR_INVALID_VALUE, "the server is not running")
                                        : cuda_fail(q, "slot server");
        }
    }
    // the descriptor as LL words (8-byte stores: data | slot number << 32), in any order:
    // the server takes it once every word carries k (bf_tc.cuh kDescWords)
    volatile unsigned long long *d = vmb(s)->desc[k % bftc::kSrvRing];
    const unsigned long long pS = reinterpret_cast<unsigned long long>(S);
    const unsigned long long pR = reinterpret_cast<unsigned long long>(R);
    d[0] = bftc::ll_word((unsigned int)pS, k);
    d[1] = bftc::ll_word((unsigned int)(pS >> 32), k);
    d[2] = bftc::ll_word((unsigned int)pR, k);
    d[3] = bftc::ll_word((unsigned int)(pR >> 32), k);
    d[4] = bftc::ll_word((unsigned int)n, k);
    d[5] = bftc::ll_word((unsigned int)stop, k);
    std::atomic_thread_fence(std::memory_order_seq_cst);
    s->next = k;
    if (ticket) *ticket = k;
    return BF_OK;
}
}  // namespace

extern "C" {

bf_status bf_server_create(bf_plan_t p, bf_server_t *out) {
    if (!p || !out) return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    if (p->f == 0) return fail(BF_ERR_UNSUPPORTED, "the slot server needs f >= 1");
    if (p->n_groups != 1) return fail(BF_ERR_UNSUPPORTED, "the slot server serves one precoder group "
                                                         "(untagged slots); got %d", p->n_groups);
    if (!p->w_in_domain)
        return fail(BF_ERR_UNSUPPORTED, "precoders outside the tensor domain: use bf_apply");
    DeviceGuard guard(p->device);
    bf_server_t s = new (std::nothrow) bf_server_s();
    if (!s) return fail(BF_ERR_OUT_OF_MEMORY, "host allocation of the server failed");
    s->plan = p;
    if (cudaHostAlloc(reinterpret_cast<void **>(&s->mb), sizeof(bftc::SrvMailbox),
                      cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void **>(&s->mb_dev), s->mb, 0) != cudaSuccess ||
        cudaMalloc(&s->dev, sizeof(bftc::SrvDev)) != cudaSuccess) {
        cudaGetLastError();
        if (s->mb) cudaFreeHost(s->mb);
        cudaFree(s->dev);
        delete s;
        return fail(BF_ERR_OUT_OF_MEMORY, "slot server mailbox allocation failed");
    }
    std::memset(s->mb, 0, sizeof(bftc::SrvMailbox));
    *out = s;
    return BF_OK;
}

bf_status bf_server_start(bf_server_t s, void *stream) {
    bfh::NvtxRange nvtx_("bf_server_start");
    if (!s) return fail(BF_ERR_INVALID_VALUE, "server is NULL");
    if (s->running) return fail(BF_ERR_INVALID_VALUE, "server already running");
    bf_plan_t p = s->plan;
    DeviceGuard guard(p->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::memset(s->mb, 0, sizeof(bftc::SrvMailbox));
    BF_CUDA(cudaMemsetAsync(s->dev, 0, sizeof(bftc::SrvDev), st));
    const BfKernelEntry &kern = g_server[p->layout];
    BF_CUDA(cudaFuncSetAttribute(kern.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kern.smem_bytes));
    bftc::TcParams tp{};
    tp.n_jobs = 0;
    tp.job[0] = tc_job(p, nullptr, nullptr, nullptr, nullptr, 0);
    tp.srv.mb = s->mb_dev;
    tp.srv.dev = s->dev;
    tp.srv.timeout_ns = 60ll * 1000 * 1000 * 1000;   // an abandoned server exits after 60 s idle
    void *args[] = {&tp};
    cudaError_t e = cudaLaunchKernel(kern.fn, dim3(sms_used(p)), dim3(bftc::kThreads), args,
                                     (size_t)kern.smem_bytes, st);
    if (e != cudaSuccess) return cuda_fail(e, "slot server launch");
    ++p->launches;
    s->stream = st;
    s->running = true;
    s->next = 0;
    return BF_OK;
}

bf_status bf_server_submit(bf_server_t s, const void *S_dev, void *R_dev, int64_t n_blocks,
                           uint64_t *ticket) {
    if (!s) return fail(BF_ERR_INVALID_VALUE, "server is NULL");
    if (!s->running) return fail(BF_ERR_INVALID_VALUE, "server is not running");
    bf_status st = validate_apply(s->plan, S_dev, nullptr, R_dev, n_blocks, true);
    if (st != BF_OK) return st;
    return server_post(s, S_dev, R_dev, n_blocks, 0, ticket);
}

bf_status bf_server_wait(bf_server_t s, uint64_t ticket, double timeout_s) {
    if (!s) return fail(BF_ERR_INVALID_VALUE, "server is NULL");
    if (ticket > s->next) return fail(BF_ERR_INVALID_VALUE, "ticket %llu was not submitted",
                                      (unsigned long long)ticket);
    const auto t0 = std::chrono::steady_clock::now();
    while (vmb(s)->done < ticket) {
        const cudaError_t q = cudaStreamQuery(s->stream);
        if (q != cudaErrorNotReady && vmb(s)->done < ticket)
            return q == cudaSuccess ? fail(BF_ERR_CUDA, "the server exited before slot %llu",
                                           (unsigned long long)ticket)
                                    : cuda_fail(q, "slot server");
        if (timeout_s > 0 && std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
            return fail(BF_ERR_CUDA, "slot %llu not done after %.1f s", (unsigned long long)ticket, timeout_s);
    }
    if (vmb(s)->error)
        return fail(BF_ERR_INVALID_VALUE, "a slot held S values outside the tensor domain "
                                          "(its R is not the contract result; use bf_apply)");
    return BF_OK;
}

bf_status bf_server_slot_time(bf_server_t s, uint64_t ticket, double *device_us) {
    if (!s || !device_us) return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    if (ticket == 0 || vmb(s)->done < ticket || s->next >= ticket + bftc::kSrvRing)
        return fail(BF_ERR_INVALID_VALUE, "slot %llu is not done or no longer in the ring",
                    (unsigned long long)ticket);
    const int e = (int)(ticket % bftc::kSrvRing);
    *device_us = (double)(vmb(s)->t_done[e] - vmb(s)->t_seen[e]) * 1e-3;
    return BF_OK;
}

bf_status bf_server_trace(bf_server_t s, double *us, int n) {
    if (!s || !us || n < 0) return fail(BF_ERR_INVALID_VALUE, "bad argument");
    const unsigned long long t0 = vmb(s)->trace[0];
    for (int i = 0; i < n && i < 8 + 2 * 160; ++i) {   // trace, then per-CTA seen / done
        const unsigned long long t = i < 8 ? vmb(s)->trace[i]
                                           : (i < 168 ? vmb(s)->cta_seen[i - 8] : vmb(s)->cta_done[i - 168]);
        us[i] = t ? (double)(long long)(t - t0) * 1e-3 : -1.0;
    }
    return BF_OK;
}

bf_status bf_server_stop(bf_server_t s) {
    bfh::NvtxRange nvtx_("bf_server_stop");
    if (!s) return fail(BF_ERR_INVALID_VALUE, "server is NULL");
    if (!s->running) return BF_OK;
    DeviceGuard guard(s->plan->device);
    bf_status st = server_post(s, nullptr, nullptr, 0, 1, nullptr);
    s->running = false;
    if (st != BF_OK) return st;
    BF_CUDA(cudaStreamSynchronize(s->stream));
    return BF_OK;
}

bf_status bf_server_destroy(bf_server_t s) {
    if (!s) return fail(BF_ERR_INVALID_VALUE, "server is NULL");
    bf_status st = s->running ? bf_server_stop(s) : BF_OK;
    DeviceGuard guard(s->plan->device);
    cudaFreeHost(s->mb);
    cudaFree(s->dev);
    delete s;
    return st;
}

bf_status bf_plan_kernel_config(bf_plan_t p, int64_t n_blocks, int *grid, int *block,
                                int *smem_bytes, int *ctas_per_sm) {
    if (!p || !grid || !block || !smem_bytes || !ctas_per_sm)
        return fail(BF_ERR_INVALID_VALUE, "NULL argument");
    const bool tensor = p->f > 0 && use_tensor(p);
    const int64_t nb = std::max<int64_t>(n_blocks, 1);
    *grid = p->f == 0 ? 0 : grid_for(p, nb, tensor);
    *block = p->f == 0 ? 0 : (tensor ? bftc::kThreads : bfk::kThreads);
    *smem_bytes = tensor ? p->kern_tc.smem_bytes : p->kern.smem_bytes;
    *ctas_per_sm = tensor ? 1 : p->ctas_per_sm;
    return BF_OK;
}

}  // extern "C"
