// bf_tc.cuh — sm_100a tensor-core (tcgen05, kind::f16 on split fp16 terms) beamforming kernel.
//
// Same operation as bf_ffma.cuh: R[n] = W[g(n)] x S[n], complex
// fp32, 64 antennas, 60 REs, F flows.  SURVEY.md §8(f) row 2: a split-precision
// tensor-core path kept only if it beats the FFMA path and meets the tolerance.
//
// Real embedding, transposed so that REs are the MMA's M rows:
//   A [m][kk]  (TMEM)  m = RE of a 2-block tile (m = 60 b + j, 120 of 128 rows),
//                      kk = 2k + c: S[blk][k][j] re (c = 0) / im (c = 1)
//   B [n][kk]  (SMEM)  n = 2i + c_out (antenna i, re / im output):
//                      n = 2i  : kk=2k -> Wr[i][k],  kk=2k+1 -> -Wi[i][k]
//                      n = 2i+1: kk=2k -> Wi[i][k],  kk=2k+1 ->  Wr[i][k]
//   D [m][n]   (TMEM)  = R[blk][i][j] re / im, fp32 accumulate.
// Split precision (error-compensated, BASELINE.json north_star item 2): every row of A
// (one RE) is scaled by 2^sg and every precoder group by 2^tau so the largest component
// lies in [2^14, 2^15); S' = S1 + S2 + S3 exactly (11-bit terms), W' = W1 + W2 + W3
// (11-bit W1, W2, |W3| <= 2^-22 |W'|, split once per bf_set_precoders), every term as
// fp16 (exact in fp16's normal range; the tensor domain bounds the rest).  Every product
// is an fp16 x fp16 product, exact in the fp32 accumulator (kind::f16, K = 16).  General
// W: S2 W1, S1 W2, then S1 W1 (dropped terms S3 W1 + S2 W2 + S W3 <= 3 2^-22 |s||w|);
// when the group is exact in one fp16 term (W2 == 0: identity, selection, small
// integers) S2 W1, S3 W1, S1 W1 = S W exactly, which makes copy-like precoders
// bit-exact.  The epilogue undoes 2^(sg + tau) with one exact multiply.
// bounds the error by 5.8e-6 T at f = 36 (complex modulus, with the accumulation model
// measured by tools/tc_acc_probe).
// Tensor domain: per row the largest element in [2^-40, 2^40), no NaN, every nonzero
// element within 2^14 of the largest component (exact W: every nonzero component within
// 2^15) — tested by the split warps as they read S; per group of W the same, tested by
// bf_set_precoders.  Blocks outside are recomputed at the end of the launch by the CTA
// that owns them with the FFMA kernel's arithmetic (fix_block), bit for bit.
//
// One CTA (18 warps) per SM, persistent over a cost-balanced range of the
// group-sorted block list (cta_range); tiles are 2 consecutive blocks of one group.
//   warp 17    producer: cp.async.bulk (TMA bulk engine) of each block's 480 F
//              contiguous bytes into a 2-4-stage shared-memory ring, completing on
//              mbarriers, up to kStages tiles ahead of the split; and the pre-split
//              B image (W) of each group segment into its W buffer (two where shared
//              memory allows: the next group's image loads while the current one's
//              MMAs run);
//   warps 0-7  split (two per TMEM lane quarter, each half of the K columns above
//              f = 16): LDS S (conflict-free, one RE column per lane), the row's
//              scale (the two halves exchange their maxima), split into the terms,
//              tcgen05.st of fp16 pairs into the A regions (one TMEM lane per RE);
//   warp 8     MMA issuer (one thread);
//   warps 9-16 epilogue (two per lane quarter, half the D columns each): tcgen05.ld
//              of the thread's D row half, release of the TMEM buffer, then the
//              tile's two R blocks written into a shared-memory stage in their
//              global layout and stored by one thread with one bulk copy per block
//              (two R stages for 16-bit outputs at f <= 16; BFTC_I16_DIRECT_MAXF builds
//              store int16 output directly from registers instead).
// Shared memory per f: TcSmem (W buffers, S ring depth, R stage).
// TMEM: two sets of A terms (fp16 pairs: KP / 2 columns per term; KP of f = 36 for the
// batch kernel) at [0, 3 KP / 2) and [3 KP / 2, 3 KP), D double buffer at [256, 384),
// [384, 512).
#pragma once
#include <cstddef>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "bf_ffma.cuh"
#include "tc_ptx.cuh"

namespace bftc {

constexpr int kSplitWarps = 8;        // two per TMEM lane quarter, half the K columns each
constexpr int kMmaWarp = 8;
constexpr int kEpiWarp0 = 9;
constexpr int kEpiWarps = 8;          // two per TMEM lane quarter, 64 D columns each
constexpr int kProdWarp = 17;
constexpr int kThreads = 32 * (kProdWarp + 1);
#ifndef BFTC_MAX_STAGES
#define BFTC_MAX_STAGES 4
#endif
constexpr int kMaxStages = BFTC_MAX_STAGES;   // S ring depth (tiles), shared memory permitting
constexpr int kSmemLimit = 232448;     // 227 KB per CTA
constexpr int kDCol0 = 256;
constexpr int kMinSmem = 120 * 1024;   // forces one CTA (and one TMEM owner) per SM
#ifndef BFTC_EARLY_RELEASE
#define BFTC_EARLY_RELEASE 0
#endif
#ifndef BFTC_DEEP_RING_MAXF
#define BFTC_DEEP_RING_MAXF 8    // S ring of kMaxStages up to this f, 2 stages above
#endif
// int16 output: direct register stores up to this f (round 1: faster than the staged epilogue
// at f <= 12), and two R stages for the staged one; round 2 (fp16 terms): staged with two R
// stages wins at every f (f = 1 0.53 -> 0.58, f = 8 0.61 -> 0.67, f = 16 0.69 -> 0.75 of copy
// BW; profiles/r02_rstage_ring.txt)
#ifndef BFTC_I16_DIRECT_MAXF
#define BFTC_I16_DIRECT_MAXF 0
#endif
#ifndef BFTC_I16_R2
#define BFTC_I16_R2 1
#endif
#ifndef BFTC_RSTAGES
#define BFTC_RSTAGES 2    // R stages where two fit (small f)
#endif
#ifndef BFTC_ABUFS
#define BFTC_ABUFS 2      // TMEM A-region buffers (2 where they fit)
#endif
// Experiments only: the runtime-f kernel with a compile-time f in some roles
// (BFTC_FIXF_ROLES bits: 1 split warps, 2 producer, 4 MMA issuer).  Results are wrong
// for any other f.
#ifndef BFTC_FIXF
#define BFTC_FIXF 0
#endif
#ifndef BFTC_FIXF_ROLES
#define BFTC_FIXF_ROLES 0
#endif
// split warps release an S ring slot as soon as their values are in registers (1), or
// after the tile's last split pass (0)
constexpr bool kEarlyRelease = BFTC_EARLY_RELEASE != 0;

// K extent of the real embedding (2F), padded to the K = 16 of a kind::f16 MMA.
__host__ __device__ constexpr int kp_of(int F) { return (2 * F + 15) / 16 * 16; }
// Relative range of the f16 path: the operands of a row of S (a group of
// W) are scaled by 2^e so their largest component lies in [2^14, 2^15); every nonzero
// element (the larger of |re|, |im|) must then be >= 1, i.e. within 2^14 of the largest
// (exponent fields: e(elem) >= e(max) - kRelRange).
constexpr int kRelRange = 14;

// One apply of a plan: blocks [0, n_items) of S -> R with the plan's precoders.
// A launch processes a list of jobs (bf_apply: one; bf_apply_batch: up to
// kMaxJobs, e.g. consecutive streaming chunks of different cells), each split
// over all CTAs; the kernel template's F is the flow count of every job, or 0
// for the batch kernel whose jobs carry their own f (1..36).
#ifndef BFTC_MAX_JOBS
#define BFTC_MAX_JOBS 16
#endif
constexpr int kMaxJobs = BFTC_MAX_JOBS;
constexpr int kOffsSlots = kMaxJobs <= 16 ? 1028 : 2052;   // shared group-offset slots: sum over jobs of (n_groups + 2)
constexpr int kFixCap = 64;            // out-of-domain blocks a CTA lists (more: rescan its range)
// Tensor domain of S and W: zero, or 2^-40 <= |x| < 2^40, as fp32 bit
// patterns without the sign.  Inside it every product of split terms is a normal fp32
// number, so the split-precision error bound holds; NaN and Inf fall outside.
constexpr uint32_t kDomLo = 0x2B800000u, kDomHi = 0x53800000u;

struct TcJob {
    const float *Wimg;        // [n_groups][2][KP/8][16][8][8] fp16 (pre-split B image)
    // Wimg per group: [W1 as fp16 core matrices (KP/8 K-chunks of 8)] then [W2, same
    // layout], both of W scaled by 2^tau (tau in wexact bits 8-15)
    const float4 *Wp;         // FFMA image of the same precoders (out-of-domain fix-up)
    const float *S;
    const int32_t *perm;      // NULL = identity order
    const int32_t *offsets;   // [n_groups + 2] group starts of the sorted order, or NULL
    const int32_t *wexact;    // [n_groups] bit 0: W exact in one fp16 term (W2 == 0);
                              //            bit 1: W outside the tensor domain;
                              //            bits 8-15: tau + 128 (the group's scale 2^tau)
    float *R;
    int64_t n_items;
    int n_groups;
    int f;
    float out_scale;          // layout 3 (int16 output): 2^e before the rounding
};

// Kernel parameters: n_jobs first, so a launch can pass a TcParams (16 jobs) to a
// kernel declared with TcParamsN<1> — cudaLaunchKernel copies the kernel's parameter
// size from the pointer, i.e. the common prefix.  The per-f kernels (bf_apply: one job)
// take the 1-job form: 1.3 KB less parameter data per launch (~1 us of launch latency,
// tools/launch_lat); the batch kernel (F = 0) takes all kMaxJobs.
// Slot server (bf_server_*: one persistent launch serving a stream of untagged applies;
// SRV kernel instantiation).  The mailbox lives in mapped pinned host memory: the host
// writes a slot descriptor and then bumps seq; CTA 0 polls it and re-broadcasts the
// descriptor through SrvDev (device memory) to the other CTAs; the last CTA to finish a
// slot publishes done = seq and the device timestamps.
constexpr int kSrvRing = 4;                // slots in flight (descriptor rings)
#ifndef BFTC_SRV_DIRECT
#define BFTC_SRV_DIRECT 0   // 1: every CTA polls the host mailbox (measured 47x slower: PCIe contention)
#endif
// Slot descriptors travel as LL words (the NCCL "LL" idea): each 8-byte word carries 32
// bits of data and the 32-bit slot number, and 8-byte aligned stores are single-copy
// atomic, so a reader that sees the expected slot number in every word holds the whole
// descriptor — no fence between data and flag on either hop (host -> CTA 0 over PCIe,
// CTA 0 -> the other CTAs through L2).
constexpr int kDescWords = 6;              // S lo, S hi, R lo, R hi, n, stop
__host__ __device__ inline unsigned long long ll_word(unsigned int data, unsigned long long k) {
    return ((unsigned long long)(unsigned int)k << 32) | data;
}
// the six words of one descriptor, three 16-byte loads issued together
template <bool SYS>
__device__ __forceinline__ void ld_ll6(const unsigned long long *w, unsigned long long (&v)[kDescWords]) {
    if (SYS)
        asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%6];\n\t"
                     "ld.relaxed.sys.global.v2.u64 {%2, %3}, [%6+16];\n\t"
                     "ld.relaxed.sys.global.v2.u64 {%4, %5}, [%6+32];"
                     : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]), "=l"(v[4]), "=l"(v[5])
                     : "l"(w) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%6];\n\t"
                     "ld.relaxed.gpu.global.v2.u64 {%2, %3}, [%6+16];\n\t"
                     "ld.relaxed.gpu.global.v2.u64 {%4, %5}, [%6+32];"
                     : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]), "=l"(v[4]), "=l"(v[5])
                     : "l"(w) : "memory");
}
__device__ __forceinline__ bool ll_complete(const unsigned long long (&v)[kDescWords], unsigned long long k) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < kDescWords; ++i) ok &= (unsigned int)(v[i] >> 32) == (unsigned int)k;
    return ok;
}
struct SrvMailbox {
    __align__(16) unsigned long long desc[kSrvRing][kDescWords];   // host-written LL words
    int error;                             // device: a slot held values outside the tensor domain
    int pad;
    unsigned long long done;               // device: last completed slot
    unsigned long long t_seen[kSrvRing];   // device globaltimer: CTA 0 saw slot k (k % ring)
    unsigned long long t_done[kSrvRing];   // device globaltimer: slot k complete
    unsigned long long trace[8];           // CTA 0, last slot: see srv_trace
    unsigned long long cta_seen[160];      // BFTC_SRV_TRACE builds: every CTA, last slot
    unsigned long long cta_done[160];
};
struct SrvDev {
    __align__(16) unsigned long long desc[kSrvRing][kDescWords];   // CTA 0's re-broadcast
    unsigned int done_cnt[kSrvRing];
};
struct SrvPtrs {
    SrvMailbox *mb;                        // device view of the mapped mailbox
    SrvDev *dev;
    long long timeout_ns;                  // a poll that waits longer than this stops the server
};

template <int NJ>
struct TcParamsN {
    int n_jobs;
    int split;                             // batch launches: 0 every job over all CTAs;
                                           // 1 one contiguous cost range of all jobs per CTA
    SrvPtrs srv;                           // SRV kernels only
    TcJob job[NJ];
};
using TcParams = TcParamsN<kMaxJobs>;
template <int F>
using TcParamsOf = TcParamsN<F == 0 ? kMaxJobs : 1>;
static_assert(offsetof(TcParamsN<1>, job) == offsetof(TcParams, job), "TcParams prefix layout");

template <int F, bool SRV = false, bool R2 = false>   // R2: a second R stage where it fits
struct TcSmem {
    static constexpr int FS = F > 0 ? F : 36;          // sizing flow count (36 for runtime f)
    static constexpr int KP = kp_of(FS);
    static constexpr int kWBytes = 2 * KP * 128 * 2;   // W1 and W2 fp16 images
    static constexpr int kSBlock = 480 * FS;           // one block of S (slot stride)
    static constexpr int kJobBytes = kMaxJobs * 96;    // per-job context (JobCtx)
    static constexpr int kFixBytes = kFixCap * 8 + 16 + 2 * kMaxStages * 4;   // fix-up list
    static constexpr int kBars = 48;                    // mbarrier slots
    static constexpr int kSigBytes = 2 * 128 * 4;       // per-row scale exponents, 2 tiles
    static constexpr int kXchBytes = 2 * 8 * 32 * 4;    // split warps' row-range exchange
    static constexpr int kMisc = kBars * 8 + 16 + kOffsSlots * 4 + kJobBytes + kFixBytes + kMaxJobs * 8 +
                                 kSigBytes + kXchBytes;
    // R staging: the epilogue writes the tile's two blocks of R into shared memory in
    // their global layout and one thread stores each block with a bulk copy (full lines,
    // no partial sectors at planar row boundaries).  Shared memory, in order of
    // preference: two W buffers (the producer prefetches the next group's image while
    // the current group's MMAs run) + R stage (f <= 25); one W buffer + R stage (above
    // f = 25 and the runtime-f batch kernel: a group change then waits for the previous
    // group's MMAs, which measured cheaper than the unstaged epilogue even for c5's
    // short, group-rich jobs: +3 %).  Each with >= 2 S stages.
    static constexpr int kRStageBytes = 2 * 30720;
    static constexpr int kFitA = (kSmemLimit - 2 * kWBytes - kMisc - kRStageBytes - 128) / (2 * kSBlock);
    static constexpr int kFitB = (kSmemLimit - kWBytes - kMisc - kRStageBytes - 128) / (2 * kSBlock);
    static constexpr bool kStageR = kFitA >= 2 || kFitB >= 2;
    // (the slot server keeps one group's image for good: one W buffer, the space to S)
    static constexpr int kWBufs = SRV || (kFitA < 2 && kFitB >= 2) ? 1 : 2;
    static constexpr int kFixed = kWBufs * kWBytes + kMisc + (kStageR ? kRStageBytes + 128 : 0);
    static constexpr int kStagesFit = (kSmemLimit - kFixed) / (2 * kSBlock);
    // S ring depth: with the staged epilogue a deeper ring measured slower above f = 12
    // (e.g. f = 20: 0.87 of the copy bandwidth with 4 stages, 0.94 with 2; f <= 12 gained
    // from 4 — tools/sweep_f.py, BFTC_MAX_STAGES builds, profiles/r01_sweep_stages_v5.txt);
    // round 2 (fp16 terms): 4 stages only up to f = 8 (f = 10-12: 0.85-0.90 with 4, 0.93
    // with 2; profiles/r02_rstage_ring.txt)
    // (fp16 output, whose stores are half the bytes, keeps the deepest ring that fits)
    // (slot server: latency, not bandwidth — every stage that fits, so a CTA's few tiles of a
    // small slot all load at once)
    static constexpr int kMaxS = (SRV || (F > 0 && F <= BFTC_DEEP_RING_MAXF)) ? kMaxStages : (kMaxStages < 2 ? kMaxStages : 2);
    static constexpr int kStagesAlloc = kStagesFit < kMaxStages ? kStagesFit : kMaxStages;
    static constexpr int kStages = kStagesFit < kMaxS ? kStagesFit : kMaxS;
    static_assert(kStages >= 2, "S ring needs two stages");
    static constexpr int kOffS = kWBufs * kWBytes;     // kStagesAlloc x 2 blocks
    static constexpr int kOffBar = kOffS + kStagesAlloc * 2 * kSBlock;   // kBars mbarrier slots
    static constexpr int kOffTmem = kOffBar + kBars * 8;
    static constexpr int kOffJobs = kOffTmem + 16;     // JobCtx[kMaxJobs]
    static constexpr int kOffOffs = kOffJobs + kJobBytes;   // group offsets of every job
    static constexpr int kOffFix = kOffOffs + kOffsSlots * 4;   // int2 list, n, overflow, last[]
    static constexpr int kOffJCost = kOffFix + kFixBytes;        // int64 per job (split = 1)
    static constexpr int kOffSig = kOffJCost + kMaxJobs * 8;       // int32 [2][128]
    static constexpr int kOffXch = kOffSig + kSigBytes;            // uint32 [2][8][32]
    static constexpr int kOffR = (kOffXch + kXchBytes + 127) / 128 * 128;
    // two R stages where they fit (small f; 16-bit outputs — R2 — only: the fp32 layouts
    // measured slower with two): the epilogue writes tile t + 1's stage while tile t's bulk
    // stores read theirs
    static constexpr int kRStages = (R2 && kStageR && F > 0 && kOffR + 2 * kRStageBytes <= kSmemLimit) ? BFTC_RSTAGES : 1;
    static constexpr int kBytesUsed = kStageR ? kOffR + kRStages * kRStageBytes : kOffXch + kXchBytes;
    static constexpr int kBytes = kBytesUsed > kMinSmem ? kBytesUsed : kMinSmem;
    static_assert(kBytesUsed <= kSmemLimit, "shared memory");
};

// A job as the roles see it (shared memory), with this CTA's share of it.
struct JobCtx {
    const float *Wimg, *S;
    const float4 *Wp;
    const int32_t *perm, *wexact;
    float *R;
    const int32_t *offs;      // shared copy of the job's offsets, or nullptr (untagged)
    int64_t begin, end;       // this CTA's item range
    int g_begin;              // group of begin
    int n_groups, f, kp;
    int wbytes;               // bytes of one group's B image
    float out_scale;          // layout 3: 2^e before the int16 rounding
};
static_assert(sizeof(JobCtx) <= 96, "JobCtx slot");

struct Tile {
    int64_t item;
    int cnt;      // 1 or 2 blocks
    int g;
    int job;
};

__device__ __forceinline__ int64_t block_of(const JobCtx &J, int64_t item) {
    return J.perm ? (int64_t)__ldg(J.perm + item) : item;
}

// Walks a CTA's item ranges, job after job, in tiles of up to 2 consecutive blocks
// of one group.  Groups come from the routing offsets copied to shared memory (no
// global loads on the critical path); every role runs the same walk, so tile t is
// the same tile everywhere.  Items with invalid tags sort last and are skipped.
struct TileIter {
    const JobCtx *jobs;
    int n_jobs;
    int j;
    const int32_t *offs;
    int G;
    int gi;
    int64_t item, end;
    int64_t gend;         // end of the current group's run of items (cached: the fast path
                          // of next() is one compare while a group lasts)
    __device__ void enter(int jj) {
        j = jj;
        gend = -1;        // forces the group lookup
        if (jj < n_jobs) {
            offs = jobs[jj].offs;
            G = jobs[jj].n_groups;
            gi = jobs[jj].g_begin;
            item = jobs[jj].begin;
            end = jobs[jj].end;
        }
    }
    __device__ bool next(Tile &t) {
        if (item < gend) {                                  // same group, same job
            t.item = item;
            t.g = offs ? gi : 0;
            t.job = j;
            t.cnt = (item + 1 < gend) ? 2 : 1;
            item += t.cnt;
            return true;
        }
        while (j < n_jobs) {
            if (item < end) {
                gend = end;
                bool ok = true;
                if (offs) {
                    while (gi < G && item >= offs[gi + 1]) ++gi;
                    if (gi >= G) ok = false;
                    else gend = min(end, (int64_t)offs[gi + 1]);
                }
                if (ok) {
                    t.item = item;
                    t.g = offs ? gi : 0;
                    t.job = j;
                    t.cnt = (item + 1 < gend) ? 2 : 1;
                    item += t.cnt;
                    return true;
                }
            }
            enter(j + 1);
        }
        return false;
    }
};

// Out-of-domain fix-up: the whole CTA recomputes block `item` of job J (group g) from
// global memory with the FFMA kernel's per-element arithmetic (k ascending; re: +wr sr,
// then -wi si; im: +wi sr, then +wr si; from +0), so a fixed block equals
// bf_ffma_kernel's result bit for bit.  Only blocks (or groups) outside the tensor
// domain get here; throughput does not matter.
template <int LAYOUT>
__device__ __forceinline__ void fix_block(const JobCtx &J, int64_t item, int g) {
    const int64_t blk = block_of(J, item);
    const int f = J.f;
    const float *Sb = J.S + blk * (int64_t)(120 * f);
    const float4 *Wg = J.Wp + (int64_t)g * f * 32;
    for (int e = threadIdx.x; e < bfk::kAnt * bfk::kB; e += blockDim.x) {
        const int i = e / bfk::kB, j = e - bfk::kB * i;
        const int ag = i >> 3, jw = (i & 7) >> 1;
        const bool odd = (i & 1) != 0;
        float re = +0.0f, im = +0.0f;
        for (int k = 0; k < f; ++k) {
            const float4 w4 = __ldg(Wg + k * 32 + jw * 8 + ag);   // bf_relayout_w's Wp layout
            const float wr = odd ? w4.y : w4.x, wi = odd ? w4.w : w4.z;
            float sr, si;
            if (LAYOUT != 1) {
                const float2 v = __ldg(reinterpret_cast<const float2 *>(Sb) + k * bfk::kB + j);
                sr = v.x;
                si = v.y;
            } else {
                sr = __ldg(Sb + k * bfk::kB + j);
                si = __ldg(Sb + (f + k) * bfk::kB + j);
            }
            re = fmaf(wr, sr, re);
            im = fmaf(wi, sr, im);
            re = fmaf(-wi, si, re);
            im = fmaf(wr, si, im);
        }
        float *Rb = J.R + blk * (int64_t)(bfk::r_block_bytes(LAYOUT) / 4);
        if (LAYOUT == 0) {
            reinterpret_cast<float2 *>(Rb)[e] = make_float2(re, im);
        } else if (LAYOUT == 1) {
            Rb[e] = re;
            Rb[bfk::kAnt * bfk::kB + e] = im;
        } else if (LAYOUT == 2) {
            reinterpret_cast<uint32_t *>(Rb)[e] = bfk::pack_half2(re, im);
        } else {
            reinterpret_cast<uint32_t *>(Rb)[e] = bfk::pack_i16x2(re, im, J.out_scale);
        }
    }
}

// Is S block `blk` inside the tensor domain (fix-up rescan; the split warps' test)?  Every
// value 0 or in [2^-40, 2^40); per row (RE j) every nonzero element within kRelRange
// binades of the row's largest component (element = max(|re|, |im|)); for exact W also
// every nonzero component.
template <int LAYOUT>
__device__ __forceinline__ bool block_in_domain(const JobCtx &J, int64_t blk, bool exact_w) {
    const uint32_t *Sb = reinterpret_cast<const uint32_t *>(J.S) + blk * (int64_t)(120 * J.f);
    bool ok = true;
    for (int jj = threadIdx.x; jj < 60; jj += blockDim.x) {
        int emax = 0, emin = 255, cmin = 255;
        for (int k = 0; k < J.f; ++k) {
            const uint32_t ur = __ldg(Sb + (LAYOUT != 1 ? 2 * (k * 60 + jj) : k * 60 + jj)) & 0x7FFFFFFFu;
            const uint32_t ui = __ldg(Sb + (LAYOUT != 1 ? 2 * (k * 60 + jj) + 1 : (J.f + k) * 60 + jj)) &
                                0x7FFFFFFFu;
            ok &= (ur == 0u || (ur >= kDomLo && ur < kDomHi)) && (ui == 0u || (ui >= kDomLo && ui < kDomHi));
            const int e = (int)(max(ur, ui) >> 23);
            if (ur | ui) { emax = max(emax, e); emin = min(emin, e); }
            if (ur) cmin = min(cmin, (int)(ur >> 23));
            if (ui) cmin = min(cmin, (int)(ui >> 23));
        }
        ok &= emax == 0 || (emin >= emax - kRelRange && (!exact_w || cmin >= emax - kRelRange));
    }
    return __syncthreads_and(ok) != 0;
}

// Cost-balanced split of the group-sorted item list over the CTAs.  Work is
// counted in tiles (2 blocks of one group; a group of m blocks is ceil(m / 2)
// tiles) plus a W reload per group segment (kWCost quarter-tiles, ~half a tile:
// the MMA issuer drains and reloads the group's B image), so a CTA whose range
// crosses group boundaries gets fewer tiles; an item-count split would make those
// CTAs, and with them the launch, slower (short launches: c5's 4096-block chunks).
// Boundaries fall on tile starts (group start + even offset); position x of the
// cost axis maps to an item monotonically, so adjacent CTAs share their boundary.
// Pure integer function of the offsets: results do not depend on it (a D row only
// depends on its own A row), only the timing does.
constexpr int64_t kTileCost = 4, kWCost = 2;
// Cost model of the contiguous split of a whole batch launch over its jobs (TcParams.split
// = 1), in units of 480 bytes: a tile of runtime f costs its two blocks' bytes, 2 (f + 64),
// plus ~29 units of per-tile overhead (fit of the per-f kernel times, c3 sweep); a W
// reload (group or job change) ~200 units (the ~3 us bubble of a one-buffer W change at
// one SM's share of the HBM bandwidth; tools/batch_exp.py).
__host__ __device__ constexpr int64_t split_tile_cost(int f) { return 2 * (f + 64) + 29; }
constexpr int64_t kSplitWCost = 200;

// item where cost position x falls inside group g (x_in = x - cost before g)
__device__ __forceinline__ int64_t item_at(const int32_t *offs, int g, int64_t x_in, int64_t tc,
                                           int64_t wc) {
    const int64_t m = offs[g + 1] - offs[g], r = x_in - wc;
    if (r <= 0) return offs[g];
    return offs[g] + min(m, 2 * ((r + tc - 1) / tc));
}

// Total cost of a job (warp-wide; lanes scan 32 groups at a time).
__device__ __forceinline__ int64_t job_cost(const int32_t *offs, int G, int64_t n, int lane,
                                            int64_t tc, int64_t wc) {
    if (!offs) return tc * ((n + 1) / 2);
    int64_t tot = 0;
    for (int base = 0; base < G; base += 32) {
        const int g = base + lane;
        const int64_t m = g < G ? offs[g + 1] - offs[g] : 0;
        int64_t c = m > 0 ? wc + tc * ((m + 1) / 2) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        tot += c;
    }
    return tot;
}

// One warp computes the items [begin, end) of the cost range [xb, xe) of a job of total
// cost tot (to_end: the range runs to the job's end, items with invalid tags included).
// Positions map to items monotonically, so adjacent ranges share their boundary.
__device__ __forceinline__ void cta_range_x(const int32_t *offs, int G, int64_t n, int lane,
                                            int64_t tc, int64_t wc, int64_t xb, int64_t xe,
                                            bool to_end, int64_t &begin, int64_t &end,
                                            int &g_begin) {
    g_begin = 0;
    if (!offs) {
        begin = min(n, 2 * ((xb + tc - 1) / tc));
        end = to_end ? n : min(n, 2 * ((xe + tc - 1) / tc));
        return;
    }
    auto cost = [&](int g) -> int64_t {
        if (g >= G) return 0;
        const int64_t m = offs[g + 1] - offs[g];
        return m > 0 ? wc + tc * ((m + 1) / 2) : 0;
    };
    begin = n;
    end = n;
    bool fb = false, fe = to_end;
    int64_t carry = 0;
    for (int base = 0; base < G && !(fb && fe); base += 32) {
        const int g = base + lane;
        const int64_t c = cost(g);
        int64_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        incl += carry;
        const int64_t excl = incl - c;
        const bool hb = !fb && c > 0 && xb >= excl && xb < incl;
        const bool he = !fe && c > 0 && xe >= excl && xe < incl;
        const int64_t ib = hb ? item_at(offs, g, xb - excl, tc, wc) : 0;
        const int64_t ie = he ? item_at(offs, g, xe - excl, tc, wc) : 0;
        const unsigned mb = __ballot_sync(0xffffffffu, hb), me = __ballot_sync(0xffffffffu, he);
        if (mb) {
            begin = __shfl_sync(0xffffffffu, ib, __ffs(mb) - 1);
            g_begin = base + __ffs(mb) - 1;
            fb = true;
        }
        if (me) { end = __shfl_sync(0xffffffffu, ie, __ffs(me) - 1); fe = true; }
        carry = __shfl_sync(0xffffffffu, incl, 31);
    }
}

// This CTA's [begin, end) of one job split over all CTAs (cost in tiles plus half a tile
// per group segment).
__device__ __forceinline__ void cta_range(const int32_t *offs, int G, int64_t n, int lane,
                                          int64_t &begin, int64_t &end, int &g_begin) {
    const int64_t bid = blockIdx.x, grid = gridDim.x;
    const int64_t tot = job_cost(offs, G, n, lane, kTileCost, kWCost);
    cta_range_x(offs, G, n, lane, kTileCost, kWCost, tot * bid / grid, tot * (bid + 1) / grid,
                bid + 1 == grid, begin, end, g_begin);
}

// Named barrier 1 over the 8 epilogue warps (256 threads).
__device__ __forceinline__ void epi_bar_sync() {
    asm volatile("bar.sync 1, 256;" ::: "memory");
}
template <int N = 0>
__device__ __forceinline__ void bulk_wait_read() {   // at most N bulk groups still reading smem
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA bulk store shared -> global (bulk-group completion), L2 cache hint.
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
        ::"l"(dst), "r"(tc::smem_u32(src)), "r"(bytes), "l"(policy) : "memory");
}

// ---- slot server helpers -------------------------------------------------------------
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Timeline of CTA 0's part of the last slot (bf_server_trace), %globaltimer ns:
// 0 doorbell seen, 1 descriptor published, 2 first S in shared memory (split), 3 first
// D ready (epilogue), 4 last bulk store issued, 5 stores complete, 6 counted.
#ifndef BFTC_SRV_TRACE
#define BFTC_SRV_TRACE 0   // 1: CTA 0 timeline of the last slot (tools/server_exp.py)
#endif
__device__ __forceinline__ void srv_trace(const SrvPtrs &sp, int i) {
    // (host-memory writes: a later fence in the same thread waits for them, so they stay
    // out of the product build)
    if (BFTC_SRV_TRACE && blockIdx.x == 0) sp.mb->trace[i] = globaltimer();
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Producer lane 0 of every CTA: wait for slot k (1-based), fill the CTA's descriptor ring
// entry jobs[k % ring] from the template job tmpl and publish it to the other roles
// (slot_full).  CTA 0 polls the host mailbox and re-broadcasts through SrvDev.  A poll
// longer than the timeout behaves as a stop.  Returns false on stop.
__device__ __forceinline__ bool srv_fill_slot(const SrvPtrs &sp, const TcJob &tmpl, JobCtx *ring,
                                              unsigned long long k, uint64_t *slot_full) {
    const int e = (int)(k % kSrvRing);
    SrvDev *dv = sp.dev;
    const unsigned long long t0 = globaltimer();
    bool stop = false;
    unsigned long long v[kDescWords];
#if BFTC_SRV_DIRECT
    // every CTA polls the host mailbox itself (one PCIe round trip, no re-broadcast hop)
    for (;;) {
        ld_ll6<true>(sp.mb->desc[e], v);
        if (ll_complete(v, k)) break;
        if ((long long)(globaltimer() - t0) > sp.timeout_ns) { stop = true; break; }
    }
    if (blockIdx.x == 0 && !stop) sp.mb->t_seen[e] = globaltimer();
    (void)dv;
#else
    if (blockIdx.x == 0) {
        for (;;) {
            ld_ll6<true>(sp.mb->desc[e], v);
            if (ll_complete(v, k)) break;
            if ((long long)(globaltimer() - t0) > sp.timeout_ns) { stop = true; break; }
        }
        const unsigned long long t_seen = globaltimer();
        if (stop)
            for (int i = 0; i < kDescWords; ++i) v[i] = ll_word(i == 5 ? 1u : 0u, k);
        // re-broadcast: relaxed 8-byte stores, the slot number in every word
        asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n\t"
                     "st.relaxed.gpu.global.v2.u64 [%0+16], {%3, %4};\n\t"
                     "st.relaxed.gpu.global.v2.u64 [%0+32], {%5, %6};"
                     ::"l"(dv->desc[e]), "l"(v[0]), "l"(v[1]), "l"(v[2]), "l"(v[3]), "l"(v[4]), "l"(v[5])
                     : "memory");
        if (!stop) {
            sp.mb->t_seen[e] = t_seen;
            if (BFTC_SRV_TRACE) sp.mb->trace[0] = t_seen;
        }
    } else {
        for (;;) {
            ld_ll6<false>(dv->desc[e], v);
            if (ll_complete(v, k)) break;
            if ((long long)(globaltimer() - t0) > sp.timeout_ns) { stop = true; break; }
        }
    }
#endif
    if (BFTC_SRV_TRACE && !stop && blockIdx.x < 160) sp.mb->cta_seen[blockIdx.x] = globaltimer();
    const unsigned long long dS = stop ? 0ull : ((v[0] & 0xFFFFFFFFull) | (v[1] << 32));
    const unsigned long long dR = stop ? 0ull : ((v[2] & 0xFFFFFFFFull) | (v[3] << 32));
    const long long dn = stop ? 0ll : (long long)(unsigned int)v[4];
    stop = stop || (unsigned int)v[5] != 0u;
    JobCtx &J = ring[e];
    J.Wimg = tmpl.Wimg;
    J.Wp = tmpl.Wp;
    J.S = reinterpret_cast<const float *>(dS);
    J.perm = nullptr;
    J.wexact = tmpl.wexact;
    J.R = reinterpret_cast<float *>(dR);
    J.offs = nullptr;
    J.n_groups = 1;
    J.f = tmpl.f;
    J.kp = kp_of(tmpl.f);
    J.wbytes = 2 * J.kp * 128 * 2;
    J.out_scale = tmpl.out_scale;
    J.g_begin = 0;
    const int64_t n = stop ? 0 : dn;
    int64_t b0 = 0, e0 = 0;
    int g0 = 0;
    cta_range(nullptr, 1, n, 0, b0, e0, g0);
    J.begin = b0;
    J.end = stop ? -1 : e0;                       // end = -1: the stop marker
    srv_trace(sp, 1);
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(slot_full + e))
                 : "memory");
    return !stop;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar))
                 : "memory");
}

// DBG (0 in the library) disables pieces for bottleneck experiments only
// (tools/tc_exp): 1 = no MMA issue, 2 = no R stores, 4 = no split/tcgen05.st,
// 8 = no S loads, 16 = main product as fp16-kind MMAs (energy experiment), 32 (with 16) =
// the split also writes S1 as packed fp16 (the instruction stream of a real fp16 main
// product, without range handling).
// Results are wrong with DBG != 0.
// SRV (F = 0 only): the slot server — one persistent launch; the jobs come one slot at a
// time from the host mailbox (p.srv) instead of the parameter block, which holds the
// plan's template job (precoders, f, output scale) in job[0].  Untagged slots, one group.
template <int F, int LAYOUT, int DBG = 0, bool SRV = false>
__global__ void __launch_bounds__(kThreads, 1) bf_tc_kernel(const TcParamsOf<F> p) {
    static_assert(!SRV || F == 0, "the slot server runs the runtime-f kernel");
    using L = TcSmem<F, SRV, LAYOUT == 2 || (BFTC_I16_R2 && LAYOUT == 3)>;   // (16-bit outputs: two R stages where they fit)
    // TMEM column stride of the three A regions: fixed across the jobs of a launch
    // (the split of a job's first tile must not overlap the previous job's regions
    // that its last MMAs may still read).
    constexpr int kARegion = L::KP / 2;      // fp16 pairs: KP / 2 columns per term
    // A regions double-buffered (the split of tile t + 1 overlaps tile t's MMAs) when both
    // sets of three terms fit below the D buffers
    constexpr int kABufs = (2 * 3 * kARegion <= kDCol0) ? BFTC_ABUFS : 1;
    // staged R (see TcSmem::kStageR); round 1 measured int16 output at f <= 12 faster with
    // the warps storing independently (0.41 vs 0.50 ms per 10^5 blocks, profiles/
    // r01_sweep_i16_v6.txt); round 2's two R stages make the staged epilogue faster at every f
    // (BFTC_I16_DIRECT_MAXF = 0; the direct path stays for experiments)
    constexpr bool kStageR = L::kStageR && (LAYOUT != 3 || F == 0 || F > BFTC_I16_DIRECT_MAXF);
    static_assert(kStageR || LAYOUT == 2 || LAYOUT == 3, "fp32 layouts always use the staged epilogue");
    // S ring depth used: 16-bit outputs (fp16, and int16 with the direct epilogue) keep the
    // deepest ring that fits (int16 f = 9-12: 0.55-0.59 of copy BW with 2 stages, 0.66-0.71
    // with 4; profiles/r02_rstage_ring.txt)
    constexpr int kRing = (LAYOUT == 2 || (LAYOUT == 3 && !kStageR)) ? L::kStagesAlloc : L::kStages;
    extern __shared__ __align__(1024) unsigned char smem[];
    float *Wsm = reinterpret_cast<float *>(smem);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L::kOffBar);
    // a_full[t] / a_free[t]: TMEM A region of split term t (0: S1, 1: S2, 2: S3)
    // a_full / a_free of A buffer 0 at bars + 0 / + 3, of A buffer 1 at bars + 36 / + 39
    uint64_t *bar_a_full = bars + 0, *bar_a_free = bars + 3, *bar_d_full = bars + 6,
             *bar_d_free = bars + 8, *bar_wfull = bars + 10, *bar_wfree = bars + 12,
             *bar_s_full = bars + 14, *bar_s_empty = bars + 14 + kRing,
             *bar_slot_full = bars + 24, *bar_slot_free = bars + 28,   // SRV: descriptor ring
             *bar_sig_full = bars + 32, *bar_sig_free = bars + 34;     // row scales, per D buffer
    float *Ss = reinterpret_cast<float *>(smem + L::kOffS);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + L::kOffTmem);
    JobCtx *jobs = reinterpret_cast<JobCtx *>(smem + L::kOffJobs);
    int32_t *soffs = reinterpret_cast<int32_t *>(smem + L::kOffOffs);
    // fix-up list of out-of-domain blocks: (item, job << 16 | group), its length, an
    // overflow flag, and per (S ring stage, block of the tile) the last tile listed + 1
    int2 *fix_list = reinterpret_cast<int2 *>(smem + L::kOffFix);
    int *fix_n = reinterpret_cast<int *>(smem + L::kOffFix + kFixCap * 8);
    int *fix_over = fix_n + 1;
    int *fix_last = fix_n + 4;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kNJ = F == 0 ? kMaxJobs : 1;
    const int n_jobs = SRV ? 0 : (p.n_jobs < kNJ ? p.n_jobs : kNJ);
    // ---- prologue: jobs and their group offsets into shared memory, then this CTA's
    //      cost-balanced range of every job (one warp each, shuffle scans).
    if ((int)threadIdx.x < n_jobs) {
        const TcJob &q = p.job[threadIdx.x];
        int base = 0;
        for (int i = 0; i < (int)threadIdx.x; ++i)
            if (p.job[i].offsets) base += p.job[i].n_groups + 2;
        JobCtx &J = jobs[threadIdx.x];
        J.Wimg = q.Wimg;
        J.Wp = q.Wp;
        J.S = q.S;
        J.perm = q.perm;
        J.wexact = q.wexact;
        J.R = q.R;
        J.offs = q.offsets ? soffs + base : nullptr;
        J.n_groups = q.n_groups;
        J.f = F > 0 ? F : q.f;
        J.kp = kp_of(J.f);
        J.wbytes = 2 * J.kp * 128 * 2;
        J.out_scale = q.out_scale;
        J.begin = J.end = 0;
        J.g_begin = 0;
    }
    __syncthreads();
    for (int jj = 0; jj < n_jobs; ++jj)
        if (jobs[jj].offs)
            for (int i = threadIdx.x; i < jobs[jj].n_groups + 2; i += blockDim.x)
                const_cast<int32_t *>(jobs[jj].offs)[i] = p.job[jj].offsets[i];
    __syncthreads();
    if (F == 0 && p.split == 1 && n_jobs > 1) {
        // one contiguous range of the concatenated jobs per CTA (cost: bytes + per-tile
        // overhead + W reloads, split_tile_cost / kSplitWCost): a CTA meets ~2 jobs per launch
        // instead of all of them, so far fewer W reloads
        int64_t *jcost = reinterpret_cast<int64_t *>(smem + L::kOffJCost);
        for (int jj = warp; jj < n_jobs; jj += kThreads / 32) {
            const int64_t c = job_cost(jobs[jj].offs, jobs[jj].n_groups, p.job[jj].n_items, lane,
                                       split_tile_cost(jobs[jj].f), kSplitWCost);
            if (lane == 0) jcost[jj] = c;
        }
        __syncthreads();
        int64_t X = 0;
        for (int jj = 0; jj < n_jobs; ++jj) X += jcost[jj];
        const int64_t bid = blockIdx.x, grid = gridDim.x;
        const int64_t Xb = X * bid / grid, Xe = bid + 1 == grid ? X : X * (bid + 1) / grid;
        for (int jj = warp; jj < n_jobs; jj += kThreads / 32) {
            int64_t P = 0;
            for (int i = 0; i < jj; ++i) P += jcost[i];
            const int64_t T = jcost[jj];
            const int64_t xb = min(max(Xb - P, (int64_t)0), T), xe = min(max(Xe - P, (int64_t)0), T);
            int64_t b0 = p.job[jj].n_items, e0 = b0;
            int g0 = 0;
            if (xb < xe || (Xe >= P + T && Xb < P + T))
                cta_range_x(jobs[jj].offs, jobs[jj].n_groups, p.job[jj].n_items, lane,
                            split_tile_cost(jobs[jj].f), kSplitWCost, xb, xe, Xe >= P + T, b0, e0, g0);
            if (lane == 0) {
                jobs[jj].begin = b0;
                jobs[jj].end = e0;
                jobs[jj].g_begin = g0;
            }
        }
    } else {
        for (int jj = warp; jj < n_jobs; jj += kThreads / 32) {
            int64_t b0, e0;
            int g0;
            cta_range(jobs[jj].offs, jobs[jj].n_groups, p.job[jj].n_items, lane, b0, e0, g0);
            if (lane == 0) {
                jobs[jj].begin = b0;
                jobs[jj].end = e0;
                jobs[jj].g_begin = g0;
            }
        }
    }
    __syncthreads();
    bool any = SRV;
    for (int jj = 0; jj < n_jobs; ++jj) any |= jobs[jj].begin < jobs[jj].end;
    if (!any) return;   // CTA-uniform, before any TMEM allocation

    if (warp == 0) tc::tmem_alloc<512>(tmem_slot);
    if (threadIdx.x < 4 + 2 * kMaxStages) fix_n[threadIdx.x] = 0;   // n, overflow, last[]
    if (threadIdx.x == 32) {
        for (int i = 0; i < 3; ++i) {
            bfk::mbar_init(bar_a_full + i, 32 * kSplitWarps);
            bfk::mbar_init(bar_a_free + i, 1);
            bfk::mbar_init(bar_a_full + 36 + i, 32 * kSplitWarps);
            bfk::mbar_init(bar_a_free + 36 + i, 1);
        }
        bfk::mbar_init(bar_d_full + 0, 1);
        bfk::mbar_init(bar_d_full + 1, 1);
        bfk::mbar_init(bar_d_free + 0, 32 * kEpiWarps);
        bfk::mbar_init(bar_d_free + 1, 32 * kEpiWarps);
        for (int i = 0; i < 2; ++i) {
            bfk::mbar_init(bar_wfull + i, 1);
            bfk::mbar_init(bar_wfree + i, 1);
        }
        for (int i = 0; i < kRing; ++i) {
            bfk::mbar_init(bar_s_full + i, 1);
            bfk::mbar_init(bar_s_empty + i, 32 * kSplitWarps);
        }
        for (int i = 0; i < 2; ++i) {
            bfk::mbar_init(bar_sig_full + i, 32 * kSplitWarps / 2);   // the K-half-0 warps write
            bfk::mbar_init(bar_sig_free + i, 32 * kEpiWarps);
        }
        if (SRV)
            for (int i = 0; i < kSrvRing; ++i) {
                bfk::mbar_init(bar_slot_full + i, 1);
                bfk::mbar_init(bar_slot_free + i, 1);
            }
        bfk::mbar_fence_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    TileIter it{jobs, n_jobs, 0, nullptr, 0, 0, 0, 0, -1};
    it.enter(0);
    Tile tl;
    // The next tile of this role.  SRV: when the current slot is exhausted, the epilogue
    // completes it (srv_done), the producer fills the next slot's descriptor, every role
    // then waits for it and restarts its walk on it; false on stop.
    enum { kRoleProd, kRoleSplit, kRoleMma, kRoleEpi };
    unsigned long long slot = 0;
    bool fresh = false;                   // SRV: the first tile of a slot (timeline trace)
    auto next_tile = [&](Tile &t2, int role) -> bool {
        if constexpr (!SRV) {
            return it.next(t2);
        } else {
            for (;;) {
                if (slot > 0 && it.next(t2)) return true;
                fresh = true;
                const unsigned long long u = slot / kSrvRing;     // use index of the next entry
                if (role == kRoleEpi && slot > 0 && warp == kEpiWarp0 && lane == 0) {
                    // slot done in this CTA: its R stores complete, then count it
                    srv_trace(p.srv, 4);
                    bulk_wait_all();
                    srv_trace(p.srv, 5);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    const int e = (int)(slot % kSrvRing);
                    if (*fix_n > 0) atomicExch(&p.srv.mb->error, 1);
                    // count the CTA (acq_rel: its R before the count; the last one sees all)
                    unsigned int old;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                                 : "=r"(old) : "l"(&p.srv.dev->done_cnt[e]) : "memory");
                    srv_trace(p.srv, 6);
                    if (BFTC_SRV_TRACE && blockIdx.x < 160) p.srv.mb->cta_done[blockIdx.x] = globaltimer();
                    if (old == (unsigned)(((slot - 1) / kSrvRing + 1) * gridDim.x) - 1u) {
                        // the last CTA: every CTA's R is ordered before its count (acq_rel), and
                        // the system-scope release of `done` makes them visible to the host
                        // (cumulativity) — no separate system fence
                        p.srv.mb->t_done[e] = globaltimer();
                        st_release_sys(&p.srv.mb->done, slot);
                    }
                    mbar_arrive(bar_slot_free + e);
                }
                ++slot;
                const int e = (int)(slot % kSrvRing);
                if (role == kRoleProd) {
                    if (lane == 0) {
                        if (slot > kSrvRing) bfk::mbar_wait(bar_slot_free + e, (uint32_t)((u - 1) & 1));
                        srv_fill_slot(p.srv, p.job[0], jobs, slot, bar_slot_full);
                    }
                    __syncwarp();
                }
                bfk::mbar_wait(bar_slot_full + e, (uint32_t)(((slot - 1) / kSrvRing) & 1));
                if (jobs[e].end < 0) return false;
                it = TileIter{jobs + e, 1, 0, nullptr, 0, 0, 0, 0, -1};
                it.enter(0);
            }
        }
    };

    if (warp < kSplitWarps) {
        // ------------------------------------------------------------ split warps
        const int m = (warp & 3) * 32 + lane;            // TMEM lane == A row
        const int ks = warp >> 2;                        // K half: chunks [0, h) or [h, end)
        const int bsel = m >= 60 ? 1 : 0, j = m - 60 * bsel;
        const uint32_t a_lane = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t *xch = reinterpret_cast<uint32_t *>(smem + L::kOffXch);   // [2][8 warps][32]
        int32_t *sig = reinterpret_cast<int32_t *>(smem + L::kOffSig);     // [2][128]
        int cur_g = -1, cur_j = -1;
        int cur_wf = 0;                                  // wexact flags of the current group
        const int32_t *cur_wk = nullptr;                // (SRV: its entry, kept across slots)
        for (int64_t t = 0; next_tile(tl, kRoleSplit); ++t) {
            const JobCtx &J = it.jobs[tl.job];
            constexpr int FXs = (BFTC_FIXF_ROLES & 1) ? BFTC_FIXF : 0;
            const int f = F > 0 ? F : (FXs ? FXs : J.f);
            const int KP = F > 0 ? L::KP : (FXs ? kp_of(FXs) : J.kp);
            const bool valid = m < 120 && bsel < tl.cnt;
            const int stage = (int)(t % kRing);
            bfk::mbar_wait(bar_s_full + stage, (uint32_t)((t / kRing) & 1));
            if (SRV && fresh) {
                if (warp == 0 && lane == 0) srv_trace(p.srv, 2);
                fresh = false;
            }
            const float *Sb = Ss + (stage * 2 + (valid ? bsel : 0)) * (L::kSBlock / 4);
            // Term order S2, S3, S1 mirrors the MMA order, so each region is rewritten
            // as soon as the previous tile's MMAs on it have completed and the tensor
            // pipe keeps running on the other terms meanwhile.
            // tcgen05.st is warp-collective: every lane stores (invalid rows store 0).
            // A buffer of this tile, its barriers and the parity of its a_free wait
            const int ab = kABufs == 2 ? (int)(t & 1) : 0;
            uint64_t *a_full = bar_a_full + 36 * ab, *a_free = bar_a_free + 36 * ab;
            const uint32_t par = kABufs == 2 ? (uint32_t)(((t >> 1) & 1) ^ 1) : (uint32_t)((t & 1) ^ 1);
            const uint32_t a_base = a_lane + (uint32_t)(ab * 3 * kARegion);
            if (tl.g != cur_g || tl.job != cur_j) {
                cur_g = tl.g;
                cur_j = tl.job;
                if (!SRV || J.wexact + tl.g != cur_wk) cur_wf = __ldg(J.wexact + tl.g);
                cur_wk = J.wexact + tl.g;
            }
            // The rest of the tile runs with a compile-time K extent: the per-f kernels pass
            // their own, the runtime-f batch kernel dispatches on the job's KP (5 classes), so
            // its loops and registers are sized per class instead of for f = 36.
            auto split_tile = [&](auto kp_const) {
                constexpr int KPc = decltype(kp_const)::value;
                // This warp's K chunks of the thread's row of S (half of them above f = 16) are
                // read from the ring once into registers and the slot is released at once; the
                // term passes split from registers.
                constexpr int kSlots = KPc <= 32 ? KPc / 8 : ((KPc / 8 + 1) >> 1);
                constexpr int c_half0 = KPc <= 32 ? KPc : ((KPc / 8 + 1) >> 1) * 8;
                const int c_beg0 = ks ? c_half0 : 0, c_end0 = ks ? KPc : c_half0;
                float xs[kSlots * 8];
                // tensor domain of the row: its largest element (max(|re|, |im|))
                // in [2^-40, 2^40), every nonzero element within kRelRange binades of it, no
                // NaN (the fma chain below turns any NaN into a NaN; Inf fails the range)
                float emx = 0.0f, nan_chk = 0.0f;
                uint32_t emn1 = 0xFFFFFFFFu;                 // smallest nonzero element bits - 1
    #pragma unroll
                for (int i = 0; i < kSlots; ++i) {
                    const int c0 = c_beg0 + 8 * i;
    #pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int k = c0 / 2 + q;
                        float re = 0.0f, im = 0.0f;
                        // (only the last chunk of a K class can pass f: fmin = KPc / 2 - 7)
                        if (c0 < c_end0 && (c0 + 8 <= KPc - 14 || k < f) && valid) {
                            if (LAYOUT != 1) {
                                const float2 v = reinterpret_cast<const float2 *>(Sb)[k * 60 + j];
                                re = v.x;
                                im = v.y;
                            } else {
                                re = Sb[k * 60 + j];
                                im = Sb[f * 60 + k * 60 + j];
                            }
                        }
                        xs[8 * i + 2 * q] = re;
                        xs[8 * i + 2 * q + 1] = im;
                        const float el = fmaxf(fabsf(re), fabsf(im));
                        emx = fmaxf(emx, el);
                        emn1 = min(emn1, __float_as_uint(el) - 1u);
                        nan_chk = fmaf(re, im, nan_chk);
                    }
                }
                // the row's other K half lives in the partner warp (warp ^ 4): exchange maxima
                // (up to f = 16 the first warp of each quarter holds whole rows: nothing to do)
                if constexpr (KPc > 32) {
                    float *xw = reinterpret_cast<float *>(xch) + (t & 1) * 256;
                    xw[warp * 32 + lane] = emx;
                    asm volatile("bar.sync %0, 64;" ::"r"(2 + (warp & 3)) : "memory");
                    emx = fmaxf(emx, xw[(warp ^ 4) * 32 + lane]);
                }
                const int emax = (int)(__float_as_uint(emx) >> 23);     // 0: all-zero row
                bool out_dom = nan_chk != nan_chk || emax >= (int)(kDomHi >> 23) ||
                               (emax != 0 && (emax < (int)(kDomLo >> 23) ||
                                              (emn1 != 0xFFFFFFFFu &&
                                               (int)((emn1 + 1u) >> 23) < emax - kRelRange)));
                // row scale 2^sg: the largest component lands in [2^14, 2^15); the epilogue
                // undoes sg + tau (the group's W scale) with one exact multiply
                const int sg = emax != 0 && !out_dom ? 141 - emax : 0;
                const float sc = __uint_as_float((uint32_t)(127 + sg) << 23);
    #pragma unroll
                for (int i = 0; i < kSlots * 4; ++i) {
                    float2 x2 = make_float2(xs[2 * i], xs[2 * i + 1]);
                    x2 = tc::mul2f(x2, make_float2(sc, sc));
                    xs[2 * i] = x2.x;
                    xs[2 * i + 1] = x2.y;
                }
                if (ks == 0) {
                    bfk::mbar_wait(bar_sig_free + (int)(t & 1), (uint32_t)(((t >> 1) & 1) ^ 1));
                    sig[(t & 1) * 128 + m] = sg + ((cur_wf >> 8) & 255) - 128;
                    mbar_arrive(bar_sig_full + (int)(t & 1));
                }
                if (kEarlyRelease) mbar_arrive(bar_s_empty + stage);    // values are in registers
                uint32_t tiny = 0xFFFFFFFFu;   // exact W: smallest nonzero scaled component - 1
                // Exact 3-term split of the scaled values, each term rounded to 11 significant
                // bits (integer add + mask, 2 ops): x = x1 + x2 + x3 exactly, |x - x1| <= 2^-11
                // |x|, |x3| <= 2^-22 |x|; packed as fp16 pairs (exact in fp16's normal range,
                // DESIGN.md §7).  One pass writes S1 and S2 (and S3 for exact W) chunk by chunk
                // — x1 computed once — into the tile's A buffer (free since tile t - 2's MMAs).
                // Up to f = 16 (<= 4 chunks) the second warp of each quarter only keeps the
                // barrier counts.
                {
                    const bool ex = (cur_wf & 1) != 0;     // S3 is only multiplied for exact W
                    bfk::mbar_wait(a_free + 1, par);
                    bfk::mbar_wait(a_free + 0, par);
                    bfk::mbar_wait(a_free + 2, par);
                    tc::fence_after_sync();
        #pragma unroll
                    for (int i = 0; i < kSlots; ++i) {
                        const int c0 = c_beg0 + 8 * i;
                        if (c0 >= c_end0) break;
                        uint32_t h1[4], h2[4];
        #pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float y1[2], y2[2];
        #pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                const float x = xs[8 * i + 2 * e + c];
                                y1[c] = tc::tf32_round(x);
                                y2[c] = tc::tf32_round(x - y1[c]);   // x - x1 exact
                            }
                            h1[e] = tc::pack_f16x2(y1[0], y1[1]);
                            h2[e] = tc::pack_f16x2(y2[0], y2[1]);
                        }
                        if constexpr (!(DBG & 4)) {
                            tc::tmem_st4(a_base + c0 / 2, h1);
                            tc::tmem_st4(a_base + kARegion + c0 / 2, h2);
                        }
                        if (ex) {
                            uint32_t h3[4];
        #pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                float y3[2];
        #pragma unroll
                                for (int c = 0; c < 2; ++c) {
                                    const float x = xs[8 * i + 2 * e + c];
                                    const float x1 = tc::tf32_round(x);
                                    const float r1 = x - x1;
                                    y3[c] = r1 - tc::tf32_round(r1);
                                    // all three terms exact in fp16 needs every nonzero scaled
                                    // component >= 2^-1 (else the block is fixed up)
                                    tiny = min(tiny, (__float_as_uint(x) & 0x7FFFFFFFu) - 1u);
                                }
                                h3[e] = tc::pack_f16x2(y3[0], y3[1]);
                            }
                            if constexpr (!(DBG & 4)) tc::tmem_st4(a_base + 2 * kARegion + c0 / 2, h3);
                        }
                    }
                    tc::tmem_st_wait();
                    tc::fence_before_sync();
                    mbar_arrive(a_full + 1);
                    mbar_arrive(a_full + 0);
                    mbar_arrive(a_full + 2);
                }
                out_dom |= tiny < 0x3EFFFFFFu;   // a nonzero scaled component below 2^-1
                if (valid && ((cur_wf & 2) || out_dom)) {
                    // rare: list the block once per tile (the first thread to see it wins; a
                    // stage's slot is reused only after every split warp finished this tile)
                    const int key = (int)(t + 1);
                    if (atomicMax(fix_last + 2 * stage + bsel, key) < key) {
                        const int idx = atomicAdd(fix_n, 1);
                        if (idx < kFixCap)
                            fix_list[idx] = make_int2((int)(it.item - tl.cnt + bsel), (it.j << 16) | tl.g);
                        else
                            atomicExch(fix_over, 1);
                    }
                }
            };
            if constexpr (F > 0) {
                split_tile(std::integral_constant<int, L::KP>{});
            } else if constexpr (FXs > 0) {
                split_tile(std::integral_constant<int, kp_of(FXs)>{});
            } else {
                switch (KP) {
                    case 16: split_tile(std::integral_constant<int, 16>{}); break;
                    case 32: split_tile(std::integral_constant<int, 32>{}); break;
                    case 48: split_tile(std::integral_constant<int, 48>{}); break;
                    case 64: split_tile(std::integral_constant<int, 64>{}); break;
                    default: split_tile(std::integral_constant<int, 80>{}); break;
                }
            }
            if (!kEarlyRelease) mbar_arrive(bar_s_empty + stage);   // ring slot may be refilled
        }
    } else if (warp == kProdWarp) {
        // ------------------------------------------------------------ S producer (TMA bulk)
        // It also loads each group segment's B image (W) into W buffer (segment mod
        // kWBufs) as it reaches the segment's first tile — up to kStages tiles ahead of
        // the MMAs — once the segment kWBufs back has released that buffer (wfree).
        const uint64_t pol = bfk::policy_evict_first();
        int cur_g = -1, cur_j = -1;
        int64_t seg = -1;
        // (SRV: untagged slots, block = item, and no look-ahead across a slot boundary)
        bool have = next_tile(tl, kRoleProd);
        int64_t blk0 = have ? block_of(it.jobs[tl.job], tl.item) : 0;
        int64_t blk1 = have && tl.cnt > 1 ? block_of(it.jobs[tl.job], tl.item + 1) : 0;
        const JobCtx *Jp = &it.jobs[tl.job];
        for (int64_t t = 0; have; ++t) {
            Tile nx;                       // next tile's block ids load while we wait
            bool have_nx = false;
            int64_t nb0 = 0, nb1 = 0;
            if constexpr (!SRV) {
                have_nx = it.next(nx);
                nb0 = have_nx ? block_of(jobs[nx.job], nx.item) : 0;
                nb1 = have_nx && nx.cnt > 1 ? block_of(jobs[nx.job], nx.item + 1) : 0;
            }
            const JobCtx &J = *Jp;
            constexpr int FXp = (BFTC_FIXF_ROLES & 2) ? BFTC_FIXF : 0;
            const int f = F > 0 ? F : (FXp ? FXp : J.f);
            const int stage = (int)(t % kRing);
            // S of this tile first: at a group change with one W buffer the producer then
            // waits for the previous group's MMAs to drain (wfree), and the S load's HBM
            // latency should overlap that wait and the W load instead of following them
            bfk::mbar_wait(bar_s_empty + stage, (uint32_t)(((t / kRing) & 1) ^ 1));
            if (DBG & 8) {
                if (lane == 0) mbar_arrive(bar_s_full + stage);
            } else if (lane == 0) {
                const uint32_t sbytes = (uint32_t)(480 * f);
                bfk::mbar_arrive_expect_tx(bar_s_full + stage, (uint32_t)tl.cnt * sbytes);
                bfk::bulk_g2s(Ss + (stage * 2) * (L::kSBlock / 4), J.S + blk0 * (int64_t)(120 * f),
                              sbytes, bar_s_full + stage, pol);
                if (tl.cnt > 1)
                    bfk::bulk_g2s(Ss + (stage * 2 + 1) * (L::kSBlock / 4),
                                  J.S + blk1 * (int64_t)(120 * f), sbytes, bar_s_full + stage, pol);
            }
            __syncwarp();
            // A new W segment at every group or job change; the slot server keeps the image
            // across slots (one plan and group; applied to batches this measured ~1 % slower).
            if ((tl.g != cur_g || tl.job != cur_j) && !(SRV && seg >= 0)) {
                cur_g = tl.g;
                cur_j = tl.job;
                ++seg;
                constexpr int NB = L::kWBufs;
                const int wb = (int)(seg % NB);
                const int wbytes = F > 0 ? L::kWBytes : J.wbytes;
                if (seg >= NB) bfk::mbar_wait(bar_wfree + wb, (uint32_t)(((seg / NB) - 1) & 1));
                if (lane == 0) {
                    bfk::mbar_arrive_expect_tx(bar_wfull + wb, (uint32_t)wbytes);
                    bfk::bulk_g2s(Wsm + wb * (L::kWBytes / 4), J.Wimg + (int64_t)tl.g * (wbytes / 4),
                                  (uint32_t)wbytes, bar_wfull + wb, bfk::policy_evict_last());
                }
            }
            __syncwarp();
            if constexpr (SRV) {
                have = next_tile(tl, kRoleProd);
                if (have) {
                    Jp = &it.jobs[tl.job];
                    blk0 = tl.item;
                    blk1 = tl.item + 1;
                }
            } else {
                tl = nx;
                have = have_nx;
                blk0 = nb0;
                blk1 = nb1;
                if (have) Jp = &jobs[tl.job];
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer
        int cur_g = -1, cur_j = -1;
        int64_t seg = -1;
        constexpr uint32_t idesc = tc::idesc_f16(128, 128);
        uint32_t w_base = tc::smem_u32(Wsm);
        bool exact = false;
        for (int64_t t = 0; next_tile(tl, kRoleMma); ++t) {
            const JobCtx &J = it.jobs[tl.job];
            constexpr int FXm = (BFTC_FIXF_ROLES & 4) ? BFTC_FIXF : 0;
            const int KP = F > 0 ? L::KP : (FXm ? kp_of(FXm) : J.kp);
            if ((tl.g != cur_g || tl.job != cur_j) && !(SRV && seg >= 0)) {   // new W segment (producer's rule)
                exact = (__ldg(J.wexact + tl.g) & 1) != 0;
                // the previous segment's buffer is free once every MMA issued so far completed
                if (seg >= 0 && lane == 0) tc::mma_commit(bar_wfree + (int)(seg % L::kWBufs));
                __syncwarp();
                ++seg;
                const int wb = (int)(seg % L::kWBufs);
                bfk::mbar_wait(bar_wfull + wb, (uint32_t)((seg / L::kWBufs) & 1));
                w_base = tc::smem_u32(Wsm + wb * (L::kWBytes / 4));
                cur_g = tl.g;
                cur_j = tl.job;
            }
            const int b = (int)(t & 1);
            const uint32_t u = (uint32_t)(t >> 1);
            const uint32_t d = tmem + kDCol0 + 128 * b;
            bfk::mbar_wait(bar_d_free + b, (u & 1) ^ 1);
            const int ab = kABufs == 2 ? b : 0;            // A buffer of this tile (split's rule)
            uint64_t *a_full = bar_a_full + 36 * ab, *a_free = bar_a_free + 36 * ab;
            const uint32_t apar = kABufs == 2 ? (uint32_t)(u & 1) : (uint32_t)(t & 1);
            const uint32_t a_tm = tmem + (uint32_t)(ab * 3 * kARegion);
            // MMA groups over K, small terms first, every one kind::f16 on fp16 terms of the
            // scaled operands (exact 11-bit x 11-bit products, fp32 accumulate):
            //   exact W (W2 == 0, e.g. identity / selection): S2 W1, S3 W1, S1 W1
            //   (= S W exactly up to accumulation rounding: copies are bit-exact);
            //   general W: S2 W1, S1 W2, S1 W1 (the S3 region is not used) — 3 KP/16 MMAs
            //   (DESIGN.md §7).  The middle group of general W reads the S1 region.
            // Each split term's TMEM region is released by a commit once read.
            // The K extent is a compile-time constant in the issue loop (the runtime-f
            // kernel dispatches on the job's KP): descriptors then come precomputed and an
            // MMA issues in ~10 instructions instead of ~16 (runtime loop: -8 % at f = 35).
            auto mma_groups = [&](auto kp_const) {
                constexpr int KPc = decltype(kp_const)::value;
    #pragma unroll
                for (int grp = 0; grp < 3; ++grp) {
                    const int at = grp == 0 ? 1 : (grp == 1 ? 2 : 0);   // barrier: S2, S3, S1
                    bfk::mbar_wait(a_full + at, apar);
                    const bool s1w2 = grp == 1 && !exact;
                    if (s1w2) bfk::mbar_wait(a_full + 0, apar);
                    tc::fence_after_sync();
                    const int areg = s1w2 ? 0 : at;                     // A region read
                    const uint32_t boff = s1w2 ? (uint32_t)(KPc / 8) : 0u;  // W2 image after W1
                    if (lane == 0) {
                        // K = 16 per MMA: 8 TMEM columns of fp16 pairs of A, two 16-byte K
                        // chunks (2 x 2048 bytes) of the B image
    #pragma unroll
                        for (int kb = 0; kb < KPc / 16; ++kb) {
                            const uint64_t desc = tc::smem_desc(
                                w_base + (uint32_t)((boff + 2 * kb) * 16 * 128), 16 * 128, 128);
                            if constexpr (!(DBG & 1))
                                tc::mma_f16_ts(d, a_tm + areg * kARegion + kb * 8, desc, idesc,
                                               (grp | kb) != 0);
                        }
                        if (grp < 2) tc::mma_commit(a_free + at);
                    }
                    __syncwarp();
                }
            };
            if constexpr (F > 0) {
                mma_groups(std::integral_constant<int, L::KP>{});
            } else if constexpr (FXm > 0) {
                mma_groups(std::integral_constant<int, kp_of(FXm)>{});
            } else {
                switch (KP) {
                    case 16: mma_groups(std::integral_constant<int, 16>{}); break;
                    case 32: mma_groups(std::integral_constant<int, 32>{}); break;
                    case 48: mma_groups(std::integral_constant<int, 48>{}); break;
                    case 64: mma_groups(std::integral_constant<int, 64>{}); break;
                    default: mma_groups(std::integral_constant<int, 80>{}); break;
                }
            }
            if (lane == 0) {
                tc::mma_commit(a_free + 0);
                tc::mma_commit(bar_d_full + b);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ epilogue warps
        // Two warps per TMEM lane quarter; each reads its 64 D columns (32 antennas)
        // of the thread's row from TMEM first, so the buffer is released (D_free)
        // before the global stores are issued; the stores then overlap the next
        // tile's MMAs.  A warp's store covers 32 consecutive REs of one antenna row:
        // 256 contiguous bytes.  Eight storing warps keep more writes in flight
        // than four (tools/write_bw).
        const int q = warp & 3;                          // TMEM lane quarter of this warp
        const int h = (warp - kEpiWarp0) >> 2;           // D columns [64 h, 64 h + 64)
        const int m = q * 32 + lane;
        const int bsel = m >= 60 ? 1 : 0, j = m - 60 * bsel;
        const bool e0 = warp == kEpiWarp0 && lane == 0;  // issues the staged bulk stores
        const int32_t *sig = reinterpret_cast<const int32_t *>(smem + L::kOffSig);   // [2][128]
        uint64_t pol_r = 0;
        if (kStageR && e0) pol_r = bfk::policy_evict_first();
        for (int64_t t = 0; next_tile(tl, kRoleEpi); ++t) {
            const JobCtx &J = it.jobs[tl.job];
            const int b = (int)(t & 1);
            const uint32_t u = (uint32_t)(t >> 1);
            const bool valid = m < 120 && bsel < tl.cnt;
            const int64_t blk = valid ? block_of(J, tl.item + bsel) : 0;
            float *Rb = J.R + blk * (int64_t)(bfk::r_block_bytes(LAYOUT) / 4);
            // the bulk-storing thread's block ids, loaded before the wait (routed order: global
            // loads whose latency would otherwise delay the stores)
            int64_t sblk[2] = {0, 0};
            if (kStageR && e0) {
                sblk[0] = block_of(J, tl.item);
                if (tl.cnt > 1) sblk[1] = block_of(J, tl.item + 1);
            }
            bfk::mbar_wait(bar_d_full + b, u & 1);
            tc::fence_after_sync();
            if (SRV && fresh) {
                if (warp == kEpiWarp0 && lane == 0) srv_trace(p.srv, 3);
                fresh = false;
            }
            // the row's scale 2^-(sg + tau) from the split warps: one exact multiply (exact
            // unless the result is subnormal)
            bfk::mbar_wait(bar_sig_full + b, u & 1);
            const float us = __uint_as_float((uint32_t)(127 - sig[b * 128 + m]) << 23);
            mbar_arrive(bar_sig_free + b);
            const uint32_t d = tmem + ((uint32_t)(q * 32) << 16) + kDCol0 + 128 * b + 64 * h;
            if constexpr (!(DBG & 2) && !kStageR && (LAYOUT == 2 || LAYOUT == 3)) {
                // 16-bit output, direct stores (int16 output in BFTC_I16_DIRECT_MAXF builds), in
                // two halves of 16 antennas to stay inside the register budget of 18 warps:
                // load 32 D columns, pack, store; the TMEM buffer is released after the
                // second load (the MMA needs it again only two tiles later).  Lane pairs
                // (j even, j + 1) trade values with one shuffle so every lane stores two
                // adjacent REs (8 bytes) at once; a half's 8 pairs are packed first — the
                // shuffles need every lane — then one branch around their stores.
                const bool odd = (j & 1) != 0;
                const float osc = J.out_scale;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    uint32_t v[32];
                    tc::tmem_ld16(d + 32 * half, *reinterpret_cast<uint32_t(*)[16]>(v));
                    tc::tmem_ld16(d + 32 * half + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
                    tc::tmem_ld_wait();
                    if (half == 1) {
                        tc::fence_before_sync();
                        mbar_arrive(bar_d_free + b);     // TMEM buffer b may be overwritten
                    }
                    uint2 pk[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int aa = 2 * i;            // antenna pair within the half
                        const float2 z0 = tc::mul2f(make_float2(__uint_as_float(v[2 * aa]), __uint_as_float(v[2 * aa + 1])),
                                                    make_float2(us, us));
                        const float2 z1 = tc::mul2f(make_float2(__uint_as_float(v[2 * aa + 2]),
                                                                __uint_as_float(v[2 * aa + 3])), make_float2(us, us));
                        const float re0 = z0.x, im0 = z0.y, re1 = z1.x, im1 = z1.y;
                        const float gr = __shfl_xor_sync(0xffffffffu, odd ? re0 : re1, 1);
                        const float gi = __shfl_xor_sync(0xffffffffu, odd ? im0 : im1, 1);
                        // even lane: antenna a, REs j, j+1; odd lane: antenna a+1, REs j-1, j
                        const float4 w4 = odd ? make_float4(gr, gi, re1, im1) : make_float4(re0, im0, gr, gi);
                        pk[i] = LAYOUT == 3
                                    ? make_uint2(bfk::pack_i16x2(w4.x, w4.y, osc), bfk::pack_i16x2(w4.z, w4.w, osc))
                                    : make_uint2(bfk::pack_half2(w4.x, w4.y), bfk::pack_half2(w4.z, w4.w));
                    }
                    if (valid) {
                        uint2 *Rw = reinterpret_cast<uint2 *>(Rb);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int a = 32 * h + 16 * half + 2 * i;
                            const int e = (a + (odd ? 1 : 0)) * 60 + j - (odd ? 1 : 0);   // element index
                            __stcs(Rw + e / 2, pk[i]);
                        }
                    }
                }
                continue;
            }
            uint32_t v[64];
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 16)
                tc::tmem_ld16(d + c0, *reinterpret_cast<uint32_t(*)[16]>(v + c0));
            tc::tmem_ld_wait();
            tc::fence_before_sync();
            mbar_arrive(bar_d_free + b);                 // TMEM buffer b may be overwritten
            if constexpr (!(DBG & 2) && kStageR) {
                // staged: both blocks of the tile in their global layout in shared memory,
                // then one bulk store per block by the first epilogue thread.  The previous
                // tile's stores must have read the stage first.
                constexpr int rbf = bfk::r_block_bytes(LAYOUT) / 4;   // floats per block
                // two R stages for fp16 output (fp32 output measured slower with two: f = 4-12
                // 0.85 vs 0.90 of copy BW; fp16 output f = 1-16 0.68-0.87 -> 0.79-0.92)
                constexpr int kRUse = L::kRStages;
                float *Rst = reinterpret_cast<float *>(smem + L::kOffR) +
                             (kRUse == 2 ? (int)(t & 1) * (L::kRStageBytes / 4) : 0);
                if (e0) bulk_wait_read<kRUse - 1>();   // this stage's previous stores read it
                epi_bar_sync();
                if (valid) {
                    float *Rt = Rst + bsel * rbf;
                    // int16 output: the row's unscale folds into the output scale (both powers
                    // of two), one multiply per value instead of two
                    const float osc = LAYOUT == 3 ? J.out_scale * us : J.out_scale;
#pragma unroll
                    for (int aa = 0; aa < 32; ++aa) {
                        const int a = 32 * h + aa;
                        const float2 raw = make_float2(__uint_as_float(v[2 * aa]), __uint_as_float(v[2 * aa + 1]));
                        const float2 z = LAYOUT == 3 ? raw : tc::mul2f(raw, make_float2(us, us));
                        const float re = z.x, im = z.y;
                        if (LAYOUT == 0)
                            *reinterpret_cast<float2 *>(Rt + 2 * (a * 60 + j)) = make_float2(re, im);
                        else if (LAYOUT == 1) {
                            Rt[a * 60 + j] = re;
                            Rt[64 * 60 + a * 60 + j] = im;
                        } else if (LAYOUT == 2)
                            reinterpret_cast<uint32_t *>(Rt)[a * 60 + j] = bfk::pack_half2(re, im);
                        else
                            reinterpret_cast<uint32_t *>(Rt)[a * 60 + j] = bfk::pack_i16x2(re, im, osc);
                    }
                }
                bfk::fence_proxy_async_smem();         // this thread's writes -> the bulk copies
                epi_bar_sync();
                if (e0) {
                    for (int b2 = 0; b2 < tl.cnt; ++b2)
                        bulk_s2g(J.R + sblk[b2] * (int64_t)rbf, Rst + b2 * rbf,
                                 (uint32_t)bfk::r_block_bytes(LAYOUT), pol_r);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            }
        }
    }
    if (kStageR && warp == kEpiWarp0 && lane == 0) {
        bulk_wait_all();                                   // stage read, stores done
        asm volatile("fence.proxy.async.global;" ::: "memory");   // before any fix-up rewrite
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after_sync();
        tc::tmem_free<512>(tmem);
    }
    // ---- fix-up of out-of-domain blocks (CTA-uniform; nothing to do in practice): the
    //      listed blocks, or after an overflow every block of this CTA's ranges rechecked.
    const int nfix = SRV ? 0 : *fix_n;   // SRV: reported per slot (mailbox error) instead
    if (nfix > 0) {
        if (*fix_over == 0) {
            for (int e = 0; e < nfix; ++e) {
                const int2 en = fix_list[e];
                fix_block<LAYOUT>(jobs[en.y >> 16], en.x, en.y & 0xFFFF);
            }
        } else {
            TileIter it2{jobs, n_jobs, 0, nullptr, 0, 0, 0, 0, -1};
            it2.enter(0);
            Tile t2;
            while (it2.next(t2)) {
                const JobCtx &J = jobs[t2.job];
                const bool wbad = (__ldg(J.wexact + t2.g) & 2) != 0;
                for (int b2 = 0; b2 < t2.cnt; ++b2)
                    if (wbad || !block_in_domain<LAYOUT>(J, block_of(J, t2.item + b2),
                                                         (__ldg(J.wexact + t2.g) & 1) != 0))
                        fix_block<LAYOUT>(J, t2.item + b2, t2.g);
            }
        }
    }
}

}  // namespace bftc
