/*
 * bf.h — C ABI of the B200 beamforming library (libbf.so).
 *
 * The operation (§III, beamforming equation):
 *   "The beam forming algorithm computes many products W x S where W the
 *    precoding matrix is constant and S the symbols matrix is changing.  A row
 *    i of W corresponds to one antenna (here there are 64).  Matrix S has f
 *    rows, one per parallel flow, and b columns, one per resource element ...
 *    where b = 60 and constant f can vary from 0 to 36."
 *
 *   For every block n with precoder group g = group_idx[n] (0 when no tags):
 *       R[n][i][j] = sum_{k<f} W[g][i][k] * S[n][k][j]     complex fp32,
 *   accumulated in fp32 from +0.0f (by CUDA-core FFMAs or by error-compensated
 *   tensor-core MMAs, see bf_variant).  Accuracy contract (BASELINE.json
 *   north_star item 4): |R - R_exact| <= 1e-5 * sum_k |W[g][i][k]| |S[n][k][j]|
 *   per element (complex modulus; DESIGN.md §7 proves it for both kernels, given
 *   finite inputs whose nonzero products |w||s| are normal fp32 numbers, i.e. no
 *   underflow); bit-exact for f = 0 (+0.0) and for identity / selection W.
 *   Non-finite inputs propagate per IEEE to the elements that use them.
 *
 * The calls follow the paper's statement: W is set once (bf_set_precoders),
 * then many S blocks are multiplied by it (bf_apply).  Multiple precoder
 * groups (per-subband W, BASELINE.json configs[3], configs[4]) extend the
 * paper's single W; blocks pick their group through group_idx.
 *
 * Element type: complex float32 = 8 bytes.  Layouts (per block, row-major):
 *   BF_LAYOUT_INTERLEAVED  W [n_groups][n_ant][f]  (re, im) pairs
 *                          S [n_blocks][f][b]       (re, im) pairs
 *                          R [n_blocks][n_ant][b]   (re, im) pairs
 *   BF_LAYOUT_PLANAR       W [n_groups][2][n_ant][f]  re plane then im plane
 *                          S [n_blocks][2][f][b]
 *                          R [n_blocks][2][n_ant][b]
 *   Both layouts move the same bytes per block: S 8*f*b, R 8*n_ant*b.
 *   BF_LAYOUT_INTERLEAVED_F16OUT: as interleaved, R in fp16 pairs (4*n_ant*b).
 *   BF_LAYOUT_INTERLEAVED_I16OUT: as interleaved, R in int16 pairs (4*n_ant*b).
 *
 * Supported domain: n_ant == 64, b == 60, 0 <= f <= 36, 1 <= n_groups <= 1024,
 * 0 <= n_blocks < 2^31.  Other shapes return BF_ERR_UNSUPPORTED (there is no
 * slow or CPU fallback).
 *
 * Ownership: the plan owns a device copy of W (re-laid out for the kernel)
 * and its workspace (routing arrays, host-pipeline staging), grown on demand.
 * The caller owns S, R and group_idx and keeps them alive until the stream
 * work completes.  R is fully overwritten, never accumulated, and must not
 * overlap S.  A plan is bound to the CUDA device current at bf_plan_create.
 *
 * Errors: every call returns a bf_status; no exception crosses the ABI.
 * Argument errors are detected synchronously before anything is enqueued.
 * Launch errors return BF_ERR_CUDA with a detail string (bf_last_error,
 * thread-local).  Device faults surface at the caller's next synchronisation.
 * Tags outside [0, n_groups) are a caller precondition violation: such blocks
 * are left unwritten (never an out-of-bounds access); with the environment
 * variable BF_CHECK=1, bf_apply synchronises and returns BF_ERR_INVALID_VALUE.
 *
 * Streams are passed as void* (a cudaStream_t; NULL = legacy default stream),
 * so callers need no CUDA headers.  All enqueueing calls are asynchronous with
 * respect to the host unless stated otherwise.
 *
 * Concurrency: distinct plans are independent.  A plan is not thread-safe: it
 * must not be used from several host threads at the same time.  bf_set_precoders must not race
 * with in-flight applies of the same plan.  Untagged applies of one plan may
 * run on several streams concurrently (read-only W); tagged applies share the
 * plan's routing workspace and must be serialised by the caller (one stream).
 */
#ifndef BF_H
#define BF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BF_VERSION 1

typedef struct bf_plan_s *bf_plan_t;

typedef enum {
    BF_LAYOUT_INTERLEAVED = 0,
    BF_LAYOUT_PLANAR = 1,
    /* W and S interleaved complex fp32 as BF_LAYOUT_INTERLEAVED, R written as
     * interleaved IEEE binary16 (re, im) pairs [n_blocks][n_ant][b], each rounded
     * once (round-to-nearest-even) from the fp32 result: 15,360 bytes per block
     * instead of 30,720 (reduced-precision fronthaul
     * output).  Accuracy: |R16 - R_exact| <= sqrt(2) 2^-11 |R_exact| + 1e-5 T. */
    BF_LAYOUT_INTERLEAVED_F16OUT = 2,
    /* W and S as BF_LAYOUT_INTERLEAVED, R written as interleaved int16 (re, im)
     * fronthaul samples [n_blocks][n_ant][b]: round-to-nearest-even of R x 2^e from
     * the fp32 result, saturated to [-32768, 32767], NaN -> 0 (SURVEY.md §8(f) row 4,
     * "int16 fronthaul samples"); e = bf_plan_set_output_exponent, default 12.
     * 15,360 bytes per block. */
    BF_LAYOUT_INTERLEAVED_I16OUT = 3
} bf_layout;

/* Kernel variant.  Both compute the same product within the same contract.
 *   BF_VARIANT_FFMA    CUDA-core kernel: 4 fp32 FFMA per complex MAC.
 *   BF_VARIANT_TENSOR  tcgen05 tensor-core kernel: every row of S (one RE) and
 *                      every precoder group scaled by a power of two into fp16's
 *                      range, S split exactly into 3 terms of 11-bit significands,
 *                      W into 2 (+ a 2^-22 residual), the terms as fp16; S2 W1 +
 *                      S1 W2 + S1 W1 as kind::f16 MMAs (S2 W1 + S3 W1 + S1 W1 when W
 *                      is exact in one fp16 term), every product exact, fp32
 *                      accumulation in TMEM, exact unscale (error-compensated split
 *                      precision, BASELINE.json north_star item 2).
 *                      Tensor domain: per row of S the largest element
 *                      max(|re|, |im|) 0 or in [2^-40, 2^40), no NaN, every nonzero
 *                      element within 2^14 of the row's largest component (for
 *                      exact W every nonzero component within 2^15); per group of W
 *                      the same with entries in [2^-40, 2^40).  Blocks with a row
 *                      outside it and blocks of groups outside it are recomputed
 *                      inside the same launch with the FFMA kernel's arithmetic
 *                      (bitwise equal to BF_VARIANT_FFMA).
 *   BF_VARIANT_AUTO    per-(f, layout) choice from the measured variant table
 *                      (default): FFMA at small f, tensor above; FFMA whenever a
 *                      precoder entry lies outside the tensor domain. */
typedef enum {
    BF_VARIANT_AUTO = 0,
    BF_VARIANT_FFMA = 1,
    BF_VARIANT_TENSOR = 2
} bf_variant;

typedef enum {
    BF_OK = 0,
    BF_ERR_INVALID_VALUE = 1,   /* NULL / negative / overlapping / wrong-device argument */
    BF_ERR_UNSUPPORTED = 2,     /* shape outside the compiled domain (n_ant, b, f, n_groups) */
    BF_ERR_NO_PRECODERS = 3,    /* bf_apply before bf_set_precoders (f > 0) */
    BF_ERR_MISALIGNED = 4,      /* device pointer not 16-byte aligned (tags: 4-byte) */
    BF_ERR_OUT_OF_MEMORY = 5,   /* device or pinned allocation failed */
    BF_ERR_CUDA = 6,            /* CUDA runtime error; see bf_last_error() */
    BF_ERR_NO_DEVICE = 7        /* no CUDA device visible */
} bf_status;

/* Create a plan for R = W x S with the given dimensions and layout.
 * n_ant: antennas (rows of W, must be 64); f: flows (0..36); b: resource
 * elements (must be 60); layout: a bf_layout.  Validates the dimensions
 * before touching the GPU (so dimension errors are reported without one).
 * *out receives the plan (unchanged on error). */
bf_status bf_plan_create(int n_ant, int f, int b, int layout, bf_plan_t *out);

/* Copy n_groups precoders from device memory W_dev (layout as above, 16-byte
 * aligned) into the plan, re-laid out for the kernel, ordered on `stream`.
 * With f == 0 W_dev may be NULL.  Replaces any previous precoders.  For f > 0
 * this call synchronises `stream` once before returning (it reads back the
 * per-group tensor-domain flags that BF_VARIANT_AUTO's choice depends on), so
 * the caller may free W_dev when it returns; not for use inside stream capture. */
bf_status bf_set_precoders(bf_plan_t p, const void *W_dev, int n_groups, void *stream);

/* R_dev = W[group_idx[n]] x S_dev[n] for n in [0, n_blocks), on `stream`.
 * S_dev, R_dev: device pointers, 16-byte aligned, layout as above.
 * group_idx_dev: device int32 per block, or NULL (every block uses group 0).
 * n_blocks == 0 is a no-op.  With f == 0, R is set to +0.0 and S_dev may be
 * NULL.  The result of block n is bitwise independent of n_blocks, of the
 * other blocks, of the stream and of the tags of other blocks. */
bf_status bf_apply(bf_plan_t p, const void *S_dev, const int32_t *group_idx_dev,
                   void *R_dev, int64_t n_blocks, void *stream);

/* Same product with HOST buffers (pinned for full speed; pageable works but
 * serialises the copies): the library pipelines chunks host->device, the same
 * kernels as bf_apply, and device->host on internal streams, ordered after
 * prior work on `stream`; `stream` waits for the last copy before returning
 * control of ordering to the caller.  The call returns after enqueueing; the
 * host buffers must stay valid until `stream` is synchronised. */
bf_status bf_apply_host(bf_plan_t p, const void *S_host, const int32_t *group_idx_host,
                        void *R_host, int64_t n_blocks, void *stream);

/* Routing step of bf_apply exposed for testing: a
 * stable counting sort of blocks by tag.  perm_dev[int32 n_blocks] receives
 * block ids ordered by (tag, block id); offsets_dev[int32 n_groups + 2]
 * receives the start of each group, then the number of valid tags, then
 * n_blocks (invalid tags sort last).  Uses the plan's precoder count. */
bf_status bf_route(bf_plan_t p, const int32_t *group_idx_dev, int64_t n_blocks,
                   int32_t *perm_dev, int32_t *offsets_dev, void *stream);

/* Apply to blocks already routed by bf_route (same tags, same plan precoder
 * count): perm_dev / offsets_dev as bf_route wrote them, or both NULL (every
 * block uses group 0).  Lets a streaming caller route the next batch on another
 * stream while this one is beamformed; the result equals bf_apply bitwise.
 * perm / offsets that did not come from bf_route are a precondition violation. */
bf_status bf_apply_routed(bf_plan_t p, const void *S_dev, const int32_t *perm_dev,
                          const int32_t *offsets_dev, void *R_dev, int64_t n_blocks,
                          void *stream);

/* One job of bf_apply_batch: bf_apply_routed(plan, S_dev, perm_dev, offsets_dev,
 * R_dev, n_blocks) — the same arguments with the same rules (alignment, R not
 * overlapping S, perm / offsets from bf_route or both NULL). */
typedef struct {
    bf_plan_t plan;
    const void *S_dev;
    const int32_t *perm_dev;
    const int32_t *offsets_dev;
    void *R_dev;
    int64_t n_blocks;
} bf_batch_job;

/* Many routed applies in one kernel launch ("many products W x S", PAPER.md:84,
 * over several precoder sets at once, e.g. consecutive streaming chunks of
 * different cells).  Equivalent to calling
 * bf_apply_routed for jobs[0..n_jobs) in order on `stream`, with bitwise equal
 * results (for a plan whose AUTO choice is the FFMA kernel, equal to that call
 * with the plan set to BF_VARIANT_TENSOR).
 *   Packing: jobs whose plan is BF_VARIANT_AUTO or _TENSOR (any f >= 1) go into
 *   tensor-core launches of up to 16 jobs, each job split over every CTA, so one
 *   kernel fill and drain is paid per pack instead of per job; f = 0 jobs and
 *   plans set to BF_VARIANT_FFMA run as their own applies, in order.
 *   Grid, profiling record and launch count follow job 0's plan
 *   (bf_plan_set_sm_share, bf_plan_set_profiling).
 *   Every plan must live on one device and share job 0's layout.  Every job is
 *   validated before anything is enqueued (BF_ERR_INVALID_VALUE /
 *   BF_ERR_MISALIGNED naming the job); a tagged job whose plan has more than
 *   1026 groups is BF_ERR_UNSUPPORTED.  n_jobs == 0 is a no-op.  Jobs may share
 *   a plan (read-only), but a job's R must not overlap another job's S or R
 *   (precondition, not checked). */
bf_status bf_apply_batch(const bf_batch_job *jobs, int n_jobs, void *stream);

/* Free the plan and everything it owns.  Call after its work has drained. */
bf_status bf_destroy(bf_plan_t p);

/* Instrumentation (used by bench.py; never changes results).
 * set_profiling(1): every bf_apply also records CUDA events around the main
 * beamforming kernel on its launching stream (at most 65,536 launches are kept
 * between two kernel_time calls).  kernel_time: synchronises those events,
 * returns the summed milliseconds and number of timed launches, and clears the
 * record.  launch_count: kernels this plan has launched so far
 * (routing, relayout and beamforming kernels; memsets and copies excluded). */
bf_status bf_plan_set_profiling(bf_plan_t p, int enable);
bf_status bf_plan_kernel_time(bf_plan_t p, double *total_ms, int64_t *n_launches);
bf_status bf_plan_launch_count(bf_plan_t p, int64_t *count);

/* Select the kernel variant (a bf_variant) used by later applies of this plan;
 * get_variant reports the variant AUTO resolves to for this plan's f
 * (BF_VARIANT_AUTO itself when f == 0, which only writes zeros). */
bf_status bf_plan_set_variant(bf_plan_t p, int variant);
bf_status bf_plan_get_variant(bf_plan_t p, int *resolved);

/* Chunk size (blocks) of bf_apply_host's pipeline; 0 selects the default. */
bf_status bf_plan_set_host_chunk(bf_plan_t p, int64_t blocks);

/* int16 output layout: later applies write sat(rne(R x 2^e)); e in [-64, 64]
 * (BF_ERR_INVALID_VALUE otherwise), default 12.  No effect on other layouts. */
bf_status bf_plan_set_output_exponent(bf_plan_t p, int e);

/* Number of SMs the beamforming kernel of later applies spreads over
 * (grid = sms x resident CTAs per SM, capped by the block count); 0 = every SM
 * of the device (the default), values above the SM count are clamped.  Keeps
 * SMs free for concurrent work on other streams (the c5 bench leaves 2 SMs to
 * its single-CTA routing kernels) or lets several plans share the GPU.  Never
 * changes results (the block -> CTA split does not enter the arithmetic).
 * BF_ERR_INVALID_VALUE if sms < 0. */
bf_status bf_plan_set_sm_share(bf_plan_t p, int sms);

/* Static description of the kernel chosen for this plan: grid and block size
 * for n_blocks, dynamic shared memory bytes and resident CTAs per SM. */
bf_status bf_plan_kernel_config(bf_plan_t p, int64_t n_blocks, int *grid, int *block,
                                int *smem_bytes, int *ctas_per_sm);

/* ---- slot server: latency-bound applies without a launch per slot ----------------
 * One persistent launch of the tensor kernel (runtime-f form, one CTA per SM of the
 * plan's SM share) stays resident and serves untagged applies ("slots", e.g. one
 * 5G NR slot of BASELINE.json configs[1]) posted through a mailbox in mapped pinned
 * host memory: no launch, no kernel prologue and no precoder load per slot, so a
 * slot costs its data movement plus the pipeline's fill and drain.  Same arithmetic
 * and results, bit for bit, as bf_apply with BF_VARIANT_TENSOR ("many
 * products W x S" with W constant).
 *   bf_server_create: plan with f >= 1, exactly one precoder group, precoders in the
 *     tensor domain (else BF_ERR_UNSUPPORTED).  The plan must outlive the server and
 *     must not be re-configured while the server runs.
 *   bf_server_start: launches the server on `stream`.  While it runs it occupies the
 *     SMs of the plan's SM share: work on other streams waits for those SMs (use
 *     bf_plan_set_sm_share to leave some free).  It exits by bf_server_stop, or by
 *     itself after 60 s without a slot.
 *   bf_server_submit: posts R_dev = W x S_dev for n_blocks (layout of the plan,
 *     validated as bf_apply); non-blocking, returns a ticket (1, 2, ...).  At most 4
 *     slots are in flight: a fifth submit waits for the oldest.  S and R must stay
 *     valid until the slot is done.
 *   bf_server_wait: returns when slot `ticket` is done (its R written and visible to
 *     the host and later stream work), BF_ERR_CUDA after timeout_s seconds (<= 0:
 *     no limit) or if the server died; BF_ERR_INVALID_VALUE if a slot held S values
 *     outside the tensor domain (the server does not run the FFMA fix-up: such data
 *     goes through bf_apply).
 *   bf_server_slot_time: device time of a done slot (among the last 4): from CTA 0
 *     seeing the slot's doorbell to the last CTA finishing it, in microseconds
 *     (%globaltimer).
 *   bf_server_stop: posts the stop slot and synchronises the server's stream. */
typedef struct bf_server_s *bf_server_t;
bf_status bf_server_create(bf_plan_t p, bf_server_t *out);
bf_status bf_server_start(bf_server_t s, void *stream);
bf_status bf_server_submit(bf_server_t s, const void *S_dev, void *R_dev, int64_t n_blocks,
                           uint64_t *ticket);
bf_status bf_server_wait(bf_server_t s, uint64_t ticket, double timeout_s);
bf_status bf_server_slot_time(bf_server_t s, uint64_t ticket, double *device_us);
bf_status bf_server_stop(bf_server_t s);
/* Instrumentation (library built with -DBFTC_SRV_TRACE=1; otherwise -1 entries): the
 * timeline of CTA 0's part of the last done slot, microseconds after CTA 0 saw its
 * doorbell: [0] 0, [1] descriptor published to the CTA, [2] first S block in shared
 * memory, [3] first D tile ready, [4] last R store issued, [5] R stores complete, [6] slot
 * counted (-1: not reached); then [8 + c] CTA c's slot start and [168 + c] its count
 * (c < 160).  us[0..min(n, 328)). */
bf_status bf_server_trace(bf_server_t s, double *us, int n);
bf_status bf_server_destroy(bf_server_t s);

const char *bf_status_string(bf_status s);
const char *bf_last_error(void);  /* thread-local detail of the last failure */
int bf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BF_H */
