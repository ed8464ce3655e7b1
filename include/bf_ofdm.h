/*
 * bf_ofdm.h — C ABI of the OFDM output stage of libbf.so: beamforming followed by the
 * per-antenna OFDM IFFT with cyclic prefix ("fuse the per-antenna
 * OFDM IFFT").
 *
 * The paper names the stages of its downlink pipeline (§II: the
 * beamformer's output goes through per-antenna OFDM modulation before the fronthaul) and the
 * 2048-point transforms of its filter (§III); it gives no formula for this
 * stage.  DESIGN.md §2 readings O1-O5 fix one (the oracle, oracle/ofdm_oracle.c, follows
 * them step by step):
 *   O1  R = W x S per block exactly as bf.h, fp32 R (the bf plan's kernels);
 *   O2  symbol m is the nb consecutive blocks m nb .. m nb + nb - 1; its Nsc = nb b
 *       subcarriers q = 0 .. Nsc - 1 are (block q / b, resource element q % b); subcarrier q
 *       sits in IDFT bin (q - Nsc/2) mod n (lower half at negative frequencies, no DC skip);
 *       the other n - Nsc bins are zero;
 *   O3  x[t] = scale * sum_bin X[bin] e^{+2 pi i bin t / n}, t < n (unnormalised inverse
 *       DFT times the caller's scale);
 *   O4  cyclic prefix: y[t'] = x[n - cp + t'] for t' < cp, y[cp + t] = x[t];
 *   O5  accuracy, per (symbol, antenna):
 *       max_t |y - y_exact| <= 1e-5 * |scale| * (sum_q T_q + sqrt(n) ||X||_2),
 *       T_q = sum_k |w||s| of subcarrier q (bf.h's per-element contract carried through the
 *       unit-modulus IDFT sum, plus the normwise FFT error scale of the filter's reading F3).
 *
 * Layouts (complex fp32 = 8 bytes, interleaved (re, im)):
 *   S  [n_sym * nb][f][b]       the bf plan's interleaved S
 *   y  [n_sym][n_ant][cp + n]   time samples of every (symbol, antenna)
 *   R  [n_sym * nb][n_ant][b]   bf_ofdm_ifft's input (the bf plan's interleaved R)
 * Supported: a bf plan with layout BF_LAYOUT_INTERLEAVED (n_ant 64, b 60), n = 2048,
 * 0 <= cp < n, 1 <= nb, nb b <= n.  Other values return BF_ERR_UNSUPPORTED /
 * BF_ERR_INVALID_VALUE before anything is enqueued.
 *
 * Ownership: the OFDM plan borrows the bf plan (which must outlive it and keeps its own
 * precoders, variant and routing) and owns a device workspace for R (grown on demand, up to
 * bf_ofdm_plan_set_chunk symbols) and its twiddle table.  The caller owns S, tags and y and
 * keeps them alive until the stream work completes.  y must not overlap S, tags or R.
 *
 * Errors: as bf.h (bf_status, bf_last_error); tags outside [0, n_groups) leave the R of
 * their blocks unwritten in the workspace (bf.h), so the samples of their symbols are
 * unspecified; BF_CHECK=1 reports them as bf_apply does.
 *
 * Concurrency: an OFDM plan uses its bf plan's routing workspace and its own R workspace:
 * calls on one plan must be serialised on one stream.
 */
#ifndef BF_OFDM_H
#define BF_OFDM_H
#include <stdint.h>

#include "bf.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bf_ofdm_plan_s *bf_ofdm_plan_t;

/* Create an OFDM output plan on top of bf plan `bf` (layout BF_LAYOUT_INTERLEAVED).
 * n: IFFT size (2048); cp: cyclic prefix samples (0 <= cp < n); nb: blocks (subbands) per
 * symbol (nb * 60 <= n); scale: the factor of O3 (e.g. 1/sqrt(n) for unit-power samples).
 * Allocates the twiddle table on the bf plan's device. */
bf_status bf_ofdm_plan_create(bf_plan_t bf, int n, int cp, int nb, float scale,
                              bf_ofdm_plan_t *out);

/* y = CP(scale * IDFT(map(W x S))) for n_sym symbols: S_dev [n_sym * nb][f][60],
 * tags_dev int32 [n_sym * nb] (precoder group per block) or NULL (group 0), y_dev
 * [n_sym][64][cp + n].  Runs in chunks of at most the plan's chunk size: bf_apply into the
 * plan's R workspace, then the IFFT kernel (bf_ofdm_ifft) from it.  n_sym == 0 is a no-op. */
bf_status bf_ofdm_apply(bf_ofdm_plan_t p, const void *S_dev, const int32_t *tags_dev,
                        int64_t n_sym, void *y_dev, void *stream);

/* The IFFT + cyclic-prefix stage alone (O2-O4) from a caller's R_dev [n_sym * nb][64][60]
 * (16-byte aligned; must not overlap y_dev). */
bf_status bf_ofdm_ifft(bf_ofdm_plan_t p, const void *R_dev, int64_t n_sym, void *y_dev,
                       void *stream);

/* Output sample format of later bf_ofdm_apply / bf_ofdm_ifft calls.
 *   BF_OFDM_OUT_F32  complex fp32 (re, im), 8 bytes per sample (the default);
 *   BF_OFDM_OUT_I16  int16 (re, im) time-domain fronthaul samples, 4 bytes per sample:
 *                    sat(rne(y * 2^exponent)) per component from the fp32 sample (the
 *                    scaling by 2^exponent is exact), saturated to [-32768, 32767], NaN -> 0;
 *                    y_dev then holds int16 pairs [n_sym][n_ant][cp + n].
 * exponent in [-126, 127] (used by BF_OFDM_OUT_I16 only; 12 is a good default for
 * scale = 1/sqrt(n): |y| < 8 at 2^-12 resolution).  BF_ERR_UNSUPPORTED when a comparison
 * IFFT kernel (BFO_OFDM_KERNEL) is selected. */
enum { BF_OFDM_OUT_F32 = 0, BF_OFDM_OUT_I16 = 1 };
bf_status bf_ofdm_plan_set_output(bf_ofdm_plan_t p, int format, int exponent);

/* Symbols per chunk of bf_ofdm_apply (0 = the default, 4096 symbols: a 3.3 GB workspace at
 * nb = 26). */
bf_status bf_ofdm_plan_set_chunk(bf_ofdm_plan_t p, int64_t symbols);

bf_status bf_ofdm_destroy(bf_ofdm_plan_t p);

/* Profiling of the IFFT kernel launches (CUDA events around each launch), as bff_*. */
bf_status bf_ofdm_plan_set_profiling(bf_ofdm_plan_t p, int enable);
bf_status bf_ofdm_plan_kernel_time(bf_ofdm_plan_t p, double *total_ms, int64_t *n_launches);
/* IFFT-stage kernels launched by this plan (the bf plan counts its own). */
bf_status bf_ofdm_plan_launch_count(bf_ofdm_plan_t p, int64_t *count);

#ifdef __cplusplus
}
#endif
#endif /* BF_OFDM_H */
