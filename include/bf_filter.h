/*
 * bf_filter.h — C ABI of the filter stage in libbf.so.
 *
 * The operation (§III): "The filter algorithm computes
 * IFFT(MULT(FFT(s))) where MULT is the pointwise multiplication by the FFT of
 * the filter sequence and FFT sizes are all 2048."
 *
 *   y = IDFT( DFT(h) . DFT(s) )   per signal s of n = 2048 complex fp32 samples,
 *   DFT unnormalised, IDFT with 1/n; equivalently the circular
 *   convolution y[k] = sum_j s[j] h[(k - j) mod n].
 *
 * Accuracy contract (DESIGN.md §2 F3; the paper states none): per signal,
 * max_k |y[k] - y_exact[k]| <= 1e-5 * ||s||_2 * max_k |DFT(h)[k]|.
 *
 * Layout: signals [n_signals][2048] complex fp32 interleaved (re, im), 16-byte
 * aligned device pointers.  y may alias s exactly (in place); partial overlap is
 * rejected.  The plan owns H = DFT(h) and the twiddle table; the caller owns s
 * and y.  Errors and streams follow bf.h (bf_status, void* cudaStream_t).
 */
#ifndef BF_FILTER_H
#define BF_FILTER_H

#include <stdint.h>

#include "bf.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bff_plan_s *bff_plan_t;

/* Create a filter plan for signals of n samples (n must be 2048, the paper's
 * size; other n return BF_ERR_UNSUPPORTED before touching the GPU). */
bf_status bff_plan_create(int n, bff_plan_t *out);

/* Set the filter sequence h (device, n complex fp32): the plan computes and
 * keeps H = DFT(h) with its own FFT kernel, ordered on `stream`. */
bf_status bff_set_taps(bff_plan_t p, const void *h_dev, void *stream);

/* y = IDFT(H . DFT(s)) for n_signals signals on `stream` (n_signals == 0: no-op). */
bf_status bff_apply(bff_plan_t p, const void *s_dev, void *y_dev, int64_t n_signals,
                    void *stream);

/* Forward DFT only (X = DFT(x), unnormalised) — the building block, exposed for
 * tests. */
bf_status bff_fft(bff_plan_t p, const void *x_dev, void *X_dev, int64_t n_signals, void *stream);

bf_status bff_destroy(bff_plan_t p);

/* Instrumentation, as bf_plan_set_profiling / bf_plan_kernel_time / launch count. */
bf_status bff_plan_set_profiling(bff_plan_t p, int enable);
bf_status bff_plan_kernel_time(bff_plan_t p, double *total_ms, int64_t *n_launches);
bf_status bff_plan_launch_count(bff_plan_t p, int64_t *count);

#ifdef __cplusplus
}
#endif
#endif /* BF_FILTER_H */
