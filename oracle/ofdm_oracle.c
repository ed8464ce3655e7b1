/*
 * ofdm_oracle.c — CPU oracle for the fused OFDM output of the beamformer
 * (second alternative: "fuse the per-antenna OFDM IFFT").
 *
 * TEST INFRASTRUCTURE ONLY (same rules as bf_oracle.c): loaded only by tests/,
 * __graft_entry__.smoke() and bench.py's baseline legs; shares nothing with the
 * CUDA path.
 *
 * What it computes (readings O1-O5; the paper names the pipeline
 * stages — PAPER.md:41, 49 — but gives no formula for this one):
 *   1. R = W x S per block, the beamforming equation of PAPER.md:84-86 (§III),
 *      kept in fp64 (no rounding to fp32: the exact product the GPU's fp32 R
 *      approximates);
 *   2. subcarrier mapping (O2): a symbol m is the nb consecutive blocks
 *      m*nb .. m*nb + nb - 1; its Nsc = nb*b subcarriers q = 0 .. Nsc-1 are
 *      block q / b, resource element q % b, and subcarrier q sits in IDFT bin
 *      (q - Nsc/2) mod n (lower half at negative frequencies); other bins are 0;
 *   3. x[t] = scale * sum_bin X[bin] e^{+2 pi i bin t / n}, t < n — the
 *      unnormalised inverse DFT (O3), written out as a sum over the active bins
 *      (the zero bins add nothing) in ascending bin order;
 *   4. cyclic prefix (O4): y[t'] = x[n - cp + t'] for t' < cp, y[cp + t] = x[t].
 * Output y [n_sym][A][cp + n] complex fp32, rounded once from fp64.
 * bound[m][a] = |scale| * (sum_q T_q + sqrt(n) * ||X||_2), T_q = sum_k |w||s| of
 * the subcarrier (O5: the beamforming contract carried through the unit-modulus
 * IDFT sum, plus the normwise FFT error scale of the filter's reading F3).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
    int A, F, B, G, nb, n, cp;
    int64_t n_sym;
    double scale;
    const float *W, *S;
    const int32_t *tags;
    float *y;
    double *bound;
    int tid, nth, rc;
} fm_job;

static void *fm_worker(void *arg) {
    fm_job *J = (fm_job *)arg;
    const int n = J->n, nsc = J->nb * J->B, half = nsc / 2, L = J->cp + n;
    const double two_pi = 6.283185307179586476925286766559;
    double *ct = (double *)malloc(sizeof(double) * n), *st = (double *)malloc(sizeof(double) * n);
    double *X = (double *)malloc(sizeof(double) * 2 * nsc), *T = (double *)malloc(sizeof(double) * nsc);
    int *bin = (int *)malloc(sizeof(int) * nsc);
    double *x = (double *)malloc(sizeof(double) * 2 * n);
    if (!ct || !st || !X || !T || !bin || !x) {
        J->rc = -1;
        free(ct); free(st); free(X); free(T); free(bin); free(x);
        return NULL;
    }
    /* e^{+2 pi i m / n} on the reduced index m (no accumulated angle error) */
    for (int i = 0; i < n; ++i) {
        ct[i] = cos(two_pi * (double)i / (double)n);
        st[i] = sin(two_pi * (double)i / (double)n);
    }
    for (int q = 0; q < nsc; ++q) bin[q] = ((q - half) % n + n) % n;
    const int64_t n_sig = J->n_sym * J->A;
    for (int64_t sig = J->tid; sig < n_sig; sig += J->nth) {
        const int64_t m = sig / J->A;
        const int a = (int)(sig % J->A);
        /* 1-2: the fp64 beamformed subcarriers of (symbol m, antenna a) */
        double xx = 0.0, tsum = 0.0;
        for (int q = 0; q < nsc; ++q) {
            const int64_t blk = m * J->nb + q / J->B;
            const int j = q % J->B;
            const int g = J->tags ? J->tags[blk] : 0;
            if (g < 0 || g >= J->G) { J->rc = -1; break; }
            const float *w = J->W + ((int64_t)g * J->A + a) * J->F * 2;
            double re = 0.0, im = 0.0, t = 0.0;
            for (int k = 0; k < J->F; ++k) {
                const float *s = J->S + ((blk * J->F + k) * J->B + j) * 2;
                const double wr = w[2 * k], wi = w[2 * k + 1], sr = s[0], si = s[1];
                re += wr * sr - wi * si;
                im += wr * si + wi * sr;
                t += hypot(wr, wi) * hypot(sr, si);
            }
            X[2 * q] = re;
            X[2 * q + 1] = im;
            T[q] = t;
            xx += re * re + im * im;
            tsum += t;
        }
        if (J->rc) break;
        /* 3: x[t] = scale * sum over active bins (ascending bin) of X e^{+2 pi i bin t / n} */
        for (int t = 0; t < n; ++t) {
            double re = 0.0, im = 0.0;
            for (int pass = 0; pass < 2; ++pass)          /* bins 0.. then the negative half */
                for (int q = pass == 0 ? half : 0; q < (pass == 0 ? nsc : half); ++q) {
                    const int idx = (int)(((int64_t)bin[q] * t) % n);
                    const double c = ct[idx], s = st[idx], xr = X[2 * q], xi = X[2 * q + 1];
                    re += xr * c - xi * s;
                    im += xr * s + xi * c;
                }
            x[2 * t] = J->scale * re;
            x[2 * t + 1] = J->scale * im;
        }
        /* 4: cyclic prefix, one rounding to fp32 */
        float *y = J->y + sig * (int64_t)L * 2;
        for (int u = 0; u < L; ++u) {
            const int t = u < J->cp ? n - J->cp + u : u - J->cp;
            y[2 * u] = (float)x[2 * t];
            y[2 * u + 1] = (float)x[2 * t + 1];
        }
        if (J->bound) J->bound[sig] = fabs(J->scale) * (tsum + sqrt((double)n) * sqrt(xx));
    }
    free(ct); free(st); free(X); free(T); free(bin); free(x);
    return NULL;
}

/* W [G][A][F], S [n_sym * nb][F][B] (complex fp32 interleaved), tags [n_sym * nb] in
 * [0, G) or NULL (group 0); y [n_sym][A][cp + n]; bound [n_sym][A] or NULL.
 * Returns 0, or -1 on invalid sizes / tags. */
int fm_ofdm(int A, int F, int B, int G, int64_t n_sym, int nb, int n, int cp, double scale,
            const float *W, const float *S, const int32_t *tags, float *y, double *bound,
            int n_threads) {
    if (A < 1 || F < 0 || B < 1 || G < 1 || n_sym < 0 || nb < 1 || n < 1 || cp < 0 || cp >= n)
        return -1;
    if ((int64_t)nb * B > n || (nb * B) % 2 != 0) return -1;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    fm_job jobs[256];
    pthread_t th[256];
    for (int t = 0; t < n_threads; ++t) {
        fm_job j = {A, F, B, G, nb, n, cp, n_sym, scale, W, S, tags, y, bound, t, n_threads, 0};
        jobs[t] = j;
    }
    for (int t = 1; t < n_threads; ++t) pthread_create(&th[t], NULL, fm_worker, &jobs[t]);
    fm_worker(&jobs[0]);
    for (int t = 1; t < n_threads; ++t) pthread_join(th[t], NULL);
    for (int t = 0; t < n_threads; ++t)
        if (jobs[t].rc) return -1;
    return 0;
}
