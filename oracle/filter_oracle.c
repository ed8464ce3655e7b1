/*
 * filter_oracle.c — CPU oracle for the filter stage.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as bf_oracle.c): loaded only by tests/,
 * __graft_entry__.smoke() and bench.py's baseline legs; shares nothing with the
 * CUDA path.
 *
 * PAPER.md:67-71 (§III): "The filter algorithm computes IFFT(MULT(FFT(s))) where
 * MULT is the pointwise multiplication by the FFT of the filter sequence and FFT
 * sizes are all 2048."
 *
 * Readings (F-readings): complex fp32 samples; unnormalised forward
 * DFT X[k] = sum_j x[j] e^{-2 pi i jk/n}; inverse with the 1/n factor
 * ("unnormalized forward, 1/n inverse"); H = DFT(h) of the
 * filter sequence h.  Then y = IDFT(H . DFT(s)) equals the circular convolution
 * y[k] = sum_j s[j] h[(k - j) mod n] (convolution theorem), which is oracle #2.
 *
 * Both are written out from their definitions in fp64 (O(n^2)); twiddles are
 * exp(-2 pi i (jk mod n)/n) evaluated with cos/sin in double on the reduced
 * index, so no accumulated angle error.  Outputs are rounded once to fp32.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

/* X[k] = sum_j x[j] * e^{sign * 2 pi i j k / n}, fp64 in and out (interleaved).
 * e^{i a} for a = 2 pi (jk mod n) / n is looked up in a table of cos/sin of the n
 * reduced angles (the same values a direct evaluation gives). */
static void dft64(const double *x, double *X, int n, int sign) {
    const double two_pi = 6.283185307179586476925286766559;
    double *ct = (double *)malloc(sizeof(double) * n), *st = (double *)malloc(sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        const double a = sign * two_pi * (double)i / (double)n;
        ct[i] = cos(a);
        st[i] = sin(a);
    }
    for (int k = 0; k < n; ++k) {
        double re = 0.0, im = 0.0;
        for (int j = 0; j < n; ++j) {
            const long long idx = ((long long)j * k) % n;
            const double c = ct[idx], s = st[idx];
            const double xr = x[2 * j], xi = x[2 * j + 1];
            re += xr * c - xi * s;
            im += xr * s + xi * c;
        }
        X[2 * k] = re;
        X[2 * k + 1] = im;
    }
    free(ct);
    free(st);
}

/* DFT / IDFT of n_sig signals (fp32 in, fp32 out).  inverse != 0 applies the
 * e^{+...} kernel and the 1/n factor. */
int fo_dft(const float *x, float *X, int n, int64_t n_sig, int inverse) {
    if (n < 1 || n_sig < 0) return -1;
    double *a = (double *)malloc(sizeof(double) * 2 * n), *b = (double *)malloc(sizeof(double) * 2 * n);
    if (!a || !b) { free(a); free(b); return -1; }
    for (int64_t q = 0; q < n_sig; ++q) {
        for (int i = 0; i < 2 * n; ++i) a[i] = x[q * 2 * n + i];
        dft64(a, b, n, inverse ? +1 : -1);
        const double scale = inverse ? 1.0 / n : 1.0;
        for (int i = 0; i < 2 * n; ++i) X[q * 2 * n + i] = (float)(b[i] * scale);
    }
    free(a); free(b);
    return 0;
}

typedef struct {
    const float *s, *h;
    float *y;
    double *bound;
    int n;
    int64_t n_sig;
    int tid, nth, mode;
} fo_job;

/* mode 0: y = IDFT(DFT(h) . DFT(s))   (the paper's IFFT(MULT(FFT(s))) in fp64)
 * mode 1: y[k] = sum_j s[j] h[(k - j) mod n]   (circular convolution, direct)
 * bound[q] = ||s_q||_2 * max_k |H[k]| (the normwise scale of the tolerance). */
static void *fo_worker(void *arg) {
    fo_job *J = (fo_job *)arg;
    const int n = J->n;
    double *H = (double *)malloc(sizeof(double) * 2 * n), *S = (double *)malloc(sizeof(double) * 2 * n);
    double *t = (double *)malloc(sizeof(double) * 2 * n), *Y = (double *)malloc(sizeof(double) * 2 * n);
    for (int i = 0; i < 2 * n; ++i) t[i] = J->h[i];
    dft64(t, H, n, -1);
    double hmax = 0.0;
    for (int k = 0; k < n; ++k) {
        const double m = hypot(H[2 * k], H[2 * k + 1]);
        if (m > hmax) hmax = m;
    }
    for (int64_t q = J->tid; q < J->n_sig; q += J->nth) {
        const float *s = J->s + q * 2 * n;
        float *y = J->y + q * 2 * n;
        double ss = 0.0;
        for (int j = 0; j < n; ++j) ss += (double)s[2 * j] * s[2 * j] + (double)s[2 * j + 1] * s[2 * j + 1];
        if (J->bound) J->bound[q] = sqrt(ss) * hmax;
        if (J->mode == 0) {
            for (int i = 0; i < 2 * n; ++i) t[i] = s[i];
            dft64(t, S, n, -1);
            for (int k = 0; k < n; ++k) {
                const double ar = S[2 * k], ai = S[2 * k + 1], br = H[2 * k], bi = H[2 * k + 1];
                t[2 * k] = ar * br - ai * bi;
                t[2 * k + 1] = ar * bi + ai * br;
            }
            dft64(t, Y, n, +1);
            for (int i = 0; i < 2 * n; ++i) y[i] = (float)(Y[i] / n);
        } else {
            for (int k = 0; k < n; ++k) {
                double re = 0.0, im = 0.0;
                for (int j = 0; j < n; ++j) {
                    const int m = ((k - j) % n + n) % n;
                    const double sr = s[2 * j], si = s[2 * j + 1];
                    const double hr = J->h[2 * m], hi = J->h[2 * m + 1];
                    re += sr * hr - si * hi;
                    im += sr * hi + si * hr;
                }
                y[2 * k] = (float)re;
                y[2 * k + 1] = (float)im;
            }
        }
    }
    free(H); free(S); free(t); free(Y);
    return NULL;
}

int fo_filter(const float *s, const float *h, float *y, double *bound, int n, int64_t n_sig,
              int mode, int n_threads) {
    if (n < 1 || n_sig < 0 || (mode != 0 && mode != 1)) return -1;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if ((int64_t)n_threads > n_sig) n_threads = n_sig > 0 ? (int)n_sig : 1;
    fo_job jobs[256];
    pthread_t th[256];
    for (int t = 0; t < n_threads; ++t) {
        fo_job j = {s, h, y, bound, n, n_sig, t, n_threads, mode};
        jobs[t] = j;
    }
    for (int t = 1; t < n_threads; ++t) pthread_create(&th[t], NULL, fo_worker, &jobs[t]);
    fo_worker(&jobs[0]);
    for (int t = 1; t < n_threads; ++t) pthread_join(th[t], NULL);
    return 0;
}
