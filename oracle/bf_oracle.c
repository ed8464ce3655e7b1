/*
 * bf_oracle.c — CPU oracle for the beamforming hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` legs may load this library.
 * The product path (paper_1810_11451_b200/, libbf.so) never links, imports or
 * calls it, and shares no code, header or table with it.
 *
 * What it computes — the definition itself, written out:
 *   PAPER.md:84-86 (§III, beamforming equation): "The beam forming algorithm
 *   computes many products W x S where W the precoding matrix is constant and
 *   S the symbols matrix is changing.  A row i of W corresponds to one antenna
 *   (here there are 64).  Matrix S has f rows, one per parallel flow, and b
 *   columns, one per resource element.  By definition of matrix product each of
 *   W's rows is multiplied by S ..." with b = 60 and 0 <= f <= 36.
 *
 *   For every block n (with precoder group g = group_idx[n], or 0), antenna i
 *   and resource element j:
 *
 *       R[n][i][j] = sum_{k=0}^{f-1} W[g][i][k] * S[n][k][j]      (complex,
 *                                                                   no conjugate)
 *
 * Readings (SURVEY.md §8(c) ledger):
 *   R1  complex fp32 in and out (BASELINE.json configs), interleaved (re, im).
 *   R2  the paper's one-row R is row i of the full n_ant x b product.
 *   R4  summation order: ascending k.
 *   R6  accumulation starts at +0.0 (f = 0 gives +0.0 exactly).
 *   Arithmetic: fp32 inputs are promoted to fp64 (each product of two fp32
 *   values is exact in fp64); the complex product is expanded in real
 *   arithmetic  re += wr*sr - wi*si ; im += wr*si + wi*sr  (4 mul,
 *   2 add, plus 2 accumulate adds per complex MAC) and the fp64 sum is rounded
 *   once to fp32 (round-to-nearest-even cast).  Compiled with
 *   -ffp-contract=off so no FMA contraction changes these roundings.
 *
 *   Per-element bound T[n][i][j] = sum_k |W[g][i][k]| * |S[n][k][j]| in fp64
 *   (|.| = complex modulus via hypot), the scale of the parity tolerance
 *   |R_gpu - R_ref| <= 1e-5 * T (BASELINE.json north_star item 4).
 *
 *   FLOP counter: 8 real FLOPs per complex MAC, incremented inside the loop
 *   (closed form 8 * n_ant * b * f per block; counting does not change
 *   results).
 *
 * Parallelism: blocks are dealt statically to threads; every element is
 * computed by exactly one thread in the fixed order above, so the output is
 * independent of the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int n_ant, f, b, n_groups;
    int64_t n_blocks;
    const float *W;          /* [n_groups][n_ant][f][2] */
    const float *S;          /* [n_blocks][f][b][2]      */
    const int32_t *gidx;     /* [n_blocks] or NULL       */
    float *R;                /* [n_blocks][n_ant][b][2]  */
    double *T;               /* [n_blocks][n_ant][b] or NULL */
    int n_threads;
} bfo_job;

typedef struct {
    const bfo_job *job;
    int tid;
    int64_t flops;
} bfo_worker;

static void bfo_one_block(const bfo_job *J, int64_t n, int64_t *flops) {
    const int A = J->n_ant, F = J->f, B = J->b;
    const int g = J->gidx ? J->gidx[n] : 0;
    const float *Wg = J->W + (size_t)g * A * F * 2;
    const float *Sn = J->S + (size_t)n * F * B * 2;
    float *Rn = J->R + (size_t)n * A * B * 2;
    double *Tn = J->T ? J->T + (size_t)n * A * B : NULL;
    for (int i = 0; i < A; ++i) {
        for (int j = 0; j < B; ++j) {
            double re = +0.0, im = +0.0, t = +0.0;
            for (int k = 0; k < F; ++k) {
                const double wr = Wg[((size_t)i * F + k) * 2 + 0];
                const double wi = Wg[((size_t)i * F + k) * 2 + 1];
                const double sr = Sn[((size_t)k * B + j) * 2 + 0];
                const double si = Sn[((size_t)k * B + j) * 2 + 1];
                re += wr * sr - wi * si;
                im += wr * si + wi * sr;
                *flops += 8;
                if (Tn) t += hypot(wr, wi) * hypot(sr, si);
            }
            Rn[((size_t)i * B + j) * 2 + 0] = (float)re;
            Rn[((size_t)i * B + j) * 2 + 1] = (float)im;
            if (Tn) Tn[(size_t)i * B + j] = t;
        }
    }
}

static void *bfo_worker_main(void *arg) {
    bfo_worker *w = (bfo_worker *)arg;
    const bfo_job *J = w->job;
    for (int64_t n = w->tid; n < J->n_blocks; n += J->n_threads)
        bfo_one_block(J, n, &w->flops);
    return NULL;
}

/* Returns 0 on success, -1 on invalid arguments (negative sizes, NULL buffers
 * with nonzero sizes, out-of-range group index).  *flops_out receives the
 * counted FLOPs. */
int bfo_beamform(int n_ant, int f, int b, int n_groups, int64_t n_blocks,
                 const float *W, const float *S, const int32_t *group_idx,
                 float *R, double *T, int n_threads, int64_t *flops_out) {
    if (n_ant < 1 || f < 0 || b < 1 || n_blocks < 0 || n_groups < 1) return -1;
    if (n_blocks > 0 && (R == NULL || (f > 0 && (W == NULL || S == NULL)))) return -1;
    if (group_idx)
        for (int64_t n = 0; n < n_blocks; ++n)
            if (group_idx[n] < 0 || group_idx[n] >= n_groups) return -1;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 1024) n_threads = 1024;
    if ((int64_t)n_threads > n_blocks) n_threads = n_blocks > 0 ? (int)n_blocks : 1;

    bfo_job J = {n_ant, f, b, n_groups, n_blocks, W, S, group_idx, R, T, n_threads};
    bfo_worker *ws = (bfo_worker *)calloc((size_t)n_threads, sizeof(bfo_worker));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!ws || !th) { free(ws); free(th); return -1; }
    for (int t = 0; t < n_threads; ++t) { ws[t].job = &J; ws[t].tid = t; ws[t].flops = 0; }
    for (int t = 1; t < n_threads; ++t) pthread_create(&th[t], NULL, bfo_worker_main, &ws[t]);
    bfo_worker_main(&ws[0]);
    int64_t total = ws[0].flops;
    for (int t = 1; t < n_threads; ++t) { pthread_join(th[t], NULL); total += ws[t].flops; }
    free(ws); free(th);
    if (flops_out) *flops_out = total;
    return 0;
}
