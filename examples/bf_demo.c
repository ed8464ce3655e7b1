/* bf_demo.c — the C ABI (include/bf.h) used from plain C99, no Python, no torch.
 *
 * Builds a plan for f = 4 flows, installs the identity-like precoder W = [I_4; 0]
 * (row i of W is antenna i), beamforms 3 blocks of S and checks
 * the result exactly: antenna rows 0..3 reproduce S's rows bit for bit and rows
 * 4..63 are +0.0 (BASELINE.json north_star item 4: bit-exact identity cases).
 * Also exercises the synchronous argument checks, and the OFDM output stage
 * (include/bf_ofdm.h): one active subcarrier through W = [I_4; 0] gives antenna 0 the
 * complex exponential e^{+2 pi i bin t / n} (readings O2-O3) behind its cyclic prefix (O4)
 * and every other antenna exact zeros.
 *
 *   gcc -std=c99 -Iinclude -I/usr/local/cuda/include examples/bf_demo.c \
 *       -Lpaper_1810_11451_b200 -lbf -L/usr/local/cuda/lib64 -lcudart -lm -o build/bf_demo
 *
 * Exit status: 0 = all checks passed, 1 = a check failed, 2 = no CUDA device.
 */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <cuda_runtime_api.h>

#include "bf.h"
#include "bf_ofdm.h"

#define N_ANT 64
#define B 60
#define F 4
#define NB 3

static int check(bf_status s, bf_status want, const char *what) {
    if (s != want) {
        fprintf(stderr, "%s: got %s, want %s (%s)\n", what, bf_status_string(s),
                bf_status_string(want), bf_last_error());
        return 1;
    }
    return 0;
}

int main(void) {
    int bad = 0;
    bf_plan_t plan = NULL;
    /* argument checks happen before the GPU is touched */
    bad |= check(bf_plan_create(N_ANT, 37, B, BF_LAYOUT_INTERLEAVED, &plan), BF_ERR_UNSUPPORTED,
                 "f = 37");
    bad |= check(bf_plan_create(N_ANT, F, B, 9, &plan), BF_ERR_INVALID_VALUE, "layout 9");
    bf_status s = bf_plan_create(N_ANT, F, B, BF_LAYOUT_INTERLEAVED, &plan);
    if (s == BF_ERR_NO_DEVICE) {
        printf("bf_demo: no CUDA device (%s)\n", bf_last_error());
        return 2;
    }
    bad |= check(s, BF_OK, "bf_plan_create");
    if (bad) return 1;

    static float W[N_ANT * F * 2], S[NB * F * B * 2], R[NB * N_ANT * B * 2];
    memset(W, 0, sizeof W);
    for (int k = 0; k < F; ++k) W[(k * F + k) * 2] = 1.0f;          /* W[k][k] = 1 + 0i */
    for (int i = 0; i < NB * F * B * 2; ++i) S[i] = (float)((i * 7919) % 1009) / 97.0f - 5.0f;
    void *dW = NULL, *dS = NULL, *dR = NULL;
    if (cudaMalloc(&dW, sizeof W) || cudaMalloc(&dS, sizeof S) || cudaMalloc(&dR, sizeof R)) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    cudaMemcpy(dW, W, sizeof W, cudaMemcpyHostToDevice);
    cudaMemcpy(dS, S, sizeof S, cudaMemcpyHostToDevice);
    cudaMemset(dR, 0x7f, sizeof R);

    bad |= check(bf_apply(plan, dS, NULL, dR, NB, NULL), BF_ERR_NO_PRECODERS, "apply before W");
    bad |= check(bf_set_precoders(plan, dW, 1, NULL), BF_OK, "bf_set_precoders");
    bad |= check(bf_apply(plan, dS, NULL, dS, NB, NULL), BF_ERR_INVALID_VALUE, "R overlaps S");
    bad |= check(bf_apply(plan, (char *)dS + 4, NULL, dR, NB, NULL), BF_ERR_MISALIGNED, "misaligned S");
    bad |= check(bf_apply(plan, dS, NULL, dR, NB, NULL), BF_OK, "bf_apply");
    if (cudaDeviceSynchronize() != cudaSuccess) {
        fprintf(stderr, "device error\n");
        return 1;
    }
    cudaMemcpy(R, dR, sizeof R, cudaMemcpyDeviceToHost);

    long mismatches = 0;
    for (int n = 0; n < NB; ++n)
        for (int i = 0; i < N_ANT; ++i)
            for (int j = 0; j < B * 2; ++j) {
                const float got = R[(n * N_ANT + i) * B * 2 + j];
                const float want = i < F ? S[(n * F + i) * B * 2 + j] : 0.0f;
                uint32_t gb, wb;
                memcpy(&gb, &got, 4);
                memcpy(&wb, &want, 4);
                mismatches += gb != wb;
            }
    if (mismatches) {
        fprintf(stderr, "identity beamforming: %ld elements differ\n", mismatches);
        bad = 1;
    }
    /* OFDM output: one symbol of NB blocks, 2048-point IFFT, 16-sample cyclic prefix; S has
     * a single 1 at flow 0 of subcarrier q0, which sits in bin (q0 - NB B / 2) mod 2048 */
    {
        enum { N = 2048, CP = 16, L = CP + N };
        const int q0 = 137, bin = ((q0 - NB * B / 2) % N + N) % N;
        static float S1[NB * F * B * 2], Y[N_ANT * L * 2];
        memset(S1, 0, sizeof S1);
        S1[((q0 / B) * F * B + q0 % B) * 2] = 1.0f;
        void *dY = NULL;
        bf_ofdm_plan_t op = NULL;
        bad |= check(bf_ofdm_plan_create(plan, 1024, CP, NB, 1.0f, &op), BF_ERR_UNSUPPORTED, "n = 1024");
        bad |= check(bf_ofdm_plan_create(plan, N, N, NB, 1.0f, &op), BF_ERR_INVALID_VALUE, "cp = n");
        bad |= check(bf_ofdm_plan_create(plan, N, CP, NB, 1.0f, &op), BF_OK, "bf_ofdm_plan_create");
        if (cudaMalloc(&dY, sizeof Y)) {
            fprintf(stderr, "cudaMalloc failed\n");
            return 1;
        }
        cudaMemcpy(dS, S1, sizeof S1, cudaMemcpyHostToDevice);
        bad |= check(bf_ofdm_apply(op, dS, NULL, 1, dY, NULL), BF_OK, "bf_ofdm_apply");
        if (cudaDeviceSynchronize() != cudaSuccess) {
            fprintf(stderr, "device error (ofdm)\n");
            return 1;
        }
        cudaMemcpy(Y, dY, sizeof Y, cudaMemcpyDeviceToHost);
        double worst = 0.0;
        long nonzero = 0, prefix = 0;
        for (int t = 0; t < N; ++t) {
            const double ang = 6.283185307179586 * (double)((long)bin * t % N) / N;
            const double dr = Y[(CP + t) * 2] - cos(ang), di = Y[(CP + t) * 2 + 1] - sin(ang);
            const double e = sqrt(dr * dr + di * di);
            if (e > worst) worst = e;
        }
        for (int u = 0; u < CP * 2; ++u) prefix += memcmp(&Y[u], &Y[N * 2 + u], 4) != 0;
        for (int i = L * 2; i < N_ANT * L * 2; ++i) nonzero += Y[i] != 0.0f;
        if (worst > 1e-5 || prefix || nonzero) {   /* O5 bound here: 1e-5 (1 + sqrt(n)) */
            fprintf(stderr, "ofdm: worst %.3e, prefix mismatches %ld, nonzero %ld\n", worst, prefix, nonzero);
            bad = 1;
        }
        bad |= check(bf_ofdm_destroy(op), BF_OK, "bf_ofdm_destroy");
        cudaFree(dY);
    }
    bad |= check(bf_destroy(plan), BF_OK, "bf_destroy");
    cudaFree(dW);
    cudaFree(dS);
    cudaFree(dR);
    printf("bf_demo: %s (libbf version %d)\n", bad ? "FAILED" : "ok", bf_version());
    return bad ? 1 : 0;
}
