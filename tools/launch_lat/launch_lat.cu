// Launch latency of empty kernels vs block size, dynamic shared memory and parameter
// size (not part of the product): which part of a short tensor-kernel launch is fixed.
#include <cstdio>
#include <cuda_runtime.h>

struct Big { char b[1344]; };
__global__ void k_small(int x) { if (x == 12345) printf("x"); }
__global__ void k_big(const Big p) { if (p.b[0] == 123 && p.b[1343] == 7) printf("x"); }
__global__ void k_smem(int x) {
    extern __shared__ char s[];
    if (x == 12345) { s[threadIdx.x] = 1; printf("%d", s[threadIdx.x ^ 1]); }
}

template <class F>
static void time_it(const char *what, F launch, int reps = 200) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    // single launch bracketed by events, median of 31
    float v[31];
    for (int i = 0; i < 31; ++i) {
        cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&v[i], a, b);
    }
    for (int i = 1; i < 31; ++i) for (int j = i; j > 0 && v[j] < v[j-1]; --j) { float t = v[j]; v[j] = v[j-1]; v[j-1] = t; }
    printf("{\"what\": \"%s\", \"back_to_back_us\": %.2f, \"single_us\": %.2f}\n", what, ms * 1e3 / reps, v[15] * 1e3);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
    Big bg{};
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    time_it("148 x 32, no smem", [] { k_small<<<148, 32>>>(0); });
    time_it("148 x 448, no smem", [] { k_small<<<148, 448>>>(0); });
    time_it("148 x 448, 1344 B params", [&] { k_big<<<148, 448>>>(bg); });
    time_it("148 x 448, 16 KB smem", [] { k_smem<<<148, 448, 16 * 1024>>>(0); });
    time_it("148 x 448, 100 KB smem", [] { k_smem<<<148, 448, 100 * 1024>>>(0); });
    time_it("148 x 448, 210 KB smem", [] { k_smem<<<148, 448, 210 * 1024>>>(0); });
    time_it("148 x 448, 220 KB smem", [] { k_smem<<<148, 448, 220 * 1024>>>(0); });
    time_it("1 x 448, 210 KB smem", [] { k_smem<<<1, 448, 210 * 1024>>>(0); });
    return 0;
}
