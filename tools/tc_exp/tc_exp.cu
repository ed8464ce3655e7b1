// Bottleneck experiments for bftc::bf_tc_kernel (not part of the product):
// the same kernel with pieces disabled (DBG bits), untagged, f = 36, timed with
// CUDA events.  tcx_run(dbg, S, R, Wimg, n, reps) -> average ms per launch.
#include <cstdio>
#include "../../paper_1810_11451_b200/csrc/bf_tc.cuh"

template <int DBG>
static float run(const float *S, float *R, const float *Wimg, long long n, int reps) {
    static int32_t *wexact = nullptr;
    if (!wexact) { cudaMalloc(&wexact, 4); const int32_t w0 = 128 << 8; cudaMemcpy(wexact, &w0, 4, cudaMemcpyHostToDevice); }  // tau = 0
    auto k = bftc::bf_tc_kernel<36, 0, DBG>;
    const int smem = bftc::TcSmem<36>::kBytes;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    bftc::TcParamsOf<36> p{};
    p.n_jobs = 1; p.job[0].Wimg = Wimg; p.job[0].S = S; p.job[0].R = R; p.job[0].n_items = n;
    p.job[0].n_groups = 1; p.job[0].wexact = wexact; p.job[0].f = 36;
    k<<<sms, bftc::kThreads, smem>>>(p);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) k<<<sms, bftc::kThreads, smem>>>(p);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
    return ms / reps;
}

// Per-launch device time of ONE launch over n blocks with the given grid, L2 flushed
// (memset of `flush`, > L2) before each of `reps` launches; returns the median in ms.
template <int DBG>
static float lat(const float *S, float *R, const float *Wimg, long long n, int grid, void *flush,
                 size_t flush_bytes, int reps) {
    static int32_t *wexact = nullptr;
    if (!wexact) { cudaMalloc(&wexact, 4); const int32_t w0 = 128 << 8; cudaMemcpy(wexact, &w0, 4, cudaMemcpyHostToDevice); }  // tau = 0
    auto k = bftc::bf_tc_kernel<36, 0, DBG>;
    const int smem = bftc::TcSmem<36>::kBytes;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bftc::TcParamsOf<36> p{};
    p.n_jobs = 1; p.job[0].Wimg = Wimg; p.job[0].S = S; p.job[0].R = R; p.job[0].n_items = n;
    p.job[0].n_groups = 1; p.job[0].wexact = wexact; p.job[0].f = 36;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float v[64];
    reps = reps > 64 ? 64 : reps;
    for (int i = 0; i < reps; ++i) {
        if (flush) cudaMemsetAsync(flush, i & 255, flush_bytes);
        cudaEventRecord(a);
        k<<<grid, bftc::kThreads, smem>>>(p);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&v[i], a, b);
    }
    cudaEventDestroy(a); cudaEventDestroy(b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
    for (int i = 1; i < reps; ++i)
        for (int j = i; j > 0 && v[j] < v[j - 1]; --j) { float t = v[j]; v[j] = v[j - 1]; v[j - 1] = t; }
    return v[reps / 2];
}

extern "C" float tcx_lat(int dbg, const float *S, float *R, const float *Wimg, long long n, int grid,
                         void *flush, long long flush_bytes, int reps) {
    switch (dbg) {
        case 0: return lat<0>(S, R, Wimg, n, grid, flush, flush_bytes, reps);
        case 1: return lat<1>(S, R, Wimg, n, grid, flush, flush_bytes, reps);
        case 2: return lat<2>(S, R, Wimg, n, grid, flush, flush_bytes, reps);
        case 4: return lat<4>(S, R, Wimg, n, grid, flush, flush_bytes, reps);
        case 8: return lat<8>(S, R, Wimg, n, grid, flush, flush_bytes, reps);
        case 15: return lat<15>(S, R, Wimg, n, grid, flush, flush_bytes, reps);
    }
    return -2;
}

extern "C" float tcx_run(int dbg, const float *S, float *R, const float *Wimg, long long n, int reps) {
    switch (dbg) {
        case 0: return run<0>(S, R, Wimg, n, reps);
        case 1: return run<1>(S, R, Wimg, n, reps);
        case 2: return run<2>(S, R, Wimg, n, reps);
        case 3: return run<3>(S, R, Wimg, n, reps);
        case 4: return run<4>(S, R, Wimg, n, reps);
        case 5: return run<5>(S, R, Wimg, n, reps);
        case 6: return run<6>(S, R, Wimg, n, reps);
        case 8: return run<8>(S, R, Wimg, n, reps);
        case 10: return run<10>(S, R, Wimg, n, reps);
        case 12: return run<12>(S, R, Wimg, n, reps);
        case 14: return run<14>(S, R, Wimg, n, reps);
        case 7: return run<7>(S, R, Wimg, n, reps);
        case 15: return run<15>(S, R, Wimg, n, reps);
    }
    return -2;
}
