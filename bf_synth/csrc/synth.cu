// synth.cu — device-side twin of bf_synth/__init__.py (S symbols, subband tags,
// per-block modulations) plus an L2-flush fill.  Bench/test infrastructure:
// NOT part of the beamforming path, holds none of its arithmetic.  The hash is
// the SplitMix64 sequence element  mix64(key + (idx + 1) * GAMMA)  with keys
// computed on the host by bf_synth.stream_key; QAM level tables come from
// bf_synth.qam_levels (host, fp64 -> fp32), so device and host agree bitwise.
#include <cuda_runtime.h>
#include <cstdint>

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t hash_at(uint64_t key, uint64_t idx) {
    uint64_t z = key + (idx + 1ull) * kGamma;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int64_t bounded(uint64_t h, int64_t n) {
    return (int64_t)(((h >> 32) * (uint64_t)n) >> 32);
}

struct Levels {
    float lv[3][8];     // QPSK (2 used), 16-QAM (4 used), 64-QAM (8 used)
};

__global__ void gen_qam(float *__restrict__ S, const int64_t *__restrict__ ids, int64_t first,
                        int64_t n, int f, int b, uint64_t key, int layout, Levels L, int mod_idx,
                        uint64_t mod_key) {
    const int64_t per = (int64_t)f * b;
    const int64_t total = n * per;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t nl = e / per;
        const int rem = (int)(e - nl * per);
        const int k = rem / b, j = rem - (rem / b) * b;
        const int64_t blk = ids ? ids[nl] : first + nl;
        int m = mod_idx;
        if (m < 0) m = (int)bounded(hash_at(mod_key, (uint64_t)blk), 3);
        const uint64_t mask = (m == 0) ? 1u : (m == 1 ? 3u : 7u);
        const uint64_t h = hash_at(key, ((uint64_t)blk * 64u + k) * 256u + j);
        const float re = L.lv[m][h & mask];
        const float im = L.lv[m][(h >> 8) & mask];
        if (layout == 0) {
            reinterpret_cast<float2 *>(S)[e] = make_float2(re, im);
        } else {
            float *Sb = S + nl * 2 * per;
            Sb[rem] = re;
            Sb[per + rem] = im;
        }
    }
}

__global__ void gen_tags(int32_t *__restrict__ out, const int64_t *__restrict__ ids,
                         int64_t first, int64_t n, uint64_t key, int n_groups) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t blk = ids ? ids[i] : first + i;
        out[i] = (int32_t)bounded(hash_at(key, (uint64_t)blk), n_groups);
    }
}

__global__ void gen_mods(int32_t *__restrict__ out, const int64_t *__restrict__ ids, int64_t first,
                         int64_t n, uint64_t key) {
    const int M[3] = {4, 16, 64};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t blk = ids ? ids[i] : first + i;
        out[i] = M[bounded(hash_at(key, (uint64_t)blk), 3)];
    }
}

__global__ void gen_signal(float2 *__restrict__ out, int64_t first, int64_t n_sig, int n,
                           uint64_t key, Levels L, int mod_idx) {
    const int64_t total = n_sig * n;
    const uint64_t mask = (mod_idx == 0) ? 1u : (mod_idx == 1 ? 3u : 7u);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = hash_at(key, (uint64_t)(first * n + e));
        out[e] = make_float2(L.lv[mod_idx][h & mask], L.lv[mod_idx][(h >> 8) & mask]);
    }
}

__global__ void fill_u32(uint32_t *__restrict__ p, int64_t n, uint32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

int grid_for(int64_t work) {
    int64_t g = (work + 255) / 256;
    if (g > 148 * 64) g = 148 * 64;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

// S for n blocks (ids[i] or first + i), f x b each; mod_idx 0/1/2 selects
// QPSK/16/64-QAM for all blocks, -1 draws it per block with mod_key.
int bfs_gen_qam(float *S, const int64_t *ids, int64_t first, int64_t n, int f, int b,
                uint64_t key, int layout, const float *levels24, int mod_idx, uint64_t mod_key,
                void *stream) {
    if (n <= 0 || f <= 0) return 0;
    Levels L;
    for (int m = 0; m < 3; ++m)
        for (int i = 0; i < 8; ++i) L.lv[m][i] = levels24[m * 8 + i];
    gen_qam<<<grid_for(n * f * b), 256, 0, (cudaStream_t)stream>>>(S, ids, first, n, f, b, key,
                                                                     layout, L, mod_idx, mod_key);
    return (int)cudaGetLastError();
}

int bfs_gen_tags(int32_t *out, const int64_t *ids, int64_t first, int64_t n, uint64_t key,
                 int n_groups, void *stream) {
    if (n <= 0) return 0;
    gen_tags<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, ids, first, n, key, n_groups);
    return (int)cudaGetLastError();
}

int bfs_gen_mods(int32_t *out, const int64_t *ids, int64_t first, int64_t n, uint64_t key,
                 void *stream) {
    if (n <= 0) return 0;
    gen_mods<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, ids, first, n, key);
    return (int)cudaGetLastError();
}

// Filter-stage signals: n_sig x n complex samples of square M-QAM, element
// index e = sig * n + k (bf_synth.filter_signals).
int bfs_gen_signals(float *out, int64_t first, int64_t n_sig, int n, uint64_t key,
                    const float *levels24, int mod_idx, void *stream) {
    if (n_sig <= 0) return 0;
    Levels L;
    for (int m = 0; m < 3; ++m)
        for (int i = 0; i < 8; ++i) L.lv[m][i] = levels24[m * 8 + i];
    gen_signal<<<grid_for(n_sig * n), 256, 0, (cudaStream_t)stream>>>((float2 *)out, first, n_sig, n,
                                                                      key, L, mod_idx);
    return (int)cudaGetLastError();
}

// Write n 32-bit words (used to flush L2 between timed iterations).
int bfs_fill_u32(void *p, int64_t n, uint32_t v, void *stream) {
    if (n <= 0) return 0;
    fill_u32<<<grid_for(n / 4 + 1), 256, 0, (cudaStream_t)stream>>>((uint32_t *)p, n, v);
    return (int)cudaGetLastError();
}

}  // extern "C"
