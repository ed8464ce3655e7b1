// Instantiations of the beamforming kernels for f = 19..24 (both layouts):
// the CUDA-core FFMA kernel (bf_ffma.cuh) and the tcgen05 split-precision kernel (bf_tc.cuh).
#include "bf_dispatch.h"
#include "bf_ffma.cuh"
#include "bf_tc.cuh"

template <int F>
static void reg(BfKernelTable &t, BfKernelTable &tc) {
    t[F][0] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 0>), bfk::Smem<F>::kBytes};
    t[F][1] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 1>), bfk::Smem<F>::kBytes};
    tc[F][0] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<F, 0>), bftc::TcSmem<F>::kBytes};
    tc[F][1] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<F, 1>), bftc::TcSmem<F>::kBytes};
    t[F][2] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 2>), bfk::Smem<F>::kBytes};
    tc[F][2] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<F, 2>), bftc::TcSmem<F, false, true>::kBytes};
    t[F][3] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 3>), bfk::Smem<F>::kBytes};
    tc[F][3] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<F, 3>), bftc::TcSmem<F, false, BFTC_I16_R2 != 0>::kBytes};
}

void bf_register_f19_24(BfKernelTable &t, BfKernelTable &tc) {
    reg<19>(t, tc);
    reg<20>(t, tc);
    reg<21>(t, tc);
    reg<22>(t, tc);
    reg<23>(t, tc);
    reg<24>(t, tc);
}
