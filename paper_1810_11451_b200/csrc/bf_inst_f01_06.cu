// Instantiations of bf_ffma_kernel for f = 1..6 (both layouts); see bf_ffma.cuh.
#include "bf_ffma.cuh"
#include "bf_dispatch.h"

template <int F>
static void reg(BfKernelTable &t) {
    t[F][0] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 0>), bfk::Smem<F>::kBytes};
    t[F][1] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 1>), bfk::Smem<F>::kBytes};
}

void bf_register_f01_06(BfKernelTable &t) {
    reg<1>(t);
    reg<2>(t);
    reg<3>(t);
    reg<4>(t);
    reg<5>(t);
    reg<6>(t);
}
