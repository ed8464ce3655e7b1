// Instantiations of bf_ffma_kernel for f = 7..12 (both layouts); see bf_ffma.cuh.
#include "bf_ffma.cuh"
#include "bf_dispatch.h"

template <int F>
static void reg(BfKernelTable &t) {
    t[F][0] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 0>), bfk::Smem<F>::kBytes};
    t[F][1] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 1>), bfk::Smem<F>::kBytes};
}

void bf_register_f07_12(BfKernelTable &t) {
    reg<7>(t);
    reg<8>(t);
    reg<9>(t);
    reg<10>(t);
    reg<11>(t);
    reg<12>(t);
}
