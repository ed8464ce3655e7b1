// Instantiations of bf_ffma_kernel for f = 25..30 (both layouts); see bf_ffma.cuh.
#include "bf_ffma.cuh"
#include "bf_dispatch.h"

template <int F>
static void reg(BfKernelTable &t) {
    t[F][0] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 0>), bfk::Smem<F>::kBytes};
    t[F][1] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 1>), bfk::Smem<F>::kBytes};
}

void bf_register_f25_30(BfKernelTable &t) {
    reg<25>(t);
    reg<26>(t);
    reg<27>(t);
    reg<28>(t);
    reg<29>(t);
    reg<30>(t);
}
