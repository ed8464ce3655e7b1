// Instantiations of bf_ffma_kernel for f = 13..18 (both layouts); see bf_ffma.cuh.
#include "bf_ffma.cuh"
#include "bf_dispatch.h"

template <int F>
static void reg(BfKernelTable &t) {
    t[F][0] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 0>), bfk::Smem<F>::kBytes};
    t[F][1] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 1>), bfk::Smem<F>::kBytes};
}

void bf_register_f13_18(BfKernelTable &t) {
    reg<13>(t);
    reg<14>(t);
    reg<15>(t);
    reg<16>(t);
    reg<17>(t);
    reg<18>(t);
}
