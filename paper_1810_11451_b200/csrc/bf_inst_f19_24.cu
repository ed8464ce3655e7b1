// Instantiations of bf_ffma_kernel for f = 19..24 (both layouts); see bf_ffma.cuh.
#include "bf_ffma.cuh"
#include "bf_dispatch.h"

template <int F>
static void reg(BfKernelTable &t) {
    t[F][0] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 0>), bfk::Smem<F>::kBytes};
    t[F][1] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 1>), bfk::Smem<F>::kBytes};
}

void bf_register_f19_24(BfKernelTable &t) {
    reg<19>(t);
    reg<20>(t);
    reg<21>(t);
    reg<22>(t);
    reg<23>(t);
    reg<24>(t);
}
