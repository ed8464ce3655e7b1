// Instantiations of bf_ffma_kernel for f = 31..36 (both layouts); see bf_ffma.cuh.
#include "bf_ffma.cuh"
#include "bf_dispatch.h"

template <int F>
static void reg(BfKernelTable &t) {
    t[F][0] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 0>), bfk::Smem<F>::kBytes};
    t[F][1] = {reinterpret_cast<const void *>(&bfk::bf_ffma_kernel<F, 1>), bfk::Smem<F>::kBytes};
}

void bf_register_f31_36(BfKernelTable &t) {
    reg<31>(t);
    reg<32>(t);
    reg<33>(t);
    reg<34>(t);
    reg<35>(t);
    reg<36>(t);
}
