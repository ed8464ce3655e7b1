// bf_dispatch.h — host-side registry of the per-f kernel instantiations.
// Each bf_inst_*.cu translation unit registers a range of f values so the 72
// instantiations (f = 1..36 x 2 layouts) compile in parallel.
#pragma once

struct BfKernelEntry {
    const void *fn;      // __global__ bfk::bf_ffma_kernel<F, LAYOUT> or bftc::bf_tc_kernel<F, LAYOUT>
    int smem_bytes;      // dynamic shared memory of that instantiation
};

using BfKernelTable = BfKernelEntry[37][4];   // [f][layout: interleaved, planar, f16 out, i16 out]
                                              // (tensor table f = 0: the batch kernel)

void bf_register_f01_06(BfKernelTable &t, BfKernelTable &tc);
void bf_register_f07_12(BfKernelTable &t, BfKernelTable &tc);
void bf_register_f13_18(BfKernelTable &t, BfKernelTable &tc);
void bf_register_f19_24(BfKernelTable &t, BfKernelTable &tc);
void bf_register_f25_30(BfKernelTable &t, BfKernelTable &tc);
void bf_register_f31_36(BfKernelTable &t, BfKernelTable &tc);
void bf_register_batch(BfKernelTable &tc);   // slot [0][layout]: runtime-f batch kernel
void bf_register_server(BfKernelEntry (&srv)[4]);   // [layout]: slot-server kernel
