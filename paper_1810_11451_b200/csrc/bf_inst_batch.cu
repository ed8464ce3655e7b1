// The runtime-f tensor-core kernel behind bf_apply_batch (bftc::bf_tc_kernel<0, LAYOUT>:
// every job carries its own f in 1..36), registered in slot f = 0 of the tensor table, and
// its slot-server form (bf_server_*).
#include "bf_dispatch.h"
#include "bf_tc.cuh"

void bf_register_batch(BfKernelTable &tc) {
    tc[0][0] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<0, 0>), bftc::TcSmem<0>::kBytes};
    tc[0][1] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<0, 1>), bftc::TcSmem<0>::kBytes};
    tc[0][2] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<0, 2>), bftc::TcSmem<0>::kBytes};
    tc[0][3] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<0, 3>), bftc::TcSmem<0>::kBytes};
}

// The slot-server instantiations (bf_server_*): the same kernel, jobs from the mailbox.
void bf_register_server(BfKernelEntry (&srv)[4]) {
    srv[0] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<0, 0, 0, true>), bftc::TcSmem<0, true>::kBytes};
    srv[1] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<0, 1, 0, true>), bftc::TcSmem<0, true>::kBytes};
    srv[2] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<0, 2, 0, true>), bftc::TcSmem<0, true>::kBytes};
    srv[3] = {reinterpret_cast<const void *>(&bftc::bf_tc_kernel<0, 3, 0, true>), bftc::TcSmem<0, true>::kBytes};
}
