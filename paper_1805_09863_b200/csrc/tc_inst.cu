// tc_inst.cu — one k-best bucket's fused tcgen05 kernels and launchers
// (compiled once per AMUN_KB in {1,2,3,4,5,6,8,12,16} by
// __graft_entry__.build(), in parallel; see launch_tc.cuh).
#define AMUN_TC_DEFINE
#include "launch_tc.cuh"

#ifndef AMUN_KB
#error "compile with -DAMUN_KB=<k-best bucket>"
#endif

template amun_status amun::launch_tc<AMUN_KB>(int, int, const CUtensorMap*, const CUtensorMap*,
                                              const CUtensorMap*, const amun::TcParams&, int,
                                              cudaStream_t, int, bool);
