// launch_tc.cuh — host launchers of the fused tcgen05 kernels.
//
// The kernels are instantiated per k-best bucket KB in separate translation
// units (tc_inst.cu compiled once per KB, in parallel, by
// __graft_entry__.build()); amun.cu sees only the declaration below.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>

#include "../../include/amun.h"
#include "tc_epi.cuh"

namespace amun {

// Records a printf-style error message (amun_last_error) and returns AMUN_ECUDA.
amun_status launch_fail(const char* fmt, ...);

template <int KB>
amun_status launch_tc(int dtype, int ng_override, const CUtensorMap* mx, const CUtensorMap* mw,
                      const CUtensorMap* mwn, const TcParams& tp, int grid, cudaStream_t st,
                      int mode, bool pairs);

}  // namespace amun

#ifdef AMUN_TC_DEFINE
#include "ol_tc.cuh"
#include "ol_tc2.cuh"

namespace amun {

#define LT_TRY(expr)                                                                    \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) return launch_fail("%s failed: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

// Launch one fused-kernel instantiation; the warpgroup register hand-off
// needs the full launch pool (see TcCfg), checked here.
template <int NG>
amun_status launch_kernel(void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams),
                          const CUtensorMap* mx, const CUtensorMap* mw, const CUtensorMap* mwn,
                          const TcParams& tp, int grid, cudaStream_t st, int smem_bytes) {
  cudaFuncAttributes fa;
  LT_TRY(cudaFuncGetAttributes(&fa, kern));
  if (fa.numRegs < TcCfg<NG>::kLaunchRegs)
    return launch_fail("fused kernel compiled with %d registers/thread, needs %d for its "
                "setmaxnreg budget", fa.numRegs, TcCfg<NG>::kLaunchRegs);
  LT_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
  const bool coop = tp.tail && !(tp.tail & TAIL_X_NOCOOP);
  if (!coop && !tp.pdl && tp.mc <= 1) {
    kern<<<grid, TcCfg<NG>::kThreads, smem_bytes, st>>>(*mx, *mw, *mwn, tp);
    LT_TRY(cudaGetLastError());
    return AMUN_OK;
  }
  // The fused tail waits on every CTA of the grid (tail.cuh): a cooperative
  // launch guarantees they are co-resident (grid <= #SMs, one CTA per SM).
  // tp.pdl: programmatic dependent launch (the kernel's prologue may overlap
  // the previous kernel's end; it waits in griddepcontrol.wait before any
  // global memory access, ol_tc.cuh).
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(TcCfg<NG>::kThreads, 1, 1);
  cfg.dynamicSmemBytes = (size_t)smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (tp.mc > 1) {   // W multicast clusters (ol_tc.cuh)
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = (unsigned)tp.mc;
    attr[na].val.clusterDim.y = 1;
    attr[na++].val.clusterDim.z = 1;
  }
  if (coop) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na++].val.cooperative = 1;
  }
  if (tp.pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  LT_TRY(cudaLaunchKernelEx(&cfg, kern, *mx, *mw, *mwn, tp));
  return AMUN_OK;
}

template <int KB, int NG>
amun_status launch_tc_ng(const CUtensorMap* mx, const CUtensorMap* mw, const CUtensorMap* mwn,
                         const TcParams& tp, int grid, cudaStream_t st, int mode, bool pairs) {
  // modes 1 (debug logits) and 4 (argmax) exist for KB = 1 only (the caller
  // dispatches them there), so other buckets do not compile them again
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams);
  if (pairs) {
    kern = mode == 2 ? ol_tc2_kernel<KB, 2, NG> : mode == 3 ? ol_tc2_kernel<KB, 3, NG>
                                                            : ol_tc2_kernel<KB, 0, NG>;
    if constexpr (KB == 1) {
      if (mode == 4) kern = ol_tc2_kernel<1, 4, NG>;
      if (mode == 1) kern = ol_tc2_kernel<1, 1, NG>;
    }
  } else {
    kern = mode == 2 ? ol_tc_kernel<KB, 2, NG> : mode == 3 ? ol_tc_kernel<KB, 3, NG>
                                                           : ol_tc_kernel<KB, 0, NG>;
    if constexpr (KB == 1) {
      if (mode == 4) kern = ol_tc_kernel<1, 4, NG>;
      if (mode == 1) kern = ol_tc_kernel<1, 1, NG>;
    }
  }
  return launch_kernel<NG>(kern, mx, mw, mwn, tp, grid, st, pairs ? TC2_SMEM : TC_SMEM);
}

// e4m3 plans: single CTAs; the full path and the two benchmark builds.
template <int KB, int NG>
amun_status launch_tc_f8(const CUtensorMap* mx, const CUtensorMap* mw, const CUtensorMap* mwn,
                         const TcParams& tp, int grid, cudaStream_t st, int mode) {
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams) =
      mode == 2 ? ol_tc_kernel<KB, 2, NG, 1> : mode == 3 ? ol_tc_kernel<KB, 3, NG, 1>
                                             : ol_tc_kernel<KB, 0, NG, 1>;
  if constexpr (KB == 1) {
    if (mode == 4) kern = ol_tc_kernel<1, 4, NG, 1>;
  }
  return launch_kernel<NG>(kern, mx, mw, mwn, tp, grid, st, TC_SMEM_F8);
}

// mxfp4 plans: single CTAs; every mode (the fused path, the test/bench
// builds and the argmax kernel).
template <int KB, int NG>
amun_status launch_tc_f4(const CUtensorMap* mx, const CUtensorMap* mw, const CUtensorMap* mwn,
                         const TcParams& tp, int grid, cudaStream_t st, int mode) {
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams) =
      mode == 2 ? ol_tc_kernel<KB, 2, NG, 3> : mode == 3 ? ol_tc_kernel<KB, 3, NG, 3>
                                             : ol_tc_kernel<KB, 0, NG, 3>;
  if constexpr (KB == 1) {
    if (mode == 1) kern = ol_tc_kernel<1, 1, NG, 3>;
    if (mode == 4) kern = ol_tc_kernel<1, 4, NG, 3>;
  }
  return launch_kernel<NG>(kern, mx, mw, mwn, tp, grid, st, TC_SMEM_F4);
}

// tf32x3 plans: single CTAs; every mode (the fused path, the test/bench
// builds and the argmax kernel).
template <int KB, int NG>
amun_status launch_tc_t3(const CUtensorMap* mx, const CUtensorMap* mw, const CUtensorMap* mwn,
                         const TcParams& tp, int grid, cudaStream_t st, int mode) {
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams) =
      mode == 2 ? ol_tc_kernel<KB, 2, NG, 2> : mode == 3 ? ol_tc_kernel<KB, 3, NG, 2>
                                             : ol_tc_kernel<KB, 0, NG, 2>;
  if constexpr (KB == 1) {
    if (mode == 1) kern = ol_tc_kernel<1, 1, NG, 2>;
    if (mode == 4) kern = ol_tc_kernel<1, 4, NG, 2>;
  }
  return launch_kernel<NG>(kern, mx, mw, mwn, tp, grid, st, TC_SMEM);
}

// Two epilogue warpgroups. bf16: measured faster than three or four (their
// extra warps cost issue slots and registers while the tensor pipe bounds;
// DESIGN.md §6.1). e4m3: four measured within run-to-run noise of two
// (cfg beam fused 80-85 vs 80-83 us). Building with -DAMUN_WITH_NG3 /
// -DAMUN_WITH_NG4 adds the other counts (env AMUN_NG).
template <int KB>
amun_status launch_tc(int dtype, int ng_override, const CUtensorMap* mx, const CUtensorMap* mw,
                      const CUtensorMap* mwn, const TcParams& tp, int grid, cudaStream_t st,
                      int mode, bool pairs) {
  if (dtype == AMUN_TF32X3) return launch_tc_t3<KB, 2>(mx, mw, mwn, tp, grid, st, mode);
  if (dtype == AMUN_MXFP4) return launch_tc_f4<KB, 2>(mx, mw, mwn, tp, grid, st, mode);
  if (dtype == AMUN_E4M3) {
#ifdef AMUN_WITH_NG4
    if (ng_override == 4) return launch_tc_f8<KB, 4>(mx, mw, mwn, tp, grid, st, mode);
#endif
    return launch_tc_f8<KB, 2>(mx, mw, mwn, tp, grid, st, mode);
  }
#ifdef AMUN_WITH_NG4
  if (ng_override == 4) return launch_tc_ng<KB, 4>(mx, mw, mwn, tp, grid, st, mode, pairs);
#endif
#ifdef AMUN_WITH_NG3
  if (ng_override == 3) return launch_tc_ng<KB, 3>(mx, mw, mwn, tp, grid, st, mode, pairs);
#endif
  (void)ng_override;
  return launch_tc_ng<KB, 2>(mx, mw, mwn, tp, grid, st, mode, pairs);
}

}  // namespace amun
#endif  // AMUN_TC_DEFINE
