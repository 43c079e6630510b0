// sim_launch.cuh -- host-side entry points of the simulate kernels.
//
// Each k_simulate<KIND, MODE> instantiation is compiled in its own
// translation unit (sim_inst.cu built once per (KIND, MODE), in parallel, by
// build_lib.py); distir.cu reaches them only through these functions.
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace distir {

struct SimArgs {
  const SpecBlock* sp;
  const DExplicit* ex;
  const Bucket* bk;
  const Item* items;
  const PCfg* perm;
  WsHeader* hdr;
  double* ms;
  int64_t* pk;
  uint32_t* rs;
  double* tp;
  SimTopk topk;
};

#define DISTIR_SIM_DECL(KD, MD)                                                    \
  cudaError_t sim_launch_##KD##_##MD(int grid, int tpb, int smem, cudaStream_t st, \
                                     const SimArgs& a);                            \
  const void* sim_fn_##KD##_##MD();
DISTIR_SIM_DECL(0, 0) DISTIR_SIM_DECL(0, 1) DISTIR_SIM_DECL(0, 2) DISTIR_SIM_DECL(0, 3)
DISTIR_SIM_DECL(0, 4) DISTIR_SIM_DECL(0, 5) DISTIR_SIM_DECL(0, 6) DISTIR_SIM_DECL(0, 7)
DISTIR_SIM_DECL(0, 8)
DISTIR_SIM_DECL(1, 0) DISTIR_SIM_DECL(1, 1) DISTIR_SIM_DECL(1, 2) DISTIR_SIM_DECL(1, 3)
DISTIR_SIM_DECL(1, 4)
#undef DISTIR_SIM_DECL
#ifdef DISTIR_INSTR
#define DISTIR_SIM_CNT(KD, MD) int sim_counters_##KD##_##MD(unsigned long long* out, int n);
DISTIR_SIM_CNT(0, 0) DISTIR_SIM_CNT(0, 1) DISTIR_SIM_CNT(0, 2) DISTIR_SIM_CNT(0, 3)
DISTIR_SIM_CNT(0, 4) DISTIR_SIM_CNT(0, 5) DISTIR_SIM_CNT(0, 6) DISTIR_SIM_CNT(0, 7)
DISTIR_SIM_CNT(0, 8)
DISTIR_SIM_CNT(1, 0) DISTIR_SIM_CNT(1, 1) DISTIR_SIM_CNT(1, 2) DISTIR_SIM_CNT(1, 3)
DISTIR_SIM_CNT(1, 4)
#undef DISTIR_SIM_CNT
#endif

}  // namespace distir
