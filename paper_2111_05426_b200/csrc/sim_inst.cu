// sim_inst.cu -- one k_simulate<SIM_KIND, SIM_MODE> instantiation per
// translation unit (built with -DSIM_KIND=k -DSIM_MODE=m by build_lib.py), so
// the heavy simulate kernels compile in parallel.
#define DISTIR_SIM_TU 1
#include "kernels.cuh"
#include "sim_launch.cuh"

#if !defined(SIM_KIND) || !defined(SIM_MODE)
#error "build with -DSIM_KIND=<kind> -DSIM_MODE=<mode>"
#endif
#define DISTIR_CAT_(a, b, c) a##b##_##c
#define DISTIR_CAT(a, b, c) DISTIR_CAT_(a, b, c)

namespace distir {

cudaError_t DISTIR_CAT(sim_launch_, SIM_KIND, SIM_MODE)(int grid, int tpb, int smem,
                                                          cudaStream_t st, const SimArgs& a) {
  k_simulate<SIM_KIND, SIM_MODE><<<grid, tpb, smem, st>>>(a.sp, a.ex, a.bk, a.items, a.perm, a.hdr,
                                                          a.ms, a.pk, a.rs, a.tp, a.topk);
  return cudaGetLastError();
}

const void* DISTIR_CAT(sim_fn_, SIM_KIND, SIM_MODE)() {
  return reinterpret_cast<const void*>(&k_simulate<SIM_KIND, SIM_MODE>);
}

#ifdef DISTIR_INSTR
// this TU's instrumentation counters: read, add into out[0..n), reset
int DISTIR_CAT(sim_counters_, SIM_KIND, SIM_MODE)(unsigned long long* out, int n) {
  unsigned long long h[40];
  if (cudaMemcpyFromSymbol(h, g_distir_instr, sizeof(h)) != cudaSuccess) return -1;
  for (int i = 0; i < n && i < 40; i++) out[i] = (i == 8 || i == 11) ? (out[i] > h[i] ? out[i] : h[i]) : out[i] + h[i];
  unsigned long long z[40] = {0};
  return cudaMemcpyToSymbol(g_distir_instr, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif

}  // namespace distir
