// tools/stepbench.cu -- cycles per wavefront step of the simulate kernel's
// fast path, isolated (not part of the product).  One warp, 2 stages per
// config (lanes 0/1 active), the step of run_gpt2: predicated task fast
// path (parity select, add, high-word bounds), a warp vote guarding a slow
// path that never triggers, the two neighbour shuffles and the send.
// Variants: V0 as the kernel; V1 without the vote/branch; V2 without the
// task (shuffles + send only); V3 task only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o sb tools/stepbench.cu && ./sb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Cache { int lo, hi; double Su0, Su1; };

template <int V>
__global__ void step_loop(double* out, long long* cyc, int steps, Cache c, double sendc,
                          volatile int* never) {
  const int lane = threadIdx.x & 31;
  const int s = lane & 1;
  double clk = 1024.0 + lane;            // inside binade 2^10
  int kk = -s;
  const unsigned K2 = 1u << 30;
  long long t0 = clock64();
  for (int w = 0; w < steps; w++) {
    const bool act = (unsigned)kk < K2 && !(kk & 1);
    const bool rcv = s > 0 && (unsigned)(kk + 1) < K2 && (kk & 1);
    kk++;
    if (V != 2) {
      const double Su = (__double2loint(clk) & 1) ? c.Su1 : c.Su0;
      const double y = __dadd_rn(clk, Su);
      const bool ok = act && __double2hiint(clk) >= c.lo && __double2hiint(y) < c.hi;
      clk = ok ? y : clk;
      const bool slow = act && !ok;
      if (V == 0 || V == 3) {
        if (__any_sync(0xffffffffu, slow)) {
          if (slow) clk = clk * (double)(*never + 1);      // never taken
        }
      }
      if (V == 4) {                                        // divergent branch, no vote
        if (__builtin_expect(slow, 0)) clk = clk * (double)(*never + 1);
      }
      if (V == 5) {                                        // vote every other step
        if ((w & 1) && __any_sync(0xffffffffu, slow)) {
          if (slow) clk = clk * (double)(*never + 1);
        }
      }
    }
    if (V != 3) {
      const double nbu = __shfl_down_sync(0xffffffffu, clk, 1);
      const double nbd = __shfl_up_sync(0xffffffffu, clk, 1);
      const bool sd = act && s == 0;
      const double nc = __dadd_rn(fmax(clk, sd ? nbu : nbd), sendc);
      clk = (sd || rcv) ? nc : clk;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = clk;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out; long long* cyc; int* never;
  cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 8); cudaMalloc(&never, 4); cudaMemset(never, 0, 4);
  Cache c{(1023 + 10) << 20, (1023 + 11) << 20, 1e-9, 1e-9};
  const int steps = 100000;
  const char* names[6] = {"kernel-like (task + vote + send)", "no vote", "send only", "task + vote only",
                          "divergent branch, no vote", "vote every other step"};
  for (int v = 0; v < 6; v++) {
    long long h = 0;
    for (int rep = 0; rep < 2; rep++) {
      if (v == 0) step_loop<0><<<1, 32>>>(out, cyc, steps, c, 1e-9, never);
      if (v == 1) step_loop<1><<<1, 32>>>(out, cyc, steps, c, 1e-9, never);
      if (v == 2) step_loop<2><<<1, 32>>>(out, cyc, steps, c, 1e-9, never);
      if (v == 3) step_loop<3><<<1, 32>>>(out, cyc, steps, c, 1e-9, never);
      if (v == 4) step_loop<4><<<1, 32>>>(out, cyc, steps, c, 1e-9, never);
      if (v == 5) step_loop<5><<<1, 32>>>(out, cyc, steps, c, 1e-9, never);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-36s %.1f cycles/step\n", names[v], (double)h / steps);
  }
  return 0;
}
