// raw.cuh -- f3: raw-program mode.  Simulates arbitrary
// explicit DistIR programs -- a list of ops, each with a device set, a cost,
// input and output values -- with the synchronous semantics of the paper:
// an op starts when all its devices are free and blocks all of them
// (P:119), end = start + cost (one IEEE add; max is exact); values
// are live from creation to last use on their device, parameters from t = 0,
// returned values never freed.  One thread per program; the per-device
// clocks and live/peak counters are thread-local, last uses are found by a
// reverse scan into the workspace.  Covers programs the model expanders do not
// generate (Fig. 3, hand-written strategies, randomized checks).
#pragma once
#include "common.cuh"

namespace distir {

__global__ void k_raw_eval(const RawProgram* __restrict__ progs, int n_progs,
                           const RawOp* __restrict__ ops, const int32_t* __restrict__ idx,
                           const RawValue* __restrict__ vals, int32_t* __restrict__ last_use,
                           double* __restrict__ makespan, double* __restrict__ clock_out,
                           int64_t* __restrict__ peak_out, double* __restrict__ op_start,
                           double* __restrict__ op_end) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_progs) return;
  const RawProgram pr = progs[p];
  const RawOp* op = ops + pr.op_base;
  const RawValue* val = vals + pr.value_base;
  int32_t* lu = last_use + pr.value_base;
  // last use of every value: reverse scan over the ops' inputs
  for (int v = 0; v < pr.n_values; v++) lu[v] = -1;
  for (int i = pr.n_ops - 1; i >= 0; i--) {
    const RawOp o = op[i];
    for (int j = 0; j < o.n_in; j++) {
      const int v = idx[o.in_off + j];
      if (lu[v] < 0) lu[v] = i;
    }
  }
  double clk[kRawMaxDev];
  int64_t live[kRawMaxDev], peak[kRawMaxDev];
  for (int d = 0; d < pr.n_dev; d++) { clk[d] = 0.0; live[d] = 0; }
  for (int v = 0; v < pr.n_values; v++)
    if (val[v].flags & 1) live[val[v].dev] += val[v].bytes;      // parameters
  for (int d = 0; d < pr.n_dev; d++) peak[d] = live[d];
  for (int i = 0; i < pr.n_ops; i++) {
    const RawOp o = op[i];
    double start = 0.0;
    for (int j = 0; j < o.n_dev; j++) start = fmax(start, clk[idx[o.dev_off + j]]);
    const double end = __dadd_rn(start, o.cost);
    for (int j = 0; j < o.n_dev; j++) clk[idx[o.dev_off + j]] = end;
    if (op_start) { op_start[pr.op_base + i] = start; op_end[pr.op_base + i] = end; }
    for (int j = 0; j < o.n_out; j++) {                           // allocate outputs
      const RawValue v = val[idx[o.out_off + j]];
      live[v.dev] += v.bytes;
    }
    for (int j = 0; j < o.n_dev; j++) {                           // peaks of members
      const int d = idx[o.dev_off + j];
      peak[d] = peak[d] > live[d] ? peak[d] : live[d];
    }
    for (int j = 0; j < o.n_in; j++) {                            // free last uses
      const int v = idx[o.in_off + j];
      bool dup = false;
      for (int t = 0; t < j; t++) dup |= idx[o.in_off + t] == v;
      if (!dup && lu[v] == i && !(val[v].flags & 2)) live[val[v].dev] -= val[v].bytes;
    }
    for (int j = 0; j < o.n_out; j++) {                           // dead outputs
      const int v = idx[o.out_off + j];
      if (lu[v] < 0 && !(val[v].flags & 2)) live[val[v].dev] -= val[v].bytes;
    }
  }
  double ms = 0.0;
  for (int d = 0; d < pr.n_dev; d++) ms = fmax(ms, clk[d]);
  makespan[p] = ms;
  if (clock_out)
    for (int d = 0; d < pr.n_dev; d++) clock_out[pr.out_base + d] = clk[d];
  if (peak_out)
    for (int d = 0; d < pr.n_dev; d++) peak_out[pr.out_base + d] = peak[d];
}

}  // namespace distir
