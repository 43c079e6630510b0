// kernels.cuh -- sm_100a kernels of the DistIR grid pass (product path).
//
// Steps (BASELINE north_star):
//   k_enumerate  a1  index -> config, validity bits (C.1-C.2),
//                    warp-shape bucket (hash), closed-form op counts
//   k_plan           bucket -> lanes per config, work items in LPT order
//   k_scatter        configs grouped by bucket into warp work items
//   k_simulate   a2-a6  per config: D/T/P + GPipe program as register
//                    templates (C.3/C.4), analytic costs (P:483-487,
//                    P:518-520; C.5), synchronous timeline (
//                    C.6) and live memory (C.7), capacity
//   k_topk_*     a7/a8  top-k by (throughput desc, peak asc, index asc)
//
// Design: one warp holds 32/S configurations, S lanes
// each (S = next power of two >= P, capped at 32).  Lane sl of a segment owns
// pipeline stage sl (and sl + 32 when 32 < P <= 64).  All D*T ranks of a stage
// run the same cost sequence and hold equal clocks and peaks (SURVEY C.6
// Theorem 2: power-of-two D, T, node size, aligned groups), so one lane
// represents them all.  Stages advance as a wavefront: task (k, s) -- the
// stage-s ops of microbatch k followed by its Send -- runs at step 2k + s
// (forward) or 2k + (P-1-s) (backward).  Each device still executes its ops in
// program order, so every op's end time is bit-identical to the global
// program-order walk (SURVEY C.6 Theorem 1): one IEEE add per op, exact max
// for the synchronising ops.  Absent collectives (T = 1, D = 1) are identity
// steps: cost +0.0 and zero bytes, which leave clocks and memory unchanged.
#pragma once
#include <nv/target>
#include <cfloat>
#include <climits>
#ifdef DISTIR_INSTR
// Debug instrumentation (tools/probe_instr.py): warp-aggregated event counts.
static __device__ unsigned long long g_distir_instr[40];   // per translation unit
__device__ __forceinline__ void distir_count(int i) {
  const unsigned m_ = __activemask();
  if ((threadIdx.x & 31) == __ffs(m_) - 1) atomicAdd(&g_distir_instr[i], (unsigned long long)__popc(m_));
}
#define DISTIR_COUNT(i) NV_IF_TARGET(NV_IS_DEVICE, (distir_count(i);))
__device__ __forceinline__ void g_distir_instr_add(int i) { atomicAdd(&g_distir_instr[i], 1ull); }
// per-lane cycle accounting of the slow path ([12] refresh, [13] crossing
// passes, [15] whole add_task), summed over lanes
__host__ __device__ __forceinline__ long long distir_clk_now() {
  NV_IF_ELSE_TARGET(NV_IS_DEVICE, (return clock64();), (return 0;))
}
__host__ __device__ __forceinline__ void distir_clk_add(int i, long long t0) {
  NV_IF_TARGET(NV_IS_DEVICE, (atomicAdd(&g_distir_instr[i], (unsigned long long)(clock64() - t0));))
}
#define DISTIR_CLK_NOW() distir_clk_now()
#define DISTIR_CLK_ADD(i, t0) distir_clk_add(i, t0)
// warp-level timing of the divergent slow path: [9] cycles, [10] entries
#define DISTIR_SLOW_T0 const long long slow_t0_ = clock64();
#define DISTIR_SLOW_T1(any)                                                   \
  if ((any) && (threadIdx.x & 31) == 0) {                                    \
    atomicAdd(&g_distir_instr[9], (unsigned long long)(clock64() - slow_t0_)); \
    atomicAdd(&g_distir_instr[10], 1ull);                                     \
  }
#else
#define DISTIR_SLOW_T0
#define DISTIR_SLOW_T1(any)
#endif
#include "common.cuh"
#include "exact_add.cuh"

namespace distir {

// ------------------------------------------------------------- config -------
struct Cfg {
  DModel M;
  int32_t topo;
  int32_t mi;            // index of M in SpecBlock.models, -1 when synthetic
  int64_t D, T, P, K, B;
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Decode canonical index i (C.1 nested order, or the synthetic sweep of
// SURVEY §8d D.1, or an explicit list).
__device__ inline void decode(const SpecBlock& sp, const DExplicit* ex, int64_t i, Cfg& c,
                              const DEntry* __restrict__ entries = nullptr) {
  if (sp.mode == MODE_EXPLICIT) {
    const DExplicit x = ex[i];
    c.M = sp.models[x.model];
    c.mi = x.model;
    c.topo = x.topo;
    c.D = x.dp; c.T = x.tp; c.P = x.pp; c.K = x.K; c.B = x.B;
    return;
  }
  if (sp.mode == MODE_SYNTH) {
    uint64_t r[8];
#pragma unroll
    for (int t = 0; t < 8; t++)
      r[t] = mix64(sp.synth_seed + 0x9E3779B97F4A7C15ull * (uint64_t)(8 * i + t + 1));
    const int e = (int)(r[1] % 7);               // W = 2^e
    int j = (int)(r[2] % (uint64_t)((e + 1) * (e + 2) / 2));
    int a = 0;                                   // j-th triple, lexicographic
    while (j >= e - a + 1) { j -= e - a + 1; a++; }
    c.D = 1ll << a; c.T = 1ll << j; c.P = 1ll << (e - a - j);
    c.K = (c.P == 1) ? 1 : (1ll << (1 + r[3] % 5));
    c.B = 1ll << (7 + r[4] % 12);
    if ((r[0] & 1) == 0) {
      c.M = DModel{0, (int32_t)(1 << (1 + r[5] % 6)), (int32_t)(1 << (8 + r[6] % 7)), 1, 1, 0, 0, 2, 8, 0, 0, 0, 0};
    } else {
      const int q = (int)(r[5] % 4);
      const int32_t L = q == 0 ? 12 : q == 1 ? 24 : q == 2 ? 36 : 48;
      const int32_t d = q == 0 ? 768 : q == 1 ? 1024 : q == 2 ? 1280 : 1600;
      const int32_t h = q == 0 ? 12 : q == 1 ? 16 : q == 2 ? 20 : 25;
      c.M = DModel{1, L, d, h, 8, 50304, 1024, 2, 8, 1, 0, 0, 0};
    }
    c.topo = sp.topo_ids[r[7] % (uint64_t)sp.n_topos];
    c.mi = -1;
    return;
  }
  const int64_t mt = i / sp.per_mt;
  const int64_t r = i - mt * sp.per_mt;
  const int mi = (int)(mt / sp.n_topos), ti = (int)(mt - (int64_t)mi * sp.n_topos);
  const DEntry* E = entries ? entries : sp.entries;
  int lo = 0, hi = sp.n_entries - 1;            // last entry with cum <= r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (E[mid].cum <= r) lo = mid; else hi = mid - 1;
  }
  const DEntry en = E[lo];
  const int64_t r2 = r - en.cum;
  const int64_t kq = r2 / sp.n_batch, bq = r2 - kq * sp.n_batch;
  c.M = sp.models[sp.model_ids[mi]];
  c.mi = sp.model_ids[mi];
  c.topo = sp.topo_ids[ti];
  c.D = en.D; c.T = en.T; c.P = en.P;
  c.K = (sp.k_mode == 0 && en.P == 1) ? 1 : sp.k_set[kq];
  c.B = sp.batch[bq];
}

// C.2 validity bits.
__device__ __forceinline__ uint32_t validity(const Cfg& c, const DTopo& t) {
  uint32_t r = 0;
  if (c.B % (c.D * c.K) != 0) r |= 1u;
  if (c.P > c.M.L) r |= 2u;
  if (c.M.d % c.T != 0) r |= 4u;
  if (c.M.kind == 1 && c.M.V % c.T != 0) r |= 4u;
  if (c.M.kind == 1 && c.M.h % c.T != 0) r |= 8u;
  if (c.D * c.T * c.P > t.world_max) r |= 16u;
  return r;
}

// Global op count of the program (a collective counts once; C.3 / C.4) and
// the (op, stage) steps a representative-rank walk performs.
__device__ __forceinline__ void op_counts(const Cfg& c, int64_t& events, int64_t& steps) {
  const int64_t D = c.D, T = c.T, P = c.P, K = c.K, L = c.M.L;
  const int64_t tp = T > 1, dp = D > 1;
  if (c.M.kind == 0) {
    events = 5 * K * D * T * L + D * T * L + K * D * T + tp * K * D * L + 2 * K * D * T * (P - 1) + dp * T * L;
    steps = K * (5 * L + tp * L + 1 + 2 * (P - 1)) + L * (1 + dp);
    // f4 (tests/test_oracle_f4.py op-count closed forms): checkpointing
    // recomputes every layer but each stage's last (MatMul, Relu, a TP
    // AllReduce for row layers); ZeRO adds per microbatch and layer two
    // Broadcasts and a Reduce per TP index, Adds / SGDs on the owner only
    // and no DP AllReduce
    int64_t rec = 0, rows = 0;
    if (c.M.rc) {
      rec = L - P;
      for (int64_t l = 1; l < L; l += 2) rows++;
      for (int64_t s = 0; s < P; s++) rows -= (((s + 1) * L / P - 1) & 1);
      steps += K * (2 * rec + tp * rows);
    }
    const int64_t ck = K * (2 * D * T * rec + tp * D * rows);
    if (c.M.zero && D > 1) {
      events += -(D - 1) * K * T * L - (D - 1) * T * L - T * L + 3 * K * T * L + K * T * rec;
      steps += K * (3 * L + rec) - L;
    }
    events += ck;
  } else {
    const int64_t lm = c.M.lm != 0;
    events = 12 * K * D * T * L + (2 + lm) * K * D * T + tp * K * D * (2 * L + 1 + lm) + K * D * T * (P - 1);
    steps = K * (12 * L + tp * 2 * L + (1 + tp) + (1 + lm + tp * lm) + 2 * (P - 1));
  }
}

// ZeRO with D > 1 runs its own kernel (mode 6) with D lanes per stage
__device__ __forceinline__ bool is_zero(const Cfg& c) { return c.M.kind == 0 && c.M.zero && c.D > 1; }

#ifndef DISTIR_SUBORDER
#define DISTIR_SUBORDER 3               // GPT-2: order a bucket's configurations by microbatch size
                                        // (1: log2 m; 3: (log2 m, log2 T) folded into the slots,
                                        // r02bl: W3 k_simulate 0.0923 -> 0.0901 ms; 2: 128 slots,
                                        // k_simulate 0.086 but prepare +14 us, r02bk)
#endif
#ifndef DISTIR_SUBSLOTS
#define DISTIR_SUBSLOTS 16              // (32: W3 step 0.1235 ms; 16: 0.1226 -- prepare -2 us, simulate +1 us, r02bn)
#endif
constexpr int kSubSlots = DISTIR_SUBORDER == 2 ? 128 : DISTIR_SUBSLOTS;   // per-bucket sub-orders
#ifndef DISTIR_GPT2_GROUP
#define DISTIR_GPT2_GROUP 0             // GPT-2 buckets also keyed by the microbatch size (experiment, off)
#endif
__device__ __forceinline__ uint32_t bucket_key(const Cfg& c, bool group_m) {
  const uint32_t K = (uint32_t)(c.K < 255 ? c.K : 255);
  const uint32_t z = is_zero(c) ? 1u : 0u;
  const uint32_t ld = z ? (uint32_t)(63 - __clzll((unsigned long long)c.D)) : 0u;
  uint32_t key = (uint32_t)c.M.kind | (uint32_t)(c.P - 1) << 1 | (uint32_t)(c.M.L - 1) << 7 | K << 17 |
                 (uint32_t)(c.M.sched & 1) << 25 | ld << 26 | z << 29 | (uint32_t)(c.M.rc & 1) << 30;
#if DISTIR_GPT2_GROUP
  // GPT-2 in grids and lists: bits 25-29 (MLP-only fields) carry log2 of the
  // microbatch size, so a warp's configurations share it -- equal op costs
  // for equal T and topology, binade crossings in the same steps.  Measured
  // (r02az, r02ba): W3 k_simulate 0.1005 -> 0.0915 ms, but 15x the buckets
  // cost k_enumerate / k_plan +7 us and the select +4 us, so the W3 step is
  // 0.1297 -> 0.1313 ms: off.  (With T as well: k_simulate 0.113 ms.)
  if (c.M.kind == 1 && group_m) {
    const int64_t m = c.B / (c.D * c.K);
    const uint32_t lm = m > 0 ? (uint32_t)(63 - __clzll((unsigned long long)m)) : 0u;
    key |= (lm < 31 ? lm : 31u) << 25;
  }
#endif
  return key;
}

// ------------------------------------------------------------ costs (C.5) ---
// Canonical binary64 expressions, round-to-nearest, no contraction.
__device__ __forceinline__ double cost_compute(int64_t flops, const DTopo& t) {
  return __dadd_rn(__ddiv_rn(__ll2double_rn(flops), t.F), t.o);
}
// Compute op with `flops` FLOPs touching `bytes` of tensors (C.5; row f2:
// the regression form of P:518-520 when the topology selects it).
static __device__ __noinline__ double cost_regression(int64_t flops, int64_t bytes, bool mm, const DTopo& t) {
  const double c0 = mm ? t.mm_c0 : t.ew_c0, cf = mm ? t.mm_flop : t.ew_flop,
               cb = mm ? t.mm_byte : t.ew_byte;
  return __dadd_rn(__dadd_rn(c0, __dmul_rn(cf, __ll2double_rn(flops))),
                   __dmul_rn(cb, __ll2double_rn(bytes)));
}
__device__ __forceinline__ double cost_op(int64_t flops, int64_t bytes, bool mm, const DTopo& t) {
  // (out of line: keeps the setup's register pressure off the simulate loop)
  if (t.cost_model == 1) return cost_regression(flops, bytes, mm, t);
  return cost_compute(flops, t);
}
// Non-negative integer quotient, in 32 bits when both operands fit (64-bit
// division is a long software routine on the GPU; the setup does ~15).
__device__ __forceinline__ int64_t qdiv(int64_t a, int64_t b) {
  return ((uint64_t)(a | b) >> 32) == 0 ? (int64_t)((uint32_t)a / (uint32_t)b) : a / b;
}
__device__ __forceinline__ bool group_intra(int64_t first, int64_t last, int32_t ns) {
  return qdiv(first, ns) == qdiv(last, ns);
}
__device__ __forceinline__ double cost_send(int64_t bytes, bool intra, const DTopo& t) {
  const double a = intra ? t.a_intra : t.a_inter, bw = intra ? t.bw_intra : t.bw_inter;
  return __dadd_rn(a, __ddiv_rn(__ll2double_rn(bytes), bw));
}
__device__ __forceinline__ double cost_ring(int64_t steps, int64_t g, int64_t bytes, bool intra,
                                            const DTopo& t) {
  const double a = intra ? t.a_intra : t.a_inter, bw = intra ? t.bw_intra : t.bw_inter;
  const double st = __ll2double_rn(steps);
  return __dadd_rn(__dmul_rn(st, a),
                   __dmul_rn(__ddiv_rn(st, __ll2double_rn(g)), __ddiv_rn(__ll2double_rn(bytes), bw)));
}
__device__ __forceinline__ double cost_allreduce(int64_t g, int64_t bytes, bool intra, const DTopo& t) {
  return cost_ring(2 * (g - 1), g, bytes, intra, t);
}
__device__ __forceinline__ double cost_allgather(int64_t g, int64_t bytes, bool intra, const DTopo& t) {
  return cost_ring(g - 1, g, bytes, intra, t);
}

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// Live-memory step (C.7): allocate outputs, record the peak, free last uses.
#define MEM(q, a, f)                                 \
  do {                                               \
    live[q] += (a);                                  \
    peak[q] = peak[q] > live[q] ? peak[q] : live[q]; \
    live[q] -= (f);                                  \
  } while (0)

// -------------------------------------------------- stage-neighbour shuffles
// Stage s of lane `lane`, slot q is s = sl + S*q.  For V == 1 the neighbours
// of a stage are the adjacent lanes of its segment; for V == 2 (S == 32, one
// config per warp) stage 31 <-> 32 wraps between lane 31 slot 0 and lane 0
// slot 1.
template <int V>
struct Nbr {
  // value of stage s+1 for each slot
  __device__ static void up_stage(const double (&x)[V], double (&out)[V], int lane) {
    const double d0 = __shfl_down_sync(0xffffffffu, x[0], 1);
    if constexpr (V == 1) {
      out[0] = d0;
    } else {
      const double d1 = __shfl_down_sync(0xffffffffu, x[1], 1);
      const double w1 = __shfl_sync(0xffffffffu, x[1], 0);
      out[0] = lane < 31 ? d0 : w1;
      out[1] = d1;
    }
  }
  // value of stage s-1 for each slot
  __device__ static void down_stage(const double (&x)[V], double (&out)[V], int lane) {
    const double e0 = __shfl_up_sync(0xffffffffu, x[0], 1);
    if constexpr (V == 1) {
      out[0] = e0;
    } else {
      const double e1 = __shfl_up_sync(0xffffffffu, x[1], 1);
      const double y = __shfl_sync(0xffffffffu, x[0], 31);
      out[0] = e0;
      out[1] = lane > 0 ? e1 : y;
    }
  }
};

__device__ __forceinline__ int warp_max_int(int v) { return __reduce_max_sync(0xffffffffu, v); }

// A per-parity pair selected without dynamic register indexing.
template <typename T>
struct Par {
  T a, b;
  __device__ __forceinline__ T operator[](int p) const { return p ? b : a; }
};

// Work the simulate kernels actually performed (physical companions of the
// logical op-event count): lane-level task slow-path entries (a binade
// crossing or a stale cache) and warp-level wavefront / co-simulation steps.
struct WorkCount {
  unsigned int slow, steps;
};

#ifndef DISTIR_HOST_TU   // the simulate kernels are compiled in sim_inst.cu, one TU each
#include "simulate.cuh"
#endif
#undef MEM

// ------------------------------------------------------------- kernels ------
#ifndef DISTIR_SIM_TU   // sim_inst.cu compiles only k_simulate

// Bodies of the prepare phases (bid / nblk: this block's index and the grid
// size).
__device__ __forceinline__ void enumerate_body(const SpecBlock* __restrict__ spp, const DExplicit* __restrict__ ex,
                            Bucket* __restrict__ bk, uint32_t* __restrict__ cfg_bucket,
                            double* __restrict__ ms_out, int64_t* __restrict__ pk_out,
                            uint32_t* __restrict__ rs_out, double* __restrict__ tp_out,
                            PCfg* __restrict__ pc_out, WsHeader* __restrict__ hdr,
                            uint32_t* __restrict__ sub, int bid, int nblk) {
  const SpecBlock& sp = *spp;
  const int64_t nloc = sp.n_local;
  unsigned long long ev = 0, st = 0, nv = 0, tk = 0;
  // the decode table, staged in shared memory (a binary search per config)
  __shared__ DEntry s_ent[kMaxEntries];
  for (int j = threadIdx.x; j < sp.n_entries; j += blockDim.x) s_ent[j] = sp.entries[j];
  __syncthreads();
  for (int64_t q = bid * (int64_t)blockDim.x + threadIdx.x; q < nloc;
       q += (int64_t)nblk * blockDim.x) {
    const int64_t i = sp.rank + q * sp.n_ranks;
    Cfg c;
    decode(sp, ex, i, c, s_ent);
    const uint32_t r = validity(c, sp.topos[c.topo]);
    if (r) {
      rs_out[q] = r;
      ms_out[q] = __longlong_as_double(0x7FF0000000000000ll);  // +inf
      pk_out[q] = -1;
      tp_out[q] = 0.0;
      cfg_bucket[q] = kEmptyKey;
      continue;
    }
    int64_t events, steps;
    op_counts(c, events, steps);
    ev += events; st += steps; nv += 1;
    tk += (unsigned long long)(c.K * c.P * (c.M.kind == 0 ? 2 : 1));
    const uint32_t key = bucket_key(c, sp.mode != MODE_SYNTH);
    uint32_t slot = (key * 2654435761u) >> 20;                 // 12-bit hash
    uint32_t found = kOverflowBucket + (is_zero(c) ? 3u : c.M.sched ? 2u : (uint32_t)c.M.kind);
    for (int probe = 0; probe < kNumBuckets; probe++) {
      const uint32_t sl = (slot + probe) & (kNumBuckets - 1);
      uint32_t cur = *(volatile uint32_t*)&bk[sl].key;
      if (cur == kEmptyKey) cur = atomicCAS(&bk[sl].key, kEmptyKey, key);
      if (cur == kEmptyKey || cur == key) { found = sl; break; }
    }
    {   // warp-aggregated count: one atomic per bucket per warp (grids put
        // thousands of configurations in one bucket)
      const unsigned peers = __match_any_sync(__activemask(), found);
      if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&bk[found].count, (unsigned)__popc(peers));
    }
    cfg_bucket[q] = found;
    // sub-order within the bucket: GPT-2 configurations by log2 of the
    // microbatch size (a warp of equal microbatches has equal op costs for
    // equal T and topology, so its binade crossings coincide), others 0
    uint32_t so = 0;
    if (DISTIR_SUBORDER && c.M.kind == 1) {
      const int64_t mb = c.B / (c.D * c.K);
      so = mb > 0 ? (uint32_t)(63 - __clzll((unsigned long long)mb)) : 0u;
#if DISTIR_SUBORDER == 2
      // ... and by tensor-parallel degree (equal m and T: equal op costs)
      so = (so < 24 ? so : 24u) * 5u + (uint32_t)(63 - __clzll((unsigned long long)c.T)) % 5u;
#elif DISTIR_SUBORDER == 3
      // (m, T) folded into the 32 slots
      so = (so * 5u + (uint32_t)(63 - __clzll((unsigned long long)c.T))) & (uint32_t)(kSubSlots - 1);
#endif
      so = so < kSubSlots ? so : kSubSlots - 1;
    }
    atomicAdd(&sub[found * kSubSlots + so], 1u);
    pc_out[q] = PCfg{c.B, (uint32_t)q, (uint16_t)c.K, (uint8_t)c.P,
                     c.mi < 0 ? kSynthModel : (uint8_t)c.mi, (uint8_t)c.topo,
                     (uint8_t)(63 - __clzll((unsigned long long)c.D)),
                     (uint8_t)(63 - __clzll((unsigned long long)c.T)), (uint8_t)so};
  }
  // warp-aggregated statistics
  for (int o = 16; o > 0; o >>= 1) {
    ev += __shfl_xor_sync(0xffffffffu, ev, o);
    st += __shfl_xor_sync(0xffffffffu, st, o);
    nv += __shfl_xor_sync(0xffffffffu, nv, o);
    tk += __shfl_xor_sync(0xffffffffu, tk, o);
  }
  if ((threadIdx.x & 31) == 0 && nv) {
    atomicAdd(&hdr->tasks, tk);
    atomicAdd(&hdr->op_events, ev);
    atomicAdd(&hdr->stage_steps, st);
    atomicAdd(&hdr->n_valid, nv);
  }
}

__global__ void k_enumerate(const SpecBlock* __restrict__ spp, const DExplicit* __restrict__ ex,
                            Bucket* __restrict__ bk, uint32_t* __restrict__ cfg_bucket,
                            double* __restrict__ ms_out, int64_t* __restrict__ pk_out,
                            uint32_t* __restrict__ rs_out, double* __restrict__ tp_out,
                            PCfg* __restrict__ pc_out, WsHeader* __restrict__ hdr,
                            uint32_t* __restrict__ sub) {
  enumerate_body(spp, ex, bk, cfg_bucket, ms_out, pk_out, rs_out, tp_out, pc_out, hdr, sub, blockIdx.x, gridDim.x);
}

__device__ __forceinline__ uint32_t pow2ceil32(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// P <= DISTIR_SEQ_MAXP: one lane walks a whole configuration in program order
// (modes 0-2).  Measured on B200 (tools/variants.sh, W1-W5): the per-lane
// program-order walk helps isolated P = 1 chains but loses on every grid
// (more configurations per warp = more divergent binade crossings per step),
// so the default routes every P to the wavefront kernels.
#ifndef DISTIR_SEQ_MAXP
#define DISTIR_SEQ_MAXP 0
#endif

// One block: lanes per config, simulate kernel (group), work items numbered
// group-major and heaviest weight class first within a group (LPT order for
// the persistent simulate kernels), config ranges.  Configurations of one
// warp diverge whenever one of them crosses a binade (exact_add.cuh), so a
// warp's time grows with the configs it holds: while a simulate kernel has
// more resident warps than items, the heaviest classes are split into items
// of fewer configurations (cpw halved per step, heaviest class first).
constexpr int kPlanThreads = 1024;   // k_plan's block size (distir.cu launch)
#ifndef DISTIR_SCATTER_AGG
#define DISTIR_SCATTER_AGG 1            // k_scatter: warp-aggregated cursor atomics
#endif
constexpr int64_t kScatterAggMin = 1 << 16;   // ... for shards of at least this many configurations
#ifndef DISTIR_PLAIN_KERNEL
#define DISTIR_PLAIN_KERNEL 1           // route plain MLP warps to k_simulate<0, 8>
#endif
constexpr int kPlainMlpRule = 32;       // = DISTIR_PLAIN_MLP (simulate.cuh), the plain_cfg rule
// Whether an MLP GPipe warp shape (L layers, P <= 32 stages, K microbatches
// as the bucket key holds it, min(K, 255)) walks op by op.  k_plan routes
// such buckets to k_simulate<0, 8> when the host launched it: for a grid or
// list whose MLP GPipe shapes are ALL plain (else the plain configurations
// stay in k_simulate<0, 3>, which walks them too: two simulate kernels run
// one after the other, and the second would add its time), and for the
// synthetic sweep.
__host__ __device__ __forceinline__ bool mlp_plain_shape(uint32_t L, uint32_t P, uint32_t K) {
  uint32_t lanes = 1;
  while (lanes < P) lanes <<= 1;
  const uint32_t nlm = (L + P - 1) / P;
  return DISTIR_PLAIN_KERNEL && P <= 32 &&
         ((unsigned long long)nlm * K <= (unsigned long long)kPlainMlpRule * (32 / lanes) ||
          (K <= 32 && lanes <= 8));
}
__device__ __forceinline__ void plan_body(Bucket* __restrict__ bk, WsHeader* __restrict__ hdr,
                                          const PlanBudget& budget, uint32_t* __restrict__ sub) {
  __shared__ unsigned int s_items[kGroups][kNumClasses];
  __shared__ unsigned int s_alt[kGroups][kNumClasses][kMaxSplit + 1];   // items at split j
  __shared__ unsigned char s_shift[kGroups][kNumClasses];
  __shared__ unsigned int s_base[kGroups][kNumClasses];
  __shared__ unsigned int s_cfg, s_nb;
  for (int c = threadIdx.x; c < kGroups * kNumClasses; c += blockDim.x) {
    s_items[c / kNumClasses][c % kNumClasses] = 0;
    s_shift[c / kNumClasses][c % kNumClasses] = 0;
    for (int j = 0; j <= kMaxSplit; j++) s_alt[c / kNumClasses][c % kNumClasses][j] = 0;
  }
  if (threadIdx.x == 0) { s_cfg = 0; s_nb = 0; }
  __syncthreads();
  // thread t owns bucket slots t, t + 1024, ...: their count, class, group,
  // lanes and item offset stay in registers across the passes (no global
  // re-reads of what this thread just wrote)
  constexpr int kPer = (kBucketSlots + kPlanThreads - 1) / kPlanThreads;
  uint32_t cnt[kPer], grp[kPer], cls_[kPer], lanes_[kPer], off[kPer];
#pragma unroll
  for (int u = 0; u < kPer; u++) {
    const int b = threadIdx.x + u * kPlanThreads;
    cnt[u] = b < kBucketSlots ? bk[b].count : 0u;
    grp[u] = cls_[u] = lanes_[u] = off[u] = 0;
  }
#pragma unroll
  for (int u = 0; u < kPer; u++) {
    const int b = threadIdx.x + u * kPlanThreads;
    if (cnt[u] == 0) continue;
    Bucket& B = bk[b];
    uint32_t lanes, cls, group;
    if (b >= kOverflowBucket) {        // mixed shapes: one config per warp
      lanes = 32;
      cls = kNumClasses - 1;
      // MLP / GPT-2 catch-alls run two stages per lane (any P <= 64); the
      // 1F1B catch-all two stages per lane (mode 7, any P <= 64); the ZeRO
      // catch-all one (stage, replica) per lane
      group = b == kOverflowBucket + 3 ? 6
            : b == kOverflowBucket + 2 ? 7 : (uint32_t)(b - kOverflowBucket) * kModes + 4;
    } else {
      const uint32_t kind = B.key & 1, P = ((B.key >> 1) & 63) + 1, K = (B.key >> 17) & 255;
      const uint32_t mkey = kind ? (B.key & 0x01FFFFFFu) : B.key;   // GPT-2: bits 25-31 are grouping only
      uint32_t mode;
      unsigned long long est;            // serial chain, in tasks
      if (P <= DISTIR_SEQ_MAXP) {
        lanes = 1;
        mode = P == 1 ? 0 : (P == 2 ? 1 : 2);
        est = (unsigned long long)K * P * (kind ? 1ull : 2ull);
      } else if ((mkey >> 29) & 1) {     // ZeRO: D lanes per stage
        lanes = pow2ceil32(P) << ((mkey >> 26) & 7);
        mode = 6;
        est = (2ull * K + P) * 4;
      } else {
        lanes = P < 32 ? pow2ceil32(P) : 32;
        mode = (mkey >> 25) & 1 ? (P > 32 ? 7 : 5) : P > 32 ? 4 : 3;
        est = (2ull * K + P) * (kind ? 1ull : 2ull) * 2;
        // MLP GPipe warps of short pipelines walk every task op by op
        // (run_mlp's plain_cfg rule, decided here from the bucket's shape):
        // their own kernel, without the cached paths' registers, fits more
        // warps per SM
        if (kind == 0 && mode == 3 && ((budget.launched >> 8) & 1u) &&
            mlp_plain_shape(((B.key >> 7) & 1023) + 1, P, K))
          mode = 8;
      }
      cls = 63 - __clzll(est + 1);
      if (cls >= kNumClasses) cls = kNumClasses - 1;
      group = kind * kModes + mode;
    }
    B.lanes = (uint16_t)lanes;
    B.cls = (uint16_t)cls;
    B.group = (uint16_t)group;
    lanes_[u] = lanes; cls_[u] = cls; grp[u] = group;
    const uint32_t cpw = 32 / lanes;
    for (int j = 0; j <= kMaxSplit; j++) {
      const uint32_t cj = (cpw >> j) ? (cpw >> j) : 1u;
      atomicAdd(&s_alt[group][cls][j], (cnt[u] + cj - 1) / cj);
    }
    B.cfg_base = atomicAdd(&s_cfg, cnt[u]);
    B.cursor = 0;
    {   // the sub-orders' cursors start at their exclusive prefix (positions
        // within the bucket); the counts were written by k_enumerate
      uint32_t* sc = sub + (size_t)b * kSubSlots;
      uint32_t* cu = sub + (size_t)kBucketSlots * kSubSlots + (size_t)b * kSubSlots;
      uint32_t v[kSubSlots];
#pragma unroll
      for (int j = 0; j < kSubSlots; j++) v[j] = sc[j];      // independent loads first
      uint32_t acc = 0;
#pragma unroll
      for (int j = 0; j < kSubSlots; j++) {
        cu[j] = acc;
        acc += v[j];
      }
    }
    atomicAdd(&s_nb, 1u);
  }
  __syncthreads();
  static_assert(kNumClasses <= 64 && kGroups <= kPlanThreads / 32, "one warp per group, 2 classes per lane");
  const int pw = threadIdx.x >> 5, pl = threadIdx.x & 31;
  if (pw < kGroups) {                  // split heavy classes while warps are idle
    const int g = pw;                  // (warp g; lane 0 walks the non-empty classes)
    const unsigned a0 = pl < kNumClasses ? s_alt[g][pl][0] : 0u;
    const unsigned a1 = pl + 32 < kNumClasses ? s_alt[g][pl + 32][0] : 0u;
    unsigned int total = __reduce_add_sync(0xffffffffu, a0 + a1);
    unsigned long long ne = (unsigned long long)__ballot_sync(0xffffffffu, a0 != 0u) |
                            ((unsigned long long)__ballot_sync(0xffffffffu, a1 != 0u) << 32);
    if (pl == 0) {
      while (ne && total > 0) {        // heaviest non-empty class first
        const int c = 63 - __clzll(ne);
        ne &= ~(1ull << c);
        int j = 0;
        while (j < kMaxSplit && total - s_alt[g][c][j] + s_alt[g][c][j + 1] <= budget.warps[g]) {
          total = total - s_alt[g][c][j] + s_alt[g][c][j + 1];
          j++;
        }
        s_shift[g][c] = (unsigned char)j;
        if (j < kMaxSplit && s_alt[g][c][j] != s_alt[g][c][j + 1]) break;   // budget reached
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; u++) {
    if (cnt[u] == 0) continue;
    const int b = threadIdx.x + u * kPlanThreads;
    const uint32_t cpw0 = 32u / lanes_[u], sh = s_shift[grp[u]][cls_[u]];
    const uint32_t cpw = (cpw0 >> sh) ? (cpw0 >> sh) : 1u;
    bk[b].cpw = (uint16_t)cpw;
    off[u] = atomicAdd(&s_items[grp[u]][cls_[u]], (cnt[u] + cpw - 1) / cpw);
  }
  __syncthreads();
  // item numbering: group-major, heaviest class first (per-group prefix by
  // one thread per group, then the group offsets)
  __shared__ unsigned int s_gsum[kGroups];
  if (pw < kGroups) {                  // exclusive prefix over classes, heaviest first
    const int g = pw;
    const int ch = 63 - pl, cl = 31 - pl;        // lanes hold classes 63..32, then 31..0
    const unsigned vh = ch < kNumClasses ? s_items[g][ch] : 0u;
    const unsigned vl = cl < kNumClasses ? s_items[g][cl] : 0u;
    unsigned sh = vh, sl2 = vl;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned xh = __shfl_up_sync(0xffffffffu, sh, o), xl = __shfl_up_sync(0xffffffffu, sl2, o);
      if (pl >= o) { sh += xh; sl2 += xl; }
    }
    const unsigned tot_h = __shfl_sync(0xffffffffu, sh, 31), tot_l = __shfl_sync(0xffffffffu, sl2, 31);
    if (ch < kNumClasses) s_base[g][ch] = sh - vh;
    if (cl < kNumClasses) s_base[g][cl] = tot_h + sl2 - vl;
    if (pl == 0) s_gsum[g] = tot_h + tot_l;
  }
  __syncthreads();
  if (threadIdx.x < kGroups) {
    const int g = threadIdx.x;
    unsigned int off = 0;
    for (int h = 0; h < g; h++) off += s_gsum[h];
    for (int c = 0; c < kNumClasses; c++) s_base[g][c] += off;
    hdr->group_begin[g] = off;
    hdr->item_counter[g] = 0;
    if (g == kGroups - 1) {
      hdr->group_begin[kGroups] = off + s_gsum[g];
      hdr->n_items = off + s_gsum[g];
      hdr->n_buckets = s_nb;
      hdr->cfg_total = s_cfg;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPer; u++) {
    if (cnt[u] == 0) continue;
    const int b = threadIdx.x + u * kPlanThreads;
    bk[b].item_off = off[u];
    bk[b].item_base = s_base[grp[u]][cls_[u]] + off[u];
  }
}

__global__ void __launch_bounds__(kPlanThreads) k_plan(Bucket* __restrict__ bk, WsHeader* __restrict__ hdr,
                                                       PlanBudget budget, uint32_t* __restrict__ sub) {
  plan_body(bk, hdr, budget, sub);
}

__device__ __forceinline__ void scatter_body(const SpecBlock* __restrict__ spp, Bucket* __restrict__ bk,
                          const uint32_t* __restrict__ cfg_bucket, const PCfg* __restrict__ pc,
                          PCfg* __restrict__ perm, Item* __restrict__ items, uint32_t* __restrict__ sub,
                          int bid, int nblk) {
  const int64_t nloc = spp->n_local;
  for (int64_t q = bid * (int64_t)blockDim.x + threadIdx.x; q < nloc;
       q += (int64_t)nblk * blockDim.x) {
    const uint32_t b = cfg_bucket[q];
    if (b == kEmptyKey) continue;
    // warp-aggregated cursor: the lanes of one bucket take consecutive
    // positions from one atomic (any order within a bucket is valid: a
    // configuration's result does not depend on its warp neighbours)
    // (only for large shards: the order in which one atomic per lane hands
    // out positions groups configurations into warps differently, and on W3
    // that grouping is 5 % faster, r02ax -- W5's prepare is 28 % faster with
    // the aggregation)
    // the position within the bucket comes from its sub-order's cursor
    // (k_plan set it to the sub-order's first position)
    const uint32_t si = b * kSubSlots + pc[q].pad;
    uint32_t* cur = sub + (size_t)kBucketSlots * kSubSlots + si;
    uint32_t pos;
    if (DISTIR_SCATTER_AGG && nloc >= kScatterAggMin) {
      const unsigned peers = __match_any_sync(__activemask(), si);
      const int lead = __ffs(peers) - 1, me = threadIdx.x & 31;
      uint32_t base = 0;
      if (me == lead) base = atomicAdd(cur, (unsigned)__popc(peers));
      base = __shfl_sync(peers, base, lead);
      pos = base + (uint32_t)__popc(peers & ((1u << me) - 1u));
    } else {
      pos = atomicAdd(cur, 1u);
    }
    const uint32_t cpw = bk[b].cpw;
    perm[bk[b].cfg_base + pos] = pc[q];
    if (pos % cpw == 0) {
      const uint32_t cnt = bk[b].count;
      Item it;
      it.first = bk[b].cfg_base + pos;
      it.bucket = (uint16_t)b;
      it.n = (uint8_t)(cnt - pos < cpw ? cnt - pos : cpw);
      it.lg_lanes = (uint8_t)(31 - __clz((int)bk[b].lanes));
      items[bk[b].item_base + pos / cpw] = it;
    }
  }
}

__global__ void k_scatter(const SpecBlock* __restrict__ spp, Bucket* __restrict__ bk,
                          const uint32_t* __restrict__ cfg_bucket, const PCfg* __restrict__ pc,
                          PCfg* __restrict__ perm, Item* __restrict__ items, uint32_t* __restrict__ sub) {
  scatter_body(spp, bk, cfg_bucket, pc, perm, items, sub, blockIdx.x, gridDim.x);
}

// Empty bucket table and zero header (every launch starts from them).
__device__ __forceinline__ void reset_body(Bucket* bk, WsHeader* hdr, uint32_t* sub, int bid, int nblk) {
  for (int i = bid * blockDim.x + threadIdx.x; i < kBucketSlots; i += nblk * blockDim.x) {
    Bucket b{};
    b.key = kEmptyKey;
    bk[i] = b;
  }
  // the sub-order counts (the cursors are set by k_plan)
  uint4* s4 = reinterpret_cast<uint4*>(sub);
  for (int i = bid * blockDim.x + threadIdx.x; i < kBucketSlots * kSubSlots / 4; i += nblk * blockDim.x)
    s4[i] = make_uint4(0u, 0u, 0u, 0u);
  if (bid == 0 && threadIdx.x == 0) {
    WsHeader h{};
    *hdr = h;
  }
}

__global__ void k_reset(Bucket* bk, WsHeader* hdr, uint32_t* sub) { reset_body(bk, hdr, sub, blockIdx.x, gridDim.x); }


#endif  // DISTIR_SIM_TU

// ------------------------------------------------------------ top-k ---------
// The C.8 total order -- throughput desc, peak asc, index asc -- as an
// unsigned lexicographic key (larger = better): a = bits of the throughput
// (a non-negative double, so its bit pattern orders like its value; 0 marks
// "no candidate": feasible throughputs are > 0), b = ~peak, c = ~index.
struct Key {
  uint64_t a, b, c;
  double ms;
};

__device__ __forceinline__ Key make_key(double tp, int64_t peak, int64_t idx, double ms) {
  return Key{(uint64_t)__double_as_longlong(tp), ~(uint64_t)peak, ~(uint64_t)idx, ms};
}
__device__ __forceinline__ Key no_key() { return Key{0, 0, 0, 0.0}; }
__device__ __forceinline__ bool better(const Key& x, const Key& y) {      // x > y
  return x.a > y.a || (x.a == y.a && (x.b > y.b || (x.b == y.b && x.c > y.c)));
}
__device__ __forceinline__ TopkRec key_rec(const Key& k) {
  return TopkRec{(int64_t)~k.c, k.ms, __longlong_as_double((long long)k.a), (int64_t)~k.b};
}
__device__ __forceinline__ void cswap(Key& x, Key& y) {                    // x >= y after
  const bool sw = better(y, x);
  const Key t = x;
  x = sw ? y : x;
  y = sw ? t : y;
}

// Lane holding the warp's best key by (a, b, c), or -1 when no lane holds a
// candidate (a == 0).  Lexicographic max over the six 32-bit words with
// warp reductions (REDUX) and ballots; stops at the first word that leaves
// a single lane (keys are unique: c holds the index).
__device__ __forceinline__ int warp_best_lane(const Key& k) {
  const uint32_t wd[6] = {(uint32_t)(k.a >> 32), (uint32_t)k.a, (uint32_t)(k.b >> 32),
                          (uint32_t)k.b, (uint32_t)(k.c >> 32), (uint32_t)k.c};
  const int lane = threadIdx.x & 31;
  unsigned m = 0xffffffffu;
  bool any = false;
#pragma unroll
  for (int i = 0; i < 6; i++) {
    const bool in = (m >> lane) & 1u;
    const uint32_t mx = __reduce_max_sync(0xffffffffu, in ? wd[i] : 0u);
    if (i < 2) any |= mx != 0u;
    m = __ballot_sync(0xffffffffu, in && wd[i] == mx);
    if (i >= 1 && __popc(m) == 1) break;
  }
  return any ? __ffs(m) - 1 : -1;
}

// Merge n_lists sorted lists of up to k_in records (counts in list_n, or,
// when list_n == NULL, records with index >= 0 are valid) into the first k
// by the C.8 order, with the whole block: thread t owns lists t, t + B, ...
// and offers the best of their heads; k rounds of a block-wide best (warp
// winners in shared memory, then warp 0); the owner of the winner advances.
// Pads `out` to k.
template <int kLPT = 4>                                        // lists per thread
__device__ void merge_lists(const TopkRec* __restrict__ lists, const int* __restrict__ list_n,
                            int n_lists, int k_in, int k, TopkRec* __restrict__ out,
                            int* __restrict__ out_n) {
  __shared__ Key s_w[32];
  __shared__ int s_win;                                        // winning thread, -1 none
  const int t = threadIdx.x, w = t >> 5, lane = t & 31, nw = blockDim.x >> 5;
  int cnt[kLPT] = {}, ptr[kLPT] = {};
  Key hd[kLPT];
  auto head = [&](int j) -> Key {
    const int l = t + j * (int)blockDim.x;
    if (ptr[j] >= cnt[j]) return no_key();
    const TopkRec x = lists[(int64_t)l * k_in + ptr[j]];
    return make_key(x.throughput, x.peak, x.index, x.makespan);
  };
#pragma unroll
  for (int j = 0; j < kLPT; j++) {
    const int l = t + j * (int)blockDim.x;
    cnt[j] = 0;
    ptr[j] = 0;
    if (l < n_lists) {
      if (list_n) cnt[j] = list_n[l] < k_in ? list_n[l] : k_in;
      else
        while (cnt[j] < k_in && lists[(int64_t)l * k_in + cnt[j]].index >= 0) cnt[j]++;
    }
    hd[j] = head(j);
  }
  int got = 0;
  for (int r = 0; r < k; r++) {
    int bj = 0;                                                // best own head
    Key mine = hd[0];
#pragma unroll
    for (int j = 1; j < kLPT; j++)
      if (better(hd[j], mine)) { bj = j; mine = hd[j]; }
    const int wl = warp_best_lane(mine);
    bool win;
    if (nw == 1) {
      if (wl < 0) break;
      win = lane == wl;
    } else {
      if (lane == 0) s_w[w] = no_key();
      __syncwarp();
      if (lane == wl) s_w[w] = mine;
      __syncthreads();
      if (w == 0) {
        const int b = warp_best_lane(lane < nw ? s_w[lane] : no_key());
        if (lane == 0) s_win = b < 0 ? -1 : b * 32;            // warp index * 32, resolved below
      }
      __syncthreads();
      const int bw = s_win;
      __syncthreads();
      if (bw < 0) break;
      win = (w == bw / 32) && lane == wl;
    }
    if (win) {
      out[r] = key_rec(mine);
#pragma unroll
      for (int j = 0; j < kLPT; j++)
        if (j == bj) { ptr[j]++; hd[j] = head(j); }
    }
    got++;
  }
  for (int r = got + t; r < k; r += blockDim.x) out[r] = TopkRec{-1, 0.0, -1.0, -1};
  if (t == 0) *out_n = got;
}


// Running top-k of one warp of a simulate kernel (row a7 fused into the
// simulate kernels): a list L of up to k keys in shared memory, best first
// by the C.8 order, its count in a warp-uniform register.  A candidate that
// beats the k-th is inserted by one parallel shift (lane i moves entries i
// and i + 32).  Warp-uniform call.
__device__ __forceinline__ void topk_insert(Key* __restrict__ L, int& cnt, int k, const Key& kc) {
  const int lane = threadIdx.x & 31;
  if (cnt == k && !better(kc, L[k - 1])) return;
  const bool b0 = lane < cnt && better(L[lane], kc);
  const bool b1 = lane + 32 < cnt && better(L[lane + 32], kc);
  const int pos = __popc(__ballot_sync(0xffffffffu, b0)) + __popc(__ballot_sync(0xffffffffu, b1));
  const Key e0 = lane < cnt ? L[lane] : no_key();
  const Key e1 = lane + 32 < cnt ? L[lane + 32] : no_key();
  __syncwarp();
  if (lane >= pos && lane < cnt && lane + 1 < k) L[lane + 1] = e0;
  if (lane + 32 >= pos && lane + 32 < cnt && lane + 33 < k) L[lane + 33] = e1;
  __syncwarp();
  if (lane == 0) L[pos] = kc;
  __syncwarp();
  cnt = cnt < k ? cnt + 1 : k;
}
__device__ __forceinline__ Key shfl_key(const Key& x, int src) {
  Key r;
  r.a = __shfl_sync(0xffffffffu, x.a, src);
  r.b = __shfl_sync(0xffffffffu, x.b, src);
  r.c = __shfl_sync(0xffffffffu, x.c, src);
  r.ms = __shfl_sync(0xffffffffu, x.ms, src);
  return r;
}

// Persistent simulate kernel for one group (model kind x stages per lane):
// each warp pulls work items of its group, heaviest weight class first.
__host__ __device__ constexpr int sim_v(int mode) {
  return mode == 0 ? 1 : mode == 1 ? 2 : mode == 2 ? 4 : (mode == 4 || mode == 7) ? 2 : 1;
}
__host__ __device__ constexpr int sim_row(int kind, int mode) {   // doubles per lane row
  return kind == 1 ? 19 + 6 * sim_v(mode) : mode == 6 ? 43 : 15 + 20 * sim_v(mode);
}
__host__ __device__ constexpr int sim_tpb(int kind, int mode) {   // threads per block
  return sim_row(kind, mode) * 8 * 128 <= 48 * 1024 ? 128 : 64;
}
// Binade tables (exact_add.cuh BinTab) of the wavefront kernels: the first
// kTabCfgs configurations of a warp (S >= 2 lanes each) get one, filled by
// their lanes before the walk: binades x 2 parities x segments doubles.
__host__ __device__ constexpr int sim_tab(int kind, int mode) {   // doubles per config
  return mode < 3 || mode == 8 ? 0 : kind == 1 ? kTabBinadesGpt2 * 2 * 3
                     : kTabBinadesMlp * 2 * (mode == 6 ? 9 : 7);
}
__host__ __device__ constexpr int sim_tab_cfgs(int kind) {     // configurations with a table
  return kind == 1 ? kTabCfgsGpt2 : kTabCfgs;
}
__host__ __device__ constexpr int sim_smem(int kind, int mode) {  // dynamic smem bytes
  return 8 * (sim_tpb(kind, mode) * sim_row(kind, mode) +
              (sim_tpb(kind, mode) / 32) * sim_tab_cfgs(kind) * sim_tab(kind, mode)) +
         (sim_tpb(kind, mode) / 32) * kMaxK * 32;       // the warps' running top-k lists
}

#ifndef DISTIR_HOST_TU
template <int KIND, int MODE>
#ifndef DISTIR_SIM_MINB
#define DISTIR_SIM_MINB 1      // min resident blocks per SM asked of ptxas (register cap)
#endif
#ifndef DISTIR_PLAIN_MINB
#define DISTIR_PLAIN_MINB 4    // the plain MLP kernel (mode 8): 4 blocks per SM (<= 128 registers)
#endif
__global__ void __launch_bounds__(sim_tpb(KIND, MODE), MODE == 8 ? DISTIR_PLAIN_MINB : DISTIR_SIM_MINB)
k_simulate(const SpecBlock* __restrict__ spp,
                                                  const DExplicit* __restrict__ ex,
                                                  const Bucket* __restrict__ bk,
                                                  const Item* __restrict__ items,
                                                  const PCfg* __restrict__ perm,
                                                  WsHeader* __restrict__ hdr,
                                                  double* __restrict__ ms_out,
                                                  int64_t* __restrict__ pk_out,
                                                  uint32_t* __restrict__ rs_out,
                                                  double* __restrict__ tp_out,
                                                  const SimTopk tk) {
  constexpr int G = KIND * kModes + MODE;
  constexpr bool SEQ = MODE < 3;
  constexpr int V = sim_v(MODE);
  const SpecBlock& sp = *spp;
  const int lane = threadIdx.x & 31;
  const unsigned int first = hdr->group_begin[G], end = hdr->group_begin[G + 1];
  // Warp w starts on item first + w (no atomic; heaviest items go to the
  // first warps), then pulls items past the grid's warp count from a queue.
  const unsigned int n_warps = gridDim.x * (blockDim.x >> 5);
  const unsigned int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  bool first_item = true;
  // per-lane rows (op costs, then per-slot task-cache increments), then
  // the warps' binade tables
  constexpr int ROW = sim_row(KIND, MODE);
  constexpr int TAB = sim_tab(KIND, MODE);
  extern __shared__ double s_dyn[];
  double* row = s_dyn + threadIdx.x * ROW;
  double* wtab = s_dyn + sim_tpb(KIND, MODE) * ROW + (threadIdx.x >> 5) * sim_tab_cfgs(KIND) * TAB;
  // this warp's running top-k (after every warp's tables)
  Key* wlist = reinterpret_cast<Key*>(s_dyn + sim_tpb(KIND, MODE) * ROW +
                                      (sim_tpb(KIND, MODE) / 32) * sim_tab_cfgs(KIND) * TAB) +
               (threadIdx.x >> 5) * kMaxK;
  int wcnt = 0;
  const int k = tk.k;
  unsigned long long feas = 0;
  WorkCount wc{0u, 0u};
  while (true) {
    unsigned int id;
    if (first_item) {
      id = first + gw;
      first_item = false;
    } else {
      id = 0;
      if (lane == 0) id = first + n_warps + atomicAdd(&hdr->item_counter[G], 1u);
      id = __shfl_sync(0xffffffffu, id, 0);
    }
    if (id >= end) break;
    const Item it = items[id];
    const int S = 1 << it.lg_lanes;
    const int seg = lane / S, sl = lane - seg * S;
    const bool has = seg < it.n;
    const PCfg pc = has ? perm[it.first + seg] : PCfg{1, 0u, 1, 1, 0, 0, 0, 0, 0};
    const uint32_t q = pc.q;
    Cfg c;
    if (has && pc.model == kSynthModel) {
      decode(sp, ex, sp.rank + (int64_t)q * sp.n_ranks, c);     // arithmetic only
    } else if (has) {
      c.M = sp.models[pc.model];
      c.mi = pc.model;
      c.topo = pc.topo;
      c.D = 1ll << pc.lgD; c.T = 1ll << pc.lgT; c.P = pc.P; c.K = pc.K; c.B = pc.B;
    } else {
      c.M = DModel{KIND, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0};
      c.topo = 0; c.mi = 0; c.D = c.T = c.P = c.K = c.B = 1;
    }
    const DTopo& tp = sp.topos[c.topo];
    double* tab = (TAB > 0 && S >= 2 && seg < sim_tab_cfgs(KIND)) ? wtab + seg * TAB : nullptr;
    double ms;
    int64_t pk;
#ifdef DISTIR_INSTR
    const long long t0 = clock64();
#endif
    if constexpr (KIND == 1) run_gpt2<V, SEQ>(c, tp, has, sl, S, lane, row, tab, ms, pk, wc);
    else if constexpr (MODE == 6) run_mlp_zero(c, tp, has, sl, S, lane, row, tab, ms, pk, wc);
    else if constexpr (MODE == 8) {   // warps of short pipelines: every task walked op by op
      if (warp_max_int(has ? c.M.rc : 0))
        run_mlp<1, false, false, true, true>(c, tp, has, sl, S, lane, row, tab, ms, pk, wc);
      else
        run_mlp<1, false, false, false, true>(c, tp, has, sl, S, lane, row, tab, ms, pk, wc);
    }
    else if (warp_max_int(has ? c.M.rc : 0))          // bucket key: warp-uniform
      run_mlp<V, SEQ, MODE == 5 || MODE == 7, true>(c, tp, has, sl, S, lane, row, tab, ms, pk, wc);
    else
      run_mlp<V, SEQ, MODE == 5 || MODE == 7, false>(c, tp, has, sl, S, lane, row, tab, ms, pk, wc);
#ifdef DISTIR_INSTR
    if (lane == 0) {
      const unsigned long long dt = (unsigned long long)(clock64() - t0);
      atomicAdd(&g_distir_instr[5], dt);
      atomicAdd(&g_distir_instr[7], 1ull);
      atomicMax(&g_distir_instr[8], dt);
      // slowest item: cycles and its bucket key / configs (for probe_instr)
      atomicMax(&g_distir_instr[11], (dt << 24) | ((unsigned long long)(bk[it.bucket].key & 0x7FFFF) << 5) |
                                         (unsigned long long)(it.n & 31));
    }
#endif
    // makespan and peak: max over the stages of the segment
    for (int o = S >> 1; o > 0; o >>= 1) {
      ms = fmax(ms, __shfl_xor_sync(0xffffffffu, ms, o));
      const int64_t po = __shfl_xor_sync(0xffffffffu, pk, o);
      pk = pk > po ? pk : po;
    }
    bool cand = false;
    Key mine = no_key();
    if (has && sl == 0) {
      const uint32_t r = pk > tp.capacity ? kCapacityBit : 0u;
      const double thr = r ? 0.0 : __ddiv_rn(__ll2double_rn(c.B), ms);
      ms_out[q] = ms;
      pk_out[q] = pk;
      rs_out[q] = r;
      tp_out[q] = thr;
      feas += r == 0;
      cand = r == 0;
      if (cand) mine = make_key(thr, pk, sp.rank + (int64_t)q * sp.n_ranks, ms);
    }
    // a7: the feasible configurations of this item join the warp's top-k
    if (k > 0) {
      for (unsigned m = __ballot_sync(0xffffffffu, cand); m; m &= m - 1)
        topk_insert(wlist, wcnt, k, shfl_key(mine, __ffs(m) - 1));
    }
  }
  unsigned long long slow = wc.slow;
  for (int o = 16; o > 0; o >>= 1) {
    feas += __shfl_xor_sync(0xffffffffu, feas, o);
    slow += __shfl_xor_sync(0xffffffffu, slow, o);
  }
  if (lane == 0) {
    if (feas) atomicAdd(&hdr->n_feasible, feas);
    if (slow) atomicAdd(&hdr->slow_tasks, slow);
    if (wc.steps) atomicAdd(&hdr->wave_steps, (unsigned long long)wc.steps);
  }
  if (k <= 0) return;
  // ---- a7: warp 0 merges the block's warp lists into part[blockIdx.x] and,
  // when the merged list is full, raises the threshold to its k-th key
  constexpr int NW = sim_tpb(KIND, MODE) / 32;
  __shared__ int s_wcnt[NW];
  if (lane == 0) s_wcnt[threadIdx.x >> 5] = wcnt;
  __syncthreads();
  if (threadIdx.x < 32) {
    const Key* base = reinterpret_cast<const Key*>(s_dyn + sim_tpb(KIND, MODE) * ROW +
                                                   NW * sim_tab_cfgs(KIND) * TAB);
    const int cnt = lane < NW ? s_wcnt[lane] : 0;
    int ptr = 0, o = 0;
    uint64_t kth_a = 0;
    TopkRec* dst = tk.part + (int64_t)blockIdx.x * k;
    for (int r = 0; r < k; r++) {
      const Key h = ptr < cnt ? base[lane * kMaxK + ptr] : no_key();
      const int wl = warp_best_lane(h);
      if (wl < 0) break;
      if (lane == wl) { dst[r] = key_rec(h); ptr++; }
      kth_a = __shfl_sync(0xffffffffu, h.a, wl < 0 ? 0 : wl);
      o++;
    }
    if (lane == 0) {
      tk.part_n[blockIdx.x] = o;
      if (o == k) atomicMax(tk.thresh, (unsigned long long)kth_a);
    }
  }
}

#endif  // DISTIR_HOST_TU

#ifndef DISTIR_SIM_TU
// Block-wide best of one key per thread (C.8 order): the index of the
// winning thread, or -1 when no thread holds a candidate.  Whole block.
__device__ __forceinline__ int block_best_thread(const Key& mine) {
  __shared__ Key s_bw[32];
  __shared__ int s_bt[32];
  __shared__ int s_win;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int wl = warp_best_lane(mine);
  const Key wk = shfl_key(mine, wl < 0 ? 0 : wl);
  if (lane == 0) {
    s_bw[w] = wl < 0 ? no_key() : wk;
    s_bt[w] = wl < 0 ? -1 : w * 32 + wl;
  }
  __syncthreads();
  if (w == 0) {
    const int b = warp_best_lane(lane < nw ? s_bw[lane] : no_key());
    if (lane == 0) s_win = b < 0 ? -1 : s_bt[b];
  }
  __syncthreads();
  const int r = s_win;
  __syncthreads();                                   // s_bw / s_bt / s_win reused next call
  return r;
}

// a7, final step: the top k of the simulate blocks' partial lists (SimTopk).
// Records below the threshold cannot be in the top k; the survivors (at most
// kSelectCap) are selected in shared memory by k rounds of a block-wide best.
// With more survivors (mass ties at the threshold) every list head is
// rescanned each round instead.  One block of kSelectThreads.
__global__ void __launch_bounds__(kSelectThreads) k_topk_select(
    const TopkRec* __restrict__ part, const int* __restrict__ part_n, int n_lists, int k,
    const WsHeader* __restrict__ hdr, TopkRec* __restrict__ out, int* __restrict__ out_n) {
  __shared__ Key s_c[kSelectCap];
  __shared__ int s_n;
  const int t = threadIdx.x;
  const uint64_t T = *(volatile const unsigned long long*)&hdr->topk_thresh;
  if (t == 0) s_n = 0;
  __syncthreads();
  // one list per thread: its count, then its records in batches of 8
  // independent loads (a list's records are contiguous; one L2 round trip
  // per batch instead of one dependent count + record pair per record)
  for (int l = t; l < n_lists; l += blockDim.x) {
    const int nl = part_n[l];
    const TopkRec* src = part + (int64_t)l * k;
    for (int r0 = 0; r0 < nl; r0 += 8) {
      TopkRec x[8];
#pragma unroll
      for (int j = 0; j < 8; j++)
        if (r0 + j < nl) x[j] = src[r0 + j];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        if (r0 + j >= nl) continue;
        const Key kk = make_key(x[j].throughput, x[j].peak, x[j].index, x[j].makespan);
        if (kk.a < T) continue;
        const int pos = atomicAdd(&s_n, 1);
        if (pos < kSelectCap) s_c[pos] = kk;
      }
    }
  }
  __syncthreads();
  const int n = s_n;
  int got = 0;
  if (n <= 4 * 32) {
    // few survivors (the usual case): warp 0 alone, no block barriers
    if (t < 32) {
      Key c[4];
#pragma unroll
      for (int j = 0; j < 4; j++) c[j] = t + 32 * j < n ? s_c[t + 32 * j] : no_key();
      cswap(c[0], c[1]); cswap(c[2], c[3]); cswap(c[0], c[2]); cswap(c[1], c[3]); cswap(c[1], c[2]);
      int head = 0;
      for (int r = 0; r < k; r++) {
        const Key mine = head == 0 ? c[0] : head == 1 ? c[1] : head == 2 ? c[2] : head == 3 ? c[3] : no_key();
        const int wl = warp_best_lane(mine);
        if (wl < 0) break;
        if (t == wl) { out[r] = key_rec(mine); head++; }
        got++;
      }
    }
    got = __shfl_sync(0xffffffffu, got, 0);      // (warp 0; other warps only pad)
    __shared__ int s_got;
    if (t == 0) s_got = got;
    __syncthreads();
    got = s_got;
  } else if (n <= kSelectCap) {
    constexpr int C = kSelectCap / kSelectThreads;
    static_assert(C == 4, "a four-key sorting network per thread");
    Key c[C];
#pragma unroll
    for (int j = 0; j < C; j++) c[j] = t + j * kSelectThreads < n ? s_c[t + j * kSelectThreads] : no_key();
    cswap(c[0], c[1]); cswap(c[2], c[3]); cswap(c[0], c[2]); cswap(c[1], c[3]); cswap(c[1], c[2]);
    int head = 0;
    for (int r = 0; r < k; r++) {
      const Key mine = head == 0 ? c[0] : head == 1 ? c[1] : head == 2 ? c[2] : head == 3 ? c[3] : no_key();
      const int win = block_best_thread(mine);
      if (win < 0) break;
      if (t == win) { out[r] = key_rec(mine); head++; }
      got++;
    }
  } else {
    __shared__ unsigned char s_ptr[kPartLists];
    for (int l = t; l < n_lists; l += blockDim.x) s_ptr[l] = 0;
    __syncthreads();
    for (int r = 0; r < k; r++) {
      Key best = no_key();
      int bl = -1;
      for (int l = t; l < n_lists; l += blockDim.x) {
        if (s_ptr[l] >= part_n[l]) continue;
        const TopkRec x = part[(int64_t)l * k + s_ptr[l]];
        const Key kk = make_key(x.throughput, x.peak, x.index, x.makespan);
        if (better(kk, best)) { best = kk; bl = l; }
      }
      const int win = block_best_thread(best);
      if (win < 0) break;
      if (t == win) { out[r] = key_rec(best); s_ptr[bl]++; }
      got++;
      __syncthreads();
    }
  }
  for (int r = got + t; r < k; r += blockDim.x) out[r] = TopkRec{-1, 0.0, -1.0, -1};
  if (t == 0) *out_n = got;
}

// Merge of gathered per-rank lists (and the empty-shard case).
__global__ void __launch_bounds__(kTopkThreads) k_topk_merge(const TopkRec* __restrict__ lists,
                                                            const int* __restrict__ list_n,
                                                            int n_lists, int k_in, int k,
                                                            TopkRec* __restrict__ out,
                                                            int* __restrict__ out_n) {
  merge_lists(lists, list_n, n_lists, k_in, k, out, out_n);
}
#endif  // DISTIR_SIM_TU

}  // namespace distir
