// simulate.cuh -- per-configuration walk of the D/T/P + GPipe program
// (rows a2-a5).  Included by kernels.cuh inside namespace distir, after the
// cost helpers, the MEM macro, Par and Nbr.
//
// Per lane = one pipeline stage (two when 32 < P <= 64).  A *task* is the
// stage's ops for one microbatch (SURVEY C.3 / C.4 emission order); its clock
// advance is applied with add_task (exact_add.cuh: bit-identical to one IEEE
// add per op, one add per task in the common case) and its live-memory
// effect with a precomputed MemProf (exact integer composition of the per-op
// alloc/peak/free steps of C.7).  Sends between stages are exact max + one
// add, exchanged with warp shuffles.  Op costs live in a per-lane row of
// shared memory (`row`), read only when a task's binade cache is refreshed
// or a task crosses a binade.

// Binade range of a configuration's clocks (for its BinTab): from the
// smallest positive op cost (every positive clock is at least one op's cost)
// to an upper bound of the makespan (P stages x the busiest stage's total
// work, doubled for rounding slack), capped at nb_max binades.  `work` is
// this lane's total work; the max runs over the configuration's S lanes.
__device__ __forceinline__ BinTab bintab_range(double* tab, int nb_max, int nu, double cmin,
                                               double work, int64_t P, int S, double slack = 2.0) {
  for (int o = S >> 1; o > 0; o >>= 1) {
    work = fmax(work, __shfl_xor_sync(0xffffffffu, work, o));
    cmin = fmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
  }
  BinTab t{reinterpret_cast<int64_t*>(tab), 0, 0, nu};
  if (tab != nullptr && cmin > 0.0 && cmin < kInf()) {
    const int32_t e0 = exp_field(cmin);
    const int32_t e1 = exp_field(__dmul_rn(work, slack * (double)P)) + 1;
    t.e0 = e0 < 53 ? 53 : e0;
    const int32_t nb = e1 - t.e0 + 1;
    t.nb = nb < 0 ? 0 : (nb > nb_max ? nb_max : nb);
  }
  return t;
}
__device__ __forceinline__ double min_pos(double m, double x) { return x > 0.0 && x < m ? x : m; }
// per-lane shared-memory storage reused for integer per-pass increments
__device__ __forceinline__ int64_t* i64(double* p) { return reinterpret_cast<int64_t*>(p); }

// Slow path entry: a warp vote and a uniform branch (DISTIR_VOTE=1), or a
// plain divergent branch (0: no vote; the slow path has no warp-collective
// operations).  Measured in isolation (tools/stepbench.cu): the vote and its
// branch cost ~110 cycles per wavefront step, the divergent branch ~50.
#ifndef DISTIR_VOTE
#ifdef DISTIR_INSTR
#define DISTIR_VOTE 1
#else
#define DISTIR_VOTE 0
#endif
#endif
#if DISTIR_VOTE
#define DISTIR_ANY(p) __any_sync(0xffffffffu, (p))
#else
#define DISTIR_ANY(p) (p)
#endif
#ifndef DISTIR_PLAIN_AFTER_MLP
#define DISTIR_PLAIN_AFTER_MLP 1   // MLP kernels: walk the rest of a task op by op after N binade crossings (W5 -16%, W2 +2%, W4 +4%)
#endif
#ifndef DISTIR_PLAIN_BLOCKS
#define DISTIR_PLAIN_BLOCKS 12
#endif
constexpr int kPlainBlocks = DISTIR_PLAIN_BLOCKS;   // GPT-2: walk tasks of <= 12 blocks op by op
                                                    // when the quick path cannot take them
#ifndef DISTIR_QUICKN
#define DISTIR_QUICKN 1     // MLP: straight-line stale-cache / single-crossing slow path
#endif
#ifndef DISTIR_PLAIN_MLP
#define DISTIR_PLAIN_MLP 32
#endif
// MLP configurations walked op by op throughout (no table, no cached
// increments): layers per stage x K <= DISTIR_PLAIN_MLP x configurations per
// warp.  A plain walk costs every lane ~4 adds per layer per task, in
// lock step; the cached fast path costs ~1 add per task plus ~20 binade
// crossings per configuration, which the configurations of a warp take one
// after another (divergent) -- so warps of many short configurations walk
// plainly (W5 2.4x faster), warps of few long ones keep the fast path.
constexpr int kPlainMlp = DISTIR_PLAIN_MLP;
#ifndef DISTIR_TIES
#define DISTIR_TIES 0       // GPT-2 tasks of > kPlainBlocks blocks with ties: closed forms
#endif                      // (task3_quick_ties) instead of add_task; measured equal on W3 (r02j), off
#ifndef DISTIR_QUICK3
#define DISTIR_QUICK3 1     // GPT-2: straight-line stale-cache / single-crossing slow path
#endif
#ifndef DISTIR_CROSS1
#define DISTIR_CROSS1 0     // straight-line single-binade-crossing slow path (task_cross1):
                            // faster single long configurations, slower grids (registers)
#endif
#if DISTIR_CROSS1 && !DISTIR_VOTE
#error "DISTIR_CROSS1 uses warp votes inside the slow path: build with DISTIR_VOTE=1"
#endif
#ifndef DISTIR_PLAIN_ALL
#define DISTIR_PLAIN_ALL 8  // GPT-2: tasks of <= N blocks walked op by op at every slow entry
                            // (A/B on one B200, r02y: W3 -2.5%, W5 -6.5%, XL P16 K128 -8%; 16: W3 +3%)
#endif
#ifndef DISTIR_JUMP
#define DISTIR_JUMP 1       // GPipe wavefronts: exact steady-state jumps (steady_jump)
#endif
#ifndef DISTIR_PLAIN_SHORT_K
#define DISTIR_PLAIN_SHORT_K 1  // MLP: warps of short pipelines walk op by op (see plain_cfg)
#endif
#ifndef DISTIR_JUMP_MLP
#define DISTIR_JUMP_MLP 0   // MLP wavefronts too: long configurations gain (MLP-1B P2 K128 -23%) but the
#endif                      // kernel's register count grows (228 -> 239) and W2 +5%, W5 +6% (r02aa): off
#ifndef DISTIR_JUMP_MLP2
#define DISTIR_JUMP_MLP2 1  // MLP GPipe wavefronts with two stages per lane (32 < P <= 64)
#endif
#ifndef DISTIR_JUMP_F1B
#define DISTIR_JUMP_F1B 1   // 1F1B slot wavefront (one stage per lane): steady-state jumps
#endif
#ifndef DISTIR_JUMP_F1B2
#define DISTIR_JUMP_F1B2 1  // ... and with two stages per lane (32 < P <= 64)
#endif
#ifndef DISTIR_JUMP_MIN_K
#define DISTIR_JUMP_MIN_K 64  // ... in warps of K >= this many microbatches (the checks cost
#endif                        // more than short pipelines gain: W5, K <= 32, +8% with them)

// Steady-state jump of a GPipe wavefront (exact).  In the pipeline's
// interior every period of two wavefront steps runs the same events on every
// stage (each stage one task, one receive, one send), so the map F over a
// window of R steps is the same function window after window.  If one window
// moved every stage clock of a configuration by the same real Delta --
// F(X) = X + Delta -- then F(X + j Delta) = F(X) + j Delta for as long as
// each clock stays in its binade and Delta is an even number of that
// binade's ulps: every IEEE add of the window is the add of some stage's
// clock whose exact result moves by j Delta inside one binade, where RN
// commutes with a shift by an even number of ulps (ties to even included),
// and max commutes with any common shift.  (Each lane's add results are its
// own clock values, which lie between its window-start and window-end
// clocks.)  So n more windows add n Delta exactly -- the same bits as walking
// them (Theorem 1 keeps the per-device program order; only clocks move).
//
// Called by every lane of the warp at the end of a window; x / snap = this
// lane's clock now / at the window's start, lane_ok = the lane holds a stage
// of the configuration, J = the configuration's stage-0 wavefront counter,
// n_max = how many more whole windows stay in the interior (<= 0: none).
// Returns the number of windows to skip (0: none), uniform over the
// configuration's S lanes; the caller adds n Delta and advances its counters.
// (lane_cond: a further condition every live lane must meet, e.g. an
// unchanged live-memory count over the window.)
__device__ __forceinline__ int64_t steady_jump(double x, double snap, bool lane_ok, bool cfg_live,
                                               int64_t n_max, int S, int lane, bool lane_cond = true) {
  const int base = lane & ~(S - 1);
  const unsigned smask = S == 32 ? 0xffffffffu : (((1u << S) - 1u) << base);
  const double dl = x - snap;                        // exact when both share a binade
  const double d0 = __shfl_sync(0xffffffffu, dl, base);
  const int64_t du = d2bits(x) - d2bits(snap);       // ulps of that binade
  const bool ok = !lane_ok || (lane_cond && snap > 0.0 && exp_field(x) == exp_field(snap) && dl == d0 &&
                               !(du & 1));
#ifdef DISTIR_INSTR
  if (cfg_live && n_max > 0) {       // jump diagnostics: attempts, and live lanes failing each test
    const int why = !lane_ok ? 0 : !(snap > 0.0 && exp_field(x) == exp_field(snap)) ? 37
                  : dl != d0 ? 38 : (du & 1) ? 39 : !lane_cond ? 31 : 0;
    if (lane == base) { DISTIR_COUNT(36); }
    if (why) { g_distir_instr_add(why); }
  }
#endif
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  const bool go = cfg_live && n_max > 0 && d0 > 0.0 && (bal & smask) == smask;
  if (!__any_sync(0xffffffffu, go)) return 0;
  int64_t n = go ? n_max : 0;
  if (go && lane_ok) {
    const int64_t room = ((int64_t)(exp_field(x) + 1) << 52) - 1 - d2bits(x);   // ulps left in the binade
    n = min(n, room / du);
  }
  for (int o = S >> 1; o > 0; o >>= 1) n = min(n, __shfl_xor_sync(0xffffffffu, n, o));
  return n;
}

// The jump check of a GPipe wavefront (one stage per lane), every 8 steps:
// windows of 4 periods (even ulp counts arise with stages one binade apart).
// kk = this lane's wavefront counter (stage s' runs task kk/2 when kk is even
// and receives when it is odd, kk = w - s' without jumps), first = the lane
// offset of the wavefront's first stage s' = 0 in the configuration's
// segment (stage 0 forward, stage P-1 backward).  J = that stage's counter
// at the next step; the window [J - 8, J) was interior iff J - 8 >= P - 1,
// and n skipped windows are iff J + 8n - 2 <= 2K - 2 (every stage s' >= 1
// receives and runs one task per period, stage 0 runs one task).  After a
// jump the warp's step bound shrinks to its configurations' remaining steps
// (a configuration ends after stage s' = P-1's task K-1, counter 2K+P-3).
__device__ __forceinline__ void wave_jump(int w, int& nsteps, double& clk, double& snap, int& kk,
                                          bool lane_ok, bool has, int64_t P, int64_t K, int S,
                                          int lane, int first) {
  if ((w & 7) != 7) return;
  const int J = __shfl_sync(0xffffffffu, kk, (lane & ~(S - 1)) + first);
  const int64_t nmax = J >= P + 7 ? (2 * K - J) / 8 : 0;
  const int64_t nj = steady_jump(clk, snap, lane_ok, has, nmax, S, lane);
  if (__any_sync(0xffffffffu, nj > 0)) {
    if (nj > 0) {
      if (lane_ok) clk = bits2d(d2bits(clk) + nj * (d2bits(clk) - d2bits(snap)));
      kk += (int)(8 * nj);
    }
    nsteps = w + 1 + warp_max_int(has ? (int)(2 * K + P - 2) - (J + (int)(8 * nj)) : 0);
  }
  snap = clk;
}

// The same check for two stages per lane (32 < P <= 64: S = 32, one
// configuration per warp; lane l holds stages l and l + 32).  Every live
// stage must show the shift of stage 0 (lane 0, first slot).
__device__ __forceinline__ void wave_jump2(int w, int& nsteps, double (&clk)[2], double (&snap)[2],
                                           int (&kk)[2], const bool (&ok)[2], bool has, int64_t P,
                                           int64_t K, int lane, int first) {
  if ((w & 7) != 7) return;
  const int k0 = __shfl_sync(0xffffffffu, kk[0], first & 31);
  const int k1 = __shfl_sync(0xffffffffu, kk[1], first & 31);
  const int J = (first >> 5) ? k1 : k0;
  const int64_t nmax = J >= P + 7 ? (2 * K - J) / 8 : 0;
  const double d0 = __shfl_sync(0xffffffffu, clk[0] - snap[0], 0);
  bool good = true;
  int64_t n = nmax;
#pragma unroll
  for (int q = 0; q < 2; q++) {
    const int64_t du = d2bits(clk[q]) - d2bits(snap[q]);
    const bool lok = snap[q] > 0.0 && exp_field(clk[q]) == exp_field(snap[q]) && clk[q] - snap[q] == d0 &&
                     !(du & 1);
    good = good && (!ok[q] || lok);
    if (ok[q] && lok && du > 0) {
      const int64_t room = ((int64_t)(exp_field(clk[q]) + 1) << 52) - 1 - d2bits(clk[q]);
      n = min(n, room / du);
    }
  }
  if (__all_sync(0xffffffffu, good) && has && nmax > 0 && d0 > 0.0) {
    for (int o = 16; o > 0; o >>= 1) n = min(n, __shfl_xor_sync(0xffffffffu, n, o));
    if (n > 0) {
#pragma unroll
      for (int q = 0; q < 2; q++) {
        if (ok[q]) clk[q] = bits2d(d2bits(clk[q]) + n * (d2bits(clk[q]) - d2bits(snap[q])));
        kk[q] += (int)(8 * n);
      }
      nsteps = w + 1 + (int)(2 * K + P - 2) - (J + (int)(8 * n));
    }
  }
  snap[0] = clk[0];
  snap[1] = clk[1];
}

// Segment -> distinct-op-list maps of the task caches (BinTab).
static __device__ constexpr int kMapId3[3] = {0, 1, 2};
// MLP backward: LossGrad, recompute (the forward lists), layers (desc)
static __device__ constexpr int kMapMlpBwd[7] = {3, 0, 1, 2, 4, 5, 6};
static __device__ constexpr int kMapMlpBwd4[4] = {3, 4, 5, 6};          // without checkpointing

__device__ __forceinline__ MemProf mem_alt(MemProf A, MemProf B, int p0, int n) {
  if (n <= 0) return mem_id();
  MemProf r = mem_id();
  if (p0) { r = B; n--; }
  r = mem_then(r, mem_rep(mem_then(A, B), n >> 1));
  if (n & 1) r = mem_then(r, A);
  return r;
}

// -------------------------------------------------- MLP training (C.3) -------
// Alternating-parity layer runs as task segments: n layers starting at
// parity p0 over per-parity op sequences A (offset oa) and B = A + na (the
// pair AB is contiguous in the row).
__device__ __forceinline__ void alt_segs(double* row, int oa, int na, int p0, int n, Seg& b, Seg& ab,
                                         Seg& a) {
  const int n1 = n - (p0 && n > 0);
  b = Seg{row + oa + na, na, (p0 && n > 0) ? 1 : 0};
  ab = Seg{row + oa, 2 * na, n1 >> 1};
  a = Seg{row + oa, na, n1 & 1};
}

template <int V, bool SEQ, bool F1B, bool RC, bool PLAIN = false>
__device__ void run_mlp(const Cfg& c, const DTopo& tp, bool has, int sl, int S, int lane,
                        double* row, double* tab, double& ms_out, int64_t& peak_out, WorkCount& wc) {
  const int64_t L = c.M.L, d = c.M.d, e = c.M.e, D = c.D, T = c.T, P = c.P, K = c.K;
  const int64_t m = has ? qdiv(c.B, D * K) : 0;
  const int32_t ns = tp.node_size;
  // Layer shapes by parity of the global layer index: even = column
  // parallel, odd = row parallel (Megatron pairing); T = 1: both full.
  const Par<int64_t> kin{d, qdiv(d, T)}, nout{qdiv(d, T), d}, dout{qdiv(d, T), d};
  const bool tp_intra = group_intra(0, T - 1, ns);
  const bool dp_intra = group_intra(0, T * (D - 1), ns);
  const int64_t w0 = kin.a * nout.a, w1 = kin.b * nout.b;
  const Par<int64_t> Wb{w0 * e, w1 * e};
  const int64_t mde = m * d * e;
  const double ar_tp = T > 1 ? cost_allreduce(T, mde, tp_intra, tp) : 0.0;
  const int64_t ar_b = T > 1 ? mde : 0;
  const int64_t dlast = dout[(L - 1) & 1];
  // LossGrad reads act_L and Y_k and writes dA (3 tensors of m x d_last)
  const double loss = cost_op(3 * m * dlast, 3 * m * dlast * e, false, tp);
  // forward / backward layer op costs (absent collectives are +0.0), in the
  // lane's row: fwd A [0,3) B [3,6), bwd A [6,10) B [10,14), LossGrad [14].
  // Bytes (regression model, DESIGN R7) = every tensor the op reads/writes:
  // MatMul act + W + Z; Relu Z + act; ReluGrad act + dA + dZ; MatMulGrad
  // act + W + dZ + dA + dW; Add G + dW + G'.
  {
    auto mm_f = [&](int64_t ki, int64_t no, int64_t w) {
      return cost_op(2 * m * w, (m * ki + w + m * no) * e, true, tp);
    };
    auto mm_b = [&](int64_t ki, int64_t no, int64_t w) {
      return cost_op(4 * m * w, (2 * m * ki + 2 * w + m * no) * e, true, tp);
    };
    row[0] = mm_f(kin.a, nout.a, w0); row[1] = 0.0;
    row[2] = cost_op(m * dout.a, 2 * m * dout.a * e, false, tp);
    row[3] = mm_f(kin.b, nout.b, w1); row[4] = ar_tp;
    row[5] = cost_op(m * dout.b, 2 * m * dout.b * e, false, tp);
    row[6] = cost_op(m * dout.a, 3 * m * dout.a * e, false, tp);
    row[7] = mm_b(kin.a, nout.a, w0); row[8] = ar_tp;
    row[9] = cost_op(w0, 3 * w0 * e, false, tp);
    row[10] = cost_op(m * dout.b, 3 * m * dout.b * e, false, tp);
    row[11] = mm_b(kin.b, nout.b, w1); row[12] = 0.0;
    row[13] = cost_op(w1, 3 * w1 * e, false, tp);
    row[14] = loss;
  }
  // live-memory profiles of one forward / backward layer (C.7)
  const MemProf lf_a = mem_then(mem_op(m * nout.a * e, 0), mem_op(m * dout.a * e, m * dout.a * e));
  const MemProf lf_b = mem_then(mem_then(mem_op(m * nout.b * e, 0), mem_op(ar_b, ar_b)),
                                mem_op(m * dout.b * e, m * dout.b * e));
  // checkpointing (f4, Fig. 8; RC = the model's `recompute`, warp-uniform):
  // a forward layer inside the stage frees its input activation at its
  // MatMul (backward uses the recomputed one)
  constexpr bool rc = RC;
  constexpr int NB = RC ? 7 : 4;               // backward task segments
  const MemProf lfk_a = mem_then(mem_op(m * nout.a * e, m * kin.a * e),
                                 mem_op(m * dout.a * e, m * dout.a * e));
  const MemProf lfk_b = mem_then(mem_then(mem_op(m * nout.b * e, m * kin.b * e), mem_op(ar_b, ar_b)),
                                 mem_op(m * dout.b * e, m * dout.b * e));
  auto lb = [&](int p, bool first, bool dead0) -> MemProf {
    const int64_t act_b = m * dout[p] * e, din = m * kin[p] * e;
    const bool col_ar = p == 0 && T > 1;
    MemProf r = mem_op(act_b, 2 * act_b);                                  // ReluGrad
    r = mem_then(r, mem_op(din + Wb[p],
                           act_b + (first ? din : 0) + ((dead0 && T == 1) ? din : 0)));  // MatMulGrad
    r = mem_then(r, mem_op(col_ar ? mde : 0, col_ar ? mde + (dead0 ? mde : 0) : 0));   // TP AR
    return mem_then(r, mem_op(Wb[p], 2 * Wb[p]));                          // Add
  };
  const MemProf lb_a = lb(0, false, false), lb_b = lb(1, false, false);

  int s[V], lo[V], hi[V];
  bool ok[V];
  double clk[V], sendf[V], sendb[V];
  int64_t live[V], peak[V];
  MemProf pf[V], pb[V];
  TaskCache cf[V], cb[V];
#pragma unroll
  for (int q = 0; q < V; q++) {
    s[q] = sl + S * q;
    ok[q] = has && s[q] < P;
    lo[q] = ok[q] ? (int)qdiv((int64_t)s[q] * L, P) : 0;
    hi[q] = ok[q] ? (int)qdiv((int64_t)(s[q] + 1) * L, P) : 0;
    const int64_t r0 = T * D * (int64_t)s[q];    // rank (0, 0, s)
    sendf[q] = (ok[q] && s[q] < P - 1)
                   ? cost_send(m * dout[(hi[q] - 1) & 1] * e, group_intra(r0, r0 + T * D, ns), tp)
                   : 0.0;
    sendb[q] = (ok[q] && s[q] > 0)
                   ? cost_send(m * kin[lo[q] & 1] * e, group_intra(r0 - T * D, r0, ns), tp)
                   : 0.0;
    const int nl = hi[q] - lo[q];
    int64_t lv = (int64_t)((nl + (lo[q] & 1)) >> 1) * 2 * Wb.b +   // odd layers in [lo, hi)
                 (int64_t)(nl - ((nl + (lo[q] & 1)) >> 1)) * 2 * Wb.a;
    if (ok[q] && s[q] == 0) lv += K * mde;                       // X_k
    if (ok[q] && s[q] == P - 1) lv += K * m * dlast * e;         // Y_k
    live[q] = ok[q] ? lv : 0; peak[q] = live[q]; clk[q] = 0.0;
    if (rc && nl > 0) {
      pf[q] = mem_then(lo[q] & 1 ? lf_b : lf_a, mem_alt(lfk_a, lfk_b, (lo[q] + 1) & 1, nl - 1));
    } else {
      pf[q] = mem_alt(lf_a, lf_b, lo[q] & 1, nl);
    }
    MemProf b = (ok[q] && s[q] == P - 1) ? mem_op(m * dlast * e, m * dlast * e) : mem_id();
    if (rc && nl > 1) b = mem_then(b, mem_alt(lf_a, lf_b, lo[q] & 1, nl - 1));   // recompute
    if (nl > 1) b = mem_then(b, mem_alt(lb_a, lb_b, (hi[q] - 1) & 1, nl - 1));
    if (nl > 0) b = mem_then(b, lb(lo[q] & 1, true, s[q] == 0 && lo[q] == 0));
    pb[q] = b;
    cf[q] = task_cache_make(i64(row + 15 + 20 * q));      // 3 fwd segments
    cb[q] = task_cache_make(i64(row + 15 + 20 * q + 6));  // 7 bwd segments
  }

  // task segments; the op lists are the same on every lane of the
  // configuration (only the repetition counts depend on the stage)
  auto fsegs = [&](int q, Seg (&sg)[3]) {
    alt_segs(row, 0, 3, lo[q] & 1, hi[q] - lo[q], sg[0], sg[1], sg[2]);
  };
  auto bsegs = [&](int q, Seg (&sg)[NB]) {    // LossGrad, [recompute], layers desc
    sg[0] = Seg{row + 14, 1, s[q] == P - 1 ? 1 : 0};
    const int nl = hi[q] - lo[q];
    if constexpr (RC) alt_segs(row, 0, 3, lo[q] & 1, nl > 1 ? nl - 1 : 0, sg[1], sg[2], sg[3]);
    alt_segs(row, 6, 4, (hi[q] - 1) & 1, nl, sg[NB - 3], sg[NB - 2], sg[NB - 1]);
  };
  bool plain_cfg;
  {
    int nlm = 0;
#pragma unroll
    for (int q = 0; q < V; q++) nlm = ok[q] && hi[q] - lo[q] > nlm ? hi[q] - lo[q] : nlm;
    for (int o = S >> 1; o > 0; o >>= 1) nlm = max(nlm, __shfl_xor_sync(0xffffffffu, nlm, o));
    const int Kw = warp_max_int(has ? (int)K : 0);
    plain_cfg = PLAIN || (int64_t)nlm * Kw <= (int64_t)kPlainMlp * (32 / S);
#if DISTIR_PLAIN_SHORT_K
    // ... and warps of >= 4 configurations of K <= 32 (their crossings come
    // one configuration after another; A/B on one B200, r02ae: W5 -11%,
    // W2 / PM / 1F1B / ZeRO grids unchanged; K <= 16 at any S: W2 +7%, W4 +8%;
    // a cycle-count model of walk vs crossings, r02ac: W2 +50%, W4 +23%)
    plain_cfg = plain_cfg || (Kw <= 32 && S <= 8);
#endif
  }
#if DISTIR_JUMP && DISTIR_JUMP_MLP2
  // two stages per lane: one configuration per warp, jumps when it is long
  const bool jump_ok2 = warp_max_int(has ? (int)K : 0) >= DISTIR_JUMP_MIN_K &&
                        __all_sync(0xffffffffu, !has || !plain_cfg);
#endif
#if DISTIR_JUMP && DISTIR_JUMP_MLP
  // steady-state jumps only in warps of long configurations (a warp of many
  // short, plainly walked ones gains less than the checks cost)
  const bool jump_ok = warp_max_int(has ? (int)K : 0) >= DISTIR_JUMP_MIN_K &&
                       __all_sync(0xffffffffu, !has || !plain_cfg);
#endif
  BinTab btf{nullptr, 0, 0, 0};
  if constexpr (!SEQ) {
    // binade table of the 7 distinct op lists (forward b / ab / a,
    // LossGrad, backward b / ab / a), filled by the configuration's lanes
    double cmin = kInf(), work = 0.0;
    for (int j = 0; j < 15; j++) cmin = min_pos(cmin, row[j]);
#pragma unroll
    for (int q = 0; q < V; q++) {
      if (!ok[q]) continue;
      cmin = min_pos(min_pos(cmin, sendf[q]), sendb[q]);
      double lay = 0.0;
      for (int j = 0; j < 14; j++) lay = lay + row[j];
      const double w = (double)(hi[q] - lo[q]) * (rc ? 2.0 : 1.0) * lay + row[14] + sendf[q] + sendb[q];
      work = fmax(work, w * (double)K);
    }
    // every task but stage 0's first starts at or after stage 0's first
    // forward task, which is at least its layers x the lighter layer's
    // forward ops: the table starts one binade below that (GPT-2 likewise)
    {
      double t0 = 0.0;
#pragma unroll
      for (int q = 0; q < V; q++)
        if (ok[q] && s[q] == 0)
          t0 = __dmul_rn(__dmul_rn((double)(hi[q] - lo[q]),
                                   fmin(row[0] + row[1] + row[2], row[3] + row[4] + row[5])), 0.5);
      for (int o = S >> 1; o > 0; o >>= 1) t0 = fmax(t0, __shfl_xor_sync(0xffffffffu, t0, o));
      if (t0 > cmin && t0 < kInf()) cmin = t0;
    }
    btf = bintab_range(has && !plain_cfg ? tab : nullptr, kTabBinadesMlp, 7, cmin, work, P, S);
    Seg f[3], g[NB], u[7];
    fsegs(0, f);
    bsegs(0, g);
    u[0] = f[0]; u[1] = f[1]; u[2] = f[2]; u[3] = g[0];
    u[4] = g[NB - 3]; u[5] = g[NB - 2]; u[6] = g[NB - 1];
    bintab_fill(btf, u, sl, S);
    __syncwarp();
  }
  // slow paths: the straight-line quick path (taskN_quick), else add_task
  // (configurations with short tasks and few microbatches are walked op by
  // op throughout -- plain_cfg, no binade table)
  auto fwd_slow = [&](int q) {
    Seg sg[3];
    fsegs(q, sg);
    if (plain_cfg) { taskN_plain(clk[q], sg); return; }
    if (DISTIR_QUICKN && clk[q] > 0.0 && taskN_quick(clk[q], sg, cf[q], btf, kMapId3) == 1) return;
    add_task(clk[q], sg, cf[q], btf, kMapId3, DISTIR_PLAIN_AFTER_MLP);
  };
  auto bwd_slow = [&](int q) {
    Seg sg[NB];
    bsegs(q, sg);
    if (plain_cfg) { taskN_plain(clk[q], sg); return; }
    if constexpr (RC) {
      if (DISTIR_QUICKN && taskN_quick(clk[q], sg, cb[q], btf, kMapMlpBwd) == 1) return;
      add_task(clk[q], sg, cb[q], btf, kMapMlpBwd, DISTIR_PLAIN_AFTER_MLP);
    } else {
      if (DISTIR_QUICKN && taskN_quick(clk[q], sg, cb[q], btf, kMapMlpBwd4) == 1) return;
      add_task(clk[q], sg, cb[q], btf, kMapMlpBwd4, DISTIR_PLAIN_AFTER_MLP);
    }
  };
  auto fwd_task = [&](int q, bool act) {
    if constexpr (SEQ) {
      if (act) mem_apply(live[q], peak[q], pf[q]);
    }
    const bool slow = task_fast_or_slow(clk[q], cf[q], act);
    wc.slow += slow;
    DISTIR_SLOW_T0
    const bool any = DISTIR_ANY(slow);
    if (any && slow) fwd_slow(q);
    DISTIR_SLOW_T1(any)
  };
  auto bwd_task = [&](int q, bool act) {
    if constexpr (SEQ) {
      if (act) mem_apply(live[q], peak[q], pb[q]);
    }
    const bool slow = task_fast_or_slow(clk[q], cb[q], act);
    wc.slow += slow;
    DISTIR_SLOW_T0
    const bool any = DISTIR_ANY(slow);
    if (any && slow) bwd_slow(q);
    DISTIR_SLOW_T1(any)
  };
  if constexpr (F1B) {
    static_assert(!SEQ, "1F1B: wavefront lanes");
    // ---- synchronous 1F1B (NEXT row f1).  Stage s's ops are the
    // PipeDream-flush sequence (w = min(P-1-s, K) warm-up forwards, then
    // F(w+i), B(i) pairs, then the remaining backwards) interleaved with its
    // Sends in the order of the unit-time schedule (DESIGN reading R6): F(k,
    // s) in slot s + k (k <= w) or 2k + s, B(k, s) in slot 2P - 1 - s + 2k; a
    // Send in the slot after its producer; in a slot, Sends before the task,
    // by lower stage of the pair, forward before backward.
    //
    // Slot wavefront: stage s runs its slot-t events at steps 3t + s + j:
    // [j = 0] the Sends on the link to s-1 (forward receive, then gradient
    // send), [1] the Sends on the link to s+1 (forward send, then gradient
    // receive), [2] the task.  The two ends of a link run its Sends at the
    // same step (stage s's j = 1 is stage s+1's j = 0); after the first Send
    // of a link both ends hold the same clock, so the second is one add.
    // Each stage runs its events in its program order and its slot blocks do
    // not overlap (3 steps per slot), so every op's end time is the
    // program-order walk's (Theorem 1); chains of Sends across stages within
    // a slot (warm-up, cool-down) pipeline along the skew.  Memory follows
    // the events in program order (C.7).
    const int Pi = (int)P, Ki = (int)K;
    int wu[V], wd[V];                              // w of this stage and of s-1
#pragma unroll
    for (int q = 0; q < V; q++) {
      wu[q] = Pi - 1 - s[q] < Ki ? Pi - 1 - s[q] : Ki;
      wd[q] = Pi - s[q] < Ki ? Pi - s[q] : Ki;
    }
    // is there a forward / backward task of stage ss in slot t (branch-free:
    // the lanes of a warp are at different sub-steps of their slots)
    auto has_f = [&](int t, int ss, int w) -> bool {
      const int dd = t - ss, h = dd >> 1;
      return (dd >= 0) & (((dd <= w) & (dd < Ki)) | (((dd & 1) == 0) & (h > w) & (h < Ki)));
    };
    auto has_b = [&](int t, int ss) -> bool {
      const int dd = t - (2 * Pi - 1 - ss);
      return (dd >= 0) & ((dd & 1) == 0) & ((dd >> 1) < Ki);
    };
    // the last task is B(K-1, 0) in slot 2P + 2K - 3, at step 3 (2P + 2K - 3) + 2
    int nsteps = warp_max_int(has ? 3 * (2 * Pi + 2 * Ki - 3) + 3 : 0);
#if DISTIR_JUMP_F1B
    const bool jump_f1b = warp_max_int(has ? Ki : 0) >= DISTIR_JUMP_MIN_K;
    double snap_c = 0.0;          // clock / live bytes at the start of the jump window
    int64_t snap_l = -1;
    double snap2c[2] = {0.0, 0.0};
    int64_t snap2l[2] = {-1, -1};
#endif
    int u[V];
#pragma unroll
    for (int q = 0; q < V; q++) u[q] = -s[q];     // step - s
    for (int step = 0; step < nsteps; step++) {
      wc.steps++;
      bool e1[V], e2[V], dn[V], tf[V], tb[V];
#pragma unroll
      for (int q = 0; q < V; q++) {
        const int uq = u[q]++;
        const int t = uq >= 0 ? uq / 3 : -1, j = uq - 3 * t;
        const int st = s[q];
        const bool lo_ok = ok[q] && st > 0 && t >= 0, hi_ok = ok[q] && st < Pi - 1 && t >= 0;
        dn[q] = j == 0;
        // the link's forward Send, then its gradient Send (slot t - 1 producers)
        e1[q] = j == 0 ? (lo_ok && has_f(t - 1, st - 1, wd[q])) : (j == 1 && hi_ok && has_f(t - 1, st, wu[q]));
        e2[q] = j == 0 ? (lo_ok && has_b(t - 1, st)) : (j == 1 && hi_ok && has_b(t - 1, st + 1));
        tf[q] = j == 2 && ok[q] && t >= 0 && has_f(t, st, wu[q]);
        tb[q] = j == 2 && ok[q] && t >= 0 && has_b(t, st);
        // the task: its memory profile, then one fast path on the forward or
        // backward cache (predicated)
        const bool act = tf[q] || tb[q];
        {
          const int64_t mp = tb[q] ? pb[q].mp : pf[q].mp, net = tb[q] ? pb[q].net : pf[q].net;
          const int64_t hi_m = live[q] + mp;
          peak[q] = (act && hi_m > peak[q]) ? hi_m : peak[q];
          live[q] += act ? net : 0;
        }
        const double x = clk[q];
        const double Su = (loword(x) & 1) ? (tb[q] ? cb[q].Su1 : cf[q].Su1) : (tb[q] ? cb[q].Su0 : cf[q].Su0);
        const double y = xadd(x, Su);
        const bool fast = act && hiword(y) < (tb[q] ? cb[q].hi : cf[q].hi);
        clk[q] = fast ? y : x;
        const bool slow = act && !fast;
        wc.slow += slow;
        if (slow) {
          if (tb[q]) bwd_slow(q);
          else fwd_slow(q);
        }
      }
      double nbu[V], nbd[V];
      Nbr<V>::up_stage(clk, nbu, lane);
      Nbr<V>::down_stage(clk, nbd, lane);
#pragma unroll
      for (int q = 0; q < V; q++) {                // predicated, no branches
        const double o = dn[q] ? nbd[q] : nbu[q];
        const double c1 = dn[q] ? sendb[q] : sendf[q];
        const double y1 = dadd(fmax(clk[q], o), c1);   // the link's first Send
        const double y2 = dadd(y1, c1);                // both ends now equal: max is the clock
        clk[q] = (e1[q] && e2[q]) ? y2 : ((e1[q] || e2[q]) ? y1 : clk[q]);
        // memory: received activation (lower link, forward), sent gradient
        // dies (lower link, backward), received gradient (upper link, backward)
        const int64_t act_b = m * kin[lo[q] & 1] * e, grd_b = m * dout[(hi[q] - 1) & 1] * e;
        const int64_t add = (dn[q] && e1[q]) ? act_b : ((!dn[q] && e2[q]) ? grd_b : 0);
        live[q] += add;
        peak[q] = peak[q] > live[q] ? peak[q] : live[q];
        live[q] -= (dn[q] && e2[q]) ? act_b : 0;
      }
#if DISTIR_JUMP_F1B
      // Steady-state jumps (as wave_jump): in slots [2P, 2K-2]
      // every stage alternates one forward and one backward task per two
      // slots (6 steps) with the same Sends, so the map over a window of
      // 24 steps (4 periods: even ulp counts with stages one binade apart)
      // repeats.  A window that moved every stage clock of a configuration
      // by the same even number of ulps inside its binade is repeated n times
      // in closed form.  Its memory events repeat too: a window that did not
      // raise a stage's live bytes (stage 0 frees a pre-split input X_k per
      // microbatch, the last stage Y_k: live falls) adds n times its change,
      // and no later window can exceed the peak it already reached.  u0 =
      // stage 0's counter at the
      // next step; the window's lowest slot is stage P-1's, the skipped
      // windows' highest stage 0's.
      if constexpr (V == 1) {
        if (jump_f1b && step % 24 == 23) {
          const int u0 = __shfl_sync(0xffffffffu, u[0], lane & ~(S - 1));
          const int64_t nmax = u0 >= 7 * Pi + 23 ? (int64_t)(6 * Ki - 3 - u0) / 24 : 0;
          const int64_t nj = steady_jump(clk[0], snap_c, ok[0], has, nmax, S, lane,
                                         snap_l >= 0 && live[0] <= snap_l);
          if (__any_sync(0xffffffffu, nj > 0)) {
            if (nj > 0) {
              if (ok[0]) {
                clk[0] = bits2d(d2bits(clk[0]) + nj * (d2bits(clk[0]) - d2bits(snap_c)));
                live[0] += nj * (live[0] - snap_l);
              }
              u[0] += (int)(24 * nj);
            }
            nsteps = step + 1 + warp_max_int(has ? 3 * (2 * Pi + 2 * Ki - 3) + 3 - (u0 + (int)(24 * nj)) : 0);
          }
          snap_c = clk[0];
          snap_l = live[0];
        }
      }
#if DISTIR_JUMP_F1B2
      if constexpr (V == 2) {           // two stages per lane (32 < P <= 64): one configuration per warp
        if (jump_f1b && step % 24 == 23) {
          const int u0 = __shfl_sync(0xffffffffu, u[0], 0);
          const int64_t nmax = u0 >= 7 * Pi + 23 ? (int64_t)(6 * Ki - 3 - u0) / 24 : 0;
          const double d0 = __shfl_sync(0xffffffffu, clk[0] - snap2c[0], 0);
          bool good = true;
          int64_t n = nmax;
#pragma unroll
          for (int q = 0; q < 2; q++) {
            const int64_t du = d2bits(clk[q]) - d2bits(snap2c[q]);
            const bool lok = snap2c[q] > 0.0 && exp_field(clk[q]) == exp_field(snap2c[q]) &&
                             clk[q] - snap2c[q] == d0 && !(du & 1) && snap2l[q] >= 0 && live[q] <= snap2l[q];
            good = good && (!ok[q] || lok);
            if (ok[q] && lok && du > 0) {
              const int64_t room = ((int64_t)(exp_field(clk[q]) + 1) << 52) - 1 - d2bits(clk[q]);
              n = min(n, room / du);
            }
          }
          if (__all_sync(0xffffffffu, good) && has && nmax > 0 && d0 > 0.0) {
            for (int o = 16; o > 0; o >>= 1) n = min(n, __shfl_xor_sync(0xffffffffu, n, o));
            if (n > 0) {
#pragma unroll
              for (int q = 0; q < 2; q++) {
                if (ok[q]) {
                  clk[q] = bits2d(d2bits(clk[q]) + n * (d2bits(clk[q]) - d2bits(snap2c[q])));
                  live[q] += n * (live[q] - snap2l[q]);
                }
                u[q] += (int)(24 * n);
              }
              nsteps = step + 1 + 3 * (2 * Pi + 2 * Ki - 3) + 3 - (u0 + (int)(24 * n));
            }
          }
#pragma unroll
          for (int q = 0; q < 2; q++) { snap2c[q] = clk[q]; snap2l[q] = live[q]; }
        }
      }
#endif
#endif
    }
  } else if constexpr (SEQ) {
    // ---- program order (one lane owns all P <= V stages)
    const int K_ = warp_max_int(has ? (int)K : 0);
    for (int k = 0; k < K_; k++) {
      wc.steps++;
#pragma unroll
      for (int q = 0; q < V; q++) {
        fwd_task(q, ok[q] && k < K);
        if (q + 1 < V && ok[q] && q + 1 < P) {                // Send q -> q+1
          const double end = dadd(fmax(clk[q], clk[q + 1 < V ? q + 1 : q]), sendf[q]);
          clk[q] = end;
          clk[q + 1 < V ? q + 1 : q] = end;
          MEM(q + 1 < V ? q + 1 : q, m * kin[lo[q + 1 < V ? q + 1 : q] & 1] * e, 0);
        }
      }
    }
    for (int k = 0; k < K_; k++) {
      wc.steps++;
#pragma unroll
      for (int q = V - 1; q >= 0; q--) {
        bwd_task(q, ok[q] && k < K);
        if (q > 0 && ok[q]) {                                  // Send q -> q-1
          const int qm = q > 0 ? q - 1 : 0;
          const double end = dadd(fmax(clk[q], clk[qm]), sendb[q]);
          clk[q] = end;
          clk[qm] = end;
          live[q] -= m * kin[lo[q] & 1] * e;                   // sent gradient dies
          MEM(qm, m * dout[(hi[qm] - 1) & 1] * e, 0);          // received gradient
        }
      }
    }
  } else {
  // Memory is time-independent (SURVEY C.7 Theorem 4): stage s's events
  // are recv act(k), fwd(k) [the Send keeps the activation for backward]
  // for every k, then recv grad(k), bwd(k), send grad(k) (the sent
  // gradient dies), composed exactly before the walk.
#pragma unroll
  for (int q = 0; q < V; q++) {
    if (!ok[q]) continue;
    const MemProf ra = s[q] > 0 ? mem_op(m * kin[lo[q] & 1] * e, 0) : mem_id();
    const MemProf rg = s[q] < P - 1 ? mem_op(m * dout[(hi[q] - 1) & 1] * e, 0) : mem_id();
    const MemProf sg = s[q] > 0 ? mem_op(0, m * kin[lo[q] & 1] * e) : mem_id();
    mem_apply(live[q], peak[q], mem_then(mem_rep(mem_then(ra, pf[q]), K),
                                         mem_rep(mem_then(mem_then(rg, pb[q]), sg), K)));
  }
  const int nsteps0 = warp_max_int(has ? (int)(2 * (K - 1) + P) : 0);
  const unsigned int K2 = (unsigned int)(2 * K);
  bool up[V], dn[V];
  double recvf[V], recvb[V];
#pragma unroll
  for (int q = 0; q < V; q++) {
    up[q] = ok[q] && s[q] < P - 1;
    dn[q] = ok[q] && s[q] > 0;
    const int64_t r0 = T * D * (int64_t)s[q];
    // costs of the Sends this stage receives: activation from s-1 (its last
    // layer is lo - 1), gradient from s+1 (its first layer is hi)
    recvf[q] = dn[q] ? cost_send(m * dout[(lo[q] - 1) & 1] * e, group_intra(r0 - T * D, r0, ns), tp) : 0.0;
    recvb[q] = up[q] ? cost_send(m * kin[hi[q] & 1] * e, group_intra(r0, r0 + T * D, ns), tp) : 0.0;
  }
  // Each Send ends at max(sender, receiver clock) + cost on both ends
  // (P:119); both ends compute it from the other's shuffled clock.
  // ---- forward wavefront: task (k, s) at step 2k + s, then Send s -> s+1
  {
    int kk[V];
#pragma unroll
    for (int q = 0; q < V; q++) kk[q] = -s[q];
    int nsteps = nsteps0;
    double snap = 0.0;   // clock at the start of the jump window
    double snap2[2] = {0.0, 0.0};
    for (int w = 0; w < nsteps; w++) {
      wc.steps++;
      bool act[V], rcv[V];
#pragma unroll
      for (int q = 0; q < V; q++) {
        act[q] = ok[q] && (unsigned int)kk[q] < K2 && !(kk[q] & 1);
        rcv[q] = dn[q] && (unsigned int)(kk[q] + 1) < K2 && (kk[q] & 1);   // stage s-1 sent
        kk[q]++;
        fwd_task(q, act[q]);
      }
      double nbu[V], nbd[V];
      Nbr<V>::up_stage(clk, nbu, lane);
      Nbr<V>::down_stage(clk, nbd, lane);
#pragma unroll
      for (int q = 0; q < V; q++) {
        const bool sd = act[q] && up[q];
        const double nc = dadd(fmax(clk[q], sd ? nbu[q] : nbd[q]), sd ? sendf[q] : recvf[q]);
        clk[q] = (sd || rcv[q]) ? nc : clk[q];
      }
#if DISTIR_JUMP && DISTIR_JUMP_MLP
      if constexpr (V == 1) {
        if (jump_ok) wave_jump(w, nsteps, clk[0], snap, kk[0], ok[0], has, P, K, S, lane, 0);
      }
#endif
#if DISTIR_JUMP && DISTIR_JUMP_MLP2
      if constexpr (V == 2) {
        if (jump_ok2) wave_jump2(w, nsteps, clk, snap2, kk, ok, has, P, K, lane, 0);
      }
#endif
    }
  }
  // ---- backward wavefront: task (k, s) at step 2k + (P-1-s), then Send s -> s-1
  {
    int kk[V];
#pragma unroll
    for (int q = 0; q < V; q++) kk[q] = -(int)(P - 1 - s[q]);
    int nsteps = nsteps0;
    double snap = 0.0;
    double snap2[2] = {0.0, 0.0};
    for (int w = 0; w < nsteps; w++) {
      wc.steps++;
      bool act[V], rcv[V];
#pragma unroll
      for (int q = 0; q < V; q++) {
        act[q] = ok[q] && (unsigned int)kk[q] < K2 && !(kk[q] & 1);
        rcv[q] = up[q] && (unsigned int)(kk[q] + 1) < K2 && (kk[q] & 1);   // stage s+1 sent
        kk[q]++;
        bwd_task(q, act[q]);
      }
      double nbu[V], nbd[V];
      Nbr<V>::up_stage(clk, nbu, lane);
      Nbr<V>::down_stage(clk, nbd, lane);
#pragma unroll
      for (int q = 0; q < V; q++) {
        const bool sd = act[q] && dn[q];
        const double nc = dadd(fmax(clk[q], sd ? nbd[q] : nbu[q]), sd ? sendb[q] : recvb[q]);
        clk[q] = (sd || rcv[q]) ? nc : clk[q];
      }
#if DISTIR_JUMP && DISTIR_JUMP_MLP
      // the backward wavefront's first stage is P-1
      if constexpr (V == 1) {
        if (jump_ok) wave_jump(w, nsteps, clk[0], snap, kk[0], ok[0], has, P, K, S, lane, (int)P - 1);
      }
#endif
#if DISTIR_JUMP && DISTIR_JUMP_MLP2
      if constexpr (V == 2) {
        if (jump_ok2) wave_jump2(w, nsteps, clk, snap2, kk, ok, has, P, K, lane, (int)P - 1);
      }
#endif
    }
  }
  }  // wavefront

  // ---- tail: DP AllReduce of the accumulated gradients, then SGD (once per
  // stage: plain op-by-op walk)
  const Par<double> ardp{D > 1 ? cost_allreduce(D, Wb.a, dp_intra, tp) : 0.0,
                         D > 1 ? cost_allreduce(D, Wb.b, dp_intra, tp) : 0.0};
  const Par<double> sgd{cost_op(2 * w0, 3 * w0 * e, false, tp),     // SGD: W + G -> W'
                        cost_op(2 * w1, 3 * w1 * e, false, tp)};
#pragma unroll
  for (int q = 0; q < V; q++) {
    if (!ok[q]) continue;
    for (int l = hi[q] - 1; l >= lo[q]; l--) {
      const int p = l & 1;
      clk[q] = dadd(clk[q], ardp[p]);
      MEM(q, D > 1 ? Wb[p] : 0, D > 1 ? Wb[p] : 0);
    }
    for (int l = lo[q]; l < hi[q]; l++) {
      const int p = l & 1;
      clk[q] = dadd(clk[q], sgd[p]);
      MEM(q, Wb[p], 2 * Wb[p]);
    }
  }
  double msx = 0.0;
  int64_t pkx = 0;
#pragma unroll
  for (int q = 0; q < V; q++) {
    if (ok[q]) { msx = fmax(msx, clk[q]); pkx = pkx > peak[q] ? pkx : peak[q]; }
  }
  ms_out = msx;
  peak_out = pkx;
}

// ------------------------------------------------ GPT-2 inference (C.4) -----
template <int V, bool SEQ>
__device__ void run_gpt2(const Cfg& c, const DTopo& tp, bool has, int sl, int S, int lane,
                         double* row, double* tab, double& ms_out, int64_t& peak_out, WorkCount& wc) {
#ifdef DISTIR_INSTR
  const long long t_entry = clock64();
#endif
  const int64_t L = c.M.L, d = c.M.d, h = c.M.h, Sq = c.M.S, Vp = c.M.V, e = c.M.e,
                ide = c.M.ide, nctx = c.M.nctx;
  const bool lm = c.M.lm != 0;
  const int64_t D = c.D, T = c.T, P = c.P, K = c.K;
  const int64_t m = has ? qdiv(c.B, D * K) : 0;
  const int64_t n = m * Sq, dT = qdiv(d, T), hT = qdiv(h, T), VT = qdiv(Vp, T);
  const int32_t ns = tp.node_size;
  const bool tp_intra = group_intra(0, T - 1, ns);
  const int64_t nde = n * d * e;
  // op costs (C.4 work per op); absent collectives are +0.0
  const double c_ar = T > 1 ? cost_allreduce(T, nde, tp_intra, tp) : 0.0;
  // Bytes (regression model, DESIGN R7) = every tensor the op reads/writes
  // (C.4 program: activations, parameters and outputs).
  const int64_t sc_b = m * hT * Sq * Sq * e, qkv_b = n * 3 * dT * e;
  const double c_ln = cost_op(5 * n * d, 2 * nde + 2 * d * e, false, tp);
  const double c_add = cost_op(n * d, 3 * nde, false, tp);
  // the lane's row: prologue [0,2), block [2,16), epilogue [16,19)
  row[0] = cost_op(2 * n * d, n * ide + VT * d * e + nctx * d * e + nde, false, tp);  // Embed
  row[1] = c_ar;                                                                     // TP AllReduce
  row[2] = c_ln;                                                                     // ln_1
  row[3] = cost_op(2 * n * d * (3 * dT) + n * (3 * dT),
                   nde + (d * 3 * dT + 3 * dT) * e + qkv_b, true, tp);              // QKV
  row[4] = cost_op(2 * m * Sq * Sq * dT, qkv_b + sc_b, true, tp);                  // scores
  row[5] = cost_op(5 * m * hT * Sq * Sq, 2 * sc_b, false, tp);                     // softmax
  row[6] = cost_op(2 * m * Sq * Sq * dT, sc_b + qkv_b + n * dT * e, true, tp);     // context
  row[7] = cost_op(2 * n * dT * d + n * d, n * dT * e + (dT * d + d) * e + nde, true, tp);  // proj
  row[8] = c_ar;                                                                     // TP AllReduce
  row[9] = c_add;                                                                    // residual
  row[10] = c_ln;                                                                    // ln_2
  row[11] = cost_op(2 * n * d * (4 * dT) + n * (4 * dT),
                    nde + (d * 4 * dT + 4 * dT) * e + n * 4 * dT * e, true, tp);    // FC1
  row[12] = cost_op(8 * n * (4 * dT), 2 * n * 4 * dT * e, false, tp);              // GeLU
  row[13] = cost_op(2 * n * (4 * dT) * d + n * d,
                    n * 4 * dT * e + (4 * dT * d + d) * e + nde, true, tp);         // FC2
  row[14] = c_ar;                                                                    // TP AllReduce
  row[15] = c_add;                                                                   // residual
  row[16] = c_ln;                                                                    // ln_f
  row[17] = lm ? cost_op(2 * n * d * VT, nde + VT * d * e + n * VT * e, true, tp) : 0.0;  // LM head
  row[18] = (lm && T > 1) ? cost_allgather(T, n * Vp * e, tp_intra, tp) : 0.0;  // AllGather
#ifdef DISTIR_INSTR
  if (lane == 0) distir_clk_add(27, t_entry);
  const long long t_mem = clock64();
#endif
  // live-memory profiles (C.7), for a normal and for the last microbatch
  // (whose ops free the parameters at their last use)
  const int64_t arb = T > 1 ? nde : 0;
  const int64_t qkvb = n * 3 * dT * e, scb = m * hT * Sq * Sq * e, ctxb = n * dT * e, fb = n * 4 * dT * e;
  const int64_t ln_p = 2 * d * e, qkv_p = (d * 3 * dT + 3 * dT) * e, prj_p = (dT * d + d) * e,
                fc1_p = (d * 4 * dT + 4 * dT) * e, fc2_p = (4 * dT * d + d) * e;
  const int64_t blk_p = 2 * ln_p + qkv_p + prj_p + fc1_p + fc2_p;
  const int64_t wte_b = VT * d * e, wpe_b = nctx * d * e;
  MemProf mblk[2], mpro[2], mepi[2];
#pragma unroll
  for (int last = 0; last < 2; last++) {
    MemProf r = mem_op(nde, last ? ln_p : 0);                       // LayerNorm ln_1
    r = mem_then(r, mem_op(qkvb, nde + (last ? qkv_p : 0)));         // QKV
    r = mem_then(r, mem_op(scb, 0));                                 // scores
    r = mem_then(r, mem_op(scb, scb));                               // softmax
    r = mem_then(r, mem_op(ctxb, scb + qkvb));                       // context
    r = mem_then(r, mem_op(nde, ctxb + (last ? prj_p : 0)));         // proj
    r = mem_then(r, mem_op(arb, arb));                               // TP AllReduce
    r = mem_then(r, mem_op(nde, 2 * nde));                           // residual
    r = mem_then(r, mem_op(nde, last ? ln_p : 0));                   // LayerNorm ln_2
    r = mem_then(r, mem_op(fb, nde + (last ? fc1_p : 0)));           // FC1
    r = mem_then(r, mem_op(fb, fb));                                 // GeLU
    r = mem_then(r, mem_op(nde, fb + (last ? fc2_p : 0)));           // FC2
    r = mem_then(r, mem_op(arb, arb));                               // TP AllReduce
    mblk[last] = mem_then(r, mem_op(nde, 2 * nde));                  // residual
    mpro[last] = mem_then(mem_op(nde, n * ide + (last ? wpe_b + ((P == 1 && lm) ? 0 : wte_b) : 0)),
                          mem_op(arb, arb));                         // Embed, TP AllReduce
    MemProf ep = mem_op(nde, nde + (last ? 2 * d * e : 0));          // final LayerNorm
    if (lm) {
      ep = mem_then(ep, mem_op(n * VT * e, nde + (last ? wte_b : 0)));           // LM head
      ep = mem_then(ep, mem_op(T > 1 ? n * Vp * e : 0, T > 1 ? n * VT * e : 0));  // AllGather
    }
    mepi[last] = ep;
  }

  int s[V], nb[V];
  bool ok[V];
  double clk[V], sendf[V];
  int64_t live[V], peak[V];
  MemProf ptask0[V], ptask1[V];   // normal / last microbatch
  TaskCache tc[V];
#pragma unroll
  for (int q = 0; q < V; q++) {
    s[q] = sl + S * q;
    ok[q] = has && s[q] < P;
    const int lo = ok[q] ? (int)qdiv((int64_t)s[q] * L, P) : 0;
    const int hi = ok[q] ? (int)qdiv((int64_t)(s[q] + 1) * L, P) : 0;
    nb[q] = hi - lo;
    const int64_t r0 = T * D * (int64_t)s[q];
    sendf[q] = (ok[q] && s[q] < P - 1) ? cost_send(nde, group_intra(r0, r0 + T * D, ns), tp) : 0.0;
    int64_t lv = (int64_t)nb[q] * blk_p;
    if (ok[q] && s[q] == 0) lv += wte_b + wpe_b + K * n * ide;
    if (ok[q] && s[q] == P - 1) lv += 2 * d * e + ((lm && P > 1) ? wte_b : 0);
    live[q] = ok[q] ? lv : 0; peak[q] = live[q]; clk[q] = 0.0;
#pragma unroll
    for (int last = 0; last < 2; last++) {
      MemProf r = (s[q] == 0) ? mpro[last] : mem_id();
      r = mem_then(r, mem_rep(mblk[last], nb[q]));
      if (s[q] == P - 1) r = mem_then(r, mepi[last]);
      if (last) ptask1[q] = r; else ptask0[q] = r;
    }
    tc[q] = task_cache_make(i64(row + 19 + 6 * q));       // 3 segments
  }
#ifdef DISTIR_INSTR
  if (lane == 0) distir_clk_add(28, t_mem);
#endif

  // the task's segments: prologue (stage 0), blocks, epilogue (stage P-1);
  // the op lists are the same on every lane of the configuration
  auto segs = [&](int q, Seg (&sg)[3]) {
    sg[0] = Seg{row, 2, s[q] == 0 ? 1 : 0};
    sg[1] = Seg{row + 2, 14, nb[q]};
    sg[2] = Seg{row + 16, 3, s[q] == P - 1 ? 1 : 0};
  };
  BinTab bt{nullptr, 0, 0, 0};
  if constexpr (!SEQ) {
    // binade table of the task segments, filled by the configuration's lanes
    // Range: every task but stage 0's first starts at a clock >= stage 0's
    // task duration t0 (after stage 0's first task), so the table starts one
    // binade below t0 (rounding slack); the makespan is at most the sum of
    // all op costs <= P x the busiest stage's K tasks and Sends.  Clocks
    // outside the table fall back to computing increments on the fly.
    double cmin = kInf(), work = 0.0;
#pragma unroll
    for (int q = 0; q < V; q++) {
      if (!ok[q]) continue;
      double w = nb[q] * (row[2] + row[3] + row[4] + row[5] + row[6] + row[7] + row[8] + row[9] +
                          row[10] + row[11] + row[12] + row[13] + row[14] + row[15]);
      if (s[q] == 0) w = w + row[0] + row[1];
      if (s[q] == P - 1) w = w + row[16] + row[17] + row[18];
      if (s[q] == 0) cmin = min_pos(cmin, __dmul_rn(w, 0.5));
      w = w + sendf[q] + sendf[q];
      work = fmax(work, w * (double)K);
    }
    bt = bintab_range(has ? tab : nullptr, kTabBinadesGpt2, 3, cmin, work, P, S, 1.0);
    Seg sg[3];
    segs(0, sg);
#ifdef DISTIR_INSTR
    const long long t_fill = clock64();
    if (lane == 0) distir_clk_add(18, t_entry);
#endif
    bintab_fill(bt, sg, sl, S);
    __syncwarp();
#ifdef DISTIR_INSTR
    if (lane == 0) distir_clk_add(20, t_fill);
#endif
  }
  auto task = [&](int q, bool act, bool last) {
    if constexpr (SEQ) {
      if (act) mem_apply(live[q], peak[q], last ? ptask1[q] : ptask0[q]);
    }
    const bool slow = task_fast_or_slow(clk[q], tc[q], act);
    wc.slow += slow;
    DISTIR_SLOW_T0
    const bool any = DISTIR_ANY(slow);
    if (any) {
      Seg sg[3];
      segs(q, sg);
      // the single-crossing path only when every slow lane qualifies (else
      // add_task runs anyway and would pay for both)
      bool s2 = slow;
      if (DISTIR_CROSS1 && __all_sync(0xffffffffu, !slow || cross1_eligible(clk[q], tc[q], bt)))
        s2 = slow && !task_cross1(clk[q], sg, tc[q], bt, kMapId3);
#if DISTIR_QUICK3
      // op by op: stage 0's first task (from zero, it climbs many binades),
      // and short tasks (few blocks) the quick path cannot take (ties)
      if (s2 && clk[q] == 0.0) {
        task3_plain(clk[q], sg);
        s2 = false;
      }
#if DISTIR_PLAIN_ALL > 0
      // short tasks: op by op, then the cache moves to the new binade
      if (s2 && nb[q] <= DISTIR_PLAIN_ALL) {
        task3_plain(clk[q], sg);
        task3_cache_to(clk[q], sg, tc[q], bt);
        s2 = false;
      }
#endif
      if (s2) {
        DISTIR_COUNT(16);
        const int r = task3_quick(clk[q], sg, tc[q], bt);
        s2 = r != 1;
        if (!s2) DISTIR_COUNT(17);
        // ties: short tasks op by op, long ones by the parity-exact closed forms
        if (s2 && nb[q] <= kPlainBlocks) {
          task3_plain(clk[q], sg);
          s2 = false;
        }
#if DISTIR_TIES
        if (s2 && r == 2) {
          s2 = !task3_quick_ties(clk[q], sg, tc[q], bt);
          if (!s2) DISTIR_COUNT(30);
        }
#endif
      }
#endif
      if (DISTIR_ANY(s2) && s2) add_task(clk[q], sg, tc[q], bt, kMapId3);
    }
    DISTIR_SLOW_T1(any)
  };
  if constexpr (SEQ) {
    // ---- program order (one lane owns all P <= V stages)
    const int K_ = warp_max_int(has ? (int)K : 0);
    for (int k = 0; k < K_; k++) {
      wc.steps++;
#pragma unroll
      for (int q = 0; q < V; q++) {
        task(q, ok[q] && k < K, k == K - 1);
        if (q + 1 < V && ok[q] && q + 1 < P) {                // Send q -> q+1
          const int qp = q + 1 < V ? q + 1 : q;
          const double end = dadd(fmax(clk[q], clk[qp]), sendf[q]);
          clk[q] = end;
          clk[qp] = end;
          live[q] -= nde;                                      // sent activation dies
          MEM(qp, nde, 0);                                     // received activation
        }
      }
    }
  } else {
  // Memory is time-independent (SURVEY C.7 Theorem 4): stage s's events
  // are recv(k), task(k), send(k) for k = 0..K-1 (the last task frees the
  // parameters), composed exactly before the walk.
#pragma unroll
  for (int q = 0; q < V; q++) {
    if (!ok[q]) continue;
    const MemProf rv = s[q] > 0 ? mem_op(nde, 0) : mem_id();          // received activation
    const MemProf sd = s[q] < P - 1 ? mem_op(0, nde) : mem_id();      // sent activation dies
    const MemProf p0 = mem_then(mem_then(rv, ptask0[q]), sd);
    const MemProf p1 = mem_then(mem_then(rv, ptask1[q]), sd);
    mem_apply(live[q], peak[q], mem_then(mem_rep(p0, K - 1), p1));
  }
  // wavefront: task (k, s) at step 2k + s, then Send s -> s+1.  Sender
  // and receiver both wait for each other and end at
  // max(their clocks) + cost; each computes it from the other's clock
  // (both neighbours' clocks are shuffled independently), bit-identically.
  int nsteps = warp_max_int(has ? (int)(2 * (K - 1) + P) : 0);
#ifdef DISTIR_INSTR
  const long long t_wave = clock64();
#endif
  double snap = 0.0;   // this lane's clock at the start of the jump window
  const bool jump_ok = warp_max_int(has ? (int)K : 0) >= DISTIR_JUMP_MIN_K;
  bool up[V], dn[V];
  int kk[V];
  double recvc[V];
  const unsigned int K2 = (unsigned int)(2 * K);
#pragma unroll
  for (int q = 0; q < V; q++) {
    up[q] = ok[q] && s[q] < P - 1;
    dn[q] = ok[q] && s[q] > 0;
    kk[q] = -s[q];
    const int64_t r0 = T * D * (int64_t)s[q];
    recvc[q] = dn[q] ? cost_send(nde, group_intra(r0 - T * D, r0, ns), tp) : 0.0;  // Send s-1 -> s
  }
  for (int w = 0; w < nsteps; w++) {
      wc.steps++;
    if (lane == 0) DISTIR_COUNT(4);
#ifdef DISTIR_INSTR
    const long long t_step = clock64();
    const unsigned slow0 = wc.slow;
#endif
    bool act[V], rcv[V];
#pragma unroll
    for (int q = 0; q < V; q++) {
      act[q] = ok[q] && (unsigned int)kk[q] < K2 && !(kk[q] & 1);
      rcv[q] = dn[q] && (unsigned int)(kk[q] + 1) < K2 && (kk[q] & 1);   // stage s-1 sent
      kk[q]++;
      task(q, act[q], false);
    }
    double nbu[V], nbd[V];
    Nbr<V>::up_stage(clk, nbu, lane);
    Nbr<V>::down_stage(clk, nbd, lane);
#pragma unroll
    for (int q = 0; q < V; q++) {
      const bool sd = act[q] && up[q];
      const double o = sd ? nbu[q] : nbd[q];
      const double nc = dadd(fmax(clk[q], o), sd ? sendf[q] : recvc[q]);
      clk[q] = (sd || rcv[q]) ? nc : clk[q];
    }
#if DISTIR_JUMP
    if constexpr (V == 1) {
      if (jump_ok) wave_jump(w, nsteps, clk[0], snap, kk[0], ok[0], has, P, K, S, lane, 0);
    }
#endif
#ifdef DISTIR_INSTR
    {   // per-step cycles, split by whether any lane of the warp took a slow path
      const bool sl_any = __any_sync(0xffffffffu, wc.slow != slow0);
      const long long dt_step = clock64() - t_step;
      if (lane == 0) {
        atomicAdd(&g_distir_instr[sl_any ? 34 : 32], (unsigned long long)dt_step);
        atomicAdd(&g_distir_instr[sl_any ? 35 : 33], 1ull);
      }
    }
#endif
  }
#ifdef DISTIR_INSTR
  if (lane == 0) distir_clk_add(19, t_wave);
#endif
  }  // wavefront
  double msx = 0.0;
  int64_t pkx = 0;
#pragma unroll
  for (int q = 0; q < V; q++) {
    if (ok[q]) { msx = fmax(msx, clk[q]); pkx = pkx > peak[q] ? pkx : peak[q]; }
  }
  ms_out = msx;
  peak_out = pkx;
}

// --------------------------------------- MLP training with ZeRO (row f4) ----
// ZeRO-2/3 (Fig. 9; DESIGN reading R9): W_l and its gradient live on
// replica l mod D of each (j, s) group.  Lane = (stage s, replica i), sl =
// i + D * s (S = next_pow2(P) * D lanes per configuration); all TP ranks of
// a replica run the same ops (Theorem 2 within the replica).  The replicas
// of a stage differ only by owner-only ops (gradient Add, SGD), and every
// forward / backward task starts with a Broadcast that synchronises them:
// a segment max over the D lanes (exact), after which the task's ops are
// the same on every replica -- including the Reduce / Add chain, because
// each Reduce waits for the previous owner's Add (max(x + add, x) = x + add,
// RN is monotone) -- up to the final Add, which only its owner performs.
// Sends pair replica i of neighbouring stages (lanes D apart).
static __device__ constexpr int kMapZeroBwd[9] = {3, 0, 1, 2, 4, 5, 6, 7, 8};

__device__ __forceinline__ double cost_chain(int64_t g, int64_t bytes, bool intra, const DTopo& t) {
  // Broadcast from / Reduce to the owner: a pipelined chain over the g
  // members, (g-1) alpha + bytes / bw (g = 2: a Send, as in Fig. 9)
  const double a = intra ? t.a_intra : t.a_inter, bw = intra ? t.bw_intra : t.bw_inter;
  return __dadd_rn(__dmul_rn(__ll2double_rn(g - 1), a), __ddiv_rn(__ll2double_rn(bytes), bw));
}

static __device__ void run_mlp_zero(const Cfg& c, const DTopo& tp, bool has, int sl, int S, int lane,
                             double* row, double* tab, double& ms_out, int64_t& peak_out, WorkCount& wc) {
  const int64_t L = c.M.L, d = c.M.d, e = c.M.e, D = c.D, T = c.T, P = c.P, K = c.K;
  const int64_t m = has ? qdiv(c.B, D * K) : 0;
  const int32_t ns = tp.node_size;
  const bool rc = c.M.rc != 0;
  const Par<int64_t> kin{d, qdiv(d, T)}, nout{qdiv(d, T), d}, dout{qdiv(d, T), d};
  const bool tp_intra = group_intra(0, T - 1, ns);
  const bool dp_intra = group_intra(0, T * (D - 1), ns);
  const int64_t w = kin.a * nout.a;              // == kin.b * nout.b (d^2 / T)
  const int64_t Wb = w * e;
  const int64_t mde = m * d * e;
  const double ar_tp = T > 1 ? cost_allreduce(T, mde, tp_intra, tp) : 0.0;
  const int64_t ar_b = T > 1 ? mde : 0;
  const int64_t dlast = dout[(L - 1) & 1];
  const double bc = D > 1 ? cost_chain(D, Wb, dp_intra, tp) : 0.0;   // Broadcast == Reduce
  {
    auto mm_f = [&](int64_t ki, int64_t no) { return cost_op(2 * m * w, (m * ki + w + m * no) * e, true, tp); };
    auto mm_b = [&](int64_t ki, int64_t no) {
      return cost_op(4 * m * w, (2 * m * ki + 2 * w + m * no) * e, true, tp);
    };
    row[0] = bc; row[1] = mm_f(kin.a, nout.a); row[2] = 0.0;
    row[3] = cost_op(m * dout.a, 2 * m * dout.a * e, false, tp);
    row[4] = bc; row[5] = mm_f(kin.b, nout.b); row[6] = ar_tp;
    row[7] = cost_op(m * dout.b, 2 * m * dout.b * e, false, tp);
    row[8] = bc; row[9] = cost_op(m * dout.a, 3 * m * dout.a * e, false, tp);
    row[10] = mm_b(kin.a, nout.a); row[11] = ar_tp;
    row[12] = bc; row[13] = cost_op(m * dout.b, 3 * m * dout.b * e, false, tp);
    row[14] = mm_b(kin.b, nout.b); row[15] = 0.0;
    row[16] = cost_op(3 * m * dlast, 3 * m * dlast * e, false, tp);            // LossGrad
    row[17] = bc;                                                            // Reduce
    row[18] = cost_op(w, 3 * w * e, false, tp);                              // Add (owner)
  }
  const double sgd = cost_op(2 * w, 3 * w * e, false, tp);

  // D is the same for every configuration of the warp (bucket key); padding
  // lanes take it from the warp so every shuffle is warp-uniform
  const int Di = warp_max_int(has ? (int)D : 1);
  const int ri = sl % Di, st = sl / Di;            // replica, stage
  const bool ok = has && st < P;
  const int lo = ok ? (int)qdiv((int64_t)st * L, P) : 0;
  const int hi = ok ? (int)qdiv((int64_t)(st + 1) * L, P) : 0;
  const int nl = hi - lo;
  const int64_t r0 = T * D * (int64_t)st;
  const double sendf = (ok && st < P - 1)
                           ? cost_send(m * dout[(hi - 1) & 1] * e, group_intra(r0, r0 + T * D, ns), tp)
                           : 0.0;
  const double sendb = (ok && st > 0) ? cost_send(m * kin[lo & 1] * e, group_intra(r0 - T * D, r0, ns), tp)
                                      : 0.0;
  // ---- live memory of replica ri (C.7), composed exactly (Theorem 4)
  auto own = [&](int l) { return (l % Di) == ri; };
  auto lfz = [&](int l, bool free_in) -> MemProf {          // [Bcast], MatMul, [AR], Relu
    const int p = l & 1;
    const int64_t cp = own(l) ? 0 : Wb;                     // the received copy
    MemProf r = mem_op(cp, 0);
    r = mem_then(r, mem_op(m * nout[p] * e, cp + (free_in ? m * kin[p] * e : 0)));
    if (p == 1) r = mem_then(r, mem_op(ar_b, ar_b));
    return mem_then(r, mem_op(m * dout[p] * e, m * dout[p] * e));
  };
  int64_t live = 0;
  for (int l = lo; l < hi; l++) live += own(l) ? 2 * Wb : 0;
  if (ok && st == 0) live += K * mde;                        // X_k
  if (ok && st == P - 1) live += K * m * dlast * e;          // Y_k
  if (!ok) live = 0;
  int64_t peak = live;
  MemProf pf = mem_id(), pb = mem_id(), tail = mem_id();
  for (int l = lo; l < hi; l++) pf = mem_then(pf, lfz(l, rc && l > lo));
  if (ok && st == P - 1) pb = mem_op(m * dlast * e, m * dlast * e);                 // LossGrad
  if (rc)
    for (int l = lo; l + 1 < hi; l++) pb = mem_then(pb, lfz(l, false));           // recompute
  for (int l = hi - 1; l >= lo; l--) {
    const int p = l & 1;
    const int64_t cp = own(l) ? 0 : Wb;
    const int64_t act_b = m * dout[p] * e, din = m * kin[p] * e;
    const bool first = l == lo, dead0 = st == 0 && l == 0, col_ar = p == 0 && T > 1;
    pb = mem_then(pb, mem_op(cp, 0));                                              // Broadcast
    pb = mem_then(pb, mem_op(act_b, 2 * act_b));                                   // ReluGrad
    pb = mem_then(pb, mem_op(din + Wb, act_b + cp + (first ? din : 0) +
                                           ((dead0 && T == 1) ? din : 0)));        // MatMulGrad
    pb = mem_then(pb, mem_op(col_ar ? mde : 0, col_ar ? mde + (dead0 ? mde : 0) : 0));  // TP AR
  }
  for (int l = lo; l < hi; l++) {
    pb = mem_then(pb, own(l) ? mem_op(Wb, Wb) : mem_op(0, Wb));                     // Reduce
    if (own(l)) pb = mem_then(pb, mem_op(Wb, 2 * Wb));                             // Add
  }
  for (int l = lo; l < hi; l++)
    if (own(l)) tail = mem_then(tail, mem_op(Wb, 2 * Wb));                         // SGD
  // the schedule (bucket key: warp-uniform); GPipe composes the stage's
  // memory events here, 1F1B applies them in its walk's order
  const bool f1b = warp_max_int(has ? (int)c.M.sched : 0) == 1;
  if (!f1b) {
    const MemProf ra = st > 0 ? mem_op(m * kin[lo & 1] * e, 0) : mem_id();
    const MemProf rg = st < P - 1 ? mem_op(m * dout[(hi - 1) & 1] * e, 0) : mem_id();
    const MemProf sg = st > 0 ? mem_op(0, m * kin[lo & 1] * e) : mem_id();
    if (ok)
      mem_apply(live, peak, mem_then(mem_then(mem_rep(mem_then(ra, pf), K),
                                              mem_rep(mem_then(mem_then(rg, pb), sg), K)), tail));
  }

  // ---- task segments and the binade table of the 9 distinct op lists
  TaskCache cf = task_cache_make(i64(row + 19)), cb = task_cache_make(i64(row + 25));
  auto fsegs = [&](Seg (&sg)[3]) { alt_segs(row, 0, 4, lo & 1, nl, sg[0], sg[1], sg[2]); };
  auto bsegs = [&](Seg (&sg)[9]) {          // LossGrad, recompute, layers desc, Reduce / Add
    sg[0] = Seg{row + 16, 1, (ok && st == P - 1) ? 1 : 0};
    alt_segs(row, 0, 4, lo & 1, (rc && nl > 1) ? nl - 1 : 0, sg[1], sg[2], sg[3]);
    alt_segs(row, 8, 4, (hi - 1) & 1, nl, sg[4], sg[5], sg[6]);
    sg[7] = Seg{row + 17, 2, nl > 0 ? nl - 1 : 0};
    sg[8] = Seg{row + 17, 1, nl > 0 ? 1 : 0};
  };
  BinTab bt{nullptr, 0, 0, 0};
  {
    double cmin = kInf(), work = 0.0;
    for (int j = 0; j < 19; j++) cmin = min_pos(cmin, row[j]);
    if (ok) {
      cmin = min_pos(min_pos(cmin, sendf), sendb);
      double lay = 0.0;
      for (int j = 0; j < 19; j++) lay = lay + row[j];
      work = (double)nl * (rc ? 2.0 : 1.0) * lay * (double)K + (sendf + sendb) * (double)K;
    }
    bt = bintab_range(has ? tab : nullptr, kTabBinadesMlp, 9, cmin, work, P, S);
    Seg f[3], g[9], u[9];
    fsegs(f);
    bsegs(g);
    u[0] = f[0]; u[1] = f[1]; u[2] = f[2];
    for (int j = 3; j < 9; j++) u[j] = g[j == 3 ? 0 : j];
    bintab_fill(bt, u, sl, S);
    __syncwarp();
  }
  double clk = 0.0;
  // the D replicas of a stage synchronise (Broadcast): exact segment max
  auto segmax = [&](double x) {
    for (int o = 1; o < Di; o <<= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
  };
  auto fwd_task = [&](bool act) {
    const double mx = segmax(clk);
    if (act) clk = mx;
    const bool slow = task_fast_or_slow(clk, cf, act);
    wc.slow += slow;
    const bool any = DISTIR_ANY(slow);
    if (any) {
      Seg sg[3];
      fsegs(sg);
      // the single-crossing path only when every slow lane qualifies (else
      // add_task runs anyway and would pay for both)
      bool s2 = slow;
      if (DISTIR_CROSS1 && __all_sync(0xffffffffu, !slow || cross1_eligible(clk, cf, bt)))
        s2 = slow && !task_cross1(clk, sg, cf, bt, kMapId3);
      if (DISTIR_ANY(s2) && s2) add_task(clk, sg, cf, bt, kMapId3);
    }
  };
  auto bwd_task = [&](bool act) {
    const double mx = segmax(clk);
    if (act) clk = mx;
    const bool slow = task_fast_or_slow(clk, cb, act);
    wc.slow += slow;
    const bool any = DISTIR_ANY(slow);
    if (any) {
      Seg sg[9];
      bsegs(sg);
      // the single-crossing path only when every slow lane qualifies (else
      // add_task runs anyway and would pay for both)
      bool s2 = slow;
      if (DISTIR_CROSS1 && __all_sync(0xffffffffu, !slow || cross1_eligible(clk, cb, bt)))
        s2 = slow && !task_cross1(clk, sg, cb, bt, kMapZeroBwd);
      if (DISTIR_ANY(s2) && s2) add_task(clk, sg, cb, bt, kMapZeroBwd);
    }
    if (act && own(hi - 1)) clk = dadd(clk, row[18]);       // the last Add: owner only
  };
  const int nsteps = warp_max_int(has ? (int)(2 * (K - 1) + P) : 0);
  const unsigned int K2 = (unsigned int)(2 * K);
  const bool up = ok && st < P - 1, dn = ok && st > 0;
  // costs of the Sends this lane receives (replica ri of stage st -/+ 1)
  const double recvf = dn ? cost_send(m * dout[(lo - 1) & 1] * e, group_intra(r0 - T * D, r0, ns), tp) : 0.0;
  const double recvb = up ? cost_send(m * kin[hi & 1] * e, group_intra(r0, r0 + T * D, ns), tp) : 0.0;
  if (f1b) {
    // ---- ZeRO under synchronous 1F1B: run_mlp's slot wavefront (DESIGN
    // reading R6; stage st's slot-t events at steps 3t + st + j: the Sends on
    // the link to st-1, those on the link to st+1, the task), with the
    // replica of this lane pairing with replica ri of the neighbouring stages
    // (lanes Di apart) and every task starting with its Broadcast (the
    // segment max over the stage's Di replicas, all at the same sub-step)
    const int Pi = (int)P, Ki = (int)K;
    const int w_s = Pi - 1 - st < Ki ? Pi - 1 - st : Ki, w_d = Pi - st < Ki ? Pi - st : Ki;
    auto has_f = [&](int t, int ss, int w) -> bool {
      const int dd = t - ss, hh = dd >> 1;
      return (dd >= 0) & (((dd <= w) & (dd < Ki)) | (((dd & 1) == 0) & (hh > w) & (hh < Ki)));
    };
    auto has_b = [&](int t, int ss) -> bool {
      const int dd = t - (2 * Pi - 1 - ss);
      return (dd >= 0) & ((dd & 1) == 0) & ((dd >> 1) < Ki);
    };
    const int n1 = warp_max_int(has ? 3 * (2 * Pi + 2 * Ki - 3) + 3 : 0);
    int uq = -st;
    const int64_t act_b = m * kin[lo & 1] * e, grd_b = m * dout[(hi - 1) & 1] * e;
    for (int step = 0; step < n1; step++) {
      wc.steps++;
      const int u = uq++;
      const int t = u >= 0 ? u / 3 : -1, j = u - 3 * t;
      const bool lo_ok = ok && st > 0 && t >= 0, hi_ok = ok && st < Pi - 1 && t >= 0;
      const bool dnl = j == 0;
      const bool e1 = dnl ? (lo_ok && has_f(t - 1, st - 1, w_d)) : (j == 1 && hi_ok && has_f(t - 1, st, w_s));
      const bool e2 = dnl ? (lo_ok && has_b(t - 1, st)) : (j == 1 && hi_ok && has_b(t - 1, st + 1));
      const bool tf = j == 2 && ok && t >= 0 && has_f(t, st, w_s);
      const bool tb = j == 2 && ok && t >= 0 && has_b(t, st);
      if (tf) mem_apply(live, peak, pf);
      if (tb) mem_apply(live, peak, pb);
      fwd_task(tf);                                // (collective: every lane, every step)
      bwd_task(tb);
      const double nbu = __shfl_down_sync(0xffffffffu, clk, Di);
      const double nbd = __shfl_up_sync(0xffffffffu, clk, Di);
      const double o = dnl ? nbd : nbu;
      const double c1 = dnl ? recvf : recvb;       // the link's cost (both directions)
      const double y1 = dadd(fmax(clk, o), c1);
      const double y2 = dadd(y1, c1);
      clk = (e1 && e2) ? y2 : ((e1 || e2) ? y1 : clk);
      const int64_t add = (dnl && e1) ? act_b : ((!dnl && e2) ? grd_b : 0);
      live += add;
      peak = peak > live ? peak : live;
      live -= (dnl && e2) ? act_b : 0;
    }
    if (ok) mem_apply(live, peak, tail);
  } else {
  {   // forward wavefront: task (k, s) at step 2k + s, then Send s -> s+1
    int kk = -st;
    for (int wv = 0; wv < nsteps; wv++) {
      wc.steps++;
      const bool act = ok && (unsigned int)kk < K2 && !(kk & 1);
      const bool rcv = dn && (unsigned int)(kk + 1) < K2 && (kk & 1);
      kk++;
      fwd_task(act);
      const double nbu = __shfl_down_sync(0xffffffffu, clk, Di);
      const double nbd = __shfl_up_sync(0xffffffffu, clk, Di);
      const bool sd = act && up;
      const double nc = dadd(fmax(clk, sd ? nbu : nbd), sd ? sendf : recvf);
      clk = (sd || rcv) ? nc : clk;
    }
  }
  {   // backward wavefront: task (k, s) at step 2k + (P-1-s), then Send s -> s-1
    int kk = -(int)(P - 1 - st);
    for (int wv = 0; wv < nsteps; wv++) {
      wc.steps++;
      const bool act = ok && (unsigned int)kk < K2 && !(kk & 1);
      const bool rcv = up && (unsigned int)(kk + 1) < K2 && (kk & 1);
      kk++;
      bwd_task(act);
      const double nbu = __shfl_down_sync(0xffffffffu, clk, Di);
      const double nbd = __shfl_up_sync(0xffffffffu, clk, Di);
      const bool sd = act && dn;
      const double nc = dadd(fmax(clk, sd ? nbd : nbu), sd ? sendb : recvb);
      clk = (sd || rcv) ? nc : clk;
    }
  }
  }   // GPipe
  // tail: the owner updates its layers (SGD); no DP AllReduce under ZeRO
  if (ok)
    for (int l = lo; l < hi; l++)
      if (own(l)) clk = dadd(clk, sgd);
  ms_out = ok ? clk : 0.0;
  peak_out = ok ? peak : 0;
}
