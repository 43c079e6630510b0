// oracle/distir_oracle.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A plain, slow, single-threaded-per-config CPU DistIR simulator written from
// the paper (arXiv 2111.05426, /root/reference/PAPER.md = "P:<line>") and the
// contract in SURVEY.md §8c (C.1-C.8).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.  It shares
// no code, header, table or constant with paper_2111_05426_b200/ (the CUDA
// path); the two meet only on the data in workloads/.
//
// What it does, literally and in the paper's order:
//   1. builds the EXPLICIT global DistIR program of one configuration: every
//      op of every rank, with its device set, input values and output values
//      (P:276-289 IR; P:301-305 device sets; P:524 D/T/P transform; SURVEY
//      C.3 MLP training under GPipe, C.4 GPT-2 inference);
//   2. gives every op its analytic cost ("N/f"; C.5);
//   3. walks the ops in program order: start = max(clock of members), end =
//      start + cost, members' clocks <- end (C.6);
//   4. tracks live bytes per device, live from creation until last use
//      (C.7), parameters live from t = 0, returned values kept;
//   5. enumerates the grid by nested loops (C.1), flags
//      validity (C.2), filters by capacity and ranks by a full stable
//      sort (C.8).
// No templates, no symmetry, no closed forms, no reordering.
//
// Parity: pinned by tests/test_oracle_*.py (Fig. 3 durations P:226-266,
// 1-rank closed form, GPipe flow-shop closed form, Table 1 grid counts,
// Table 1 MLP parameter bytes, hand-traced peak, brute force on random
// programs).  Build: g++ -std=c++17 -O2 -ffp-contract=off (no FMA contraction,
// C.5 / C.9 A27).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <atomic>
#include <thread>
#include <vector>

namespace {

// ---------------------------------------------------------------- inputs ----
struct Model {          // workloads/ model dict, in this order
  int64_t kind;         // 0 MLP training, 1 GPT-2 inference
  int64_t n_layer, d_model, n_head, seq_len, vocab_pad, n_ctx;
  int64_t dtype_bytes, id_bytes, lm_head;
  int64_t schedule;     // MLP training pipeline schedule: 0 GPipe, 1 1F1B
  // memory-saving variants of the training program (NEXT row f4; Appendix
  // Figs. 8/9): gradient checkpointing and ZeRO-2/3 partitioning
  int64_t recompute;    // 1: discard in-stage activations, recompute in backward
  int64_t zero;         // 1: W_l and its gradient owned by replica l mod D
};
struct Topo {
  int64_t world_max, node_size, capacity;
  double F, o, a_intra, bw_intra, a_inter, bw_inter;
  // cost model (C.5; NEXT row f2): 0 analytic flops/F + o; 1 the paper's
  // linear-regression cost functions, t = c0 + c_flop * flops +
  // c_byte * bytes, one coefficient set for MatMul-type ops, one for the rest
  int64_t cost_model;
  double mm_c0, mm_flop, mm_byte, ew_c0, ew_flop, ew_byte;
};

Model model_from(const int64_t* f) {
  Model m;
  m.kind = f[0]; m.n_layer = f[1]; m.d_model = f[2]; m.n_head = f[3];
  m.seq_len = f[4]; m.vocab_pad = f[5]; m.n_ctx = f[6]; m.dtype_bytes = f[7];
  m.id_bytes = f[8]; m.lm_head = f[9]; m.schedule = f[10];
  m.recompute = f[11]; m.zero = f[12];
  return m;
}
Topo topo_from(const int64_t* i, const double* d) {
  Topo t;
  t.world_max = i[0]; t.node_size = i[1]; t.capacity = i[2];
  t.F = d[0]; t.o = d[1]; t.a_intra = d[2]; t.bw_intra = d[3];
  t.a_inter = d[4]; t.bw_inter = d[5];
  t.cost_model = i[3];
  t.mm_c0 = d[6]; t.mm_flop = d[7]; t.mm_byte = d[8];
  t.ew_c0 = d[9]; t.ew_flop = d[10]; t.ew_byte = d[11];
  return t;
}

// ---------------------------------------------------------- the program ----
// a function is a list of ops over SSA values.
enum Cls { COMPUTE = 0, SEND = 1, ALLREDUCE = 2, ALLGATHER = 3, BROADCAST = 4, REDUCE = 5 };

struct Value {
  int dev;          // the device the value lives on (P:410 type carries device)
  int64_t bytes;    // elements x element bytes
  bool param;       // function parameter: live from t = 0 (C.7)
  bool returned;    // returned values are never freed (C.7)
};

struct Op {
  Cls cls;
  std::vector<int> devs;   // device set
  std::vector<int> in, out;
  int64_t work;            // FLOPs (compute) or bytes (communication)
  double cost;             // seconds (C.5)
  bool mm = false;         // MatMul-type compute op (Gemm / MatMul / MatMulGrad)
};

struct Program {
  int n_dev = 0;
  std::vector<Value> vals;
  std::vector<Op> ops;
  int new_val(int dev, int64_t bytes, bool param = false, bool ret = false) {
    vals.push_back(Value{dev, bytes, param, ret});
    return (int)vals.size() - 1;
  }
};

// ------------------------------------------------------------ cost model ----
// C.5: the link class of a group is intra iff every member shares
// floor(rank / node_size).
bool intra(const Topo& t, const std::vector<int>& devs) {
  for (int d : devs)
    if (d / t.node_size != devs[0] / t.node_size) return false;
  return true;
}

double op_cost(const Topo& t, const Program& pr, const Op& op) {
  if (op.cls == COMPUTE && t.cost_model == 1) {
    // "linear regression models in terms of the sizes of the
    // input tensors" for MatMul, analytic-style ones for the rest; the
    // features are the op's FLOPs and the bytes of every tensor it reads or
    // writes (its typed inputs and outputs), evaluated left to right.
    int64_t bytes = 0;
    for (int v : op.in) bytes += pr.vals[v].bytes;
    for (int v : op.out) bytes += pr.vals[v].bytes;
    const double c0 = op.mm ? t.mm_c0 : t.ew_c0;
    const double cf = op.mm ? t.mm_flop : t.ew_flop;
    const double cb = op.mm ? t.mm_byte : t.ew_byte;
    return (c0 + cf * (double)op.work) + cb * (double)bytes;
  }
  if (op.cls == COMPUTE)  // P:487 "N / f", plus the fixed overhead o
    return ((double)op.work) / t.F + t.o;
  const bool in_node = intra(t, op.devs);
  const double a = in_node ? t.a_intra : t.a_inter;
  const double bw = in_node ? t.bw_intra : t.bw_inter;
  const int64_t g = (int64_t)op.devs.size();
  if (op.cls == SEND)  // alpha-beta
    return a + ((double)op.work) / bw;
  if (op.cls == ALLREDUCE)  // ring: 2(g-1) steps of bytes/g
    return ((double)(2 * (g - 1))) * a +
           (((double)(2 * (g - 1))) / ((double)g)) * (((double)op.work) / bw);
  if (op.cls == ALLGATHER)  // ring: (g-1) steps; work = gathered bytes
    return ((double)(g - 1)) * a +
           (((double)(g - 1)) / ((double)g)) * (((double)op.work) / bw);
  // BROADCAST from the owner / REDUCE to the owner (ZeRO, Fig. 9):
  // a pipelined chain over the g members, (g-1) hops of latency and the
  // whole tensor once over a link; g = 2 is exactly a Send (Fig. 9 sends
  // w1, w2 between its two devices).  DESIGN reading R9.
  return ((double)(g - 1)) * a + ((double)op.work) / bw;
}

// ------------------------------------------------ C.3 MLP training, GPipe ---
struct Cfg { int64_t D, T, P, K, B; };

int64_t rank_of(const Cfg& c, int64_t i, int64_t j, int64_t s) {
  return j + c.T * (i + c.D * s);  // C.3 rank layout (C.9 A19)
}

Program build_mlp(const Model& M, const Cfg& c) {
  Program pr;
  const int64_t L = M.n_layer, d = M.d_model, e = M.dtype_bytes;
  const int64_t D = c.D, T = c.T, P = c.P, K = c.K;
  const int64_t m = c.B / (D * K);      // microbatch size per replica
  const int64_t W = D * T * P;
  pr.n_dev = (int)W;
  enum { FULL, COL, ROW };
  auto mode = [&](int64_t l) { return T == 1 ? FULL : (l % 2 == 0 ? COL : ROW); };
  auto k_in = [&](int64_t l) { return mode(l) == ROW ? d / T : d; };
  auto n_out = [&](int64_t l) { return mode(l) == COL ? d / T : d; };
  auto d_out = [&](int64_t l) { return mode(l) == COL ? d / T : d; };
  auto lo = [&](int64_t s) { return (s * L) / P; };  // balanced split (C.2)
  auto stage_ranks = [&](int64_t s) {
    std::vector<int> r;
    for (int64_t i = 0; i < D; i++)
      for (int64_t j = 0; j < T; j++) r.push_back((int)rank_of(c, i, j, s));
    return r;  // ascending
  };
  auto stage_of = [&](int r) { return (int64_t)r / (D * T); };
  auto emit = [&](Cls cls, std::vector<int> devs, std::vector<int> in,
                  std::vector<int> out, int64_t work, bool mm = false) {
    pr.ops.push_back(Op{cls, std::move(devs), std::move(in), std::move(out), work, 0.0, mm});
  };
  // NEXT row f4 (Appendix; DESIGN readings R8/R9).
  // Gradient checkpointing (Fig. 8): a stage keeps its input and output
  // activations; the activations inside the stage die after their forward
  // use and are recomputed at the start of the stage's backward (after
  // LossGrad, as as_b follows dp in Fig. 8).
  const bool ckpt = M.recompute != 0;
  // ZeRO-2/3 (Fig. 9): W_l and its gradient belong to replica l mod D of the
  // layer's (j, s) group; the owner broadcasts W_l before each forward and
  // backward use (w2_1_f, w2_1_b), the replicas' gradients are reduced to the
  // owner after the stage's backward (MPIReduce dw1, dw2), which accumulates
  // and updates them alone.  With D = 1 the owner is the only replica.
  const bool zero = M.zero != 0 && D > 1;
  auto owner = [&](int64_t l) { return l % D; };
  auto replica_of = [&](int r) { return ((int64_t)r / T) % D; };
  auto wbytes = [&](int64_t l) { return k_in(l) * n_out(l) * e; };

  // Parameters (C.3): W_l and a zero gradient buffer G_l per local layer
  // (ZeRO: on the owner only); X_k on stage 0, Y_k on stage P-1.
  std::vector<int> Wv(W * L, -1), Gv(W * L, -1), X(W * K, -1), Y(W * K, -1);
  for (int r = 0; r < W; r++) {
    int64_t s = stage_of(r);
    for (int64_t l = lo(s); l < lo(s + 1); l++) {
      if (zero && replica_of(r) != owner(l)) continue;
      Wv[r * L + l] = pr.new_val(r, wbytes(l), true);
      Gv[r * L + l] = pr.new_val(r, wbytes(l), true);
    }
    for (int64_t k = 0; k < K; k++) {
      if (s == 0) X[r * K + k] = pr.new_val(r, m * d * e, true);
      if (s == P - 1) Y[r * K + k] = pr.new_val(r, m * d_out(L - 1) * e, true);
    }
  }
  // the weight of layer l each rank of stage s reads: its own, or (ZeRO) a
  // copy broadcast from the owner of its (*, j, s) group just before use
  auto weights = [&](int64_t l, int64_t s) {
    std::vector<int> Wu(W, -1);
    if (!zero) {
      for (int r : stage_ranks(s)) Wu[r] = Wv[r * L + l];
      return Wu;
    }
    for (int64_t j = 0; j < T; j++) {
      std::vector<int> g, out;
      const int src = (int)rank_of(c, owner(l), j, s);
      for (int64_t i = 0; i < D; i++) {
        const int r = (int)rank_of(c, i, j, s);
        g.push_back(r);
        if (r == src) { Wu[r] = Wv[r * L + l]; continue; }
        const int v = pr.new_val(r, wbytes(l));
        out.push_back(v);
        Wu[r] = v;
      }
      emit(BROADCAST, g, {Wv[src * L + l]}, out, wbytes(l));
    }
    return Wu;
  };
  // acts[(k*W + r)*(L+1) + l] = input activation of layer l (output of l-1);
  // racts: the same for activations recomputed in backward (checkpointing).
  std::vector<int> acts(K * W * (L + 1), -1), racts(K * W * (L + 1), -1);
  auto act = [&](int64_t k, int r, int64_t l) -> int& { return acts[(k * W + r) * (L + 1) + l]; };
  auto ract = [&](int64_t k, int r, int64_t l) -> int& { return racts[(k * W + r) * (L + 1) + l]; };
  std::vector<int> fwd_recv(K * W, -1), bwd_recv(K * W, -1);

  // one forward layer on stage s: [ZeRO Broadcast], MatMul, [TP AllReduce
  // if row], Relu; A[r] = input activation, replaced by the output
  auto fwd_layer = [&](int64_t s, int64_t l, std::vector<int>& A) {
    std::vector<int> R = stage_ranks(s);
    std::vector<int> Wu = weights(l, s);
    std::vector<int> Z(W, -1);
    for (int r : R) {
      Z[r] = pr.new_val(r, m * n_out(l) * e);
      emit(COMPUTE, {r}, {A[r], Wu[r]}, {Z[r]}, 2 * m * k_in(l) * n_out(l), true);
    }
    if (mode(l) == ROW) {  // partial sums -> TP AllReduce over (i, *, s)
      for (int64_t i = 0; i < D; i++) {
        std::vector<int> g, in, out;
        for (int64_t j = 0; j < T; j++) {
          int r = (int)rank_of(c, i, j, s);
          int z2 = pr.new_val(r, m * d * e);
          g.push_back(r); in.push_back(Z[r]); out.push_back(z2); Z[r] = z2;
        }
        emit(ALLREDUCE, g, in, out, m * d * e);
      }
    }
    for (int r : R) {
      int a = pr.new_val(r, m * d_out(l) * e);
      emit(COMPUTE, {r}, {Z[r]}, {a}, m * d_out(l));  // Relu
      A[r] = a;
    }
  };

  // ---- the four kinds of pipeline events of one microbatch k on stage s
  auto fwd_task = [&](int64_t k, int64_t s) {        // per layer: MatMul, [TP AllReduce], Relu
    std::vector<int> A(W, -1);
    for (int r : stage_ranks(s)) {
      A[r] = (s == 0) ? X[r * K + k] : fwd_recv[k * W + r];
      act(k, r, lo(s)) = A[r];
    }
    for (int64_t l = lo(s); l < lo(s + 1); l++) {
      fwd_layer(s, l, A);
      for (int r : stage_ranks(s)) act(k, r, l + 1) = A[r];
    }
  };
  auto fwd_send = [&](int64_t k, int64_t s) {        // stage s -> s+1
    for (int r : stage_ranks(s)) {
      int dst = r + (int)(T * D);
      int64_t bytes = m * d_out(lo(s + 1) - 1) * e;
      int v = pr.new_val(dst, bytes);
      emit(SEND, {r, dst}, {act(k, r, lo(s + 1))}, {v}, bytes);
      fwd_recv[k * W + dst] = v;
    }
  };
  std::vector<int> Gcur = Gv;
  std::vector<int> bwd_out(K * W, -1);                // dA leaving stage s (first layer)
  auto bwd_task = [&](int64_t k, int64_t s) {        // [LossGrad], [recompute], per layer desc
    std::vector<int> R = stage_ranks(s);
    std::vector<int> dA(W, -1);
    for (int r : R) {
      if (s == P - 1) {  // LossGrad (MSE gradient, C.9 A22)
        dA[r] = pr.new_val(r, m * d_out(L - 1) * e);
        emit(COMPUTE, {r}, {act(k, r, L), Y[r * K + k]}, {dA[r]}, 3 * m * d_out(L - 1));
      } else {
        dA[r] = bwd_recv[k * W + r];
      }
    }
    // checkpointing: recompute the activations inside the stage
    auto a_in = [&](int r, int64_t l) { return (ckpt && l > lo(s)) ? ract(k, r, l) : act(k, r, l); };
    auto a_out = [&](int r, int64_t l) {
      return (ckpt && l + 1 < lo(s + 1)) ? ract(k, r, l + 1) : act(k, r, l + 1);
    };
    if (ckpt) {
      std::vector<int> A(W, -1);
      for (int r : R) A[r] = act(k, r, lo(s));
      for (int64_t l = lo(s); l + 1 < lo(s + 1); l++) {
        fwd_layer(s, l, A);
        for (int r : R) ract(k, r, l + 1) = A[r];
      }
    }
    std::vector<std::vector<int>> pend(L);            // ZeRO: gradients to reduce
    for (int64_t l = lo(s + 1) - 1; l >= lo(s); l--) {
      std::vector<int> Wu = weights(l, s);
      std::vector<int> dZ(W, -1), dW(W, -1);
      for (int r : R) {  // ReluGrad
        dZ[r] = pr.new_val(r, m * d_out(l) * e);
        emit(COMPUTE, {r}, {a_out(r, l), dA[r]}, {dZ[r]}, m * d_out(l));
      }
      for (int r : R) {  // MatMulGrad -> (dA_l, dW_l)
        int da = pr.new_val(r, m * k_in(l) * e);
        dW[r] = pr.new_val(r, wbytes(l));
        emit(COMPUTE, {r}, {a_in(r, l), Wu[r], dZ[r]}, {da, dW[r]},
             4 * m * k_in(l) * n_out(l), true);
        dA[r] = da;
      }
      if (mode(l) == COL) {  // partial dA_l (m x d) -> TP AllReduce
        for (int64_t i = 0; i < D; i++) {
          std::vector<int> g, in, out;
          for (int64_t j = 0; j < T; j++) {
            int r = (int)rank_of(c, i, j, s);
            int v = pr.new_val(r, m * d * e);
            g.push_back(r); in.push_back(dA[r]); out.push_back(v); dA[r] = v;
          }
          emit(ALLREDUCE, g, in, out, m * d * e);
        }
      }
      if (zero) { pend[l] = dW; continue; }
      for (int r : R) {  // gradient accumulation (C.9 A20)
        int gn = pr.new_val(r, wbytes(l));
        emit(COMPUTE, {r}, {Gcur[r * L + l], dW[r]}, {gn}, k_in(l) * n_out(l));
        Gcur[r * L + l] = gn;
      }
    }
    if (zero) {  // reduce each layer's gradient to its owner, who accumulates it
      for (int64_t l = lo(s); l < lo(s + 1); l++) {
        std::vector<int> red(W, -1);
        for (int64_t j = 0; j < T; j++) {
          std::vector<int> g, in;
          const int dst = (int)rank_of(c, owner(l), j, s);
          for (int64_t i = 0; i < D; i++) {
            const int r = (int)rank_of(c, i, j, s);
            g.push_back(r); in.push_back(pend[l][r]);
          }
          red[dst] = pr.new_val(dst, wbytes(l));
          emit(REDUCE, g, in, {red[dst]}, wbytes(l));
        }
        for (int64_t j = 0; j < T; j++) {
          const int o = (int)rank_of(c, owner(l), j, s);
          int gn = pr.new_val(o, wbytes(l));
          emit(COMPUTE, {o}, {Gcur[o * L + l], red[o]}, {gn}, k_in(l) * n_out(l));
          Gcur[o * L + l] = gn;
        }
      }
    }
    for (int r : R) bwd_out[k * W + r] = dA[r];
  };
  auto bwd_send = [&](int64_t k, int64_t s) {        // stage s -> s-1
    for (int r : stage_ranks(s)) {
      int dst = r - (int)(T * D);
      int64_t bytes = m * k_in(lo(s)) * e;
      int v = pr.new_val(dst, bytes);
      emit(SEND, {r, dst}, {bwd_out[k * W + r]}, {v}, bytes);
      bwd_recv[k * W + dst] = v;
    }
  };

  if (M.schedule == 0) {
    // GPipe (north_star; C.3): all forwards microbatch-major, then all
    // backwards.
    for (int64_t k = 0; k < K; k++)
      for (int64_t s = 0; s < P; s++) {
        fwd_task(k, s);
        if (s < P - 1) fwd_send(k, s);
      }
    for (int64_t k = 0; k < K; k++)
      for (int64_t s = P - 1; s >= 0; s--) {
        bwd_task(k, s);
        if (s > 0) bwd_send(k, s);
      }
  } else {
    // Synchronous 1F1B (PipeDream-flush): stage s runs w_s =
    // min(P-1-s, K) warm-up forwards, then alternates F(w_s + i), B(i), then
    // the remaining backwards.  The global program order (DESIGN reading R6)
    // is the order of the unit-time schedule of these per-stage sequences
    // (F and B take one unit, a task waits for its stage and for its
    // producer on the neighbour stage): ops sorted by time, each Send at the
    // time its producer finishes, Sends before tasks at equal times, Sends by
    // lower stage of the pair then forward-before-backward, tasks by stage.
    // For P = K = 2 this is exactly the program of Fig. 2/3.
    struct Ev { int64_t t; int cls; int64_t key, kind, k, s; };
    std::vector<std::vector<std::pair<int, int64_t>>> seq(P);   // (0 = F / 1 = B, k)
    for (int64_t s = 0; s < P; s++) {
      const int64_t w = std::min<int64_t>(P - 1 - s, K);
      for (int64_t k = 0; k < w; k++) seq[s].push_back({0, k});
      for (int64_t i = 0; i < K - w; i++) { seq[s].push_back({0, w + i}); seq[s].push_back({1, i}); }
      for (int64_t k = K - w; k < K; k++) seq[s].push_back({1, k});
    }
    // unit-time schedule by relaxation over the per-stage sequences
    std::vector<int64_t> endF(K * P, -1), endB(K * P, -1);
    std::vector<Ev> ev;
    std::vector<size_t> ptr(P, 0);
    std::vector<int64_t> freeT(P, 0);
    bool progress = true;
    while (progress) {
      progress = false;
      for (int64_t s = 0; s < P; s++) {
        while (ptr[s] < seq[s].size()) {
          const int kind = seq[s][ptr[s]].first;
          const int64_t k = seq[s][ptr[s]].second;
          int64_t dep = 0;
          if (kind == 0 && s > 0) { if (endF[k * P + s - 1] < 0) break; dep = endF[k * P + s - 1]; }
          if (kind == 1 && s < P - 1) { if (endB[k * P + s + 1] < 0) break; dep = endB[k * P + s + 1]; }
          const int64_t st = std::max(freeT[s], dep);
          (kind == 0 ? endF : endB)[k * P + s] = st + 1;
          freeT[s] = st + 1;
          ev.push_back(Ev{st, 1, s, kind, k, s});                       // the task
          if (kind == 0 && s < P - 1) ev.push_back(Ev{st + 1, 0, s, 0, k, s});      // F send
          if (kind == 1 && s > 0) ev.push_back(Ev{st + 1, 0, s - 1, 1, k, s});      // B send
          ptr[s]++;
          progress = true;
        }
      }
    }
    std::stable_sort(ev.begin(), ev.end(), [](const Ev& x, const Ev& y) {
      if (x.t != y.t) return x.t < y.t;
      if (x.cls != y.cls) return x.cls < y.cls;
      if (x.key != y.key) return x.key < y.key;
      return x.kind < y.kind;
    });
    for (const Ev& v : ev) {
      if (v.cls == 1) {
        if (v.kind == 0) fwd_task(v.k, v.s); else bwd_task(v.k, v.s);
      } else {
        if (v.kind == 0) fwd_send(v.k, v.s); else bwd_send(v.k, v.s);
      }
    }
  }
  // Tail: DP AllReduce of the accumulated gradients, then SGD (C.9 A23);
  // ZeRO: the owner updates its layers alone (w1_new, w2_new of Fig. 9).
  for (int64_t s = P - 1; s >= 0; s--) {
    std::vector<int> R = stage_ranks(s);
    if (D > 1 && !zero) {
      for (int64_t l = lo(s + 1) - 1; l >= lo(s); l--) {
        for (int64_t j = 0; j < T; j++) {
          std::vector<int> g, in, out;
          for (int64_t i = 0; i < D; i++) {
            int r = (int)rank_of(c, i, j, s);
            int v = pr.new_val(r, wbytes(l));
            g.push_back(r); in.push_back(Gcur[r * L + l]); out.push_back(v);
            Gcur[r * L + l] = v;
          }
          emit(ALLREDUCE, g, in, out, wbytes(l));
        }
      }
    }
    for (int64_t l = lo(s); l < lo(s + 1); l++) {
      for (int r : R) {
        if (zero && replica_of(r) != owner(l)) continue;
        int wn = pr.new_val(r, wbytes(l), false, true);  // returned
        emit(COMPUTE, {r}, {Wv[r * L + l], Gcur[r * L + l]}, {wn}, 2 * k_in(l) * n_out(l));
      }
    }
  }
  return pr;
}

// ---------------------------------------------- C.4 GPT-2 inference, GPipe --
Program build_gpt2(const Model& M, const Cfg& c) {
  Program pr;
  const int64_t L = M.n_layer, d = M.d_model, h = M.n_head, S = M.seq_len;
  const int64_t V = M.vocab_pad, e = M.dtype_bytes, ide = M.id_bytes;
  const int64_t D = c.D, T = c.T, P = c.P, K = c.K;
  const int64_t m = c.B / (D * K);
  const int64_t n = m * S;             // tokens per microbatch
  const int64_t dT = d / T, hT = h / T, VT = V / T;
  const int64_t W = D * T * P;
  pr.n_dev = (int)W;
  auto lo = [&](int64_t s) { return (s * L) / P; };
  auto stage_ranks = [&](int64_t s) {
    std::vector<int> r;
    for (int64_t i = 0; i < D; i++)
      for (int64_t j = 0; j < T; j++) r.push_back((int)rank_of(c, i, j, s));
    return r;
  };
  auto stage_of = [&](int r) { return (int64_t)r / (D * T); };
  auto emit = [&](Cls cls, std::vector<int> devs, std::vector<int> in,
                  std::vector<int> out, int64_t work, bool mm = false) {
    pr.ops.push_back(Op{cls, std::move(devs), std::move(in), std::move(out), work, 0.0, mm});
  };
  // Per-block parameters (Megatron shards; C.4), one value per tensor.
  enum { LN1 = 0, WQKV, BQKV, WPROJ, BPROJ, LN2, WFC1, BFC1, WFC2, BFC2, NPB };
  const int64_t pbytes[NPB] = {2 * d * e, d * 3 * dT * e, 3 * dT * e, dT * d * e, d * e,
                               2 * d * e, d * 4 * dT * e, 4 * dT * e, 4 * dT * d * e, d * e};
  std::vector<int> bp(W * L * NPB, -1);
  auto bpar = [&](int r, int64_t l, int which) { return bp[(r * L + l) * NPB + which]; };
  std::vector<int> wte(W, -1), wpe(W, -1), wte_last(W, -1), lnf(W, -1), ids(W * K, -1);
  for (int r = 0; r < W; r++) {
    int64_t s = stage_of(r);
    for (int64_t l = lo(s); l < lo(s + 1); l++)
      for (int q = 0; q < NPB; q++) bp[(r * L + l) * NPB + q] = pr.new_val(r, pbytes[q], true);
    if (s == 0) {
      wte[r] = pr.new_val(r, VT * d * e, true);
      wpe[r] = pr.new_val(r, M.n_ctx * d * e, true);
      for (int64_t k = 0; k < K; k++) ids[r * K + k] = pr.new_val(r, n * ide, true);
    }
    if (s == P - 1) {
      lnf[r] = pr.new_val(r, 2 * d * e, true);
      if (M.lm_head) wte_last[r] = (P == 1) ? wte[r] : pr.new_val(r, VT * d * e, true);
    }
  }
  std::vector<int> recv(K * W, -1);
  auto tp_allreduce = [&](int64_t s, std::vector<int>& x, int64_t bytes) {
    for (int64_t i = 0; i < D; i++) {
      std::vector<int> g, in, out;
      for (int64_t j = 0; j < T; j++) {
        int r = (int)rank_of(c, i, j, s);
        int v = pr.new_val(r, bytes);
        g.push_back(r); in.push_back(x[r]); out.push_back(v); x[r] = v;
      }
      emit(ALLREDUCE, g, in, out, bytes);
    }
  };
  for (int64_t k = 0; k < K; k++) {
    for (int64_t s = 0; s < P; s++) {
      std::vector<int> R = stage_ranks(s);
      std::vector<int> x(W, -1);
      if (s == 0) {  // prologue: vocab-parallel embedding
        for (int r : R) {
          x[r] = pr.new_val(r, n * d * e);
          emit(COMPUTE, {r}, {ids[r * K + k], wte[r], wpe[r]}, {x[r]}, 2 * n * d);
        }
        if (T > 1) tp_allreduce(s, x, n * d * e);
      } else {
        for (int r : R) x[r] = recv[k * W + r];
      }
      for (int64_t l = lo(s); l < lo(s + 1); l++) {
        std::vector<int> h1(W), qkv(W), sc(W), pb(W), ctx(W), o(W), x2(W), h2(W), f(W), g(W), f2(W), x3(W);
        for (int r : R) {  // 1 LayerNorm ln_1
          h1[r] = pr.new_val(r, n * d * e);
          emit(COMPUTE, {r}, {x[r], bpar(r, l, LN1)}, {h1[r]}, 5 * n * d);
        }
        for (int r : R) {  // 2 Gemm QKV (column parallel)
          qkv[r] = pr.new_val(r, n * 3 * dT * e);
          emit(COMPUTE, {r}, {h1[r], bpar(r, l, WQKV), bpar(r, l, BQKV)}, {qkv[r]},
               2 * n * d * (3 * dT) + n * (3 * dT), true);
        }
        for (int r : R) {  // 3 attention scores
          sc[r] = pr.new_val(r, m * hT * S * S * e);
          emit(COMPUTE, {r}, {qkv[r]}, {sc[r]}, 2 * m * S * S * dT, true);
        }
        for (int r : R) {  // 4 softmax
          pb[r] = pr.new_val(r, m * hT * S * S * e);
          emit(COMPUTE, {r}, {sc[r]}, {pb[r]}, 5 * m * hT * S * S);
        }
        for (int r : R) {  // 5 attention context
          ctx[r] = pr.new_val(r, n * dT * e);
          emit(COMPUTE, {r}, {pb[r], qkv[r]}, {ctx[r]}, 2 * m * S * S * dT, true);
        }
        for (int r : R) {  // 6 Gemm proj (row parallel) -> partial
          o[r] = pr.new_val(r, n * d * e);
          emit(COMPUTE, {r}, {ctx[r], bpar(r, l, WPROJ), bpar(r, l, BPROJ)}, {o[r]},
               2 * n * dT * d + n * d, true);
        }
        if (T > 1) tp_allreduce(s, o, n * d * e);  // 7
        for (int r : R) {  // 8 residual add
          x2[r] = pr.new_val(r, n * d * e);
          emit(COMPUTE, {r}, {x[r], o[r]}, {x2[r]}, n * d);
        }
        for (int r : R) {  // 9 LayerNorm ln_2
          h2[r] = pr.new_val(r, n * d * e);
          emit(COMPUTE, {r}, {x2[r], bpar(r, l, LN2)}, {h2[r]}, 5 * n * d);
        }
        for (int r : R) {  // 10 Gemm FC1 (column parallel)
          f[r] = pr.new_val(r, n * 4 * dT * e);
          emit(COMPUTE, {r}, {h2[r], bpar(r, l, WFC1), bpar(r, l, BFC1)}, {f[r]},
               2 * n * d * (4 * dT) + n * (4 * dT), true);
        }
        for (int r : R) {  // 11 GeLU
          g[r] = pr.new_val(r, n * 4 * dT * e);
          emit(COMPUTE, {r}, {f[r]}, {g[r]}, 8 * n * (4 * dT));
        }
        for (int r : R) {  // 12 Gemm FC2 (row parallel) -> partial
          f2[r] = pr.new_val(r, n * d * e);
          emit(COMPUTE, {r}, {g[r], bpar(r, l, WFC2), bpar(r, l, BFC2)}, {f2[r]},
               2 * n * (4 * dT) * d + n * d, true);
        }
        if (T > 1) tp_allreduce(s, f2, n * d * e);  // 13
        for (int r : R) {  // 14 residual add
          x3[r] = pr.new_val(r, n * d * e);
          emit(COMPUTE, {r}, {x2[r], f2[r]}, {x3[r]}, n * d);
        }
        for (int r : R) x[r] = x3[r];
      }
      if (s == P - 1) {  // epilogue
        for (int r : R) {
          int hf = pr.new_val(r, n * d * e, false, M.lm_head == 0);
          emit(COMPUTE, {r}, {x[r], lnf[r]}, {hf}, 5 * n * d);
          x[r] = hf;
        }
        if (M.lm_head) {
          for (int r : R) {  // vocab-parallel LM head (tied wte shard)
            int lg = pr.new_val(r, n * VT * e, false, T == 1);
            emit(COMPUTE, {r}, {x[r], wte_last[r]}, {lg}, 2 * n * d * VT, true);
            x[r] = lg;
          }
          if (T > 1) {  // gather the logits on every TP rank
            for (int64_t i = 0; i < D; i++) {
              std::vector<int> gr, in, out;
              for (int64_t j = 0; j < T; j++) {
                int r = (int)rank_of(c, i, j, s);
                int v = pr.new_val(r, n * V * e, false, true);
                gr.push_back(r); in.push_back(x[r]); out.push_back(v);
              }
              emit(ALLGATHER, gr, in, out, n * V * e);
            }
          }
        }
      } else {
        for (int r : R) {
          int dst = r + (int)(T * D);
          int v = pr.new_val(dst, n * d * e);
          emit(SEND, {r, dst}, {x[r]}, {v}, n * d * e);
          recv[k * W + dst] = v;
        }
      }
    }
  }
  return pr;
}

// --------------------------------------------------- C.6 + C.7 simulate ----
struct SimOut {
  double makespan = 0.0;
  std::vector<double> clock;       // per device, final
  std::vector<int64_t> peak, live; // per device
  bool ready_ok = true;            // ready <= start for every op (C.6 check)
  bool placement_ok = true;        // compute ops on one device with local values
};

SimOut simulate(const Program& pr, std::vector<double>* op_start = nullptr,
                std::vector<double>* op_end = nullptr) {
  const int nd = pr.n_dev;
  const size_t nv = pr.vals.size();
  SimOut r;
  // last_use(v): last op in program order that reads v (reverse scan, C.7).
  std::vector<int64_t> last_use(nv, -1);
  for (int64_t i = (int64_t)pr.ops.size() - 1; i >= 0; i--)
    for (int v : pr.ops[i].in)
      if (last_use[v] < 0) last_use[v] = i;
  std::vector<double> ready(nv, 0.0);
  r.clock.assign(nd, 0.0);
  r.live.assign(nd, 0);
  for (const Value& v : pr.vals)
    if (v.param) r.live[v.dev] += v.bytes;  // parameters live from t = 0
  r.peak = r.live;
  if (op_start) op_start->assign(pr.ops.size(), 0.0);
  if (op_end) op_end->assign(pr.ops.size(), 0.0);
  std::vector<int> seen;
  for (size_t i = 0; i < pr.ops.size(); i++) {
    const Op& op = pr.ops[i];
    // placement: a compute op runs where all its values live.
    if (op.cls == COMPUTE) {
      for (int v : op.in) if (pr.vals[v].dev != op.devs[0]) r.placement_ok = false;
      for (int v : op.out) if (pr.vals[v].dev != op.devs[0]) r.placement_ok = false;
    }
    // time (C.6): wait until every member device is free.
    double start = 0.0;
    for (int d : op.devs) start = std::max(start, r.clock[d]);
    double rdy = 0.0;
    for (int v : op.in) rdy = std::max(rdy, ready[v]);
    if (rdy > start) r.ready_ok = false;
    const double end = start + op.cost;
    for (int d : op.devs) r.clock[d] = end;
    for (int v : op.out) ready[v] = end;
    if (op_start) (*op_start)[i] = start;
    if (op_end) (*op_end)[i] = end;
    // memory (C.7): allocate outputs, record peaks, free last uses.
    for (int v : op.out) r.live[pr.vals[v].dev] += pr.vals[v].bytes;
    for (int d : op.devs) r.peak[d] = std::max(r.peak[d], r.live[d]);
    seen.clear();
    for (int v : op.in) {
      if (std::find(seen.begin(), seen.end(), v) != seen.end()) continue;
      seen.push_back(v);
      if (last_use[v] == (int64_t)i && !pr.vals[v].returned) r.live[pr.vals[v].dev] -= pr.vals[v].bytes;
    }
    for (int v : op.out)
      if (last_use[v] < 0 && !pr.vals[v].returned) r.live[pr.vals[v].dev] -= pr.vals[v].bytes;
  }
  for (double c : r.clock) r.makespan = std::max(r.makespan, c);
  return r;
}

// ------------------------------------------------------ C.2 validity bits --
enum {
  R_BATCH = 1u << 0,     // B mod (D*K) != 0
  R_STAGES = 1u << 1,    // P > n_layer (an empty stage)
  R_TP_DIM = 1u << 2,    // d (or the padded vocab) not divisible by T
  R_TP_HEADS = 1u << 3,  // GPT-2: heads not divisible by T
  R_WORLD = 1u << 4,     // W > topology world_max
  R_CAPACITY = 1u << 5,  // valid but peak > capacity
};

uint32_t validity(const Model& M, const Topo& t, const Cfg& c) {
  uint32_t r = 0;
  if (c.B % (c.D * c.K) != 0) r |= R_BATCH;
  if (c.P > M.n_layer) r |= R_STAGES;
  if (M.d_model % c.T != 0) r |= R_TP_DIM;
  if (M.kind == 1 && M.vocab_pad % c.T != 0) r |= R_TP_DIM;
  if (M.kind == 1 && M.n_head % c.T != 0) r |= R_TP_HEADS;
  if (c.D * c.T * c.P > t.world_max) r |= R_WORLD;
  return r;
}

struct Result {
  double makespan;
  int64_t peak;
  uint32_t reason;
  int64_t n_ops;
};

Result eval_config(const Model& M, const Topo& t, const Cfg& c,
                   std::vector<int64_t>* peaks = nullptr,
                   std::vector<double>* clocks = nullptr, int* err = nullptr) {
  Result res{std::numeric_limits<double>::infinity(), -1, validity(M, t, c), 0};
  if (res.reason) return res;
  Program pr = (M.kind == 0) ? build_mlp(M, c) : build_gpt2(M, c);
  for (Op& op : pr.ops) op.cost = op_cost(t, pr, op);
  SimOut so = simulate(pr);
  if (err && (!so.ready_ok || !so.placement_ok)) *err = 1;
  res.makespan = so.makespan;
  res.peak = 0;
  for (int64_t p : so.peak) res.peak = std::max(res.peak, p);
  res.n_ops = (int64_t)pr.ops.size();
  if (res.peak > t.capacity) res.reason |= R_CAPACITY;
  if (peaks) *peaks = so.peak;
  if (clocks) *clocks = so.clock;
  return res;
}

// ------------------------------------------------------- C.1 enumeration ---
struct Spec {
  std::vector<Model> models;   // candidate models (handle table)
  std::vector<Topo> topos;
  std::vector<int64_t> model_ids, topo_ids, world, batch, k_set;
  int64_t k_mode = 0, dp_mask = 0xFF, tp_mask = 0xFF, pp_mask = 0xFF;
  uint64_t synth_seed = 0;
  int64_t synth_count = 0;
};

struct Decoded {
  Model M;
  int64_t model_slot, topo_slot;  // spec positions (synth: model_slot = -1)
  Cfg c;
};

int ilog2(int64_t x) { int e = 0; while ((int64_t(1) << (e + 1)) <= x) e++; return e; }

std::vector<Cfg> triples(const Spec& sp, int64_t W) {
  std::vector<Cfg> out;
  for (int64_t D = 1; D <= W; D *= 2)
    for (int64_t T = 1; D * T <= W; T *= 2) {
      int64_t P = W / (D * T);
      if (D * T * P != W) continue;
      if (!((sp.dp_mask >> ilog2(D)) & 1) || !((sp.tp_mask >> ilog2(T)) & 1) ||
          !((sp.pp_mask >> ilog2(P)) & 1))
        continue;
      out.push_back(Cfg{D, T, P, 0, 0});
    }
  return out;  // lexicographic in (D, T, P)
}

// Counter-based generator for the synthetic sweep, written
// independently of the CUDA enumerator.
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

Decoded synth(const Spec& sp, int64_t index) {
  uint64_t r[8];
  for (int t = 0; t < 8; t++)
    r[t] = mix64(sp.synth_seed + 0x9E3779B97F4A7C15ull * (uint64_t)(8 * index + t + 1));
  Decoded dc;
  const int64_t kind = (int64_t)(r[0] & 1);
  const int64_t W = int64_t(1) << (r[1] % 7);
  // all power-of-two triples of W, lexicographic
  std::vector<Cfg> tr;
  for (int64_t D = 1; D <= W; D *= 2)
    for (int64_t T = 1; D * T <= W; T *= 2) tr.push_back(Cfg{D, T, W / (D * T), 0, 0});
  Cfg c = tr[r[2] % tr.size()];
  c.K = (c.P == 1) ? 1 : (int64_t(1) << (1 + r[3] % 5));
  c.B = int64_t(1) << (7 + r[4] % 12);
  Model M;
  static const int64_t HF[4][3] = {{12, 768, 12}, {24, 1024, 16}, {36, 1280, 20}, {48, 1600, 25}};
  if (kind == 0) {
    M = Model{0, int64_t(1) << (1 + r[5] % 6), int64_t(1) << (8 + r[6] % 7), 1, 1, 0, 0, 2, 8, 0, 0};
  } else {
    const int64_t* hf = HF[r[5] % 4];
    M = Model{1, hf[0], hf[1], hf[2], 8, 50304, 1024, 2, 8, 1, 0};
  }
  dc.M = M;
  dc.model_slot = -1;
  dc.topo_slot = (int64_t)(r[7] % sp.topo_ids.size());
  dc.c = c;
  return dc;
}

// Nested-loop enumeration in the canonical order (C.1); returns all configs.
std::vector<Decoded> enumerate(const Spec& sp) {
  std::vector<Decoded> out;
  if (sp.synth_count > 0) {
    for (int64_t i = 0; i < sp.synth_count; i++) out.push_back(synth(sp, i));
    return out;
  }
  for (size_t mi = 0; mi < sp.model_ids.size(); mi++)
    for (size_t ti = 0; ti < sp.topo_ids.size(); ti++)
      for (int64_t W : sp.world)
        for (Cfg c : triples(sp, W)) {
          std::vector<int64_t> ks;
          if (sp.k_mode == 0 && c.P == 1) ks = {1};
          else ks = sp.k_set;
          for (int64_t K : ks)
            for (int64_t B : sp.batch) {
              Decoded dc;
              dc.M = sp.models[sp.model_ids[mi]];
              dc.model_slot = (int64_t)mi;
              dc.topo_slot = (int64_t)ti;
              dc.c = c; dc.c.K = K; dc.c.B = B;
              out.push_back(dc);
            }
        }
  return out;
}

Spec spec_from(int32_t n_model_table, const int64_t* model_table,
               int32_t n_topo_table, const int64_t* topo_i, const double* topo_d,
               const int64_t* hdr, const int64_t* lists) {
  // hdr: n_models, n_topos, n_world, n_batch, n_k, k_mode, dp_mask, tp_mask,
  //      pp_mask, synth_seed, synth_count; lists: the lists concatenated.
  Spec sp;
  for (int i = 0; i < n_model_table; i++) sp.models.push_back(model_from(model_table + 13 * i));
  for (int i = 0; i < n_topo_table; i++) sp.topos.push_back(topo_from(topo_i + 4 * i, topo_d + 12 * i));
  const int64_t* p = lists;
  sp.model_ids.assign(p, p + hdr[0]); p += hdr[0];
  sp.topo_ids.assign(p, p + hdr[1]); p += hdr[1];
  sp.world.assign(p, p + hdr[2]); p += hdr[2];
  sp.batch.assign(p, p + hdr[3]); p += hdr[3];
  sp.k_set.assign(p, p + hdr[4]); p += hdr[4];
  sp.k_mode = hdr[5]; sp.dp_mask = hdr[6]; sp.tp_mask = hdr[7]; sp.pp_mask = hdr[8];
  sp.synth_seed = (uint64_t)hdr[9]; sp.synth_count = hdr[10];
  return sp;
}

}  // namespace

// =========================================================== extern "C" =====
extern "C" {

// Simulate an arbitrary explicit program (raw DistIR ops with given costs).
// value_flags: bit0 parameter, bit1 returned.  Per-op arrays are flattened
// with counts.  Returns 0, or 1 if an op's inputs were produced after it
// started (impossible under P:303; reported, not fatal).
int oracle_simulate_raw(int32_t n_dev, int32_t n_values, const int32_t* value_dev,
                        const int64_t* value_bytes, const uint8_t* value_flags,
                        int32_t n_ops, const int32_t* op_ndev, const int32_t* op_devs,
                        const int32_t* op_nin, const int32_t* op_ins,
                        const int32_t* op_nout, const int32_t* op_outs,
                        const double* op_cost, double* op_start, double* op_end,
                        double* clock_end, int64_t* peak, int64_t* live_end,
                        double* makespan) {
  Program pr;
  pr.n_dev = n_dev;
  for (int i = 0; i < n_values; i++)
    pr.new_val(value_dev[i], value_bytes[i], value_flags[i] & 1, (value_flags[i] >> 1) & 1);
  const int32_t *pd = op_devs, *pi = op_ins, *po = op_outs;
  for (int i = 0; i < n_ops; i++) {
    Op op;
    op.cls = COMPUTE;
    op.devs.assign(pd, pd + op_ndev[i]); pd += op_ndev[i];
    op.in.assign(pi, pi + op_nin[i]); pi += op_nin[i];
    op.out.assign(po, po + op_nout[i]); po += op_nout[i];
    op.work = 0;
    op.cost = op_cost[i];
    pr.ops.push_back(op);
  }
  std::vector<double> st, en;
  SimOut so = simulate(pr, &st, &en);
  for (int i = 0; i < n_ops; i++) { op_start[i] = st[i]; op_end[i] = en[i]; }
  for (int d = 0; d < n_dev; d++) { clock_end[d] = so.clock[d]; peak[d] = so.peak[d]; live_end[d] = so.live[d]; }
  *makespan = so.makespan;
  return so.ready_ok ? 0 : 1;
}

// One configuration: builds the explicit program, simulates it.  Returns 0 on
// success, 2 if the program violated a self-check (placement / readiness).
// peak_per_rank / clock_per_rank: [D*T*P] or NULL.
int oracle_eval_config(const int64_t* model, const int64_t* topo_i, const double* topo_d,
                       int64_t D, int64_t T, int64_t P, int64_t K, int64_t B,
                       double* makespan, int64_t* peak, uint32_t* reason, int64_t* n_ops,
                       int64_t* peak_per_rank, double* clock_per_rank) {
  Model M = model_from(model);
  Topo t = topo_from(topo_i, topo_d);
  std::vector<int64_t> pk;
  std::vector<double> ck;
  int err = 0;
  Result r = eval_config(M, t, Cfg{D, T, P, K, B}, &pk, &ck, &err);
  *makespan = r.makespan; *peak = r.peak; *reason = r.reason; *n_ops = r.n_ops;
  if (r.n_ops > 0) {
    if (peak_per_rank) for (size_t i = 0; i < pk.size(); i++) peak_per_rank[i] = pk[i];
    if (clock_per_rank) for (size_t i = 0; i < ck.size(); i++) clock_per_rank[i] = ck[i];
  }
  return err ? 2 : 0;
}

// Per-op listing of one configuration's program (debug / trace / tests):
// fills up to cap ops: class, n_devs, first device, work, cost, start, end.
int64_t oracle_program_ops(const int64_t* model, const int64_t* topo_i, const double* topo_d,
                           int64_t D, int64_t T, int64_t P, int64_t K, int64_t B,
                           int64_t cap, int32_t* cls, int32_t* ndev, int32_t* dev0,
                           int64_t* work, double* cost, double* start, double* end) {
  Model M = model_from(model);
  Topo t = topo_from(topo_i, topo_d);
  Cfg c{D, T, P, K, B};
  if (validity(M, t, c) & ~(uint32_t)R_CAPACITY) return -1;
  Program pr = (M.kind == 0) ? build_mlp(M, c) : build_gpt2(M, c);
  for (Op& op : pr.ops) op.cost = op_cost(t, pr, op);
  std::vector<double> st, en;
  simulate(pr, &st, &en);
  int64_t n = (int64_t)pr.ops.size();
  for (int64_t i = 0; i < n && i < cap; i++) {
    cls[i] = pr.ops[i].cls; ndev[i] = (int32_t)pr.ops[i].devs.size();
    dev0[i] = pr.ops[i].devs[0]; work[i] = pr.ops[i].work; cost[i] = pr.ops[i].cost;
    start[i] = st[i]; end[i] = en[i];
  }
  return n;
}

// Export the explicit program of one configuration (for the Python
// brute-force checkers).  Two-phase: call with caps = 0 to get the sizes
// (sizes[0] = n_values, sizes[1] = n_ops, sizes[2] = total devs,
// sizes[3] = total ins, sizes[4] = total outs), then with arrays.
int oracle_export_program(const int64_t* model, const int64_t* topo_i, const double* topo_d,
                          int64_t D, int64_t T, int64_t P, int64_t K, int64_t B,
                          int64_t* sizes, int32_t* value_dev, int64_t* value_bytes,
                          uint8_t* value_flags, int32_t* op_cls, double* op_costs,
                          int32_t* op_ndev, int32_t* op_devs, int32_t* op_nin,
                          int32_t* op_ins, int32_t* op_nout, int32_t* op_outs) {
  Model M = model_from(model);
  Topo t = topo_from(topo_i, topo_d);
  Cfg c{D, T, P, K, B};
  if (validity(M, t, c) & ~(uint32_t)R_CAPACITY) return -1;
  Program pr = (M.kind == 0) ? build_mlp(M, c) : build_gpt2(M, c);
  for (Op& op : pr.ops) op.cost = op_cost(t, pr, op);
  int64_t nd = 0, ni = 0, no = 0;
  for (const Op& op : pr.ops) { nd += op.devs.size(); ni += op.in.size(); no += op.out.size(); }
  const bool fill = value_dev != nullptr;
  sizes[0] = (int64_t)pr.vals.size(); sizes[1] = (int64_t)pr.ops.size();
  sizes[2] = nd; sizes[3] = ni; sizes[4] = no;
  if (!fill) return 0;
  for (size_t v = 0; v < pr.vals.size(); v++) {
    value_dev[v] = pr.vals[v].dev; value_bytes[v] = pr.vals[v].bytes;
    value_flags[v] = (pr.vals[v].param ? 1 : 0) | (pr.vals[v].returned ? 2 : 0);
  }
  int64_t a = 0, b = 0, q = 0;
  for (size_t i = 0; i < pr.ops.size(); i++) {
    const Op& op = pr.ops[i];
    op_cls[i] = op.cls; op_costs[i] = op.cost;
    op_ndev[i] = (int32_t)op.devs.size(); op_nin[i] = (int32_t)op.in.size();
    op_nout[i] = (int32_t)op.out.size();
    for (int d : op.devs) op_devs[a++] = d;
    for (int v : op.in) op_ins[b++] = v;
    for (int v : op.out) op_outs[q++] = v;
  }
  return 0;
}

// Canonical enumeration: number of configs and their decoded fields.
int64_t oracle_enumerate(int32_t n_model_table, const int64_t* model_table,
                         int32_t n_topo_table, const int64_t* topo_i, const double* topo_d,
                         const int64_t* hdr, const int64_t* lists, int64_t cap,
                         int64_t* fields /* [cap][9]: model_slot, topo_slot, W, D, T, P, K, B, kind */,
                         int64_t* model_out /* [cap][13] or NULL */) {
  Spec sp = spec_from(n_model_table, model_table, n_topo_table, topo_i, topo_d, hdr, lists);
  std::vector<Decoded> all = enumerate(sp);
  for (int64_t i = 0; i < (int64_t)all.size() && i < cap; i++) {
    const Decoded& dc = all[i];
    int64_t* f = fields + 9 * i;
    f[0] = dc.model_slot; f[1] = dc.topo_slot; f[2] = dc.c.D * dc.c.T * dc.c.P;
    f[3] = dc.c.D; f[4] = dc.c.T; f[5] = dc.c.P; f[6] = dc.c.K; f[7] = dc.c.B; f[8] = dc.M.kind;
    if (model_out) {
      const Model& M = dc.M;
      int64_t* mo = model_out + 13 * i;
      mo[0] = M.kind; mo[1] = M.n_layer; mo[2] = M.d_model; mo[3] = M.n_head; mo[4] = M.seq_len;
      mo[5] = M.vocab_pad; mo[6] = M.n_ctx; mo[7] = M.dtype_bytes; mo[8] = M.id_bytes; mo[9] = M.lm_head;
      mo[10] = M.schedule; mo[11] = M.recompute; mo[12] = M.zero;
    }
  }
  return (int64_t)all.size();
}

// Evaluate the configs at the given canonical indices (or all when
// idx == NULL), with n_threads worker threads taking configs one at a time.
// Outputs are indexed like idx.  Returns the number of configs that failed a
// self-check (0 expected).
int64_t oracle_grid_eval(int32_t n_model_table, const int64_t* model_table,
                         int32_t n_topo_table, const int64_t* topo_i, const double* topo_d,
                         const int64_t* hdr, const int64_t* lists,
                         const int64_t* idx, int64_t n_idx, int32_t n_threads,
                         double* makespan, int64_t* peak, uint32_t* reason, int64_t* n_ops) {
  Spec sp = spec_from(n_model_table, model_table, n_topo_table, topo_i, topo_d, hdr, lists);
  std::vector<Decoded> all = enumerate(sp);
  if (!idx) n_idx = (int64_t)all.size();
  std::vector<int64_t> bad(std::max(1, n_threads), 0);
  auto work = [&](int tid, int64_t a, int64_t b) {
    for (int64_t q = a; q < b; q++) {
      const int64_t i = idx ? idx[q] : q;
      if (i < 0 || i >= (int64_t)all.size()) { reason[q] = 0xFFFFFFFFu; continue; }
      const Decoded& dc = all[i];
      const Topo& t = sp.topos[sp.topo_ids[dc.topo_slot]];
      int err = 0;
      Result r = eval_config(dc.M, t, dc.c, nullptr, nullptr, &err);
      makespan[q] = r.makespan; peak[q] = r.peak; reason[q] = r.reason; n_ops[q] = r.n_ops;
      bad[tid] += err;
    }
  };
  if (n_threads <= 1) {
    work(0, 0, n_idx);
  } else {
    // configurations differ in size by orders of magnitude: threads take
    // them one at a time from a shared counter (dynamic distribution)
    std::atomic<int64_t> next{0};
    auto worker = [&](int tid) {
      for (int64_t q; (q = next.fetch_add(1)) < n_idx;) work(tid, q, q + 1);
    };
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; t++) th.emplace_back(worker, t);
    for (auto& x : th) x.join();
  }
  int64_t nb = 0;
  for (int64_t b : bad) nb += b;
  return nb;
}

// Validity bits (C.2) of every enumerated config, without simulating.
int64_t oracle_grid_validity(int32_t n_model_table, const int64_t* model_table,
                             int32_t n_topo_table, const int64_t* topo_i, const double* topo_d,
                             const int64_t* hdr, const int64_t* lists, int64_t cap,
                             uint32_t* reason) {
  Spec sp = spec_from(n_model_table, model_table, n_topo_table, topo_i, topo_d, hdr, lists);
  std::vector<Decoded> all = enumerate(sp);
  for (int64_t i = 0; i < (int64_t)all.size() && i < cap; i++)
    reason[i] = validity(all[i].M, sp.topos[sp.topo_ids[all[i].topo_slot]], all[i].c);
  return (int64_t)all.size();
}

// Top-k by a full stable sort (C.8): feasible = reason == 0; order by
// throughput = B / makespan descending, then peak ascending, then index
// ascending.  Writes up to k positions into out_pos; returns how many.
int32_t oracle_topk(int64_t n, const int64_t* index, const int64_t* batch,
                    const double* makespan, const int64_t* peak, const uint32_t* reason,
                    int32_t k, int64_t* out_pos, double* out_throughput) {
  std::vector<int64_t> pos;
  std::vector<double> tp(n, 0.0);
  for (int64_t i = 0; i < n; i++)
    if (reason[i] == 0) { pos.push_back(i); tp[i] = ((double)batch[i]) / makespan[i]; }
  std::stable_sort(pos.begin(), pos.end(), [&](int64_t a, int64_t b) {
    if (tp[a] != tp[b]) return tp[a] > tp[b];
    if (peak[a] != peak[b]) return peak[a] < peak[b];
    return index[a] < index[b];
  });
  int32_t nk = (int32_t)std::min<int64_t>(k, (int64_t)pos.size());
  for (int32_t i = 0; i < nk; i++) { out_pos[i] = pos[i]; out_throughput[i] = tp[pos[i]]; }
  return nk;
}

}  // extern "C"
