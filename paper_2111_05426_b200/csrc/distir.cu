// distir.cu -- libdistir.so: C ABI (include/distir.h) + host planner.
//
// The host side only validates arguments, lays out the caller's workspace,
// builds the grid decode table (<= 96 entries), uploads it, and launches the
// kernels of kernels.cuh on the caller's stream.  Every step of the method
// (enumerate, expand, cost, timeline, memory, feasibility, top-k, merge) runs
// on the GPU; there is no CPU fallback.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/distir.h"
#define DISTIR_HOST_TU 1   // k_simulate lives in sim_inst.cu (one TU per instantiation)
#include "kernels.cuh"
#include "raw.cuh"
#include "sim_launch.cuh"

using namespace distir;

static_assert(sizeof(distir_topk_entry) == sizeof(TopkRec), "top-k record layout");
static_assert(sizeof(distir_config) == sizeof(DExplicit), "config layout");
static_assert(sizeof(distir_raw_op) == sizeof(RawOp), "raw op layout");
static_assert(sizeof(distir_raw_value) == sizeof(RawValue), "raw value layout");
static_assert(sizeof(distir_raw_program) == sizeof(RawProgram), "raw program layout");

namespace {

thread_local std::string g_err;
// bumped by every NCCL communicator create / destroy: a cached graph that
// captured an all-gather on a communicator is replayed only while no
// communicator changed since
std::atomic<uint64_t> g_comm_gen{0};

distir_status fail(distir_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      return fail(DISTIR_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));   \
  } while (0)

bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

int ilog2(int64_t x) {
  int e = 0;
  while ((int64_t(1) << (e + 1)) <= x) e++;
  return e;
}

// ------------------------------------------------------------ layout -------
struct Layout {
  size_t hdr, spec, ex, bk, sub, cfg_bucket, pc, perm, items, ms, pk, rs, tp, part, part_n, gath, fin,
      fin_n, out, out_n, total;
};

Layout layout(int64_t n_local, int64_t n_explicit) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t n = (size_t)(n_local > 0 ? n_local : 1);
  L.spec = take(sizeof(SpecBlock));
  L.ex = take((size_t)(n_explicit > 0 ? n_explicit : 1) * sizeof(DExplicit));
  L.bk = take(kBucketSlots * sizeof(Bucket));
  L.sub = take((size_t)2 * kBucketSlots * kSubSlots * 4);    // sub-order counts, cursors
  L.cfg_bucket = take(n * 4);
  L.pc = take(n * sizeof(PCfg));
  L.perm = take(n * sizeof(PCfg));
  L.items = take(n * sizeof(Item));
  L.ms = take(n * 8);
  L.pk = take(n * 8);
  L.rs = take(n * 4);
  L.tp = take(n * 8);
  L.part = take((size_t)kPartLists * kMaxK * sizeof(TopkRec));
  L.part_n = take((size_t)kPartLists * 4);
  L.gath = take((size_t)kMaxRanks * kMaxK * sizeof(TopkRec));
  L.fin = take((size_t)kMaxK * sizeof(TopkRec));
  L.fin_n = take(16);
  // final top-k, its count and the header contiguous: the host-buffer path
  // fetches all three with one copy
  L.out = take((size_t)kMaxK * sizeof(TopkRec));
  L.out_n = take(16);
  L.hdr = take(sizeof(WsHeader));
  L.total = off;
  return L;
}

// ------------------------------------------------------------ NCCL ---------
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { api.why = "dlopen(libnccl.so.2) failed"; return; }
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
    api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
    api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
    api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy;
    if (!api.ok) api.why = "NCCL symbols missing";
  });
  return api;
}

}  // namespace

// ------------------------------------------------------------- handle ------
struct GraphCache {
  cudaGraph_t graph = nullptr;    // kept alive: its node handles address exec's nodes
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  cudaEvent_t ph[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // placeholders
  cudaGraphNode_t evnode[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  bool ev_ring = false;          // event nodes currently point into the ring
  int64_t kernels = 0;
  // key
  const void* ws = nullptr;
  double* ms = nullptr;
  int64_t* pk = nullptr;
  uint32_t* rs = nullptr;
  TopkRec* topk = nullptr;
  int* ntopk = nullptr;
  int k = -1;
  void* comm = nullptr;
  uint64_t comm_gen = 0;         // g_comm_gen at capture (a freed communicator's
                                 // address may be reused by a new one)
  int64_t n_local = -1, n_total = -1;
  int32_t mode = -1;
  uint32_t f1b = 0xFFFFFFFFu;
};

struct distir_sim {
  int device = 0;
  double plan_x = 1.0;
  cudaStream_t stream = nullptr;
  std::vector<DModel> models;
  std::vector<DTopo> topos;
  int num_sms = 0;
  int sim_grid[kGroups] = {};
  int enum_grid = 0;
  SpecBlock spec{};
  bool uploaded = false;
  const void* uploaded_ws = nullptr;
  int64_t h2d = 0, d2h = 0;      // bytes copied by the last upload / eval
  // profiling (distir_profile)
  bool prof = false;
  std::vector<cudaEvent_t> ev;   // 5 per recorded launch
  size_t ev_used = 0;            // launches recorded in ev
  distir_profile_data acc{};     // totals folded in from ev
  int64_t kernels = 0, launches = 0;
  GraphCache graph[2];            // [0] plain, [1] with the profiling event nodes
  bool use_graph = true;
  // pinned host staging of the per-call small copies (spec H2D; top-k,
  // its count and the statistics header D2H), so they are true async DMA
  struct Pinned {
    SpecBlock spec;
    // image of the workspace's [out | out_n | hdr] sections (Layout)
    alignas(256) unsigned char tail[kMaxK * sizeof(TopkRec) + 256 + sizeof(WsHeader)];
  };
  Pinned* pin = nullptr;
  cudaEvent_t pin_ev = nullptr;     // the last H2D from pin->spec
  bool pin_pending = false;
  // side streams and events of the concurrent simulate kernels (fork / join)
  cudaStream_t side[kGroups] = {};
  cudaEvent_t fork_ev = nullptr, join_ev[kGroups] = {};
  ~distir_sim() {
    for (int i = 0; i < kGroups; i++) {
      if (side[i]) cudaStreamDestroy(side[i]);
      if (join_ev[i]) cudaEventDestroy(join_ev[i]);
    }
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (pin) cudaFreeHost(pin);
    if (pin_ev) cudaEventDestroy(pin_ev);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    for (GraphCache& g : graph) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      if (g.graph) cudaGraphDestroy(g.graph);
      for (cudaEvent_t e : g.ph)
        if (e) cudaEventDestroy(e);
      if (g.cap) cudaStreamDestroy(g.cap);
    }
  }
};

namespace {

// bit of simulate kernel (kind, mode) in SpecBlock.f1b
constexpr uint32_t gbit(int kind, int mode) { return 1u << (kind * kModes + mode); }
#ifndef DISTIR_PLAIN_MIXED
#define DISTIR_PLAIN_MIXED 0   // grids mixing plain and cached MLP shapes: both kernels (concurrent)
#endif

distir_status check_handle(const distir_sim* sim) {
  if (!sim) return fail(DISTIR_E_INVALID_ARG, "sim is NULL");
  return DISTIR_OK;
}

distir_status validate_model(const distir_model& m, int i) {
  auto bad = [&](const char* what) {
    return fail(DISTIR_E_INVALID_ARG, "model " + std::to_string(i) + ": " + what);
  };
  if (m.kind != DISTIR_MODEL_MLP_TRAIN && m.kind != DISTIR_MODEL_GPT2_INFER) return bad("kind");
  if (m.n_layer < 1 || m.d_model < 1 || m.dtype_bytes < 1) return bad("n_layer/d_model/dtype_bytes");
  if (m.n_layer > 1024) return fail(DISTIR_E_UNSUPPORTED, "n_layer > 1024");
  if (m.kind == DISTIR_MODEL_MLP_TRAIN && m.schedule != DISTIR_SCHED_GPIPE &&
      m.schedule != DISTIR_SCHED_1F1B)
    return bad("schedule");
  if (m.kind == DISTIR_MODEL_MLP_TRAIN && ((m.recompute != 0 && m.recompute != 1) ||
                                           (m.zero != 0 && m.zero != 1)))
    return bad("recompute / zero must be 0 or 1");
  if (m.d_model > (1 << 20)) return fail(DISTIR_E_UNSUPPORTED, "d_model > 2^20");
  if (m.kind == DISTIR_MODEL_GPT2_INFER) {
    if (m.n_head < 1 || m.seq_len < 1 || m.vocab_pad < 1 || m.n_ctx < 0 || m.id_bytes < 1)
      return bad("n_head/seq_len/vocab_pad/n_ctx/id_bytes");
  }
  return DISTIR_OK;
}

distir_status validate_topo(const distir_topology& t, int i) {
  auto bad = [&](const char* what) {
    return fail(DISTIR_E_INVALID_ARG, "topology " + std::to_string(i) + ": " + what);
  };
  if (t.world_max < 1) return bad("world_max");
  if (!is_pow2(t.node_size)) return fail(DISTIR_E_UNSUPPORTED, "node_size must be a power of two");
  if (!(t.flops_per_s > 0) || !(t.bw_intra_Bps > 0) || !(t.bw_inter_Bps > 0)) return bad("rates");
  if (!(t.op_overhead_s >= 0) || !(t.alpha_intra_s >= 0) || !(t.alpha_inter_s >= 0))
    return bad("overheads");
  if (t.capacity_bytes < 0) return bad("capacity");
  if (t.cost_model != DISTIR_COST_ANALYTIC && t.cost_model != DISTIR_COST_REGRESSION)
    return bad("cost_model");
  if (t.reserved != 0) return bad("reserved");
  if (t.cost_model == DISTIR_COST_REGRESSION) {
    const double cs[6] = {t.mm_c0_s, t.mm_s_per_flop, t.mm_s_per_byte,
                          t.ew_c0_s, t.ew_s_per_flop, t.ew_s_per_byte};
    for (double v : cs)
      if (!(v >= 0) || !(v < INFINITY)) return bad("regression coefficients");
  }
  return DISTIR_OK;
}

// Largest per-op integer work must fit in int64 (checked with 128-bit math):
// MLP 4 m d^2, GPT-2 2 n d V and the n V e gathered logits.
bool work_fits(const DModel& M, int64_t B) {
  const __int128 d = M.d, b = B;
  __int128 w;
  if (M.kind == 0) {
    w = 4 * b * d * d;
  } else {
    const __int128 n = b * M.S;
    w = 2 * n * d * ((__int128)M.V + 4 * d) + n * M.V * M.e;
  }
  return w < ((__int128)1 << 62);
}

// Build the SpecBlock for a grid spec (host, O(#triples)).
distir_status build_spec(const distir_sim* sim, const distir_grid_spec* g, SpecBlock& sp,
                         int64_t& n_total) {
  std::memset(&sp, 0, sizeof(sp));
  for (size_t i = 0; i < sim->models.size(); i++) sp.models[i] = sim->models[i];
  for (size_t i = 0; i < sim->topos.size(); i++) sp.topos[i] = sim->topos[i];
  if (g->n_topos < 1 || g->n_topos > 8) return fail(DISTIR_E_INVALID_ARG, "spec.n_topos");
  for (int i = 0; i < g->n_topos; i++) {
    if (g->topos[i] < 0 || g->topos[i] >= (int)sim->topos.size())
      return fail(DISTIR_E_INVALID_ARG, "spec.topos index");
    sp.topo_ids[i] = g->topos[i];
  }
  sp.n_topos = g->n_topos;
  if (g->synth_count > 0) {
    if (g->synth_count > (int64_t(1) << 31) - 1) return fail(DISTIR_E_UNSUPPORTED, "synth_count");
    sp.mode = MODE_SYNTH;
    sp.synth_seed = g->synth_seed;
    n_total = g->synth_count;
    // synthetic sweep: GPipe MLP and GPT-2, P up to 64
    sp.f1b = gbit(0, 3) | gbit(0, 8) | gbit(0, 4) | gbit(1, 3) | gbit(1, 4);
    return DISTIR_OK;
  }
  sp.mode = MODE_GRID;
  if (g->n_models < 1 || g->n_models > 8) return fail(DISTIR_E_INVALID_ARG, "spec.n_models");
  for (int i = 0; i < g->n_models; i++) {
    if (g->models[i] < 0 || g->models[i] >= (int)sim->models.size())
      return fail(DISTIR_E_INVALID_ARG, "spec.models index");
    sp.model_ids[i] = g->models[i];
  }
  sp.n_models = g->n_models;
  if (g->n_world < 1 || g->n_world > 8) return fail(DISTIR_E_INVALID_ARG, "spec.n_world");
  if (g->n_batch < 1 || g->n_batch > 32) return fail(DISTIR_E_INVALID_ARG, "spec.n_batch");
  if (g->n_k < 0 || g->n_k > 16) return fail(DISTIR_E_INVALID_ARG, "spec.n_k");
  if (g->k_mode != 0 && g->k_mode != 1) return fail(DISTIR_E_INVALID_ARG, "spec.k_mode");
  bool any_zero = false;
  for (int mi = 0; mi < g->n_models; mi++) {
    any_zero |= sim->models[g->models[mi]].kind == 0 && sim->models[g->models[mi]].zero != 0;
  }
  for (int i = 0; i < g->n_world; i++) {
    if (!is_pow2(g->world[i]) || (i && g->world[i] <= g->world[i - 1]))
      return fail(DISTIR_E_INVALID_ARG, "spec.world: ascending powers of two");
    if (g->world[i] > kMaxWorld) return fail(DISTIR_E_UNSUPPORTED, "world size > 64");
  }
  for (int i = 0; i < g->n_batch; i++) {
    if (g->batch[i] < 1 || (i && g->batch[i] <= g->batch[i - 1]))
      return fail(DISTIR_E_INVALID_ARG, "spec.batch: ascending positive");
    if (g->batch[i] > (int64_t(1) << 40)) return fail(DISTIR_E_UNSUPPORTED, "batch > 2^40");
    for (int mi = 0; mi < g->n_models; mi++)
      if (!work_fits(sim->models[g->models[mi]], g->batch[i]))
        return fail(DISTIR_E_UNSUPPORTED, "per-op work overflows int64");
  }
  for (int i = 0; i < g->n_k; i++) {
    if (g->k_set[i] < 1 || (i && g->k_set[i] <= g->k_set[i - 1]))
      return fail(DISTIR_E_INVALID_ARG, "spec.k_set: ascending positive");
    if (g->k_set[i] > 4096) return fail(DISTIR_E_UNSUPPORTED, "microbatches > 4096");
  }
  sp.k_mode = g->k_mode;
  // simulate kernels this grid can need (k_plan's group choice, bucket_key):
  // the wavefront kernel of each model kind, its two-stages-per-lane variant
  // when P > 32 is possible, 1F1B and ZeRO when a model uses them (a grid
  // has far fewer than 4096 warp shapes, so the catch-all buckets stay empty)
  {
    const int32_t wmax = g->world[g->n_world - 1];
    uint32_t m = 0;
    for (int mi = 0; mi < g->n_models; mi++) {
      const DModel& M = sim->models[g->models[mi]];
      if (M.kind == 0 && M.zero) m |= gbit(0, 6);   // ZeRO with D > 1, either schedule
      if (M.kind == 0 && M.sched == 1) { m |= gbit(0, 5) | (wmax > 32 ? gbit(0, 7) : 0); continue; }
      if (M.kind == 0) {
        // the plain-walk kernel or the cached one, as the grid's (P, K)
        // shapes need (k_plan's mlp_plain_shape on every P <= 32)
        for (int32_t P = 1; P <= (wmax < 32 ? wmax : 32); P <<= 1) {
          const int nk = (sp.k_mode == 0 && P == 1) ? 1 : g->n_k;
          for (int i = 0; i < nk; i++) {
            const int32_t K = (sp.k_mode == 0 && P == 1) ? 1 : g->k_set[i];
            m |= mlp_plain_shape((uint32_t)M.L, (uint32_t)P, (uint32_t)(K < 255 ? K : 255))
                     ? gbit(0, 8) : gbit(0, 3);
          }
        }
      } else {
        m |= gbit(M.kind, 3);
      }
      if (!DISTIR_PLAIN_MIXED && (m & gbit(0, 3))) m &= ~gbit(0, 8);   // mixed shapes: one kernel walks both
      if (wmax > 32) m |= gbit(M.kind, 4);
      if (M.kind == 0 && M.zero) m |= gbit(0, 6);
    }
    sp.f1b = m;
  }
  sp.n_k = g->n_k;
  for (int i = 0; i < g->n_k; i++) sp.k_set[i] = g->k_set[i];
  sp.n_batch = g->n_batch;
  for (int i = 0; i < g->n_batch; i++) sp.batch[i] = g->batch[i];
  int64_t cum = 0;
  int ne = 0;
  for (int wi = 0; wi < g->n_world; wi++) {
    const int e = ilog2(g->world[wi]);
    for (int a = 0; a <= e; a++)
      for (int b = 0; a + b <= e; b++) {
        const int c = e - a - b;
        if (!((g->dp_mask >> a) & 1) || !((g->tp_mask >> b) & 1) || !((g->pp_mask >> c) & 1)) continue;
        const int nK = (g->k_mode == 0 && c == 0) ? 1 : g->n_k;
        if (nK == 0) continue;
        if (ne >= kMaxEntries) return fail(DISTIR_E_UNSUPPORTED, "too many (D,T,P) triples");
        // ZeRO's kernel holds one (stage, replica) per lane: D > 1 needs
        // next_pow2(P) * D = 2^(a + c) <= 32 (D = 1 runs the plain kernels)
        if (any_zero && a > 0 && a + c > 5)
          return fail(DISTIR_E_UNSUPPORTED, "ZeRO needs next_pow2(pp) * dp <= 32");
        sp.entries[ne] = DEntry{1 << a, 1 << b, 1 << c, nK, cum};
        cum += (int64_t)nK * g->n_batch;
        ne++;
      }
  }
  sp.n_entries = ne;
  sp.per_mt = cum;
  n_total = (int64_t)g->n_models * g->n_topos * cum;
  if (n_total > (int64_t(1) << 31) - 1) return fail(DISTIR_E_UNSUPPORTED, "grid > 2^31 configs");
  return DISTIR_OK;
}

distir_status validate_configs(const distir_sim* sim, const distir_config* cf, int64_t n) {
  for (int64_t i = 0; i < n; i++) {
    const distir_config& c = cf[i];
    auto bad = [&](const char* w) {
      return fail(DISTIR_E_INVALID_ARG, "config " + std::to_string(i) + ": " + w);
    };
    if (c.model < 0 || c.model >= (int)sim->models.size()) return bad("model index");
    if (c.topo < 0 || c.topo >= (int)sim->topos.size()) return bad("topo index");
    if (c.dp < 1 || c.tp < 1 || c.pp < 1 || c.microbatches < 1 || c.batch < 1) return bad("degrees");
    if (!is_pow2(c.dp) || !is_pow2(c.tp))
      return fail(DISTIR_E_UNSUPPORTED, "config dp/tp must be powers of two (stage symmetry)");
    if ((int64_t)c.dp * c.tp * c.pp > kMaxWorld) return fail(DISTIR_E_UNSUPPORTED, "world size > 64");
    if (sim->models[c.model].kind == 0 && sim->models[c.model].zero && c.dp > 1) {
      int64_t p2 = 1;
      while (p2 < c.pp) p2 <<= 1;
      if (p2 * c.dp > 32) return fail(DISTIR_E_UNSUPPORTED, "ZeRO needs next_pow2(pp) * dp <= 32");
    }
    if (c.microbatches > 4096) return fail(DISTIR_E_UNSUPPORTED, "microbatches > 4096");
    if (!work_fits(sim->models[c.model], c.batch))
      return fail(DISTIR_E_UNSUPPORTED, "per-op work overflows int64");
  }
  return DISTIR_OK;
}

distir_status check_ws(void* ws, size_t have, size_t need) {
  if (!ws) return fail(DISTIR_E_WORKSPACE, "workspace is NULL");
  if (((uintptr_t)ws & 255) != 0) return fail(DISTIR_E_WORKSPACE, "workspace not 256-byte aligned");
  if (have < need)
    return fail(DISTIR_E_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  return DISTIR_OK;
}

template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

// Merge n_lists sorted top-k lists on the device (k_topk_merge): one warp
// covers up to 128 lists (4 per lane), a full block up to kMergeMaxLists.
void enqueue_merge(cudaStream_t st, const TopkRec* lists, const int* list_n, int n_lists, int k_in,
                   int k, TopkRec* out, int* out_n) {
  const int threads = n_lists <= 4 * 32 ? 32 : kTopkThreads;
  k_topk_merge<<<1, threads, 0, st>>>(lists, list_n, n_lists, k_in, k, out, out_n);
}

// Fold the recorded launch events into the accumulated totals.
distir_status prof_fold(distir_sim* sim) {
  if (sim->ev_used == 0) return DISTIR_OK;
  CUDA_TRY(cudaEventSynchronize(sim->ev[5 * (sim->ev_used - 1) + 4]));
  for (size_t i = 0; i < sim->ev_used; i++) {
    float t[4];
    for (int j = 0; j < 4; j++)
      CUDA_TRY(cudaEventElapsedTime(&t[j], sim->ev[5 * i + j], sim->ev[5 * i + j + 1]));
    sim->acc.ms_prepare += t[0];
    sim->acc.ms_simulate += t[1];
    sim->acc.ms_topk += t[2];
    sim->acc.ms_merge += t[3];
  }
  sim->ev_used = 0;
  return DISTIR_OK;
}

// Enqueue a1-a7 (+ a8 when comm != NULL) of the uploaded shard on stream st;
// the (global) top-k goes to (topk, ntopk).  ev[0..4] (or NULL) are recorded
// between the phases; with `external` they become event-record nodes of a
// captured graph.  Returns the number of kernels enqueued in *kernels.
distir_status enqueue_all(distir_sim* sim, cudaStream_t st, const cudaEvent_t* ev, bool external,
                          int k, void* comm, void* ws, double* ms, int64_t* pk, uint32_t* rs,
                          TopkRec* topk, int* ntopk, int64_t* kernels_out) {
  const SpecBlock& sp = sim->spec;
  int64_t kernels = 0;
  auto mark = [&](int j) -> cudaError_t {
    if (!ev) return cudaSuccess;
    return external ? cudaEventRecordWithFlags(ev[j], st, cudaEventRecordExternal)
                    : cudaEventRecord(ev[j], st);
  };
  CUDA_TRY(mark(0));
  const Layout L = layout(sp.n_local, sp.mode == MODE_EXPLICIT ? sp.n_total : 0);
  ms = ms ? ms : at<double>(ws, L.ms);
  pk = pk ? pk : at<int64_t>(ws, L.pk);
  rs = rs ? rs : at<uint32_t>(ws, L.rs);
  const SpecBlock* dsp = at<SpecBlock>(ws, L.spec);
  const DExplicit* dex = at<DExplicit>(ws, L.ex);
  Bucket* bk = at<Bucket>(ws, L.bk);
  WsHeader* hdr = at<WsHeader>(ws, L.hdr);
  uint32_t* cb = at<uint32_t>(ws, L.cfg_bucket);
  PCfg* pc = at<PCfg>(ws, L.pc);
  PCfg* perm = at<PCfg>(ws, L.perm);
  Item* items = at<Item>(ws, L.items);
  double* tpv = at<double>(ws, L.tp);
  const int64_t n = sp.n_local;
  PlanBudget pb;
  for (int g = 0; g < kGroups; g++)
    pb.warps[g] = (uint32_t)(sim->plan_x * sim->sim_grid[g] * (sim_tpb(g / kModes, g % kModes) / 32));
  pb.launched = sp.f1b;
  // (one cooperative kernel with grid barriers instead of these four was
  // measured 10 us slower per launch on a B200 and dropped)
  uint32_t* sub = at<uint32_t>(ws, L.sub);
  k_reset<<<(kBucketSlots * kSubSlots / 4 + 255) / 256, 256, 0, st>>>(bk, hdr, sub);
  kernels++;
  if (n > 0) {
    const int eg = (int)std::min<int64_t>((n + 255) / 256, sim->enum_grid);
    k_enumerate<<<eg, 256, 0, st>>>(dsp, dex, bk, cb, ms, pk, rs, tpv, pc, hdr, sub);
    k_plan<<<1, kPlanThreads, 0, st>>>(bk, hdr, pb, sub);
    k_scatter<<<eg, 256, 0, st>>>(dsp, bk, cb, pc, perm, items, sub);
    kernels += 3;
  }
  CUDA_TRY(mark(1));
  TopkRec* fin = at<TopkRec>(ws, L.fin);
  int* fin_n = at<int>(ws, L.fin_n);
  TopkRec* loc = comm ? fin : topk;   // local list (padded) when merging
  int* loc_n = comm ? fin_n : ntopk;
  TopkRec* part = at<TopkRec>(ws, L.part);
  int* part_n = at<int>(ws, L.part_n);
  // the simulate kernels the grid can need (SpecBlock.f1b mask, plus the
  // program-order variants when built in); a7 runs inside them, the last one
  // launched merging the per-kernel top-k lists
  // Several simulate kernels run CONCURRENTLY, one per stream (fork / join
  // on the library's stream): each is persistent and sized to the whole GPU,
  // so the next one's blocks start as the previous one's retire -- in its
  // tail, where its heaviest items leave most SMs idle -- instead of after
  // it.  Longest pipelines first (they set the tail).
  static const int kOrder[] = {0 * kModes + 4, 0 * kModes + 7, 1 * kModes + 4, 0 * kModes + 5,
                               0 * kModes + 6, 1 * kModes + 3, 0 * kModes + 3, 0 * kModes + 8,
                               0, 1, 2, kModes + 0, kModes + 1, kModes + 2};
  int groups[kGroups], ng = 0;
  if (n > 0) {
    for (int g : kOrder) {
      const int md = g % kModes;
      const bool seq = md < 3 && md < DISTIR_SEQ_MAXP && g / kModes <= 1;
      if (seq || (md >= 3 && (sp.f1b & (1u << g)))) groups[ng++] = g;
    }
  }
  const bool fork = ng > 1 && sim->fork_ev != nullptr;
  if (fork) CUDA_TRY(cudaEventRecord(sim->fork_ev, st));
  int n_lists = 0;                    // partial top-k lists (one per simulate block)
  for (int i = 0; i < ng; i++) {
    const int g = groups[i];
    if (n_lists + sim->sim_grid[g] > kPartLists)
      return fail(DISTIR_E_UNSUPPORTED, "simulate grids exceed the partial top-k lists");
    SimArgs sa{dsp, dex, bk, items, perm, hdr, ms, pk, rs, tpv,
               SimTopk{k, part + (int64_t)n_lists * (k > 0 ? k : 1), part_n + n_lists,
                       &hdr->topk_thresh}};
    n_lists += sim->sim_grid[g];
    const int kd = g / kModes, md = g % kModes, grid = sim->sim_grid[g];
    const int tpb = sim_tpb(kd, md), sm = sim_smem(kd, md);
    cudaStream_t ks = st;
    if (fork && i > 0) {
      ks = sim->side[i];
      CUDA_TRY(cudaStreamWaitEvent(ks, sim->fork_ev, 0));
    }
    cudaError_t e = cudaErrorInvalidValue;
    switch (g) {
#define DISTIR_CASE(KD, MD) case KD * kModes + MD: e = sim_launch_##KD##_##MD(grid, tpb, sm, ks, sa); break;
      DISTIR_CASE(0, 0) DISTIR_CASE(0, 1) DISTIR_CASE(0, 2) DISTIR_CASE(0, 3) DISTIR_CASE(0, 4)
      DISTIR_CASE(0, 5) DISTIR_CASE(0, 6) DISTIR_CASE(0, 7) DISTIR_CASE(0, 8)
      DISTIR_CASE(1, 0) DISTIR_CASE(1, 1) DISTIR_CASE(1, 2) DISTIR_CASE(1, 3) DISTIR_CASE(1, 4)
#undef DISTIR_CASE
      default: break;
    }
    CUDA_TRY(e);
    kernels++;
    if (fork && i > 0) {
      CUDA_TRY(cudaEventRecord(sim->join_ev[i], ks));
      CUDA_TRY(cudaStreamWaitEvent(st, sim->join_ev[i], 0));
    }
  }
  CUDA_TRY(mark(2));
  if (k > 0) {                        // a7: the top k of the blocks' lists
    // (programmatic dependent launches of the simulate and select kernels
    // were measured: no change in the step time, dropped)
    k_topk_select<<<1, kSelectThreads, 0, st>>>(part, part_n, n_lists, k, hdr, loc, loc_n);
    kernels++;
  }
  CUDA_TRY(mark(3));
  if (k > 0 && comm) {
    NcclApi& api = nccl();
    if (!api.ok) return fail(DISTIR_E_NCCL, api.why);
    TopkRec* gath = at<TopkRec>(ws, L.gath);
    ncclResult_t r = api.allGather(fin, gath, (size_t)k * sizeof(TopkRec), ncclUint8,
                                   static_cast<ncclComm_t>(comm), st);
    if (r != ncclSuccess)
      return fail(DISTIR_E_NCCL, std::string("ncclAllGather: ") +
                                     (api.getErrorString ? api.getErrorString(r) : "error"));
    enqueue_merge(st, gath, nullptr, sp.n_ranks, k, k, topk, ntopk);
    kernels++;
  }
  CUDA_TRY(mark(4));
  CUDA_TRY(cudaGetLastError());
  *kernels_out = kernels;
  return DISTIR_OK;
}

// Launch the pipeline on the handle's stream.  The kernel sequence is captured
// once into a CUDA graph per (workspace, outputs, k, comm, shard size) and
// replayed (one launch instead of 7-8); the profiling event-record nodes are
// re-pointed at the next ring entry before each replay.  DISTIR_NO_GRAPH=1
// launches the kernels directly.
distir_status launch_all(distir_sim* sim, int k, void* comm, void* ws, double* ms, int64_t* pk,
                         uint32_t* rs, TopkRec* topk, int* ntopk) {
  distir_status s;
  // without profiling, a graph with no event-record nodes at all
  GraphCache& G = sim->graph[sim->prof ? 1 : 0];
  const bool key_ok = G.exec && G.ws == ws && G.ms == ms && G.pk == pk && G.rs == rs &&
                      G.topk == topk && G.ntopk == ntopk && G.k == k && G.comm == comm &&
                      (comm == nullptr || G.comm_gen == g_comm_gen.load()) &&
                      G.n_local == sim->spec.n_local && G.n_total == sim->spec.n_total &&
                      G.mode == sim->spec.mode && G.f1b == sim->spec.f1b;
  if (sim->use_graph && !key_ok) {
    if (G.exec) { cudaGraphExecDestroy(G.exec); G.exec = nullptr; }
    if (G.graph) { cudaGraphDestroy(G.graph); G.graph = nullptr; }
    if (!G.cap) CUDA_TRY(cudaStreamCreateWithFlags(&G.cap, cudaStreamNonBlocking));
    if (!G.ph[0])
      for (int j = 0; j < 5; j++) CUDA_TRY(cudaEventCreate(&G.ph[j]));
    CUDA_TRY(cudaStreamBeginCapture(G.cap, cudaStreamCaptureModeThreadLocal));
    int64_t kern = 0;
    s = enqueue_all(sim, G.cap, sim->prof ? G.ph : nullptr, true, k, comm, ws, ms, pk, rs, topk,
                    ntopk, &kern);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(G.cap, &g);
    if (s != DISTIR_OK) { if (g) cudaGraphDestroy(g); return s; }
    if (e != cudaSuccess || !g) {
      // capture unsupported here (e.g. NCCL build): launch directly from now on
      cudaGetLastError();
      sim->use_graph = false;
    } else {
      e = cudaGraphInstantiate(&G.exec, g, 0);
      size_t nn = 0;
      if (e == cudaSuccess) e = cudaGraphGetNodes(g, nullptr, &nn);
      std::vector<cudaGraphNode_t> nodes(nn);
      if (e == cudaSuccess && nn) e = cudaGraphGetNodes(g, nodes.data(), &nn);
      for (int j = 0; j < 5; j++) G.evnode[j] = nullptr;
      for (size_t i = 0; e == cudaSuccess && i < nn; i++) {
        cudaGraphNodeType t;
        if (cudaGraphNodeGetType(nodes[i], &t) != cudaSuccess || t != cudaGraphNodeTypeEventRecord)
          continue;
        cudaEvent_t ev;
        if (cudaGraphEventRecordNodeGetEvent(nodes[i], &ev) != cudaSuccess) continue;
        for (int j = 0; j < 5; j++)
          if (ev == G.ph[j]) G.evnode[j] = nodes[i];
      }
      G.graph = g;
      CUDA_TRY(e);
      G.ws = ws; G.ms = ms; G.pk = pk; G.rs = rs; G.topk = topk; G.ntopk = ntopk; G.k = k;
      G.comm = comm; G.comm_gen = g_comm_gen.load(); G.n_local = sim->spec.n_local; G.n_total = sim->spec.n_total;
      G.mode = sim->spec.mode; G.f1b = sim->spec.f1b; G.kernels = kern; G.ev_ring = false;
    }
  }
  if (sim->use_graph && G.exec) {
    if (sim->prof) {
      if (5 * (sim->ev_used + 1) > sim->ev.size() && (s = prof_fold(sim)) != DISTIR_OK) return s;
      for (int j = 0; j < 5; j++)
        if (G.evnode[j])
          CUDA_TRY(cudaGraphExecEventRecordNodeSetEvent(G.exec, G.evnode[j],
                                                        sim->ev[5 * sim->ev_used + j]));
      G.ev_ring = true;
    } else if (G.ev_ring) {
      for (int j = 0; j < 5; j++)
        if (G.evnode[j]) CUDA_TRY(cudaGraphExecEventRecordNodeSetEvent(G.exec, G.evnode[j], G.ph[j]));
      G.ev_ring = false;
    }
    CUDA_TRY(cudaGraphLaunch(G.exec, sim->stream));
    if (sim->prof) { sim->ev_used++; sim->kernels += G.kernels; sim->launches++; }
    return DISTIR_OK;
  }
  // direct launches
  const cudaEvent_t* ev = nullptr;
  if (sim->prof) {
    if (5 * (sim->ev_used + 1) > sim->ev.size() && (s = prof_fold(sim)) != DISTIR_OK) return s;
    ev = &sim->ev[5 * sim->ev_used];
  }
  int64_t kern = 0;
  if ((s = enqueue_all(sim, sim->stream, ev, false, k, comm, ws, ms, pk, rs, topk, ntopk, &kern)) !=
      DISTIR_OK)
    return s;
  if (sim->prof) { sim->ev_used++; sim->kernels += kern; sim->launches++; }
  return DISTIR_OK;
}

distir_status upload(distir_sim* sim, const distir_grid_spec* spec, const distir_config* configs,
                     int64_t n_configs, int32_t rank, int32_t n_ranks, void* ws, size_t ws_bytes,
                     int64_t* n_local_out) {
  if (n_ranks < 1 || n_ranks > kMaxRanks || rank < 0 || rank >= n_ranks)
    return fail(DISTIR_E_INVALID_ARG, "rank / n_ranks");
  if ((spec == nullptr) == (configs == nullptr))
    return fail(DISTIR_E_INVALID_ARG, "exactly one of spec / configs");
  SpecBlock& sp = sim->spec;
  int64_t n_total = 0;
  distir_status s;
  if (spec) {
    if ((s = build_spec(sim, spec, sp, n_total)) != DISTIR_OK) return s;
  } else {
    if (n_configs < 0 || n_configs > (int64_t(1) << 31) - 1)
      return fail(DISTIR_E_INVALID_ARG, "n_configs");
    if ((s = validate_configs(sim, configs, n_configs)) != DISTIR_OK) return s;
    std::memset(&sp, 0, sizeof(sp));
    for (size_t i = 0; i < sim->models.size(); i++) sp.models[i] = sim->models[i];
    for (size_t i = 0; i < sim->topos.size(); i++) sp.topos[i] = sim->topos[i];
    sp.mode = MODE_EXPLICIT;
    n_total = n_configs;
    // simulate kernels the configurations need (k_plan's group choice);
    // with more configurations than hash buckets, the catch-alls too
    uint32_t m = 0, kinds = 0;
    for (int64_t i = 0; i < n_configs; i++) {
      const DModel& M = sim->models[configs[i].model];
      const bool zero = M.kind == 0 && M.zero && configs[i].dp > 1;    // ZeRO lanes, either schedule
      kinds |= 1u << (zero ? 3 : M.kind == 0 && M.sched == 1 ? 2 : M.kind);
      if (zero) m |= gbit(0, 6);
      else if (M.kind == 0 && M.sched == 1) m |= configs[i].pp > 32 ? gbit(0, 7) : gbit(0, 5);
      else if (configs[i].pp > 32) m |= gbit(M.kind, 4);
      else if (M.kind == 0 && mlp_plain_shape((uint32_t)M.L, (uint32_t)configs[i].pp,
                                              (uint32_t)(configs[i].microbatches < 255 ? configs[i].microbatches : 255)))
        m |= gbit(0, 8);
      else m |= gbit(M.kind, 3);
    }
    if (!DISTIR_PLAIN_MIXED && (m & gbit(0, 3))) m &= ~gbit(0, 8);   // mixed shapes: one kernel walks both
    if (n_configs > kNumBuckets / 2)
      m |= ((kinds & 1) ? gbit(0, 4) : 0) | ((kinds & 2) ? gbit(1, 4) : 0) |
           ((kinds & 4) ? gbit(0, 7) : 0);
    sp.f1b = m;
  }
  sp.n_total = n_total;
  sp.rank = rank;
  sp.n_ranks = n_ranks;
  sp.n_local = n_total > rank ? (n_total - rank + n_ranks - 1) / n_ranks : 0;
  const Layout L = layout(sp.n_local, sp.mode == MODE_EXPLICIT ? n_total : 0);
  if ((s = check_ws(ws, ws_bytes, L.total)) != DISTIR_OK) return s;
  CUDA_TRY(cudaSetDevice(sim->device));
  if (sim->pin) {
    // the staging buffer may still feed the previous upload's copy
    if (sim->pin_pending) CUDA_TRY(cudaEventSynchronize(sim->pin_ev));
    std::memcpy(&sim->pin->spec, &sp, sizeof(SpecBlock));
    CUDA_TRY(cudaMemcpyAsync(at<SpecBlock>(ws, L.spec), &sim->pin->spec, sizeof(SpecBlock),
                             cudaMemcpyHostToDevice, sim->stream));
    CUDA_TRY(cudaEventRecord(sim->pin_ev, sim->stream));
    sim->pin_pending = true;
  } else {
    CUDA_TRY(cudaMemcpyAsync(at<SpecBlock>(ws, L.spec), &sp, sizeof(SpecBlock),
                             cudaMemcpyHostToDevice, sim->stream));
  }
  if (sp.mode == MODE_EXPLICIT && n_total > 0)
    CUDA_TRY(cudaMemcpyAsync(at<DExplicit>(ws, L.ex), configs, n_total * sizeof(DExplicit),
                             cudaMemcpyHostToDevice, sim->stream));
  sim->uploaded = true;
  sim->uploaded_ws = ws;
  sim->h2d = (int64_t)sizeof(SpecBlock) +
             (sp.mode == MODE_EXPLICIT ? n_total * (int64_t)sizeof(DExplicit) : 0);
  sim->d2h = 0;
  if (n_local_out) *n_local_out = sp.n_local;
  return DISTIR_OK;
}

distir_status fetch_stats(distir_sim* sim, void* ws, distir_stats* out) {
  const Layout L = layout(sim->spec.n_local, sim->spec.mode == MODE_EXPLICIT ? sim->spec.n_total : 0);
  WsHeader h;
  CUDA_TRY(cudaMemcpyAsync(&h, at<WsHeader>(ws, L.hdr), sizeof(h), cudaMemcpyDeviceToHost,
                           sim->stream));
  CUDA_TRY(cudaStreamSynchronize(sim->stream));
  out->n_configs = sim->spec.n_local;
  out->n_valid = (int64_t)h.n_valid;
  out->n_feasible = (int64_t)h.n_feasible;
  out->op_events = (int64_t)h.op_events;
  out->stage_steps = (int64_t)h.stage_steps;
  out->n_buckets = h.n_buckets;
  out->n_items = h.n_items;
  out->h2d_bytes = sim->h2d;
  out->d2h_bytes = sim->d2h + (int64_t)sizeof(WsHeader);
  out->tasks = (int64_t)h.tasks;
  out->slow_tasks = (int64_t)h.slow_tasks;
  out->wave_steps = (int64_t)h.wave_steps;
  return DISTIR_OK;
}

}  // namespace

// ================================================================== ABI =====
extern "C" {

const char* distir_last_error(void) { return g_err.c_str(); }

const char* distir_version(void) { return "distir-b200 0.1 (sm_100a)"; }



distir_status distir_sim_create(const distir_model* models, int32_t n_models,
                                const distir_topology* topos, int32_t n_topos, int32_t cuda_device,
                                void* cuda_stream, distir_sim** out) {
  g_err.clear();
  if (!out) return fail(DISTIR_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!models || n_models < 1 || n_models > kMaxModels)
    return fail(DISTIR_E_INVALID_ARG, "models / n_models in [1, 64]");
  if (!topos || n_topos < 1 || n_topos > kMaxTopos)
    return fail(DISTIR_E_INVALID_ARG, "topos / n_topos in [1, 64]");
  distir_status s;
  for (int i = 0; i < n_models; i++)
    if ((s = validate_model(models[i], i)) != DISTIR_OK) return s;
  for (int i = 0; i < n_topos; i++)
    if ((s = validate_topo(topos[i], i)) != DISTIR_OK) return s;
  distir_sim* sim = new (std::nothrow) distir_sim();
  if (!sim) return fail(DISTIR_E_OUT_OF_MEMORY, "handle");
  for (int i = 0; i < n_models; i++) {
    const distir_model& m = models[i];
    sim->models.push_back(DModel{m.kind, m.n_layer, m.d_model, m.n_head, m.seq_len, m.vocab_pad,
                                 m.n_ctx, m.dtype_bytes, m.id_bytes, m.lm_head,
                                 m.kind == DISTIR_MODEL_MLP_TRAIN ? m.schedule : 0,
                                 m.kind == DISTIR_MODEL_MLP_TRAIN ? m.recompute : 0,
                                 m.kind == DISTIR_MODEL_MLP_TRAIN ? m.zero : 0});
  }
  for (int i = 0; i < n_topos; i++) {
    const distir_topology& t = topos[i];
    sim->topos.push_back(DTopo{t.world_max, t.node_size, t.flops_per_s, t.op_overhead_s,
                               t.alpha_intra_s, t.bw_intra_Bps, t.alpha_inter_s, t.bw_inter_Bps,
                               t.capacity_bytes, t.cost_model, t.mm_c0_s, t.mm_s_per_flop,
                               t.mm_s_per_byte, t.ew_c0_s, t.ew_s_per_flop, t.ew_s_per_byte});
  }
  sim->device = cuda_device;
  sim->stream = static_cast<cudaStream_t>(cuda_stream);
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sim->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  int per_sm[kGroups] = {};
  const void* fns[kGroups] = {};
  {
    const void* k0[] = {sim_fn_0_0(), sim_fn_0_1(), sim_fn_0_2(), sim_fn_0_3(), sim_fn_0_4(),
                        sim_fn_0_5(), sim_fn_0_6(), sim_fn_0_7(), sim_fn_0_8()};
    const void* k1[] = {sim_fn_1_0(), sim_fn_1_1(), sim_fn_1_2(), sim_fn_1_3(), sim_fn_1_4()};
    for (int m = 0; m < 9; m++) fns[m] = k0[m];
    for (int m = 0; m < 5; m++) fns[kModes + m] = k1[m];
  }
  for (int g = 0; g < kGroups && e == cudaSuccess; g++) {
    if (!fns[g]) continue;
    const int smem = sim_smem(g / kModes, g % kModes);
    e = cudaFuncSetAttribute(fns[g], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[g], fns[g], sim_tpb(g / kModes, g % kModes), smem);
  }
  if (e != cudaSuccess) {
    delete sim;
    return fail(DISTIR_E_CUDA, std::string("device setup: ") + cudaGetErrorString(e));
  }
  // resident blocks per SM of the persistent simulate kernels (occupancy
  // limit; DISTIR_SIM_BLOCKS_PER_SM caps it for experiments)
  const char* bps = getenv("DISTIR_SIM_BLOCKS_PER_SM");
  const int cap = bps ? atoi(bps) : 0;
  for (int g = 0; g < kGroups; g++) {
    int b = per_sm[g] > 0 ? per_sm[g] : 1;
    if (cap > 0 && b > cap) b = cap;
    // (one partial top-k list per block; kPartLists per launch)
    const int gr = sim->num_sms * b;
    const int lim = kPartLists / kGroups;
    sim->sim_grid[g] = gr < lim ? gr : lim;
  }
  // work-item budget of k_plan's splitting, in resident warps of each
  // simulate kernel (DISTIR_PLAN_BUDGET_X scales it for experiments)
  const char* px = getenv("DISTIR_PLAN_BUDGET_X");
  sim->plan_x = px ? atof(px) : kPlanBudgetX;
  if (cudaMallocHost(&sim->pin, sizeof(distir_sim::Pinned)) != cudaSuccess ||
      cudaEventCreateWithFlags(&sim->pin_ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();            // pageable fallback
    if (sim->pin) cudaFreeHost(sim->pin);
    sim->pin = nullptr;
    sim->pin_ev = nullptr;
  }
  const char* ng = getenv("DISTIR_NO_GRAPH");
  sim->use_graph = !(ng && ng[0] == '1');
  sim->enum_grid = sim->num_sms * 8;
  {   // concurrent simulate kernels (DISTIR_CONCURRENT=0: one after another)
    const char* cc = getenv("DISTIR_CONCURRENT");
    bool ok = !(cc && cc[0] == '0') &&
              cudaEventCreateWithFlags(&sim->fork_ev, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < kGroups; i++)
      ok = cudaStreamCreateWithFlags(&sim->side[i], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&sim->join_ev[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      if (sim->fork_ev) cudaEventDestroy(sim->fork_ev);
      sim->fork_ev = nullptr;
    }
  }
  *out = sim;
  return DISTIR_OK;
}

void distir_sim_destroy(distir_sim* sim) { delete sim; }

distir_status distir_grid_size(const distir_sim* sim, const distir_grid_spec* spec, int64_t* n) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  if (!spec || !n) return fail(DISTIR_E_INVALID_ARG, "spec / n_configs is NULL");
  SpecBlock* sp = new (std::nothrow) SpecBlock();
  if (!sp) return fail(DISTIR_E_OUT_OF_MEMORY, "spec");
  int64_t total = 0;
  s = build_spec(sim, spec, *sp, total);
  delete sp;
  if (s == DISTIR_OK) *n = total;
  return s;
}

distir_status distir_workspace_size(const distir_sim* sim, int64_t n_configs, size_t* bytes) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  if (!bytes || n_configs < 0) return fail(DISTIR_E_INVALID_ARG, "bytes / n_configs");
  *bytes = layout(n_configs, n_configs).total;
  return DISTIR_OK;
}

distir_status distir_result_layout(const distir_sim* sim, int64_t n_configs, int64_t offsets[3],
                                   size_t* bytes) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  if (!offsets || !bytes || n_configs < 0) return fail(DISTIR_E_INVALID_ARG, "offsets / bytes / n_configs");
  // the device sections ms | pk | rs of the workspace (Layout), back to back
  const Layout L = layout(n_configs, 0);
  offsets[0] = 0;
  offsets[1] = (int64_t)(L.pk - L.ms);
  offsets[2] = (int64_t)(L.rs - L.ms);
  *bytes = (L.rs - L.ms) + (size_t)(n_configs > 0 ? n_configs : 1) * 4;
  return DISTIR_OK;
}

distir_status distir_grid_upload(distir_sim* sim, const distir_grid_spec* spec,
                                 const distir_config* configs, int64_t n_configs, int32_t rank,
                                 int32_t n_ranks, void* d_workspace, size_t ws_bytes,
                                 int64_t* n_local_out) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  return upload(sim, spec, configs, n_configs, rank, n_ranks, d_workspace, ws_bytes, n_local_out);
}

distir_status distir_grid_launch(distir_sim* sim, int32_t k, void* nccl_comm, void* d_workspace,
                                 size_t ws_bytes, double* d_makespan, int64_t* d_peak,
                                 uint32_t* d_reason, distir_topk_entry* d_topk,
                                 int32_t* d_n_topk) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  if (!sim->uploaded || sim->uploaded_ws != d_workspace)
    return fail(DISTIR_E_INVALID_ARG, "no grid uploaded to this workspace");
  if (k < 0 || k > kMaxK) return fail(DISTIR_E_INVALID_ARG, "k in [0, 64]");
  if (k > 0 && (!d_topk || !d_n_topk)) return fail(DISTIR_E_INVALID_ARG, "d_topk / d_n_topk");
  const Layout L = layout(sim->spec.n_local, sim->spec.mode == MODE_EXPLICIT ? sim->spec.n_total : 0);
  if ((s = check_ws(d_workspace, ws_bytes, L.total)) != DISTIR_OK) return s;
  CUDA_TRY(cudaSetDevice(sim->device));
  return launch_all(sim, k, nccl_comm, d_workspace, d_makespan, d_peak, d_reason,
                    reinterpret_cast<TopkRec*>(d_topk), d_n_topk);
}

distir_status distir_profile(distir_sim* sim, int32_t enable, distir_profile_data* out) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  CUDA_TRY(cudaSetDevice(sim->device));
  if (out) {
    if ((s = prof_fold(sim)) != DISTIR_OK) return s;
    *out = sim->acc;
    out->launches = sim->launches;
    out->kernels = sim->kernels;
    sim->acc = distir_profile_data{};
    sim->launches = sim->kernels = 0;
  }
  if (enable && sim->ev.empty()) {
    sim->ev.resize(5 * 4096);
    for (cudaEvent_t& e : sim->ev) CUDA_TRY(cudaEventCreate(&e));
  }
  sim->prof = enable != 0;
  return DISTIR_OK;
}

distir_status distir_last_stats(distir_sim* sim, void* d_workspace, distir_stats* out) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  if (!out || !d_workspace) return fail(DISTIR_E_INVALID_ARG, "out / workspace");
  CUDA_TRY(cudaSetDevice(sim->device));
  return fetch_stats(sim, d_workspace, out);
}

distir_status distir_grid_eval_sharded(distir_sim* sim, const distir_grid_spec* spec,
                                       const distir_config* configs, int64_t n_configs,
                                       int32_t rank, int32_t n_ranks, void* nccl_comm, int32_t k,
                                       void* d_workspace, size_t ws_bytes, double* makespan_out,
                                       int64_t* peak_out, uint32_t* reason_out,
                                       distir_topk_entry* topk_out, int32_t* n_topk_out,
                                       distir_stats* stats_out) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  if (k < 0 || k > kMaxK) return fail(DISTIR_E_INVALID_ARG, "k in [0, 64]");
  if (k > 0 && (!topk_out || !n_topk_out)) return fail(DISTIR_E_INVALID_ARG, "topk_out / n_topk_out");
  if (n_ranks > 1 && !nccl_comm) return fail(DISTIR_E_INVALID_ARG, "nccl_comm is NULL");
  if ((s = upload(sim, spec, configs, n_configs, rank, n_ranks, d_workspace, ws_bytes, nullptr)) !=
      DISTIR_OK)
    return s;
  const SpecBlock& sp = sim->spec;
  const Layout L = layout(sp.n_local, sp.mode == MODE_EXPLICIT ? sp.n_total : 0);
  TopkRec* fin = at<TopkRec>(d_workspace, L.out);
  int* fin_n = at<int>(d_workspace, L.out_n);
  if ((s = launch_all(sim, k, nccl_comm, d_workspace, nullptr, nullptr, nullptr, fin, fin_n)) !=
      DISTIR_OK)
    return s;
  const int64_t n = sp.n_local;
  sim->d2h = n * ((makespan_out ? 8 : 0) + (peak_out ? 8 : 0) + (reason_out ? 4 : 0)) +
             (k > 0 ? (int64_t)k * (int64_t)sizeof(TopkRec) + 4 : 0);
  if (n > 0) {
    // per-config results straight into the caller's (pinned) buffers; a
    // strided copy only when shards interleave
    const size_t pitch = (size_t)n_ranks;
    auto get = [&](void* dst, const void* src, size_t w) -> cudaError_t {
      if (n_ranks == 1) return cudaMemcpyAsync(dst, src, w * n, cudaMemcpyDeviceToHost, sim->stream);
      return cudaMemcpy2DAsync(dst, pitch * w, src, w, w, n, cudaMemcpyDeviceToHost, sim->stream);
    };
    const char* m0 = reinterpret_cast<const char*>(makespan_out);
    const bool packed = n_ranks == 1 && makespan_out && peak_out && reason_out &&
                        reinterpret_cast<const char*>(peak_out) - m0 == (ptrdiff_t)(L.pk - L.ms) &&
                        reinterpret_cast<const char*>(reason_out) - m0 == (ptrdiff_t)(L.rs - L.ms);
    if (packed) {          // distir_result_layout: one copy of ms | pk | rs
      CUDA_TRY(cudaMemcpyAsync(makespan_out, at<double>(d_workspace, L.ms), (L.rs - L.ms) + (size_t)n * 4,
                               cudaMemcpyDeviceToHost, sim->stream));
    } else {
      if (makespan_out) CUDA_TRY(get(makespan_out + rank, at<double>(d_workspace, L.ms), 8));
      if (peak_out) CUDA_TRY(get(peak_out + rank, at<int64_t>(d_workspace, L.pk), 8));
      if (reason_out) CUDA_TRY(get(reason_out + rank, at<uint32_t>(d_workspace, L.rs), 4));
    }
  }
  distir_sim::Pinned* P = sim->pin;
  // top-k, its count and the header: one copy of the contiguous workspace
  // tail [out | out_n | hdr] into the pinned image
  const size_t t_n = L.out_n - L.out, t_h = L.hdr - L.out;
  static_assert(sizeof(((distir_sim::Pinned*)nullptr)->tail) >= kMaxK * sizeof(TopkRec) + 256 + sizeof(WsHeader),
                "pinned tail image");
  if (P && (k > 0 || stats_out)) {
    CUDA_TRY(cudaMemcpyAsync(P->tail, fin, t_h + sizeof(WsHeader), cudaMemcpyDeviceToHost, sim->stream));
  } else if (k > 0) {
    CUDA_TRY(cudaMemcpyAsync(topk_out, fin, (size_t)k * sizeof(TopkRec), cudaMemcpyDeviceToHost, sim->stream));
    CUDA_TRY(cudaMemcpyAsync(n_topk_out, fin_n, sizeof(int32_t), cudaMemcpyDeviceToHost, sim->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(sim->stream));
  if (P && k > 0) {
    std::memcpy(topk_out, P->tail, (size_t)k * sizeof(TopkRec));
    std::memcpy(n_topk_out, P->tail + t_n, sizeof(int32_t));
  }
  if (stats_out) {
    if (P) {
      WsHeader h;
      std::memcpy(&h, P->tail + t_h, sizeof(WsHeader));
      stats_out->n_configs = sp.n_local;
      stats_out->n_valid = (int64_t)h.n_valid;
      stats_out->n_feasible = (int64_t)h.n_feasible;
      stats_out->op_events = (int64_t)h.op_events;
      stats_out->stage_steps = (int64_t)h.stage_steps;
      stats_out->n_buckets = h.n_buckets;
      stats_out->n_items = h.n_items;
      stats_out->h2d_bytes = sim->h2d;
      stats_out->d2h_bytes = sim->d2h + (int64_t)sizeof(WsHeader);
      stats_out->tasks = (int64_t)h.tasks;
      stats_out->slow_tasks = (int64_t)h.slow_tasks;
      stats_out->wave_steps = (int64_t)h.wave_steps;
    } else if ((s = fetch_stats(sim, d_workspace, stats_out)) != DISTIR_OK) {
      return s;
    }
  }
  return DISTIR_OK;
}

distir_status distir_grid_eval(distir_sim* sim, const distir_grid_spec* spec,
                               const distir_config* configs, int64_t n_configs, int32_t k,
                               void* d_workspace, size_t ws_bytes, double* makespan_out,
                               int64_t* peak_out, uint32_t* reason_out, distir_topk_entry* topk_out,
                               int32_t* n_topk_out, distir_stats* stats_out) {
  return distir_grid_eval_sharded(sim, spec, configs, n_configs, 0, 1, nullptr, k, d_workspace,
                                  ws_bytes, makespan_out, peak_out, reason_out, topk_out,
                                  n_topk_out, stats_out);
}

distir_status distir_topk_merge(distir_sim* sim, const distir_topk_entry* d_lists,
                                const int32_t* d_list_n, int32_t n_lists, int32_t k_in,
                                int32_t k, distir_topk_entry* d_out, int32_t* d_n_out) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  if (n_lists < 1 || n_lists > kMergeMaxLists)
    return fail(DISTIR_E_INVALID_ARG, "n_lists in [1, 1024]");
  if (k_in < 0 || k_in > kMaxK || k < 0 || k > kMaxK)
    return fail(DISTIR_E_INVALID_ARG, "k_in / k in [0, 64]");
  if (!d_lists || !d_out || !d_n_out) return fail(DISTIR_E_INVALID_ARG, "NULL device buffer");
  const char* lo = reinterpret_cast<const char*>(d_lists);
  const char* oo = reinterpret_cast<const char*>(d_out);
  if (oo < lo + (size_t)n_lists * k_in * sizeof(TopkRec) && lo < oo + (size_t)k * sizeof(TopkRec))
    return fail(DISTIR_E_INVALID_ARG, "d_out overlaps d_lists");
  CUDA_TRY(cudaSetDevice(sim->device));
  enqueue_merge(sim->stream, reinterpret_cast<const TopkRec*>(d_lists), d_list_n, n_lists, k_in, k,
                reinterpret_cast<TopkRec*>(d_out), d_n_out);
  CUDA_TRY(cudaGetLastError());
  return DISTIR_OK;
}

distir_status distir_nccl_unique_id(uint8_t id_out[128]) {
  g_err.clear();
  if (!id_out) return fail(DISTIR_E_INVALID_ARG, "id_out is NULL");
  NcclApi& api = nccl();
  if (!api.ok) return fail(DISTIR_E_NCCL, api.why);
  ncclUniqueId id;
  ncclResult_t r = api.getUniqueId(&id);
  if (r != ncclSuccess) return fail(DISTIR_E_NCCL, "ncclGetUniqueId failed");
  std::memcpy(id_out, &id, 128);
  return DISTIR_OK;
}

distir_status distir_nccl_comm_init(const uint8_t id[128], int32_t n_ranks, int32_t rank,
                                    int32_t cuda_device, void** comm_out) {
  g_err.clear();
  if (!id || !comm_out || n_ranks < 1 || rank < 0 || rank >= n_ranks)
    return fail(DISTIR_E_INVALID_ARG, "id / comm_out / rank");
  NcclApi& api = nccl();
  if (!api.ok) return fail(DISTIR_E_NCCL, api.why);
  CUDA_TRY(cudaSetDevice(cuda_device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t comm = nullptr;
  ncclResult_t r = api.commInitRank(&comm, n_ranks, uid, rank);
  if (r != ncclSuccess)
    return fail(DISTIR_E_NCCL, std::string("ncclCommInitRank: ") +
                                   (api.getErrorString ? api.getErrorString(r) : "error"));
  g_comm_gen.fetch_add(1);
  *comm_out = comm;
  return DISTIR_OK;
}

distir_status distir_nccl_comm_destroy(void* comm) {
  g_err.clear();
  if (!comm) return DISTIR_OK;
  NcclApi& api = nccl();
  if (!api.ok) return fail(DISTIR_E_NCCL, api.why);
  g_comm_gen.fetch_add(1);
  api.commDestroy(static_cast<ncclComm_t>(comm));
  return DISTIR_OK;
}

#ifdef DISTIR_INSTR
// Debug: read and reset the instrumentation counters (not part of distir.h).
// The counters live per translation unit (one per simulate kernel); maxima
// ([8], [11]) are combined by max, the rest summed.
int distir_debug_counters(unsigned long long* out, int n) {
  for (int i = 0; i < n; i++) out[i] = 0;
  int r = 0;
  r |= sim_counters_0_0(out, n); r |= sim_counters_0_1(out, n); r |= sim_counters_0_2(out, n);
  r |= sim_counters_0_3(out, n); r |= sim_counters_0_4(out, n); r |= sim_counters_0_5(out, n);
  r |= sim_counters_0_6(out, n); r |= sim_counters_0_7(out, n); r |= sim_counters_0_8(out, n);
  r |= sim_counters_1_0(out, n);
  r |= sim_counters_1_1(out, n); r |= sim_counters_1_2(out, n); r |= sim_counters_1_3(out, n);
  r |= sim_counters_1_4(out, n);
  return r;
}
#endif

// ---------------------------------------------------------- raw programs --
namespace {
struct RawLayout {
  size_t progs, ops, idx, vals, lu, ms, clk, pk, st, en, total;
};
RawLayout raw_layout(int64_t np, int64_t no, int64_t ni, int64_t nv, int64_t nout) {
  RawLayout L{};
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~size_t(255); return o; };
  auto n1 = [](int64_t x) { return (size_t)(x > 0 ? x : 1); };
  L.progs = take(n1(np) * sizeof(RawProgram));
  L.ops = take(n1(no) * sizeof(RawOp));
  L.idx = take(n1(ni) * 4);
  L.vals = take(n1(nv) * sizeof(RawValue));
  L.lu = take(n1(nv) * 4);
  L.ms = take(n1(np) * 8);
  L.clk = take(n1(nout) * 8);
  L.pk = take(n1(nout) * 8);
  L.st = take(n1(no) * 8);
  L.en = take(n1(no) * 8);
  L.total = off;
  return L;
}
}  // namespace

distir_status distir_raw_workspace_size(int32_t n_programs, int64_t n_ops, int64_t n_idx,
                                        int64_t n_values, int64_t n_out, size_t* bytes) {
  g_err.clear();
  if (!bytes || n_programs < 0 || n_ops < 0 || n_idx < 0 || n_values < 0 || n_out < 0)
    return fail(DISTIR_E_INVALID_ARG, "sizes / bytes");
  *bytes = raw_layout(n_programs, n_ops, n_idx, n_values, n_out).total;
  return DISTIR_OK;
}

distir_status distir_raw_eval(distir_sim* sim, const distir_raw_program* programs,
                              int32_t n_programs, const distir_raw_op* ops, int64_t n_ops,
                              const int32_t* idx, int64_t n_idx, const distir_raw_value* values,
                              int64_t n_values, int64_t n_out, void* d_workspace, size_t ws_bytes,
                              double* makespan_out, double* clock_out, int64_t* peak_out,
                              double* op_start_out, double* op_end_out) {
  g_err.clear();
  distir_status s;
  if ((s = check_handle(sim)) != DISTIR_OK) return s;
  if (n_programs < 0 || (n_programs > 0 && (!programs || !makespan_out)))
    return fail(DISTIR_E_INVALID_ARG, "programs / makespan_out");
  if ((op_start_out == nullptr) != (op_end_out == nullptr))
    return fail(DISTIR_E_INVALID_ARG, "op_start_out and op_end_out go together");
  // validate every id and offset (host)
  for (int32_t p = 0; p < n_programs; p++) {
    const distir_raw_program& pr = programs[p];
    auto bad = [&](const char* w) {
      return fail(DISTIR_E_INVALID_ARG, "program " + std::to_string(p) + ": " + w);
    };
    if (pr.n_dev < 1 || pr.n_dev > kRawMaxDev) return bad("n_dev in [1, 64]");
    if (pr.n_ops < 0 || pr.op_base < 0 || (int64_t)pr.op_base + pr.n_ops > n_ops) return bad("op range");
    if (pr.n_values < 0 || pr.value_base < 0 || (int64_t)pr.value_base + pr.n_values > n_values)
      return bad("value range");
    if (pr.out_base < 0 || (int64_t)pr.out_base + pr.n_dev > n_out) return bad("out range");
    for (int32_t v = 0; v < pr.n_values; v++) {
      const distir_raw_value& x = values[pr.value_base + v];
      if (x.dev < 0 || x.dev >= pr.n_dev || x.bytes < 0) return bad("value device / bytes");
    }
    for (int32_t i = 0; i < pr.n_ops; i++) {
      const distir_raw_op& o = ops[pr.op_base + i];
      if (!(o.cost >= 0.0) || std::isinf(o.cost)) return bad("op cost must be finite and >= 0");
      if (o.n_dev < 1 || o.n_in < 0 || o.n_out < 0) return bad("op counts");
      if (o.dev_off < 0 || (int64_t)o.dev_off + o.n_dev > n_idx || o.in_off < 0 ||
          (int64_t)o.in_off + o.n_in > n_idx || o.out_off < 0 || (int64_t)o.out_off + o.n_out > n_idx)
        return bad("op index range");
      for (int j = 0; j < o.n_dev; j++)
        if (idx[o.dev_off + j] < 0 || idx[o.dev_off + j] >= pr.n_dev) return bad("op device id");
      for (int j = 0; j < o.n_in; j++)
        if (idx[o.in_off + j] < 0 || idx[o.in_off + j] >= pr.n_values) return bad("op input id");
      for (int j = 0; j < o.n_out; j++)
        if (idx[o.out_off + j] < 0 || idx[o.out_off + j] >= pr.n_values) return bad("op output id");
    }
    // program semantics the kernel relies on: every input
    // is a parameter or an earlier op's output, every value is defined once,
    // and an output lives on one of its op's devices
    std::vector<uint8_t> defined(pr.n_values);
    for (int32_t v = 0; v < pr.n_values; v++) defined[v] = values[pr.value_base + v].flags & 1;
    for (int32_t i = 0; i < pr.n_ops; i++) {
      const distir_raw_op& o = ops[pr.op_base + i];
      for (int j = 0; j < o.n_in; j++)
        if (!defined[idx[o.in_off + j]]) return bad("op input used before it is defined");
      for (int j = 0; j < o.n_out; j++) {
        const int32_t v = idx[o.out_off + j];
        if (defined[v]) return bad("value defined twice (a parameter or an earlier output)");
        defined[v] = 1;
        bool on = false;
        for (int t = 0; t < o.n_dev; t++) on |= idx[o.dev_off + t] == values[pr.value_base + v].dev;
        if (!on) return bad("output value not on one of its op's devices");
      }
    }
  }
  // one thread per program writes its value, output and op ranges: they
  // must not overlap across programs
  {
    auto disjoint = [&](auto base, auto len) {
      std::vector<std::pair<int64_t, int64_t>> r;
      for (int32_t p = 0; p < n_programs; p++)
        if (len(programs[p]) > 0) r.push_back({base(programs[p]), len(programs[p])});
      std::sort(r.begin(), r.end());
      for (size_t i = 1; i < r.size(); i++)
        if (r[i - 1].first + r[i - 1].second > r[i].first) return false;
      return true;
    };
    if (!disjoint([](const distir_raw_program& q) { return (int64_t)q.value_base; },
                  [](const distir_raw_program& q) { return (int64_t)q.n_values; }) ||
        !disjoint([](const distir_raw_program& q) { return (int64_t)q.out_base; },
                  [](const distir_raw_program& q) { return (int64_t)q.n_dev; }) ||
        !disjoint([](const distir_raw_program& q) { return (int64_t)q.op_base; },
                  [](const distir_raw_program& q) { return (int64_t)q.n_ops; }))
      return fail(DISTIR_E_INVALID_ARG, "programs' op / value / output ranges overlap");
  }
  const RawLayout L = raw_layout(n_programs, n_ops, n_idx, n_values, n_out);
  if ((s = check_ws(d_workspace, ws_bytes, L.total)) != DISTIR_OK) return s;
  if (n_programs == 0) return DISTIR_OK;
  CUDA_TRY(cudaSetDevice(sim->device));
  cudaStream_t st = sim->stream;
  void* ws = d_workspace;
  CUDA_TRY(cudaMemcpyAsync(at<void>(ws, L.progs), programs, n_programs * sizeof(RawProgram),
                           cudaMemcpyHostToDevice, st));
  if (n_ops)
    CUDA_TRY(cudaMemcpyAsync(at<void>(ws, L.ops), ops, n_ops * sizeof(RawOp), cudaMemcpyHostToDevice, st));
  if (n_idx)
    CUDA_TRY(cudaMemcpyAsync(at<void>(ws, L.idx), idx, n_idx * 4, cudaMemcpyHostToDevice, st));
  if (n_values)
    CUDA_TRY(cudaMemcpyAsync(at<void>(ws, L.vals), values, n_values * sizeof(RawValue),
                             cudaMemcpyHostToDevice, st));
  k_raw_eval<<<(n_programs + 127) / 128, 128, 0, st>>>(
      at<RawProgram>(ws, L.progs), n_programs, at<RawOp>(ws, L.ops), at<int32_t>(ws, L.idx),
      at<RawValue>(ws, L.vals), at<int32_t>(ws, L.lu), at<double>(ws, L.ms),
      clock_out ? at<double>(ws, L.clk) : nullptr, peak_out ? at<int64_t>(ws, L.pk) : nullptr,
      op_start_out ? at<double>(ws, L.st) : nullptr, op_end_out ? at<double>(ws, L.en) : nullptr);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(makespan_out, at<double>(ws, L.ms), n_programs * 8, cudaMemcpyDeviceToHost, st));
  if (clock_out && n_out)
    CUDA_TRY(cudaMemcpyAsync(clock_out, at<double>(ws, L.clk), n_out * 8, cudaMemcpyDeviceToHost, st));
  if (peak_out && n_out)
    CUDA_TRY(cudaMemcpyAsync(peak_out, at<int64_t>(ws, L.pk), n_out * 8, cudaMemcpyDeviceToHost, st));
  if (op_start_out && n_ops) {
    CUDA_TRY(cudaMemcpyAsync(op_start_out, at<double>(ws, L.st), n_ops * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(op_end_out, at<double>(ws, L.en), n_ops * 8, cudaMemcpyDeviceToHost, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return DISTIR_OK;
}

int64_t distir_shard_indices(int64_t n_configs, int32_t rank, int32_t n_ranks, int64_t* out,
                             int64_t cap) {
  if (n_configs <= 0 || n_ranks < 1 || rank < 0 || rank >= n_ranks) return 0;
  const int64_t n = n_configs > rank ? (n_configs - rank + n_ranks - 1) / n_ranks : 0;
  for (int64_t q = 0; q < n && q < cap && out; q++) out[q] = rank + q * n_ranks;
  return n;
}

}  // extern "C"
