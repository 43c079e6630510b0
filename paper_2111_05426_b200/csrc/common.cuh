// common.cuh -- device-side data layout of the DistIR grid pass (product).
//
// Everything the kernels read lives in the caller-owned workspace (HBM):
//   WsHeader | SpecBlock | explicit configs | bucket table | per-config
//   bucket ids | permutation | work items | per-config results | top-k
// Offsets are computed by the host planner (distir.cu, ws_layout()).
#pragma once
#include <cstdint>

namespace distir {

constexpr int kMaxModels = 64;      // models / topologies copied at create
constexpr int kMaxTopos = 64;
constexpr int kMaxEntries = 96;     // (W, D, T, P) triples of a grid spec
constexpr int kMaxWorld = 64;       // world size limit (2 stages per lane)
constexpr int kMaxK = 64;           // top-k width
constexpr int kMaxRanks = 8;        // GPUs merged by the all-gather
constexpr int kNumBuckets = 4096;   // hash slots for warp-shape buckets
constexpr int kOverflowBucket = kNumBuckets;  // catch-alls: + kind (1 config / warp)
constexpr int kBucketSlots = kNumBuckets + 4;   // + MLP, GPT-2, MLP-1F1B, MLP-ZeRO catch-alls
// Simulate kernels ("groups"): model kind x schedule mode.  Modes 0-2: one
// lane walks a whole configuration in program order, P <= 1 / 2 / 4 stages;
// modes 3-4: wavefront, one lane per stage (mode 4: two stages per lane,
// 32 < P <= 64, and the catch-all buckets); mode 5 (MLP only): the 1F1B
// co-simulation, one lane per stage, P <= 32; mode 6 (MLP only): ZeRO (f4),
// one lane per (stage, replica), next_pow2(P) * D <= 32; mode 7 (MLP only):
// 1F1B with two stages per lane, 32 < P <= 64, and the 1F1B catch-all;
// mode 8 (MLP only): mode 3 for warps that walk every task op by op
// (mlp_plain_shape), without the cached paths -- fewer registers, more
// warps per SM.
constexpr int kModes = 9;
constexpr int kGroups = 2 * kModes;
constexpr int kNumClasses = 40;     // weight classes (LPT order of items)
constexpr int kMaxSplit = 5;        // configs per item divided by up to 2^5
constexpr double kPlanBudgetX = 1.0; // k_plan splits while items <= X x resident warps
struct PlanBudget {                 // resident warps of each simulate kernel
  uint32_t warps[kGroups];
  uint32_t launched;                  // the simulate kernels enqueued (SpecBlock.f1b)
};
// Binade tables (exact_add.cuh BinTab) of the wavefront simulate kernels:
// the first kTabCfgs configurations of a warp get one.
constexpr int kTabCfgs = 4;          // MLP kernels: tables for the first 4 configurations
constexpr int kTabCfgsGpt2 = 16;     // GPT-2 kernels: every configuration of a warp (S >= 2)
constexpr int kTabBinadesGpt2 = 16;   // 3 task segments; from the binade below the
                                      // first task to the makespan bound
constexpr int kTabBinadesMlp = 24;    // 3 forward + 4 backward task segments
constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;
constexpr uint32_t kCapacityBit = 1u << 5;   // DISTIR_R_CAPACITY
constexpr int kTopkThreads = 256;   // threads of a block-wide top-k merge (k_topk_merge)
constexpr int kMergeMaxLists = 4 * kTopkThreads;   // distir_topk_merge: 4 lists per thread
constexpr int kPartLists = 8192;     // simulate blocks' partial top-k lists per launch
constexpr int kSelectThreads = 256;  // k_topk_select: one block
constexpr int kSelectCap = 1024;     // candidates it selects from in shared memory

enum Mode : int32_t { MODE_GRID = 0, MODE_SYNTH = 1, MODE_EXPLICIT = 2 };

struct DModel {          // distir_model, int32
  int32_t kind, L, d, h, S, V, nctx, e, ide, lm, sched;
  int32_t rc, zero;      // f4: gradient checkpointing, ZeRO-2/3 (MLP training)
};

struct DTopo {           // distir_topology
  int32_t world_max, node_size;
  double F, o, a_intra, bw_intra, a_inter, bw_inter;
  int64_t capacity;
  int32_t cost_model;    // 0 analytic, 1 regression
  double mm_c0, mm_flop, mm_byte, ew_c0, ew_flop, ew_byte;
};

struct DEntry {          // one (D, T, P) triple of the grid, canonical order
  int32_t D, T, P, nK;
  int64_t cum;           // configs of this (model, topo) before this entry
};

struct DExplicit {       // distir_config (32 bytes, same layout)
  int32_t dp, tp, pp, K;
  int64_t B;
  int32_t model, topo;
};

struct SpecBlock {
  int32_t mode;
  int32_t n_models, n_topos;          // spec lists (grid / synth)
  int32_t model_ids[8], topo_ids[8];
  int32_t n_entries;
  DEntry entries[kMaxEntries];
  int32_t k_mode, n_k;
  int32_t k_set[16];
  int32_t n_batch;
  int64_t batch[32];
  int64_t per_mt;                     // configs per (model, topo) pair
  uint64_t synth_seed;
  int64_t n_total;                    // configs of the whole grid
  int32_t rank, n_ranks;              // shard: global i = rank + q * n_ranks
  int64_t n_local;
  uint32_t f1b;                       // simulate kernels to launch: bit kind * kModes
                                      // + mode (distir.cu gbit)
  DModel models[kMaxModels];          // handle tables
  DTopo topos[kMaxTopos];
};

struct WsHeader {
  unsigned int item_counter[kGroups]; // persistent-kernel work queues
  unsigned int group_begin[kGroups + 1];  // item ranges per simulate kernel
  unsigned int n_items;
  unsigned int n_buckets;
  unsigned long long op_events;
  unsigned long long stage_steps;
  unsigned long long n_valid;
  unsigned long long n_feasible;
  unsigned long long tasks;           // (microbatch, stage) tasks of the valid configs
  unsigned long long slow_tasks;      // lane-level slow-path entries (k_simulate)
  unsigned long long wave_steps;      // warp-level wavefront steps (k_simulate)
  unsigned int cfg_total;
  unsigned long long topk_thresh;      // max over simulate blocks of their k-th throughput bits
};

struct Bucket {          // per hash slot (plus one overflow slot)
  uint32_t key;          // kind | (P-1) << 1 | (L-1) << 7 | min(K,255) << 17 |
                         // sched << 25 | log2(D) << 26 | ZeRO << 29 | recompute << 30
  uint32_t count;        // configs in the bucket
  uint32_t cfg_base;     // first position in perm
  uint32_t item_base;    // first work item
  uint32_t cursor;       // scatter cursor
  uint16_t lanes;        // lanes per config S (power of two <= 32)
  uint16_t cpw;          // configs per work item (<= 32 / lanes)
  uint16_t cls;          // weight class
  uint16_t group;        // simulate kernel: kind * kModes + mode
  uint32_t item_off;     // offset within (group, class)
};

struct Item {            // one warp's worth of configs of one bucket
  uint32_t first;        // position in the permuted config list
  uint16_t bucket;
  uint8_t n;             // configs in this item
  uint8_t lg_lanes;      // log2(lanes per config)
};

// A decoded configuration as k_enumerate packs it and k_scatter permutes it
// into warp order, so k_simulate reads each config with one load instead of
// re-decoding (the grid decode is a binary search over a table in HBM).
struct PCfg {
  int64_t B;
  uint32_t q;            // shard position (output index)
  uint16_t K;
  uint8_t P;
  uint8_t model;         // index into SpecBlock.models; kSynthModel: synthetic
  uint8_t topo;
  uint8_t lgD, lgT;
  uint8_t pad;
};
constexpr uint8_t kSynthModel = 0xFF;   // model drawn by the synthetic sweep (re-decoded)

struct TopkRec {         // == distir_topk_entry
  int64_t index;
  double makespan;
  double throughput;
  int64_t peak;
};

// Row a7 inside the simulate kernels: each warp keeps a running top-k, each
// block merges its warps' lists into part[blockIdx] (k records, count in
// part_n) and, when that list is full, raises *thresh to its k-th key's
// throughput bits; k_topk_select then picks the top k of the records at or
// above the threshold (every global top-k record is: the block holding the
// largest k-th throughput alone has k records at least that good).
struct SimTopk {
  int k;
  TopkRec* part;        // this kernel's gridDim.x lists of k records
  int* part_n;
  unsigned long long* thresh;
};

}  // namespace distir

namespace distir {
// ----------------------------------------------------- raw programs (f3) ----
struct RawOp {           // == distir_raw_op (32 bytes)
  int32_t n_dev, dev_off, n_in, in_off, n_out, out_off;
  double cost;
};
struct RawValue {        // == distir_raw_value (16 bytes)
  int32_t dev, flags;    // flags: bit0 parameter, bit1 returned
  int64_t bytes;
};
struct RawProgram {      // == distir_raw_program (24 bytes)
  int32_t n_dev, n_ops, op_base, n_values, value_base, out_base;
};
constexpr int kRawMaxDev = 64;
}  // namespace distir
