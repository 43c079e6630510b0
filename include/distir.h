/*
 * distir.h -- C ABI of libdistir.so, the B200-native grid-search simulator
 * pass of DistIR (arXiv 2111.05426).
 *
 * "P:<n>" cites /root/reference/PAPER.md line n; "§8c C.x" cites SURVEY.md.
 *
 * The problem: given a model, a hardware
 * description and the D/T/P/K(/batch) space, predict every configuration's
 * runtime and peak memory by simulating its distributed program, drop the
 * configurations over the per-GPU memory limit, and return the top k.
 *
 * One call evaluates a whole grid on the GPU:
 *   a1 enumerate  -- canonical index -> (model, topology, D, T, P, K, B) and
 *                    validity bits (§8c C.1-C.2)
 *   a2 expand     -- D/T/P transform + GPipe schedule (§8c C.3-C.4)
 *   a3 cost       -- FLOPs / F + o; alpha-beta Send, ring AllReduce /
 *                    AllGather (§8c C.5)
 *   a4 timeline   -- start = max(member clocks); end = start + cost
 *                    (§8c C.6)
 *   a5 memory     -- live from creation until last use, per-rank peak
 *                    (§8c C.7)
 *   a6 feasible   -- valid and peak <= capacity; throughput = B / makespan
 *
 *   a7 top-k      -- (throughput desc, peak asc, index asc)
 *   a8 merge      -- across GPUs: one all-gather of the per-GPU top-k
 *
 * Conventions
 *   * Every call returns distir_status; nothing throws or aborts across the
 *     ABI.  A human-readable reason for the last failure on this thread is
 *     returned by distir_last_error().
 *   * Per-configuration outcomes are DATA, not errors: an invalid config
 *     (reason bits 0-4) has makespan = +inf, peak = -1; a valid config over
 *     capacity (bit 5) keeps its simulated makespan and peak; both are
 *     excluded from the top-k.
 *   * Outputs are bit-identical for any sharding, launch shape or GPU count.
 *   * fp64 arithmetic is IEEE binary64 round-to-nearest without FMA
 *     contraction, in the order of §8c C.5.
 *   * A handle is bound to one CUDA device and one stream (when a grid needs
 *     several simulate kernels they run on the handle's private side
 *     streams, forked from and joined back into that stream: the caller sees
 *     stream order as usual); it is not
 *     thread-safe.  Distinct handles are independent.
 *   * The library owns the handle; model/topology arrays are copied at
 *     create.  The caller owns every output buffer and the device workspace
 *     (e.g. a torch uint8 tensor of distir_workspace_size() bytes).
 *   * Limits (DISTIR_E_UNSUPPORTED beyond them): world size <= 64, n_layer
 *     <= 1024, microbatches <= 4096, node_size a power of two, k <= 64,
 *     dp and tp powers of two in explicit configs (stage symmetry); ZeRO
 *     configurations with dp > 1: next_pow2(pp) * dp <= 32 (distir_model).
 */
#ifndef DISTIR_H_
#define DISTIR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DISTIR_OK = 0,
  DISTIR_E_INVALID_ARG = 1,   /* NULL / out-of-range argument, bad spec       */
  DISTIR_E_UNSUPPORTED = 2,   /* outside the limits above                     */
  DISTIR_E_OUT_OF_MEMORY = 3, /* host allocation failed                        */
  DISTIR_E_CUDA = 4,          /* a CUDA runtime call or kernel failed          */
  DISTIR_E_NCCL = 5,          /* NCCL missing or an NCCL call failed           */
  DISTIR_E_WORKSPACE = 6      /* workspace NULL, misaligned or too small       */
} distir_status;

/* Model families: synthetic MLP training, GPT-2 inference. */
enum { DISTIR_MODEL_MLP_TRAIN = 0, DISTIR_MODEL_GPT2_INFER = 1 };

/* Validity / feasibility reason bits (§8c C.2). 0 = feasible. */
enum {
  DISTIR_R_BATCH = 1u << 0,    /* B mod (D*K) != 0                            */
  DISTIR_R_STAGES = 1u << 1,   /* P > n_layer: an empty pipeline stage        */
  DISTIR_R_TP_DIM = 1u << 2,   /* d_model (GPT-2: or vocab_pad) mod T != 0    */
  DISTIR_R_TP_HEADS = 1u << 3, /* GPT-2: n_head mod T != 0                    */
  DISTIR_R_WORLD = 1u << 4,    /* D*T*P > topology.world_max                  */
  DISTIR_R_CAPACITY = 1u << 5  /* valid, but peak bytes > capacity    */
};

/* A model (Table 1).  MLP: n_layer square bias-free layers of
 * width d_model; GPT-2: HF shapes with seq_len tokens per sample, a
 * padded vocabulary and an optional LM head.  dtype_bytes = 2 (16-bit values,
 * P:543); id_bytes = bytes per token id.  schedule (MLP training only): the
 * pipeline schedule of the D/T/P transform, DISTIR_SCHED_GPIPE (north_star)
 * or DISTIR_SCHED_1F1B (the paper's synchronous 1F1B).
 * recompute / zero (MLP training only, 0 or 1, DESIGN
 * readings R8 / R9): the memory-saving variants of the Appendix --
 *   recompute: gradient checkpointing (Fig. 8): a stage keeps its
 *              input and output activations; the activations inside it are
 *              recomputed at the start of its backward, after LossGrad;
 *   zero:      ZeRO-2/3 partitioning (Fig. 9): W_l and its gradient
 *              live on replica l mod D of its (tp, stage) group, which
 *              broadcasts W_l before each forward / backward use and
 *              receives the gradients by a reduce after the stage's backward;
 *              either schedule; configs with D > 1 need next_pow2(pp) * dp
 *              <= 32 (DISTIR_E_UNSUPPORTED).
 *              Broadcast / Reduce cost (g-1) alpha + bytes / bw.
 * Unused fields are ignored. */
enum { DISTIR_SCHED_GPIPE = 0, DISTIR_SCHED_1F1B = 1 };
typedef struct {
  int32_t kind;
  int32_t n_layer, d_model, n_head, seq_len, vocab_pad, n_ctx;
  int32_t dtype_bytes, id_bytes, lm_head;
  int32_t schedule;
  int32_t recompute, zero;
} distir_model;

/* Hardware description ("GPU DRAM bandwidth, kernel launch overhead,
 * and network bandwidths"; §8d D.2).  A group is intra-node iff all members
 * share floor(rank / node_size). */
typedef struct {
  int32_t world_max, node_size;
  double flops_per_s;     /* F: device throughput ("f")               */
  double op_overhead_s;   /* o: fixed per-op overhead               */
  double alpha_intra_s, bw_intra_Bps;
  double alpha_inter_s, bw_inter_Bps;
  int64_t capacity_bytes; /* per-GPU memory limit                   */
  /* Compute-op cost model.  DISTIR_COST_ANALYTIC:
   * flops / F + o.  DISTIR_COST_REGRESSION: the paper's linear-regression
   * cost functions, t = (c0 + s_per_flop * flops) + s_per_byte *
   * bytes, evaluated left to right in binary64 without contraction, where
   * bytes = the sizes of every tensor the op reads or writes (DESIGN R7);
   * the mm_* set applies to MatMul-type ops (Gemm, MatMul, MatMulGrad), the
   * ew_* set to every other compute op.  Coefficients must be finite and
   * >= 0 (ignored under ANALYTIC).  Communication keeps the alpha-beta forms. */
  int32_t cost_model;
  int32_t reserved;       /* must be 0                                      */
  double mm_c0_s, mm_s_per_flop, mm_s_per_byte;
  double ew_c0_s, ew_s_per_flop, ew_s_per_byte;
} distir_topology;
enum { DISTIR_COST_ANALYTIC = 0, DISTIR_COST_REGRESSION = 1 };

/* One explicit configuration (D, T, P, K; P:567 batch).  model and
 * topo index the arrays given to distir_sim_create. */
typedef struct {
  int32_t dp, tp, pp, microbatches;
  int64_t batch;
  int32_t model, topo;
} distir_config;

/* A grid (§8c C.1).  Canonical order: for model in models, for topo in topos,
 * for W in world (ascending powers of two), for (D,T,P) powers of two with
 * D*T*P == W in lexicographic order (masked by dp/tp/pp_mask: bit e allows
 * degree 2^e), for K in Kset(P) ascending, for B in batch ascending.
 * k_mode 0: Kset = {1} if P == 1 else k_set; 1: k_set for every P.
 * synth_count > 0 selects the counter-based synthetic sweep of §8d D.1
 * instead (seed synth_seed, topology topos[r7 mod n_topos]); models/world/
 * batch/k lists are then ignored. */
typedef struct {
  int32_t n_world;
  int32_t world[8];
  int32_t k_mode;
  int32_t n_k;
  int32_t k_set[16];
  int32_t n_batch;
  int64_t batch[32];
  int32_t n_models;
  int32_t models[8];
  int32_t n_topos;
  int32_t topos[8];
  uint32_t dp_mask, tp_mask, pp_mask;
  uint64_t synth_seed;
  int64_t synth_count;
} distir_grid_spec;

/* One top-k record (32 bytes). index = canonical grid index (spec mode) or
 * array position (explicit configs). throughput = batch / makespan. */
typedef struct {
  int64_t index;
  double makespan_s;
  double throughput;
  int64_t peak_bytes;
} distir_topk_entry;

/* Per-evaluation statistics (all over the evaluated shard). */
typedef struct {
  int64_t n_configs;      /* configurations evaluated                        */
  int64_t n_valid;        /* reason bits 0-4 clear                           */
  int64_t n_feasible;     /* reason == 0                                     */
  int64_t op_events;      /* sum over valid configs of the global op count   */
                          /* (a collective counts once; §8c C.3/C.4)         */
  int64_t stage_steps;    /* (op, stage) steps the kernel walked             */
  int64_t n_buckets;      /* distinct warp-shape buckets                     */
  int64_t n_items;        /* warp work items                                 */
  int64_t h2d_bytes;      /* host->device bytes the last eval/upload copied   */
  int64_t d2h_bytes;      /* device->host bytes the last eval copied          */
  /* work the simulate kernels actually performed (physical companions of  */
  /* op_events, which count the logical program):                          */
  int64_t tasks;          /* (microbatch, stage) tasks of the valid configs   */
  int64_t slow_tasks;     /* tasks that left the one-add fast path (a binade  */
                          /* crossing or a stale increment cache)            */
  int64_t wave_steps;     /* warp-level wavefront / co-simulation steps       */
} distir_stats;

typedef struct distir_sim distir_sim;

/* Create a handle: copies models/topologies, validates them, selects
 * cuda_device and binds cuda_stream (a cudaStream_t; NULL = legacy default
 * stream).  *out is set on success.  Errors: INVALID_ARG (NULL, counts,
 * nonsensical fields), UNSUPPORTED (limits), CUDA. */
distir_status distir_sim_create(const distir_model* models, int32_t n_models,
                                const distir_topology* topos, int32_t n_topos,
                                int32_t cuda_device, void* cuda_stream,
                                distir_sim** out);

/* Destroy a handle (NULL is a no-op).  Does not free caller memory. */
void distir_sim_destroy(distir_sim* sim);

/* Number of configurations of a grid spec (host arithmetic, no GPU work). */
distir_status distir_grid_size(const distir_sim* sim, const distir_grid_spec* spec,
                               int64_t* n_configs);

/* Bytes of device workspace needed to evaluate up to n_configs configs with
 * top-k width up to 64 on up to 8 ranks.  The workspace must be 256-byte
 * aligned. */
distir_status distir_workspace_size(const distir_sim* sim, int64_t n_configs,
                                    size_t* bytes);

/* Packed host layout of the per-configuration results for n_configs
 * configurations: byte offsets of makespan / peak / reason (offsets[0..2],
 * offsets[0] == 0) in one host buffer of *bytes bytes.  When the three
 * output pointers of distir_grid_eval / _sharded (single rank) sit at these
 * offsets of one buffer, the results arrive in ONE device->host copy, which
 * also writes the (unspecified) padding between the arrays; any other
 * placement is copied array by array.  Pure host arithmetic. */
distir_status distir_result_layout(const distir_sim* sim, int64_t n_configs, int64_t offsets[3],
                                   size_t* bytes);

/* Evaluate a grid (spec != NULL, configs == NULL) or an explicit list
 * (spec == NULL, configs/n_configs) on this handle's GPU, synchronously.
 * All outputs are HOST buffers owned by the caller:
 *   makespan_out [n] / peak_out [n] / reason_out [n]  (each may be NULL),
 *   topk_out [k], *n_topk_out = min(k, #feasible), stats_out (may be NULL).
 * Host->device copies of the spec/configs and device->host copies of the
 * results happen inside the call.  k in [0, 64]. */
distir_status distir_grid_eval(distir_sim* sim, const distir_grid_spec* spec,
                               const distir_config* configs, int64_t n_configs,
                               int32_t k, void* d_workspace, size_t ws_bytes,
                               double* makespan_out, int64_t* peak_out,
                               uint32_t* reason_out, distir_topk_entry* topk_out,
                               int32_t* n_topk_out, distir_stats* stats_out);

/* Device-resident pipeline, split in two so a timed region can start with
 * every input already in HBM:
 *   distir_grid_upload  copies the spec (or explicit configs) and the decode
 *                       tables into d_workspace (async on the stream) and
 *                       records the shard (rank of n_ranks, round-robin over
 *                       canonical indices: index i belongs to rank i mod n).
 *   distir_grid_launch  runs a1-a7 on the uploaded grid, writing DEVICE
 *                       buffers: d_makespan / d_peak / d_reason indexed by
 *                       shard position q (global index rank + q*n_ranks;
 *                       each may be NULL) and d_topk[k] + *d_n_topk.  Fully
 *                       asynchronous on the stream; no host synchronisation.
 *                       With nccl_comm != NULL (an ncclComm_t whose ranks are
 *                       the upload's n_ranks), the local top-k lists are
 *                       all-gathered and merged on the device as in
 *                       distir_grid_eval_sharded, so d_topk is global.
 * The launch uses the grid most recently uploaded by this handle. */
distir_status distir_grid_upload(distir_sim* sim, const distir_grid_spec* spec,
                                 const distir_config* configs, int64_t n_configs,
                                 int32_t rank, int32_t n_ranks, void* d_workspace,
                                 size_t ws_bytes, int64_t* n_local_out);
distir_status distir_grid_launch(distir_sim* sim, int32_t k, void* nccl_comm,
                                 void* d_workspace, size_t ws_bytes, double* d_makespan,
                                 int64_t* d_peak, uint32_t* d_reason,
                                 distir_topk_entry* d_topk, int32_t* d_n_topk);

/* Kernel-level timing of launches, measured with CUDA events recorded on
 * the handle's stream around each phase of every launch while enabled.
 * distir_profile(sim, enable, out): if out != NULL, synchronises, writes the
 * totals accumulated since the previous read and resets them; then turns
 * recording on (enable = 1) or off (0). */
typedef struct {
  int64_t launches;     /* distir_grid_launch / eval calls recorded          */
  int64_t kernels;      /* kernels this library launched in them             */
  double ms_prepare;    /* reset + enumerate + plan + scatter                 */
  double ms_simulate;   /* k_simulate: expand, cost, timeline, memory (a2-a6) */
  double ms_topk;       /* local top-k (a7)                                   */
  double ms_merge;      /* all-gather + merge (a8), 0 without NCCL            */
} distir_profile_data;

distir_status distir_profile(distir_sim* sim, int32_t enable, distir_profile_data* out);

/* Read the statistics of the last launch (synchronises the stream). */
distir_status distir_last_stats(distir_sim* sim, void* d_workspace, distir_stats* out);

/* Multi-GPU evaluation (one process per GPU).  This rank evaluates indices
 * i with i mod n_ranks == rank, then all-gathers the k-entry local top-k
 * lists over the NCCL communicator nccl_comm (an ncclComm_t of n_ranks
 * ranks, this process = rank) and merges them on the device with the same
 * total order, so every rank returns the identical global top-k.  Per-config
 * host outputs are GLOBAL-indexed [grid size]; only this rank's indices are
 * written.  nccl_comm may be NULL only when n_ranks == 1. */
distir_status distir_grid_eval_sharded(distir_sim* sim, const distir_grid_spec* spec,
                                       const distir_config* configs, int64_t n_configs,
                                       int32_t rank, int32_t n_ranks, void* nccl_comm,
                                       int32_t k, void* d_workspace, size_t ws_bytes,
                                       double* makespan_out, int64_t* peak_out,
                                       uint32_t* reason_out, distir_topk_entry* topk_out,
                                       int32_t* n_topk_out, distir_stats* stats_out);

/* Device merge of top-k lists (row a8: the step distir_grid_launch /
 * distir_grid_eval_sharded run after the NCCL all-gather of the per-rank
 * lists; north_star "only the final top-k merged").  Selects the first k
 * records of the union of n_lists sorted lists by the C.8 order --
 * throughput descending, then peak_bytes ascending, then index ascending
 * -- on this handle's device, asynchronously on its stream.
 *   d_lists   DEVICE, n_lists x k_in records, list l at d_lists[l * k_in],
 *             each sorted by the C.8 order (as distir_grid_launch writes its
 *             d_topk); records are identified by index, which must be
 *             distinct across the lists.
 *   d_list_n  DEVICE, n_lists counts (clamped to k_in), or NULL: then list
 *             l's records are its leading entries with index >= 0 (the
 *             padding distir_grid_launch writes past *d_n_topk is index -1).
 *   d_out     DEVICE, k records: the merged list, padded with index -1;
 *   d_n_out   DEVICE, the number of real records, min(k, sum of counts).
 * Limits: 1 <= n_lists <= 1024, 0 <= k_in, k <= 64.  d_out must not overlap
 * d_lists.  Errors: INVALID_ARG, CUDA. */
distir_status distir_topk_merge(distir_sim* sim, const distir_topk_entry* d_lists,
                                const int32_t* d_list_n, int32_t n_lists, int32_t k_in,
                                int32_t k, distir_topk_entry* d_out, int32_t* d_n_out);

/* NCCL bootstrap helpers (NCCL is loaded at run time with dlopen, so the
 * library itself has no link-time NCCL dependency).  The unique id is 128
 * opaque bytes to broadcast from rank 0 (e.g. through torch.distributed). */
distir_status distir_nccl_unique_id(uint8_t id_out[128]);
distir_status distir_nccl_comm_init(const uint8_t id[128], int32_t n_ranks, int32_t rank,
                                    int32_t cuda_device, void** comm_out);
distir_status distir_nccl_comm_destroy(void* comm);

/* Shard planner (host arithmetic, no GPU): the number of global indices of a
 * grid of n_configs that rank owns, and the first cap of them in order. */
int64_t distir_shard_indices(int64_t n_configs, int32_t rank, int32_t n_ranks,
                             int64_t* out, int64_t cap);

/* ---------------------------------------------- raw-program mode (f3) ----
 * Simulate arbitrary explicit DistIR programs (straight-line ops,
 * each on a device set; an op starts when all its devices are free and blocks
 * them all; values live from creation to last use), e.g. the Fig. 3
 * traces or hand-written strategies.  All arrays are HOST arrays:
 *   programs[i]: n_dev devices (1..64); its ops are ops[op_base, op_base +
 *   n_ops); its values are values[value_base, value_base + n_values); its
 *   per-device outputs go to clock_out / peak_out[out_base, out_base + n_dev).
 *   ops[j]: cost in seconds (>= 0); device ids idx[dev_off, dev_off + n_dev),
 *   input value ids idx[in_off, ...+n_in), output ids idx[out_off, ...+n_out)
 *   -- ids are local to the program.
 *   values[v]: device, flags (bit 0 parameter: live from t = 0; bit 1
 *   returned: never freed), bytes.
 * Outputs (host; any but makespan_out may be NULL): makespan per program,
 * final clock and peak live bytes per device, start and end time per op.
 * Programs are checked on the host before any GPU work: every op input
 * must be a parameter or an earlier op's output, every value is defined at
 * most once, an op's outputs must live on one of its devices, and the
 * programs' op, value and output ranges must not overlap.
 * Synchronous.  Errors: INVALID_ARG for out-of-range ids/offsets or a
 * program that breaks these rules. */
typedef struct {
  int32_t n_dev, dev_off, n_in, in_off, n_out, out_off;
  double cost;
} distir_raw_op;
typedef struct {
  int32_t dev, flags;
  int64_t bytes;
} distir_raw_value;
typedef struct {
  int32_t n_dev, n_ops, op_base, n_values, value_base, out_base;
} distir_raw_program;

distir_status distir_raw_workspace_size(int32_t n_programs, int64_t n_ops, int64_t n_idx,
                                        int64_t n_values, int64_t n_out, size_t* bytes);
distir_status distir_raw_eval(distir_sim* sim, const distir_raw_program* programs,
                              int32_t n_programs, const distir_raw_op* ops, int64_t n_ops,
                              const int32_t* idx, int64_t n_idx, const distir_raw_value* values,
                              int64_t n_values, int64_t n_out, void* d_workspace, size_t ws_bytes,
                              double* makespan_out, double* clock_out, int64_t* peak_out,
                              double* op_start_out, double* op_end_out);

/* Thread-local description of the last error ("" if none). */
const char* distir_last_error(void);

/* Library version string. */
const char* distir_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DISTIR_H_ */
