/*
 * hzp_b200.h — C-ABI of the B200-native AsyncHZP hot path.
 *
 * One shared library (paper_2510_20111_b200/libhzp_b200.so) exports these
 * symbols.  Plain C types only (no torch, no C++); every call returns an
 * int status (HZP_OK or an HZP_ERR_* code mirroring the reference's C++
 * exception codes) and hzp_last_error() gives a thread-local message.
 *
 * The reference (arxiv 2510.20111 artifact, /root/reference/proj) has no C
 * ABI; it is a C++ namespace API.  Each entry point below cites the
 * reference interface it replaces.  The C++ drop-in (same names/types as the
 * reference) lives in paper_2510_20111_b200/csrc/hzp/{config,sched}.hpp and
 * is what these wrappers call for the host-side pieces.
 */
#ifndef HZP_B200_H_
#define HZP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
/* Mirrors ValidationError::Code (include/hzp/config.hpp:68-77),
 * CollectiveError::Code (include/hzp/collective.hpp:18-27),
 * SchedError::Code (include/hzp/sched.hpp:55-64), MemoryError
 * (include/hzp/memory.hpp:26-35) and EquivalenceFailure (train.hpp:94-98). */
enum {
  HZP_OK = 0,
  HZP_ERR_NON_DIVISIBLE = 1,     /* ValidationError::NonDivisible */
  HZP_ERR_EMPTY_MODEL = 2,       /* ValidationError::EmptyModel */
  HZP_ERR_BAD_FIELD = 3,         /* ValidationError::BadField */
  HZP_ERR_SHAPE_MISMATCH = 4,    /* CollectiveError::ShapeMismatch */
  HZP_ERR_DTYPE_UNSUPPORTED = 5, /* CollectiveError::DTypeUnsupported */
  HZP_ERR_INVALID_POLICY = 6,    /* SchedError::InvalidPolicy */
  HZP_ERR_DEADLOCK = 7,          /* SchedError::DeadlockDetected */
  HZP_ERR_MEMORY = 8,            /* MemoryError / device allocation */
  HZP_ERR_EQUIVALENCE = 9,       /* EquivalenceFailure */
  HZP_ERR_CUDA = 10,             /* any CUDA runtime / driver failure */
  HZP_ERR_ARG = 11               /* null pointer / out-of-range argument */
};

const char* hzp_last_error(void);
const char* hzp_version(void);

/* ---- domain (include/hzp/config.hpp:16-66) ------------------------------ */
typedef struct {
  int dp, z1, z2, z3; /* ParallelConfig: data-parallel size, optimizer /   */
  int pp, vpp, cp, tp; /* gradient / parameter sharding group sizes, outer */
} hzp_parallel;        /* dims (pp, vpp, cp, tp >= 1)                       */

typedef struct {
  int64_t num_layers, params_per_layer, embedding_params;
  int64_t seq_len, micro_batch_size, num_microbatches;
  double flops_per_token_per_layer;
  int64_t hidden_size;
} hzp_model_spec; /* ModelSpec (config.hpp:16-31) */

typedef struct {
  int num_nodes, ranks_per_node;
  double intra_bw, inter_bw, intra_latency, inter_latency;
  double device_flops;
} hzp_cost; /* Topology (config.hpp:44-54) + CostModel::device_flops (collective.hpp:63-67) */

enum { HZP_GROUP_Z1 = 0, HZP_GROUP_Z2 = 1, HZP_GROUP_Z3 = 2, HZP_GROUP_DZP = 3 };

/* shard_elems (include/hzp/memory.hpp:37-38): ceil(n / parts). */
int64_t hzp_shard_elems(int64_t n, int64_t parts);

/* validate_config (include/hzp/config.hpp:89-91). */
int hzp_validate(const hzp_model_spec* spec, const hzp_parallel* par, const hzp_cost* topo);

/* build_process_groups (include/hzp/config.hpp:96-97) for one GroupKind:
 * writes groups back to back into ranks_out (cap ints), *group_size and
 * *n_groups.  Ranks of group g are ranks_out[g*group_size ...]. */
int hzp_groups(const hzp_parallel* par, int kind, int* ranks_out, int cap, int* group_size,
               int* n_groups);

/* ---- scheduler (include/hzp/sched.hpp:20-137) --------------------------- */
/* TaskKind order matches sched.hpp:20-29. */
enum {
  HZP_TASK_FWD = 0, HZP_TASK_BWD = 1, HZP_TASK_FWD_RECOMPUTE = 2, HZP_TASK_AG_PARAM = 3,
  HZP_TASK_RS_GRAD = 4, HZP_TASK_AR_DZP = 5, HZP_TASK_OPT_STEP = 6, HZP_TASK_AG_POST = 7
};
enum { HZP_STREAM_COMPUTE = 0, HZP_STREAM_AG = 1, HZP_STREAM_RS = 2 };
enum { HZP_MODE_VANILLA = 0, HZP_MODE_ASYNC = 1 };

typedef struct hzp_graph hzp_graph;

typedef struct {
  int id, kind, layer, microbatch, virtual_stage, pass;
  double duration;
  int64_t bytes;
  int num_deps;
  const int* deps; /* valid until the graph is destroyed */
} hzp_task;        /* Task (sched.hpp:35-45) */

/* build_task_graph (sched.hpp:90-91).  defer_rs / rank mirror GraphPolicy
 * (sched.hpp:66-76) with the default one-F-one-B-per-microbatch order. */
int hzp_graph_build(const hzp_model_spec* spec, const hzp_parallel* par, const hzp_cost* cost,
                    int defer_rs, int rank, hzp_graph** out);

/* ReuseReport (pipeline.hpp:57). */
typedef struct {
  int r1_eliminated_ag, r2_merged_rs, r3_eliminated_ag;
  int64_t extra_cached_bytes;
} hzp_reuse_report;

/* The CLI's graph (hzpsim.cpp:111-127): build_task_graph over `rank`'s slot
 * order of the pipeline schedule (build_schedule, pipeline.cpp:84-105: 1F1B,
 * interleaved when par->vpp > 1), then apply_reuse (pipeline.cpp:167-279)
 * when `reuse`, then recompute_rule (pipeline.cpp:281-318) when `recompute`.
 * `report` (optional) receives the reuse counters. */
int hzp_graph_build_pipeline(const hzp_model_spec* spec, const hzp_parallel* par, const hzp_cost* cost,
                             int defer_rs, int rank, int reuse, int recompute, hzp_reuse_report* report,
                             hzp_graph** out);
void hzp_graph_destroy(hzp_graph* g);
int hzp_graph_size(const hzp_graph* g);
int hzp_graph_task(const hzp_graph* g, int i, hzp_task* out);
int64_t hzp_graph_ag_slot_bytes(const hzp_graph* g); /* TaskGraph::ag_slot_bytes */
int64_t hzp_graph_grad_buf_bytes(const hzp_graph* g); /* TaskGraph::grad_buf_bytes */

/* derive_prelaunch_depth (sched.hpp:110-112). */
int hzp_derive_prelaunch_depth(const hzp_graph* g, int64_t free_budget);

/* make_pools (sched.hpp:108): AG pool = depth slots of ag_slot_bytes,
 * RS pool = rs_slots slots of grad_buf_bytes. */
typedef struct {
  int64_t capacity;
  int slot_count;
  int64_t slot_bytes;
} hzp_pool;
int hzp_make_pools(const hzp_graph* g, int depth, int rs_slots, hzp_pool* ag, hzp_pool* rs);

/* simulate (sched.hpp:137): start/end per task (arrays of hzp_graph_size). */
typedef struct {
  double makespan, compute_idle, compute_busy;
} hzp_sim_summary;
int hzp_simulate(const hzp_graph* g, int depth, int rs_slots, int mode, double* start,
                 double* end, hzp_sim_summary* summary);

/* Static-memory ledger (replaces hzp::ledger, memory.hpp:47 / memory.cpp:35-45):
 * per-rank bytes of bf16 params / fp32 grads / master / m / v shards. */
typedef struct {
  int64_t params_bf16, grads_fp32, replica_fp32, momentum_fp32, variance_fp32, total_static;
} hzp_ledger;
int hzp_memory_ledger(const hzp_model_spec* spec, const hzp_parallel* par, hzp_ledger* out);

/* Pool occupancy / fragmentation / peak gradient-buffer bytes of a timeline
 * (replaces hzp::memory_trace, sched.hpp:139-149 / sched.cpp:389-466).  With
 * start == end == NULL the timeline is simulate(g, depth, rs_slots, mode);
 * otherwise start[i] / end[i] are MEASURED task times (e.g. hzp_timeline) and
 * the release points, busy time and memory samples are derived from them by
 * the same rules.  static_bytes = ledger.total_static.  Samples (time, bytes
 * incl. static) are written up to cap; n_samples is the full count. */
typedef struct {
  int64_t peak_bytes;             /* static + peak dynamic */
  double fragmentation;           /* (reserved pools - max live pools) / reserved */
  int64_t peak_grad_buffer_bytes; /* live unsharded-gradient buffers x rs slot bytes */
  int64_t peak_memory;            /* Timeline::peak_memory (dynamic only) */
  double makespan;
  int n_samples;
} hzp_memory_report;
int hzp_memory_trace(const hzp_graph* g, int depth, int rs_slots, int mode, const double* start,
                     const double* end, int64_t static_bytes, hzp_memory_report* out, double* sample_t,
                     int64_t* sample_bytes, int cap);
/* Model FLOPs / (makespan x peak_flops) (replaces hzp::utilization_report,
 * sched.hpp:151-152 / sched.cpp:468-477); timeline chosen as above. */
int hzp_utilization_report(const hzp_graph* g, int depth, int rs_slots, int mode, const double* start,
                           const double* end, double peak_flops, double* out);

/* LaunchPlan (new): the per-task issue record the device executor follows.
 * slot = k % depth for the k-th AG-pool task, k % rs_slots for the k-th RS
 * task, -1 otherwise; ring_wait = the task whose completion frees that slot
 * (sched.cpp:285-309 rule), -1 if none. */
typedef struct {
  int id, kind, layer, microbatch, stream, slot, ring_wait;
  int num_waits;
  const int* waits; /* deps + ring_wait; valid until the graph is destroyed */
} hzp_plan_entry;
int hzp_plan_entry_get(const hzp_graph* g, int depth, int rs_slots, int i, hzp_plan_entry* out);

/* Host-side work decomposition of the P2P passes for one rank (no GPU):
 * tiles of the layer-wise AG (per layer), the RS (per layer) and the fused
 * Z1 stage, exactly as the device kernels consume them.  layer_off/size: the
 * model's flat layer ranges (train.cpp:42-53 layout); working_bytes 2|4.
 * ag_off/rs_off receive L+1 prefix offsets into `out`; *z1_off / *z1_n the
 * Z1 range.  *n_out = total tiles (call with out=NULL to size). */
typedef struct {
  int64_t a_off, b_off, c_off;
  uint64_t mask;
  int32_t len;
  int16_t local, src;
  int32_t vec, pad_;
} hzp_comm_tile;
int hzp_comm_tiles(const hzp_parallel* par, int64_t P, const int64_t* layer_off,
                   const int64_t* layer_size, int num_layers, int rank, int working_bytes,
                   hzp_comm_tile* out, int cap, int* n_out, int* ag_off, int* rs_off,
                   int* z1_off, int* z1_n);

/* ---- device engine ------------------------------------------------------ */
/* Model families.  HZP_MODEL_MLP is the reference's model (tanh MLP, loss
 * sum(y^2)/(2*B*out), flat W|b layout per layer, train.cpp:29-150).
 * HZP_MODEL_GPT is the GPU-scale decoder (pre-LN, GELU MLP, causal MHA,
 * untied LM head) whose flat layout is documented in DESIGN.md. */
enum { HZP_MODEL_MLP = 0, HZP_MODEL_GPT = 1 };
enum { HZP_PREC_FP32 = 0, HZP_PREC_BF16 = 1 };

typedef struct {
  int model;          /* HZP_MODEL_* */
  int precision;      /* HZP_PREC_FP32: fp32 working copy + fp32 GEMMs (parity tier B);
                         HZP_PREC_BF16: bf16 working copy + tcgen05 bf16 GEMMs */
  int num_dims;       /* MLP: dims[0..num_dims-1] (input width first) */
  int dims[32];
  int gpt_layers, gpt_hidden, gpt_heads, gpt_ffn, gpt_vocab, gpt_seq;
  int batch;          /* MLP: rows per microbatch; GPT: sequences per microbatch */
  int num_microbatches;
  hzp_parallel par;
  int prelaunch_depth; /* AG ring slots (reference default 2, hzpsim.cpp:95) */
  int rs_slots;        /* RS ring slots (reference default 1, hzpsim.cpp:96) */
  int wgrad_slots;     /* physical gradient buffers peers pull from (>= 2) */
  int mode;            /* HZP_MODE_ASYNC or HZP_MODE_VANILLA */
  double lr, beta1, beta2, eps; /* AdamParams (train.hpp:22-27) */
  double grad_scale;   /* RS cast/scale factor; 1.0 = reference semantics */
  int device;          /* CUDA ordinal this process drives */
  int my_rank;         /* global rank driven by this process, or -1 = emulate all
                          dp ranks on `device` (single-process parity mode) */
  int timeline;        /* record per-task CUDA events (measured timeline) */
  /* GPT only: mixture-of-experts feed-forward (0 = dense).  Each block's FFN
   * becomes gpt_experts GELU experts of width gpt_ffn with a top-gpt_topk
   * router; gpt_capacity = slots per expert per microbatch (0 = 1.25 x
   * topk x tokens / experts, rounded up to 128). */
  int gpt_experts, gpt_topk, gpt_capacity;
  /* 1 = apply the CLI's parameter reuse to the step's graph (apply_reuse,
   * pipeline.cpp:167-279; hzpsim.cpp:126).  At pp = 1 only R3 fires: every
   * forward after the first reads microbatch 0's forward all-gather, which
   * lands in a per-layer side cache (full bf16 layer per layer) instead of a
   * ring slot; backward all-gathers keep the ring. */
  int reuse;
  /* 1 = activation recomputation (recompute_rule, pipeline.cpp:281-318): a
   * FWD-recompute task before every BWD.  GPT blocks then keep only their
   * input and share one activation set, rebuilt by the recompute (the
   * embedding / head keep their outputs: their recompute is a no-op). */
  int recompute;
  /* GPT only: 1 = SwiGLU feed-forward (LLaMA-style: fc1 [2 gpt_ffn, h] = gate
   * | up, act = silu(gate) * up, fc2 [h, gpt_ffn], no FFN biases), for the
   * dense blocks and every MoE expert. */
  int gpt_swiglu;
} hzp_engine_config;

typedef struct hzp_ctx hzp_ctx;

int hzp_ctx_create(const hzp_engine_config* cfg, hzp_ctx** out);
void hzp_ctx_destroy(hzp_ctx* ctx);

/* Layout facts of the ctx's model: P, s1, s2, s3, layer count and each
 * layer's [offset, size) in the flat vector (layer_views, train.cpp:42-53). */
int hzp_ctx_layout(const hzp_ctx* ctx, int64_t* P, int64_t* s1, int64_t* s2, int64_t* s3,
                   int* num_layers);
int hzp_ctx_layer_range(const hzp_ctx* ctx, int layer, int64_t* offset, int64_t* size);

/* Multi-process wiring (one process per GPU): hzp_ctx_ipc_handle writes this
 * rank's share record (pid + POSIX fds of its cuMem arena and, on a group's
 * first rank, of the Z3 / Z2 NVLS multicast objects; opaque bytes to the
 * caller); after an all-gather of the records over the control plane,
 * hzp_ctx_open_peers maps every peer's arena (pidfd_getfd +
 * cuMemImportFromShareableHandle) and binds this rank's AG / gradient rings
 * into its groups' multicast objects.  All ranks must call it concurrently. */
int hzp_ctx_ipc_handle(hzp_ctx* ctx, void* buf, size_t* len);
int hzp_ctx_open_peers(hzp_ctx* ctx, const void* handles, size_t handle_len, int n_ranks);

/* ShardedState mirror (train.hpp:73-83).  field: 0 param_shard (working
 * dtype: fp32 or bf16 bits), 1 grad_shard (fp32), 2 master, 3 momentum,
 * 4 variance (fp32).  Host buffers; rank must be driven by this ctx. */
enum { HZP_F_PARAM = 0, HZP_F_GRAD = 1, HZP_F_MASTER = 2, HZP_F_MOM = 3, HZP_F_VAR = 4 };
int hzp_state_upload(hzp_ctx* ctx, int rank, int field, const void* host, int64_t n);
int hzp_state_download(hzp_ctx* ctx, int rank, int field, void* host, int64_t n);
int hzp_state_set_step(hzp_ctx* ctx, int rank, int adam_step);
/* The Adam step counter of a driven rank (checkpointing). */
int hzp_state_get_step(const hzp_ctx* ctx, int rank, int* adam_step);
/* shard_init (train.cpp:224-253) done on the host by the caller and
 * uploaded, or seeded on the device for throughput runs: */
int hzp_state_init_random(hzp_ctx* ctx, uint64_t seed, double scale);

/* train_step_hzp (train.hpp:114-119) on the device, walking the LaunchPlan.
 * inputs: MLP → fp32 [local_ranks][num_mb][batch][dims0];
 *         GPT → int32 token ids [local_ranks][num_mb][batch][seq+1].
 * inputs_on_device != 0: `inputs` is a device pointer; else a host pointer
 * (copied H2D on the ctx's stream inside the step).  losses_out
 * (host, [local_ranks], optional) receives per-rank summed losses (D2H). */
/* Reference-faithful synthetic inputs (replace shard_init / seeded_uniform /
 * run_case seeding, train.cpp:17-27, 224-253, 501-508):
 *   hzp_seeded_span: out[i] = float(seeded_uniform(P, seed)[first + i]) * scale
 *     (0 past P: the zero padding of the flat vector);
 *   hzp_state_init_seeded: every driven rank's master chunk = that vector's
 *     Z1 chunk, working copy = its Z3 shard (bf16 RNE in bf16 mode), m = v =
 *     grad = 0, step 0 (scale 1 = the reference's shard_init bit for bit);
 *   hzp_make_tokens: the run_case stream of (step, rank, microbatch),
 *     mt19937_64(seed ^ 0x9E3779B97F4A7C15 * (step*1024 + rank*32 + mb + 1)),
 *     token = floor(((raw >> 11) * 2^-53) * vocab). */
int hzp_seeded_span(uint64_t seed, int64_t P, int64_t first, int64_t n, double scale, float* out);
int hzp_state_init_seeded(hzp_ctx* ctx, uint64_t seed, double scale);
int hzp_make_tokens(uint64_t seed, int step, int rank, int microbatch, int64_t n, int vocab, int32_t* out);

int hzp_step(hzp_ctx* ctx, const void* inputs, int inputs_on_device, float* losses_out);
int hzp_sync(hzp_ctx* ctx);

/* Launch log: the kernels issued by the last step, in issue order, each with
 * the reference task ids it covers (SURVEY §7.3-8 parity of launch order). */
typedef struct {
  int task_id;   /* reference task id (first covered) */
  int kind;      /* HZP_TASK_* */
  int layer, microbatch, stream, slot;
  int covered_first, covered_last; /* fused kernels cover a task id range */
} hzp_launch_rec;
int hzp_launch_log(const hzp_ctx* ctx, hzp_launch_rec* out, int cap, int* n);

/* Measured timeline of the last step (requires cfg.timeline): per task
 * start/end in ms relative to step start, and the compute-stream idle
 * (= last compute end - sum compute busy, sched.cpp:341-350). */
int hzp_timeline(const hzp_ctx* ctx, double* start_ms, double* end_ms, int cap, int* n,
                 double* compute_idle_ms, double* compute_busy_ms, double* makespan_ms);
/* Per-layer optimizer (Z1) times of the last step (requires cfg.timeline;
 * async mode: *n = layers, vanilla: *n = 0 — one tail kernel): ms from step
 * start when the layer's gradient was final on this rank, when every rank it
 * reads from / pushes into had posted GradReady, and when its kernel ended. */
int hzp_z1_timeline(const hzp_ctx* ctx, double* ready_ms, double* start_ms, double* end_ms, int cap, int* n);
/* Turn per-task event recording on/off for the following steps (events are
 * created on first use), so a timed run can be measured untouched and one
 * extra step recorded for hzp_timeline. */
int hzp_set_timeline(hzp_ctx* ctx, int on);

/* Extra device work counters (kernels launched by the last step). */
int hzp_ctx_launch_count(const hzp_ctx* ctx, int64_t* kernels);
/* Total kernels this library has launched in the process (every launch site
 * counts itself) — the bench's gpu_launches evidence. */
uint64_t hzp_kernel_launches(void);
/* The ctx's CUDA streams (which: HZP_STREAM_*) as cudaStream_t, so callers
 * can time the step with events on the stream the work runs on. */
int hzp_ctx_stream(const hzp_ctx* ctx, int which, void** stream);
/* Per-GEMM timing for the roofline: while on, every tcgen05 GEMM launch is
 * bracketed by CUDA events; read returns (and clears) the summed algorithmic
 * FLOPs, summed kernel milliseconds and launch count. */
int hzp_gemm_profile(int on);
int hzp_gemm_profile_read(double* flops, double* ms, int* launches);
/* Same, plus a per-shape text table (count, ms, TFLOP/s) into text[cap]. */
int hzp_gemm_profile_dump(double* flops, double* ms, int* launches, char* text, int cap);
/* As read / dump, plus busy_ms = the union of the launch intervals (GEMMs on
 * concurrent streams overlap: sum(ms) >= busy_ms). */
int hzp_gemm_profile_read_busy(double* flops, double* ms, double* busy_ms, int* launches);
int hzp_gemm_profile_dump_ex(double* flops, double* ms, double* busy_ms, int* launches, char* text, int cap);

/* ---- kernel-level entry points (single ctx, its streams) ---------------- */
/* Layer-wise P2P-pull all-gather of layer `layer` into AG ring slot `slot`
 * for every rank the ctx drives (collective.cpp:44-67 semantics). */
int hzp_ag_layer(hzp_ctx* ctx, int layer, int slot);
/* Read back one rank's AG slot (working dtype bytes, layer size elems). */
int hzp_ag_slot_download(hzp_ctx* ctx, int rank, int slot, void* host, int64_t n);
/* Upload a rank's unsharded gradient of `layer` into its gradient ring
 * buffer `wslot` (fp32 host data, cast to the wire dtype). */
int hzp_wgrad_upload(hzp_ctx* ctx, int rank, int layer, int wslot, const float* host, int64_t n);
/* P2P-pull reduce-scatter of `layer` from ring buffer `wslot` into the Z2
 * grad shards, ascending-rank fp32 sum, cast/scale, += (collective.cpp:69-97
 * then train.cpp:313-322). */
int hzp_rs_layer(hzp_ctx* ctx, int layer, int wslot);
/* Fused Z1 stage: pull-reduce across DZP replicas (collective.cpp:99-115),
 * Adam (train.cpp:171-189) on the Z1 chunk, round-to-bf16 and P2P-store the
 * working copy into the Z3 owners (train.cpp:361-379).  grad_out (device
 * or NULL) optionally receives each driven rank's reduced Z1 gradient chunk. */
/* Device-timed (CUDA events on the collective's own stream, no host sync
 * between iterations) back-to-back runs of the step's own collective for one
 * layer: kind 0 = AG (the layer-wise all-gather into ring slots), 1 = RS
 * (reduce-scatter into the grad shard; accumulates, so measurement only).
 * Starts with a device-side barrier of all ranks. */
int hzp_collective_time(hzp_ctx* ctx, int kind, int layer, int iters, double* ms_per_iter);
int hzp_z1_adam_step(hzp_ctx* ctx);
int hzp_zero_grads(hzp_ctx* ctx);
/* Device-wide barrier over all dp ranks (no-op in emulation mode). */
int hzp_barrier(hzp_ctx* ctx);

/* Standalone tcgen05 GEMM for tests and benches: C[M,N] = sum_k A[m,k] B[n,k]
 * with A, B bf16; a_mn / b_mn select MN-major storage (A[k*lda+m],
 * B[k*ldb+n]) instead of K-major (A[m*lda+k], B[n*ldb+k]).  epi: 0 store
 * bf16, 1 store fp32, 2 accumulate into fp32 C. stream = cudaStream_t. */
int hzp_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int lda, int ldb,
                  int ldc, int a_mn, int b_mn, int epi, void* stream);
/* Extended epilogue (tests): mode 0 store / 1 accumulate (fp32 C) / 2 assign 0+acc;
 * act 0 none, 1 tanh, 2 gelu (aux <- pre-activation, bf16), 3 tanh' (aux in),
 * 4 gelu' (aux in), 5 softmax-grad alpha*aux*(acc - rowvec[m]); bias bf16 [N]
 * or NULL; resid bf16 [M, ldres] added last or NULL; alpha scales acc. */
int hzp_gemm_bf16_ex(const void* A, const void* B, void* C, int M, int N, int K, int lda, int ldb,
                     int ldc, int a_mn, int b_mn, int mode, int out_bf16, int act,
                     const void* bias_bf16, void* aux, int ldaux, const void* resid, int ldres,
                     const float* rowvec, float alpha, void* stream);
/* Fused causal attention (head dim 128) on bf16 device buffers: qkv [b,S,3h],
 * O [b,S,h], lse [b*nh,S] fp32; backward from dO [b,S,h] and
 * workspace D [2,b*nh,S] fp32 (filled here with -rowsum(dO*O)/sqrt(128) and
 * -lse*log2(e), the backward's per-query vectors) writes dQ, dK, dV into
 * dqkv [b,S,3h].  dsT = a [b*nh,S,S] bf16 buffer: dS^T leaves the backward
 * kernel by TMA stores and dQ is one causal GEMM over it (what the GPT step
 * uses: 0.28 ms at b 4, 16 heads, S 2048); dsT = NULL: dQ by a query-tile
 * pass that recomputes P / dS in TMEM, no S^2 buffer (0.34 ms). */
int hzp_attention_fwd(const void* qkv, void* O, float* lse, int b, int nh, int S, int h, void* stream);
int hzp_attention_bwd(const void* qkv, const void* O, const void* dO, const float* lse, float* D,
                      void* dqkv, void* dsT, int b, int nh, int S, int h, void* stream);
/* Same contract, fp32 operands on the CUDA cores (fp32 parity tier): each
 * output a left fold over k in ascending order, separately rounded multiply
 * and add (train.cpp:68-79).  epi 1 = store, 2 = accumulate, 3 = store
 * tanh(acc) with the host libm's tanhf bit for bit (the hidden-layer
 * activation of the reference's MLP). */
int hzp_gemm_f32(const float* A, const float* B, float* C, int M, int N, int K, int lda,
                 int ldb, int ldc, int a_mn, int b_mn, int epi, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HZP_B200_H_ */
