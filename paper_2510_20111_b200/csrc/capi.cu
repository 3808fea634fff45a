// C-ABI of libhzp_b200.so (declared in include/hzp_b200.h).  Thin marshalling
// over the C++ drop-in (hzp/config.hpp, hzp/sched.hpp) and the device engine;
// C++ exceptions never cross this boundary: they become HZP_ERR_* codes with
// a thread-local message (hzp_last_error).
#include <algorithm>
#include <array>
#include <cstdio>
#include <map>
#include <random>
#include <cstring>
#include <string>

#include "engine/attn.cuh"
#include "engine/engine.hpp"
#include "engine/gpt_ops.cuh"
#include "engine/gemm.cuh"
#include "hzp_b200.h"

using namespace hzp;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HZP_OK;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const SchedError& e) {
    g_err = e.what();
    return e.code() == SchedError::Code::InvalidPolicy ? HZP_ERR_INVALID_POLICY : HZP_ERR_DEADLOCK;
  } catch (const CudaError& e) {
    g_err = e.what();
    return HZP_ERR_CUDA;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return HZP_ERR_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HZP_ERR_ARG;
  }
}

ParallelConfig to_cfg(const hzp_parallel* p) {
  ParallelConfig c;
  c.dp = p->dp;
  c.z1 = p->z1;
  c.z2 = p->z2;
  c.z3 = p->z3;
  c.pp = p->pp > 0 ? p->pp : 1;
  c.vpp = p->vpp > 0 ? p->vpp : 1;
  c.cp = p->cp > 0 ? p->cp : 1;
  c.tp = p->tp > 0 ? p->tp : 1;
  return c;
}

ModelSpec to_spec(const hzp_model_spec* s) {
  ModelSpec m;
  m.num_layers = s->num_layers;
  m.params_per_layer = s->params_per_layer;
  m.embedding_params = s->embedding_params;
  m.seq_len = s->seq_len;
  m.micro_batch_size = s->micro_batch_size;
  m.num_microbatches = s->num_microbatches;
  m.flops_per_token_per_layer = s->flops_per_token_per_layer;
  m.hidden_size = s->hidden_size;
  return m;
}

Topology to_topo(const hzp_cost* c) {
  Topology t;
  t.num_nodes = c->num_nodes;
  t.ranks_per_node = c->ranks_per_node;
  t.intra_bw = c->intra_bw;
  t.inter_bw = c->inter_bw;
  t.intra_latency = c->intra_latency;
  t.inter_latency = c->inter_latency;
  return t;
}

}  // namespace

struct hzp_graph {
  TaskGraph g;
  // LaunchPlans cached per (depth, rs_slots)
  int plan_depth = -1, plan_rs = -1;
  LaunchPlan plan;
};

struct hzp_ctx {
  Engine* e = nullptr;
};

extern "C" {

const char* hzp_last_error(void) { return g_err.c_str(); }
const char* hzp_version(void) { return "hzp-b200 0.1 (sm_100a)"; }

int64_t hzp_shard_elems(int64_t n, int64_t parts) { return shard_elems(n, parts); }

int hzp_validate(const hzp_model_spec* spec, const hzp_parallel* par, const hzp_cost* topo) {
  if (!spec || !par || !topo) return HZP_ERR_ARG;
  return guarded([&] { validate_config(to_spec(spec), to_cfg(par), to_topo(topo)); });
}

int hzp_groups(const hzp_parallel* par, int kind, int* ranks_out, int cap, int* group_size,
               int* n_groups) {
  if (!par || !ranks_out || !group_size || !n_groups) return HZP_ERR_ARG;
  return guarded([&] {
    Topology t;
    t.ranks_per_node = par->dp * (par->pp > 0 ? par->pp : 1) * (par->cp > 0 ? par->cp : 1) *
                       (par->tp > 0 ? par->tp : 1);
    const GroupMap m = build_process_groups(to_cfg(par), t);
    static const GroupKind kinds[] = {GroupKind::Z1, GroupKind::Z2, GroupKind::Z3, GroupKind::DzpReplica};
    if (kind < 0 || kind > 3) throw std::invalid_argument("bad group kind");
    const auto& gs = m.at(kinds[kind]);
    int k = 0;
    for (const auto& g : gs)
      for (int r : g.ranks) {
        if (k >= cap) throw std::invalid_argument("ranks_out too small");
        ranks_out[k++] = r;
      }
    *n_groups = static_cast<int>(gs.size());
    *group_size = gs.empty() ? 0 : gs.front().size();
  });
}

int hzp_graph_build(const hzp_model_spec* spec, const hzp_parallel* par, const hzp_cost* cost,
                    int defer_rs, int rank, hzp_graph** out) {
  if (!spec || !par || !cost || !out) return HZP_ERR_ARG;
  return guarded([&] {
    CostModel cm;
    cm.topo = to_topo(cost);
    cm.device_flops = cost->device_flops;
    GraphPolicy pol;
    pol.defer_rs = defer_rs != 0;
    pol.rank = rank;
    auto* g = new hzp_graph();
    try {
      g->g = build_task_graph(to_spec(spec), to_cfg(par), cm, pol);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int hzp_graph_build_pipeline(const hzp_model_spec* spec, const hzp_parallel* par, const hzp_cost* cost,
                             int defer_rs, int rank, int reuse, int recompute, hzp_reuse_report* report,
                             hzp_graph** out) {
  if (!spec || !par || !cost || !out) return HZP_ERR_ARG;
  return guarded([&] {
    CostModel cm;
    cm.topo = to_topo(cost);
    cm.device_flops = cost->device_flops;
    const ModelSpec ms = to_spec(spec);
    const ParallelConfig pc = to_cfg(par);
    GraphPolicy pol;
    pol.defer_rs = defer_rs != 0;
    pol.rank = rank;
    pol.order = pipeline_order(pc.pp, pc.vpp, int(ms.num_microbatches), rank);
    auto* g = new hzp_graph();
    try {
      g->g = build_task_graph(ms, pc, cm, pol);
      ReuseReport rep;
      if (reuse) rep = apply_reuse(g->g);
      if (recompute) recompute_rule(g->g);
      if (report) *report = {rep.r1_eliminated_ag, rep.r2_merged_rs, rep.r3_eliminated_ag, rep.extra_cached_bytes};
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

void hzp_graph_destroy(hzp_graph* g) { delete g; }
int hzp_graph_size(const hzp_graph* g) { return g ? static_cast<int>(g->g.tasks.size()) : 0; }
int64_t hzp_graph_ag_slot_bytes(const hzp_graph* g) { return g ? g->g.ag_slot_bytes : 0; }
int64_t hzp_graph_grad_buf_bytes(const hzp_graph* g) { return g ? g->g.grad_buf_bytes : 0; }

int hzp_graph_task(const hzp_graph* g, int i, hzp_task* out) {
  if (!g || !out || i < 0 || i >= static_cast<int>(g->g.tasks.size())) return HZP_ERR_ARG;
  const Task& t = g->g.tasks[i];
  out->id = t.id;
  out->kind = static_cast<int>(t.kind);
  out->layer = t.layer;
  out->microbatch = t.microbatch;
  out->virtual_stage = t.virtual_stage;
  out->pass = static_cast<int>(t.pass);
  out->duration = t.duration;
  out->bytes = t.bytes;
  out->num_deps = static_cast<int>(t.deps.size());
  out->deps = t.deps.data();
  return HZP_OK;
}

int hzp_derive_prelaunch_depth(const hzp_graph* g, int64_t free_budget) {
  return g ? derive_prelaunch_depth(g->g, free_budget) : 1;
}

int hzp_make_pools(const hzp_graph* g, int depth, int rs_slots, hzp_pool* ag, hzp_pool* rs) {
  if (!g || !ag || !rs) return HZP_ERR_ARG;
  const PoolSet p = make_pools(g->g, depth, rs_slots);
  *ag = {p.ag.capacity, p.ag.slot_count, p.ag.slot_bytes};
  *rs = {p.rs.capacity, p.rs.slot_count, p.rs.slot_bytes};
  return HZP_OK;
}

int hzp_simulate(const hzp_graph* g, int depth, int rs_slots, int mode, double* start,
                 double* end, hzp_sim_summary* summary) {
  if (!g) return HZP_ERR_ARG;
  return guarded([&] {
    const Timeline tl = simulate(g->g, make_pools(g->g, depth, rs_slots),
                                 mode == HZP_MODE_VANILLA ? SchedMode::Vanilla : SchedMode::Async);
    for (size_t i = 0; i < tl.entries.size(); ++i) {
      if (start) start[i] = tl.entries[i].start;
      if (end) end[i] = tl.entries[i].end;
    }
    if (summary) *summary = {tl.makespan, tl.compute_idle, tl.compute_busy};
  });
}

int hzp_memory_ledger(const hzp_model_spec* spec, const hzp_parallel* par, hzp_ledger* out) {
  if (!spec || !par || !out) return HZP_ERR_ARG;
  return guarded([&] {
    const MemoryLedger m = ledger(to_spec(spec), to_cfg(par));
    *out = {m.params_bf16, m.grads_fp32, m.replica_fp32, m.momentum_fp32, m.variance_fp32, m.total_static};
  });
}

namespace {
// simulate() or the measured start / end times, with derived fields
Timeline timeline_of(const hzp_graph* g, const PoolSet& pools, int mode, const double* start, const double* end) {
  if (!start != !end) throw std::invalid_argument("start and end must both be given or both be NULL");
  if (!start) return simulate(g->g, pools, mode == HZP_MODE_VANILLA ? SchedMode::Vanilla : SchedMode::Async);
  Timeline tl;
  tl.mode = mode == HZP_MODE_VANILLA ? SchedMode::Vanilla : SchedMode::Async;
  tl.entries.resize(g->g.tasks.size());
  for (size_t i = 0; i < tl.entries.size(); ++i) {
    tl.entries[i].start = start[i];
    tl.entries[i].end = end[i];
  }
  finish_timeline(g->g, pools, tl);
  return tl;
}
}  // namespace

int hzp_memory_trace(const hzp_graph* g, int depth, int rs_slots, int mode, const double* start,
                     const double* end, int64_t static_bytes, hzp_memory_report* out, double* sample_t,
                     int64_t* sample_bytes, int cap) {
  if (!g || !out) return HZP_ERR_ARG;
  return guarded([&] {
    const PoolSet pools = make_pools(g->g, depth, rs_slots);
    const Timeline tl = timeline_of(g, pools, mode, start, end);
    MemoryLedger led;
    led.total_static = static_bytes;
    const MemoryTraceResult m = memory_trace(tl, led, pools);
    *out = {m.peak_bytes, m.fragmentation, m.peak_grad_buffer_bytes, tl.peak_memory, tl.makespan,
            static_cast<int>(m.samples.size())};
    for (int i = 0; i < cap && i < static_cast<int>(m.samples.size()); ++i) {
      if (sample_t) sample_t[i] = m.samples[i].first;
      if (sample_bytes) sample_bytes[i] = m.samples[i].second;
    }
  });
}

int hzp_utilization_report(const hzp_graph* g, int depth, int rs_slots, int mode, const double* start,
                           const double* end, double peak_flops, double* out) {
  if (!g || !out) return HZP_ERR_ARG;
  return guarded([&] {
    const PoolSet pools = make_pools(g->g, depth, rs_slots);
    *out = utilization_report(timeline_of(g, pools, mode, start, end), g->g.spec, peak_flops);
  });
}

int hzp_plan_entry_get(const hzp_graph* cg, int depth, int rs_slots, int i, hzp_plan_entry* out) {
  auto* g = const_cast<hzp_graph*>(cg);
  if (!g || !out) return HZP_ERR_ARG;
  return guarded([&] {
    if (g->plan_depth != depth || g->plan_rs != rs_slots) {
      g->plan = build_launch_plan(g->g, make_pools(g->g, depth, rs_slots));
      g->plan_depth = depth;
      g->plan_rs = rs_slots;
    }
    if (i < 0 || i >= static_cast<int>(g->plan.entries.size())) throw std::invalid_argument("index");
    const PlanEntry& e = g->plan.entries[i];
    out->id = e.id;
    out->kind = static_cast<int>(e.kind);
    out->layer = e.layer;
    out->microbatch = e.microbatch;
    out->stream = static_cast<int>(e.stream);
    out->slot = e.slot;
    out->ring_wait = e.ring_wait;
    out->num_waits = static_cast<int>(e.waits.size());
    out->waits = e.waits.data();
  });
}

int hzp_comm_tiles(const hzp_parallel* par, int64_t P, const int64_t* layer_off,
                   const int64_t* layer_size, int num_layers, int rank, int working_bytes,
                   hzp_comm_tile* out, int cap, int* n_out, int* ag_off, int* rs_off,
                   int* z1_off, int* z1_n) {
  static_assert(sizeof(hzp_comm_tile) == sizeof(CommTile), "tile ABI");
  if (!par || !layer_off || !layer_size || !n_out) return HZP_ERR_ARG;
  return guarded([&] {
    const ParallelConfig c = to_cfg(par);
    if (rank < 0 || rank >= c.dp || c.dp > kMaxRanks) throw std::invalid_argument("rank / dp out of range");
    std::vector<Range64> lr;
    for (int l = 0; l < num_layers; ++l) lr.push_back({layer_off[l], layer_size[l]});
    const TileTables T = build_comm_tiles(ShardGeom(P, c), lr, {rank}, working_bytes, c.z2 == 1);
    *n_out = static_cast<int>(T.tiles.size());
    if (out) std::memcpy(out, T.tiles.data(), sizeof(CommTile) * std::min<size_t>(cap, T.tiles.size()));
    if (ag_off) std::copy(T.ag_off.begin(), T.ag_off.end(), ag_off);
    if (rs_off) std::copy(T.rs_off.begin(), T.rs_off.end(), rs_off);
    if (z1_off) *z1_off = T.z1_off;
    if (z1_n) *z1_n = T.z1_n;
  });
}

// ---- engine ---------------------------------------------------------------
int hzp_ctx_create(const hzp_engine_config* cfg, hzp_ctx** out) {
  if (!cfg || !out) return HZP_ERR_ARG;
  return guarded([&] {
    auto* c = new hzp_ctx();
    try {
      c->e = new Engine(*cfg);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void hzp_ctx_destroy(hzp_ctx* ctx) {
  if (!ctx) return;
  delete ctx->e;
  delete ctx;
}

int hzp_ctx_layout(const hzp_ctx* ctx, int64_t* P, int64_t* s1, int64_t* s2, int64_t* s3,
                   int* num_layers) {
  if (!ctx) return HZP_ERR_ARG;
  const Engine& e = *ctx->e;
  if (P) *P = e.geom.P;
  if (s1) *s1 = e.geom.s1;
  if (s2) *s2 = e.geom.s2;
  if (s3) *s3 = e.geom.s3;
  if (num_layers) *num_layers = static_cast<int>(e.layers.size());
  return HZP_OK;
}

int hzp_ctx_layer_range(const hzp_ctx* ctx, int layer, int64_t* offset, int64_t* size) {
  if (!ctx || layer < 0 || layer >= static_cast<int>(ctx->e->layers.size())) return HZP_ERR_ARG;
  if (offset) *offset = ctx->e->layers[layer].off;
  if (size) *size = ctx->e->layers[layer].size;
  return HZP_OK;
}

int hzp_ctx_ipc_handle(hzp_ctx* ctx, void* buf, size_t* len) {
  if (!ctx || !len) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    if (!buf || *len < sizeof(ShareRecord)) {
      *len = sizeof(ShareRecord);
      throw std::invalid_argument("buffer too small");
    }
    const ShareRecord r = e.share_record();
    std::memcpy(buf, &r, sizeof(r));
    *len = sizeof(r);
  });
}

int hzp_ctx_open_peers(hzp_ctx* ctx, const void* handles, size_t handle_len, int n_ranks) {
  if (!ctx || !handles) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    if (e.emulate) return;
    if (handle_len != sizeof(ShareRecord)) throw std::invalid_argument("need one share record per dp rank");
    std::vector<ShareRecord> recs(n_ranks);
    for (int r = 0; r < n_ranks; ++r)
      std::memcpy(&recs[r], static_cast<const char*>(handles) + r * handle_len, sizeof(ShareRecord));
    e.open_peers(recs.data(), n_ranks);
  });
}

static void* field_ptr(Engine& e, int li, int field, size_t* elem, int64_t* count) {
  const int r = e.locals[li].rank;
  switch (field) {
    case HZP_F_PARAM: *elem = e.bf16 ? 2 : 4; *count = e.geom.s3; return e.arenas[r].param;
    case HZP_F_GRAD: *elem = 4; *count = e.geom.s2; return e.arenas[r].grad;
    case HZP_F_MASTER: *elem = 4; *count = e.geom.s1; return e.locals[li].master;
    case HZP_F_MOM: *elem = 4; *count = e.geom.s1; return e.locals[li].mom;
    case HZP_F_VAR: *elem = 4; *count = e.geom.s1; return e.locals[li].var;
    default: throw std::invalid_argument("bad field");
  }
}

int hzp_state_upload(hzp_ctx* ctx, int rank, int field, const void* host, int64_t n) {
  if (!ctx || !host) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    const int li = e.local_index(rank);
    if (li < 0) throw std::invalid_argument("rank not driven by this ctx");
    size_t es;
    int64_t cnt;
    void* p = field_ptr(e, li, field, &es, &cnt);
    if (n != cnt) throw std::invalid_argument("element count mismatch");
    HZP_CUDA(cudaSetDevice(e.cfg.device));
    // the engine's streams are non-blocking: a step issued with step_async may
    // still be reading / writing this buffer
    HZP_CUDA(cudaDeviceSynchronize());
    HZP_CUDA(cudaMemcpy(p, host, size_t(n) * es, cudaMemcpyHostToDevice));
  });
}

int hzp_state_download(hzp_ctx* ctx, int rank, int field, void* host, int64_t n) {
  if (!ctx || !host) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    const int li = e.local_index(rank);
    if (li < 0) throw std::invalid_argument("rank not driven by this ctx");
    size_t es;
    int64_t cnt;
    void* p = field_ptr(e, li, field, &es, &cnt);
    if (n != cnt) throw std::invalid_argument("element count mismatch");
    HZP_CUDA(cudaSetDevice(e.cfg.device));
    HZP_CUDA(cudaDeviceSynchronize());
    HZP_CUDA(cudaMemcpy(host, p, size_t(n) * es, cudaMemcpyDeviceToHost));
  });
}

int hzp_state_set_step(hzp_ctx* ctx, int rank, int adam_step) {
  if (!ctx) return HZP_ERR_ARG;
  const int li = ctx->e->local_index(rank);
  if (li < 0) return HZP_ERR_ARG;
  ctx->e->locals[li].adam_step = adam_step;
  return HZP_OK;
}

int hzp_state_get_step(const hzp_ctx* ctx, int rank, int* adam_step) {
  if (!ctx || !adam_step) return HZP_ERR_ARG;
  const int li = ctx->e->local_index(rank);
  if (li < 0) return HZP_ERR_ARG;
  *adam_step = ctx->e->locals[li].adam_step;
  return HZP_OK;
}

namespace {
__device__ __forceinline__ float hash_uniform(uint64_t e, uint64_t seed) {
  uint64_t x = e * 0x9E3779B97F4A7C15ull ^ seed;
  x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 33;
  return float(x >> 40) * (1.0f / 16777216.0f) - 0.5f;
}
// Device-side shard_init for throughput runs: element e of the flat master
// copy is hash_uniform(e) * scale; every rank materialises exactly its own
// Z1 chunk and its Z3 working-copy segment (train.cpp:224-253 layout).
__global__ void init_rank_kernel(void* param, int bf16, float* master, int64_t s1, int64_t s3,
                                 int64_t i1, int64_t i3, int64_t P, uint64_t seed, float scale) {
  const int64_t n = s1 > s3 ? s1 : s3;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    if (i < s1) {
      const int64_t e = i1 * s1 + i;
      master[i] = e < P ? hash_uniform(e, seed) * scale : 0.f;
    }
    if (i < s3) {
      const int64_t e = i3 * s3 + i;
      const float w = e < P ? hash_uniform(e, seed) * scale : 0.f;
      if (bf16) static_cast<uint16_t*>(param)[i] = f32_to_bf16_bits(w);
      else static_cast<float*>(param)[i] = w;
    }
  }
}
}  // namespace

int hzp_state_init_random(hzp_ctx* ctx, uint64_t seed, double scale) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    HZP_CUDA(cudaSetDevice(e.cfg.device));
    for (auto& l : e.locals) {
      const int r = l.rank;
      init_rank_kernel<<<4 * kNumSMs, 256>>>(e.arenas[r].param, e.bf16, l.master, e.geom.s1, e.geom.s3,
                                              r % e.geom.z1, r % e.geom.z3, e.geom.P, seed, float(scale));
      HZP_LAUNCH_CHECK();
      HZP_CUDA(cudaMemset(l.mom, 0, size_t(e.geom.s1) * 4));
      HZP_CUDA(cudaMemset(l.var, 0, size_t(e.geom.s1) * 4));
      HZP_CUDA(cudaMemset(e.arenas[r].grad, 0, size_t(e.geom.s2) * 4));
      l.adam_step = 0;
    }
    HZP_CUDA(cudaDeviceSynchronize());
  });
}

// ---- reference-faithful synthetic state / inputs (train.cpp:17-27, 224-253, 501-508) ----
namespace {
inline float seeded_value(std::mt19937_64& rng) {
  // seeded_uniform<float>: (raw >> 11) * 2^-53 - 0.5 in double, then float
  return static_cast<float>(static_cast<double>(rng() >> 11) * 0x1p-53 - 0.5);
}
inline uint16_t bf16_rne_host(float f) {  // bf16_round (kernels.hpp:37-50), non-NaN inputs
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
}  // namespace

int hzp_seeded_span(uint64_t seed, int64_t P, int64_t first, int64_t n, double scale, float* out) {
  if (!out || first < 0 || n < 0) return HZP_ERR_ARG;
  return guarded([&] {
    std::mt19937_64 rng(seed);
    rng.discard(static_cast<unsigned long long>(std::min(first, P)));
    const float sc = static_cast<float>(scale);
    for (int64_t i = 0; i < n; ++i) out[i] = first + i < P ? seeded_value(rng) * sc : 0.0f;
  });
}

int hzp_state_init_seeded(hzp_ctx* ctx, uint64_t seed, double scale) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    HZP_CUDA(cudaSetDevice(e.cfg.device));
    HZP_CUDA(cudaDeviceSynchronize());
    const ShardGeom& g = e.geom;
    const float sc = static_cast<float>(scale);
    constexpr int64_t kChunk = int64_t(1) << 24;
    std::vector<float> buf(kChunk);
    std::vector<uint16_t> bbuf(kChunk);
    for (auto& l : e.locals) {
      const int r = l.rank;
      // this rank's Z1 master chunk and Z3 working-copy shard of the padded
      // flat vector seeded_uniform(P, seed) * scale, streamed in one pass
      const int64_t m0 = int64_t(r % g.z1) * g.s1, p0 = int64_t(r % g.z3) * g.s3;
      const int64_t lo = std::min(m0, p0), hi = std::max(m0 + g.s1, p0 + g.s3);
      std::mt19937_64 rng(seed);
      rng.discard(static_cast<unsigned long long>(std::min(lo, g.P)));
      auto* master = l.master;
      auto* param = static_cast<char*>(e.arenas[r].param);
      for (int64_t c0 = lo; c0 < hi; c0 += kChunk) {
        const int64_t n = std::min(kChunk, hi - c0);
        for (int64_t i = 0; i < n; ++i) buf[i] = c0 + i < g.P ? seeded_value(rng) * sc : 0.0f;
        const int64_t a = std::max(c0, m0), b = std::min(c0 + n, m0 + g.s1);
        if (a < b) HZP_CUDA(cudaMemcpy(master + (a - m0), buf.data() + (a - c0), size_t(b - a) * 4, cudaMemcpyHostToDevice));
        const int64_t x = std::max(c0, p0), y = std::min(c0 + n, p0 + g.s3);
        if (x < y) {
          if (e.bf16) {
            for (int64_t i = x; i < y; ++i) bbuf[i - x] = bf16_rne_host(buf[i - c0]);
            HZP_CUDA(cudaMemcpy(param + (x - p0) * 2, bbuf.data(), size_t(y - x) * 2, cudaMemcpyHostToDevice));
          } else {
            HZP_CUDA(cudaMemcpy(param + (x - p0) * 4, buf.data() + (x - c0), size_t(y - x) * 4, cudaMemcpyHostToDevice));
          }
        }
      }
      HZP_CUDA(cudaMemset(l.mom, 0, size_t(g.s1) * 4));
      HZP_CUDA(cudaMemset(l.var, 0, size_t(g.s1) * 4));
      HZP_CUDA(cudaMemset(e.arenas[r].grad, 0, size_t(g.s2) * 4));
      l.adam_step = 0;
    }
    HZP_CUDA(cudaDeviceSynchronize());
  });
}

int hzp_make_tokens(uint64_t seed, int step, int rank, int microbatch, int64_t n, int vocab, int32_t* out) {
  if (!out || n < 0 || vocab < 1) return HZP_ERR_ARG;
  // run_case's per-(step, rank, microbatch) stream (train.cpp:506-507);
  // token = floor(u * vocab), u = (raw >> 11) * 2^-53
  std::mt19937_64 rng(seed ^ (0x9E3779B97F4A7C15ull * (uint64_t(step) * 1024ull + uint64_t(rank) * 32ull +
                                                       uint64_t(microbatch) + 1)));
  for (int64_t i = 0; i < n; ++i) {
    const int t = static_cast<int>(static_cast<double>(rng() >> 11) * 0x1p-53 * vocab);
    out[i] = t < vocab ? t : vocab - 1;
  }
  return HZP_OK;
}

int hzp_step(hzp_ctx* ctx, const void* inputs, int inputs_on_device, float* losses_out) {
  if (!ctx || !inputs) return HZP_ERR_ARG;
  return guarded([&] { ctx->e->step(inputs, inputs_on_device != 0, losses_out); });
}

int hzp_sync(hzp_ctx* ctx) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    HZP_CUDA(cudaSetDevice(ctx->e->cfg.device));
    HZP_CUDA(cudaDeviceSynchronize());
  });
}

int hzp_launch_log(const hzp_ctx* ctx, hzp_launch_rec* out, int cap, int* n) {
  if (!ctx || !n) return HZP_ERR_ARG;
  const auto& log = ctx->e->log;
  *n = static_cast<int>(log.size());
  if (out)
    for (int i = 0; i < *n && i < cap; ++i) out[i] = log[i];
  return HZP_OK;
}

int hzp_set_timeline(hzp_ctx* ctx, int on) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    HZP_CUDA(cudaSetDevice(e.cfg.device));
    HZP_CUDA(cudaDeviceSynchronize());
    e.timeline_events(on != 0);
    e.cfg.timeline = on ? 1 : 0;
  });
}

int hzp_timeline(const hzp_ctx* ctx, double* start_ms, double* end_ms, int cap, int* n,
                 double* compute_idle_ms, double* compute_busy_ms, double* makespan_ms) {
  if (!ctx || !n) return HZP_ERR_ARG;
  return guarded([&] {
    const Engine& e = *ctx->e;
    if (!e.cfg.timeline) throw std::invalid_argument("ctx created without timeline");
    HZP_CUDA(cudaEventSynchronize(e.ev_step1));
    const int cnt = static_cast<int>(e.plan.entries.size());
    *n = cnt;
    double busy = 0, last_c = 0, mk = 0;
    for (int i = 0; i < cnt; ++i) {
      float a = 0, b = 0;
      HZP_CUDA(cudaEventElapsedTime(&a, e.ev_step0, e.tev0[i]));
      HZP_CUDA(cudaEventElapsedTime(&b, e.ev_step0, e.tev1[i]));
      if (i < cap) {
        if (start_ms) start_ms[i] = a;
        if (end_ms) end_ms[i] = b;
      }
      if (e.plan.entries[i].stream == StreamId::Compute) {
        busy += b - a;
        last_c = last_c > b ? last_c : b;
      }
      mk = mk > b ? mk : b;
    }
    if (compute_idle_ms) *compute_idle_ms = last_c - busy;
    if (compute_busy_ms) *compute_busy_ms = busy;
    if (makespan_ms) *makespan_ms = mk;
  });
}

int hzp_z1_timeline(const hzp_ctx* ctx, double* ready_ms, double* start_ms, double* end_ms, int cap, int* n) {
  if (!ctx || !n) return HZP_ERR_ARG;
  return guarded([&] {
    const Engine& e = *ctx->e;
    HZP_CUDA(cudaEventSynchronize(e.ev_step1));
    *n = e.z1_timed ? static_cast<int>(e.layers.size()) : 0;
    for (int l = 0; l < *n && l < cap; ++l) {
      float a = 0, b = 0, c = 0;
      HZP_CUDA(cudaEventElapsedTime(&a, e.ev_step0, e.zev_ready[l]));
      HZP_CUDA(cudaEventElapsedTime(&b, e.ev_step0, e.zev_start[l]));
      HZP_CUDA(cudaEventElapsedTime(&c, e.ev_step0, e.zev_end[l]));
      if (ready_ms) ready_ms[l] = a;
      if (start_ms) start_ms[l] = b;
      if (end_ms) end_ms[l] = c;
    }
  });
}

int hzp_ctx_launch_count(const hzp_ctx* ctx, int64_t* kernels) {
  if (!ctx || !kernels) return HZP_ERR_ARG;
  *kernels = ctx->e->launches;
  return HZP_OK;
}

uint64_t hzp_kernel_launches(void) { return launch_counter(); }

int hzp_ctx_stream(const hzp_ctx* ctx, int which, void** stream) {
  if (!ctx || !stream || which < 0 || which > 2) return HZP_ERR_ARG;
  *stream = ctx->e->st[which];
  return HZP_OK;
}

int hzp_gemm_profile(int on) {
  gemm_profile().on = on != 0;
  return HZP_OK;
}

int hzp_gemm_profile_read(double* flops, double* ms, int* launches) {
  return hzp_gemm_profile_dump(flops, ms, launches, nullptr, 0);
}

int hzp_gemm_profile_read_busy(double* flops, double* ms, double* busy_ms, int* launches) {
  return hzp_gemm_profile_dump_ex(flops, ms, busy_ms, launches, nullptr, 0);
}

int hzp_gemm_profile_dump(double* flops, double* ms, int* launches, char* text, int cap) {
  return hzp_gemm_profile_dump_ex(flops, ms, nullptr, launches, text, cap);
}

int hzp_gemm_profile_dump_ex(double* flops, double* ms, double* busy_ms, int* launches, char* text, int cap) {
  return guarded([&] {
    GemmProfile& p = gemm_profile();
    std::map<std::string, std::array<double, 3>> agg;  // shape -> {count, ms, flops}
    double f = 0, t = 0;
    std::vector<std::pair<float, float>> iv;  // launch [start, end] relative to the first
    for (size_t i = 0; i < p.ev.size(); ++i) {
      HZP_CUDA(cudaEventSynchronize(p.ev[i].second));
      float x = 0, t0 = 0;
      HZP_CUDA(cudaEventElapsedTime(&x, p.ev[i].first, p.ev[i].second));
      HZP_CUDA(cudaEventElapsedTime(&t0, p.ev[0].first, p.ev[i].first));
      iv.emplace_back(t0, t0 + x);
      t += x;
      f += p.flops[i];
      if (i < p.shape.size()) {
        auto& a = agg[p.shape[i]];
        a[0] += 1;
        a[1] += x;
        a[2] += p.flops[i];
      }
    }
    for (auto& e : p.ev) {
      cudaEventDestroy(e.first);
      cudaEventDestroy(e.second);
    }
    if (busy_ms) {  // union of the launch intervals (concurrent streams overlap)
      std::sort(iv.begin(), iv.end());
      double busy = 0, s0 = -1, e0 = -1;
      for (const auto& [a, b] : iv) {
        if (a > e0) {
          if (e0 > s0) busy += e0 - s0;
          s0 = a;
          e0 = b;
        } else if (b > e0) {
          e0 = b;
        }
      }
      if (e0 > s0) busy += e0 - s0;
      *busy_ms = busy;
    }
    if (flops) *flops = f;
    if (ms) *ms = t;
    if (launches) *launches = static_cast<int>(p.ev.size());
    p.ev.clear();
    p.flops.clear();
    p.shape.clear();
    if (text && cap > 0) {
      std::string out;
      for (const auto& [k, a] : agg) {
        char line[256];
        std::snprintf(line, sizeof line, "%-48s n=%4.0f ms=%9.3f TF/s=%7.1f\n", k.c_str(), a[0], a[1],
                      a[1] > 0 ? a[2] / (a[1] * 1e9) : 0.0);
        out += line;
      }
      std::snprintf(text, size_t(cap), "%s", out.c_str());
    }
  });
}

int hzp_ag_layer(hzp_ctx* ctx, int layer, int slot) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    if (layer < 0 || layer >= static_cast<int>(e.layers.size()) || slot < 0 || slot >= e.depth)
      throw std::invalid_argument("layer/slot out of range");
    e.ag_layer(layer, slot, e.st[1]);
    HZP_CUDA(cudaStreamSynchronize(e.st[1]));
  });
}

int hzp_ag_slot_download(hzp_ctx* ctx, int rank, int slot, void* host, int64_t n) {
  if (!ctx || !host) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    const int li = e.local_index(rank);
    if (li < 0 || slot < 0 || slot >= e.depth || n > e.slot_elems) throw std::invalid_argument("bad args");
    const int es = e.bf16 ? 2 : 4;
    HZP_CUDA(cudaDeviceSynchronize());
    HZP_CUDA(cudaMemcpy(host, static_cast<char*>(e.arenas[rank].ag) + int64_t(slot) * e.slot_elems * es,
                        size_t(n) * es, cudaMemcpyDeviceToHost));
  });
}

namespace {
__global__ void cast_to_wire_kernel(const float* in, void* out, int64_t n, int bf16) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    if (bf16) static_cast<uint16_t*>(out)[i] = f32_to_bf16_bits(in[i]);
    else static_cast<float*>(out)[i] = in[i];
  }
}
}  // namespace

int hzp_wgrad_upload(hzp_ctx* ctx, int rank, int layer, int wslot, const float* host, int64_t n) {
  if (!ctx || !host) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    const int li = e.local_index(rank);
    if (li < 0 || e.direct_grad || wslot < 0 || wslot >= e.wslots ||
        n != e.layers.at(layer).size)
      throw std::invalid_argument("bad args (z2 == 1 has no gradient ring)");
    float* tmp = nullptr;
    HZP_CUDA(cudaMalloc(&tmp, size_t(n) * 4));
    HZP_CUDA(cudaMemcpy(tmp, host, size_t(n) * 4, cudaMemcpyHostToDevice));
    const int es = e.bf16 ? 2 : 4;
    void* dst = static_cast<char*>(e.arenas[rank].wgrad) + int64_t(wslot) * e.slot_elems * es;
    cast_to_wire_kernel<<<256, 256>>>(tmp, dst, n, e.bf16);
    HZP_LAUNCH_CHECK();
    HZP_CUDA(cudaDeviceSynchronize());
    cudaFree(tmp);
  });
}

int hzp_rs_layer(hzp_ctx* ctx, int layer, int wslot) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    if (e.direct_grad) throw std::invalid_argument("z2 == 1: the reduce-scatter is fused into wgrad");
    e.rs_layer(layer, wslot, false, ++e.rs_seq, e.st[2]);
    HZP_CUDA(cudaStreamSynchronize(e.st[2]));
  });
}

int hzp_collective_time(hzp_ctx* ctx, int kind, int layer, int iters, double* ms_per_iter) {
  if (!ctx || !ms_per_iter || iters < 1) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    if (layer < 0 || layer >= static_cast<int>(e.layers.size())) throw std::invalid_argument("layer out of range");
    if (kind == 0 && e.zero_copy_ag) throw std::invalid_argument("z3 == 1: the all-gather is the identity");
    if (kind == 1 && e.direct_grad) throw std::invalid_argument("z2 == 1: the reduce-scatter is fused into wgrad");
    if (kind != 0 && kind != 1) throw std::invalid_argument("kind: 0 = AG, 1 = RS");
    HZP_CUDA(cudaSetDevice(e.cfg.device));
    cudaStream_t s = e.st[kind == 0 ? 1 : 2];
    HZP_CUDA(cudaDeviceSynchronize());
    e.barrier(s);  // all ranks start together
    cudaEvent_t a, b;
    HZP_CUDA(cudaEventCreate(&a));
    HZP_CUDA(cudaEventCreate(&b));
    HZP_CUDA(cudaEventRecord(a, s));
    for (int i = 0; i < iters; ++i) {
      if (kind == 0) e.ag_layer(layer, i % e.depth, s);
      else e.rs_layer(layer, 0, false, ++e.rs_seq, s);
    }
    HZP_CUDA(cudaEventRecord(b, s));
    HZP_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    HZP_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms_per_iter = ms / iters;
  });
}

int hzp_z1_adam_step(hzp_ctx* ctx) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    e.barrier(e.st[0]);
    e.z1_adam(e.st[0]);
    e.barrier(e.st[0]);
    HZP_CUDA(cudaStreamSynchronize(e.st[0]));
  });
}

int hzp_zero_grads(hzp_ctx* ctx) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    Engine& e = *ctx->e;
    HZP_CUDA(cudaSetDevice(e.cfg.device));
    HZP_CUDA(cudaDeviceSynchronize());  // see hzp_state_upload
    for (auto& l : e.locals) HZP_CUDA(cudaMemset(e.arenas[l.rank].grad, 0, size_t(e.geom.s2) * 4));
    HZP_CUDA(cudaDeviceSynchronize());
  });
}

int hzp_barrier(hzp_ctx* ctx) {
  if (!ctx) return HZP_ERR_ARG;
  return guarded([&] {
    ctx->e->barrier(ctx->e->st[0]);
    HZP_CUDA(cudaStreamSynchronize(ctx->e->st[0]));
  });
}

int hzp_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int lda, int ldb,
                  int ldc, int a_mn, int b_mn, int epi, void* stream) {
  return guarded([&] {
    GemmShape s{M, N, K, lda, ldb, a_mn, b_mn};
    Epilogue e;
    e.ldc = ldc;
    e.out_bf16 = epi == 0;
    e.mode = epi == 2 ? kEpiAccum : kEpiStore;
    gemm_tc_bf16(A, B, C, s, e, static_cast<cudaStream_t>(stream));
  });
}

int hzp_gemm_bf16_ex(const void* A, const void* B, void* C, int M, int N, int K, int lda, int ldb,
                     int ldc, int a_mn, int b_mn, int mode, int out_bf16, int act,
                     const void* bias_bf16, void* aux, int ldaux, const void* resid, int ldres,
                     const float* rowvec, float alpha, void* stream) {
  return guarded([&] {
    GemmShape s{M, N, K, lda, ldb, a_mn, b_mn};
    Epilogue e;
    e.ldc = ldc;
    e.out_bf16 = out_bf16;
    e.mode = mode;
    e.act = act;
    e.bias_any = bias_bf16;
    e.aux = aux;
    e.ldaux = ldaux;
    e.aux_bf16 = 1;
    e.resid = resid;
    e.ldres = ldres;
    e.rowvec = rowvec;
    e.alpha = alpha;
    gemm_tc_bf16(A, B, C, s, e, static_cast<cudaStream_t>(stream));
  });
}

int hzp_attention_fwd(const void* qkv, void* O, float* lse, int b, int nh, int S, int h, void* stream) {
  return guarded([&] {
    attention_fwd_tc(static_cast<const uint16_t*>(qkv), static_cast<uint16_t*>(O), nullptr, lse, b, nh, S, h,
                     static_cast<cudaStream_t>(stream));
  });
}

int hzp_attention_bwd(const void* qkv, const void* O, const void* dO, const float* lse, float* D,
                      void* dqkv, void* dsT, int b, int nh, int S, int h, void* stream) {
  return guarded([&] {
    auto st = static_cast<cudaStream_t>(stream);
    const auto* q = static_cast<const uint16_t*>(qkv);
    auto* dq = static_cast<uint16_t*>(dqkv);
    auto* ds = static_cast<uint16_t*>(dsT);
    attn_rowdot(static_cast<const uint16_t*>(dO), static_cast<const uint16_t*>(O), lse, D, b, nh, S, 128, st);
    if (ds) {  // legacy: dS^T through HBM + GEMM dQ
      attention_bwd_tc(q, static_cast<const uint16_t*>(dO), lse, D, dq, ds, b, nh, S, h, st);
      attention_dq(q, ds, dq, b, nh, S, h, st);
    } else {   // production: dQ pass recomputing P / dS in TMEM
      attention_bwd_tc(q, static_cast<const uint16_t*>(dO), lse, D, dq, nullptr, b, nh, S, h, st);
      attention_dq_tc(q, static_cast<const uint16_t*>(dO), D, dq, b, nh, S, h, st);
    }
  });
}

int hzp_gemm_f32(const float* A, const float* B, float* C, int M, int N, int K, int lda, int ldb,
                 int ldc, int a_mn, int b_mn, int epi, void* stream) {
  return guarded([&] {
    GemmShape s{M, N, K, lda, ldb, a_mn, b_mn};
    Epilogue e;
    e.ldc = ldc;
    e.out_bf16 = 0;
    e.mode = epi == 2 ? kEpiAccum : kEpiStore;
    if (epi == 3) e.act = kActTanh;
    gemm_f32_ordered(A, B, C, s, e, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
