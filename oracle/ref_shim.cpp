// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT PATH.
//
// extern "C" shim around the UNMODIFIED reference library (the sources under
// /root/reference/proj/src, compiled by oracle/Makefile into
// oracle/_ref/libhzpref.so).  It lets the Python tests and bench.py's
// `--impl reference` arm call the reference's own hot-path functions through
// ctypes.  No reference source is copied; this file only marshals arguments.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "hzp/collective.hpp"
#include "hzp/config.hpp"
#include "hzp/kernels.hpp"
#include "hzp/memory.hpp"
#include "hzp/pipeline.hpp"
#include "hzp/sched.hpp"
#include "hzp/train.hpp"

namespace {

thread_local std::string g_err;

hzp::MlpShape shape_of(const int* dims, int nl) {
  hzp::MlpShape s;
  s.dims.assign(dims, dims + nl + 1);
  return s;
}

hzp::ParallelConfig cfg_of(int dp, int z1, int z2, int z3) {
  hzp::ParallelConfig c;
  c.dp = dp;
  c.z1 = z1;
  c.z2 = z2;
  c.z3 = z3;
  return c;
}

template <typename T>
hzp::RankBatches<T> batches_for(const hzp::MlpShape& shape, int dp, int mbs, int batch,
                                std::uint64_t seed, int step) {
  // run_case's per-(step, rank, mb) seeding (src/train.cpp:501-508).
  hzp::RankBatches<T> b(dp);
  for (int r = 0; r < dp; ++r)
    for (int mb = 0; mb < mbs; ++mb)
      b[r].push_back(hzp::seeded_uniform<T>(
          static_cast<std::size_t>(batch) * shape.dims[0],
          seed ^ (0x9E3779B97F4A7C15ull * (step * 1024ull + r * 32ull + mb + 1))));
  return b;
}

template <typename T>
int run_states(const int* dims, int nl, int dp, int z1, int z2, int z3, int mbs, int batch,
               std::uint64_t seed, int steps, int bf16_working, T* param, T* grad, T* master,
               T* mom, T* var, T* losses, T* baseline_working) {
  const auto shape = shape_of(dims, nl);
  const auto cfg = cfg_of(dp, z1, z2, z3);
  auto states = hzp::shard_init<T>(shape, cfg, seed, bf16_working != 0);
  auto base = hzp::baseline_init<T>(shape, seed, bf16_working != 0);
  const hzp::AdamParams adam;
  std::vector<T> l;
  for (int step = 0; step < steps; ++step) {
    const auto b = batches_for<T>(shape, dp, mbs, batch, seed, step);
    l = hzp::train_step_hzp(states, shape, cfg, b, batch, adam, bf16_working != 0);
    hzp::train_step_baseline(base, shape, b, batch, adam, hzp::ReductionOrder{dp, z2},
                             bf16_working != 0);
  }
  const std::int64_t p = shape.param_count();
  const std::int64_t s1 = hzp::shard_elems(p, z1), s2 = hzp::shard_elems(p, z2),
                     s3 = hzp::shard_elems(p, z3);
  for (int r = 0; r < dp; ++r) {
    std::memcpy(param + r * s3, states[r].param_shard.data(), sizeof(T) * s3);
    std::memcpy(grad + r * s2, states[r].grad_shard.data(), sizeof(T) * s2);
    std::memcpy(master + r * s1, states[r].master_shard.data(), sizeof(T) * s1);
    std::memcpy(mom + r * s1, states[r].momentum_shard.data(), sizeof(T) * s1);
    std::memcpy(var + r * s1, states[r].variance_shard.data(), sizeof(T) * s1);
    losses[r] = l.empty() ? T(0) : l[r];
  }
  std::memcpy(baseline_working, base.working.data(), sizeof(T) * p);
  return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

long long ref_shard_elems(long long n, long long parts) { return hzp::shard_elems(n, parts); }

float ref_bf16_round(float x) { return hzp::kernels::bf16_round(x); }

// impl: 0 = scalar, 1 = active (AVX2 where available)
void ref_bf16_round_vec(float* v, long long n, int impl) {
  const auto& k = impl ? hzp::kernels::active_impl() : hzp::kernels::scalar_impl();
  k.bf16_round_f32(v, static_cast<std::size_t>(n));
}

void ref_seeded_uniform_f64(double* out, long long n, unsigned long long seed) {
  auto v = hzp::seeded_uniform<double>(static_cast<std::size_t>(n), seed);
  std::memcpy(out, v.data(), sizeof(double) * n);
}

void ref_seeded_uniform_f32(float* out, long long n, unsigned long long seed) {
  auto v = hzp::seeded_uniform<float>(static_cast<std::size_t>(n), seed);
  std::memcpy(out, v.data(), sizeof(float) * n);
}

// Run shard_init + `steps` x train_step_hzp with run_case inputs; dump the
// per-rank ShardedState (flat [dp][s]) and the baseline's working copy.
int ref_run_states_f32(const int* dims, int nl, int dp, int z1, int z2, int z3, int mbs,
                       int batch, unsigned long long seed, int steps, int bf16_working,
                       float* param, float* grad, float* master, float* mom, float* var,
                       float* losses, float* base_working) {
  try {
    return run_states<float>(dims, nl, dp, z1, z2, z3, mbs, batch, seed, steps, bf16_working,
                             param, grad, master, mom, var, losses, base_working);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_run_states_f64(const int* dims, int nl, int dp, int z1, int z2, int z3, int mbs,
                       int batch, unsigned long long seed, int steps, double* param,
                       double* grad, double* master, double* mom, double* var,
                       double* losses, double* base_working) {
  try {
    return run_states<double>(dims, nl, dp, z1, z2, z3, mbs, batch, seed, steps, 0, param,
                              grad, master, mom, var, losses, base_working);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Reference mlp_loss_grad on one batch.
float ref_mlp_loss_grad_f32(const int* dims, int nl, const float* params, const float* in,
                            int batch, float* grad) {
  const auto shape = shape_of(dims, nl);
  std::vector<float> p(params, params + shape.param_count());
  std::vector<float> x(in, in + static_cast<std::size_t>(batch) * dims[0]);
  auto lg = hzp::mlp_loss_grad(shape, p, x, batch);
  std::memcpy(grad, lg.grad.data(), sizeof(float) * lg.grad.size());
  return lg.loss;
}

// Process groups (src/config.cpp:127-170).  kind: 0=Z1 1=Z2 2=Z3 3=DZP.
// Writes the groups' ranks back to back into out (dp ints); returns group count.
int ref_groups(int dp, int z1, int z2, int z3, int kind, int* out) {
  hzp::Topology topo;
  topo.num_nodes = 1;
  topo.ranks_per_node = dp;
  const auto map = hzp::build_process_groups(cfg_of(dp, z1, z2, z3), topo);
  const hzp::GroupKind kinds[] = {hzp::GroupKind::Z1, hzp::GroupKind::Z2, hzp::GroupKind::Z3,
                                  hzp::GroupKind::DzpReplica};
  const auto& groups = map.at(kinds[kind]);
  int k = 0;
  for (const auto& g : groups)
    for (int r : g.ranks) out[k++] = r;
  return static_cast<int>(groups.size());
}

// validate_config error code: 0 ok, 1 NonDivisible, 2 EmptyModel, 3 BadField.
int ref_validate(long long layers, long long ppl, int dp, int z1, int z2, int z3, int ranks) {
  hzp::ModelSpec spec;
  spec.num_layers = layers;
  spec.params_per_layer = ppl;
  hzp::Topology topo;
  topo.num_nodes = 1;
  topo.ranks_per_node = ranks;
  try {
    hzp::validate_config(spec, cfg_of(dp, z1, z2, z3), topo);
    return 0;
  } catch (const hzp::ValidationError& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  }
}

// Collectives over flat buffers (src/collective.cpp:44-115).
void ref_all_gather_f64(const double* shards, int g, long long per, double* out) {
  hzp::ProcessGroup grp;
  for (int r = 0; r < g; ++r) grp.ranks.push_back(r);
  std::vector<hzp::RankTensor<double>> s(g);
  for (int r = 0; r < g; ++r)
    s[r] = {r, r, hzp::Dtype::FP64, std::vector<double>(shards + r * per, shards + (r + 1) * per)};
  auto f = hzp::all_gather(grp, s);
  std::memcpy(out, f[0].elems.data(), sizeof(double) * g * per);
}

int ref_reduce_scatter_f32(const float* fulls, int g, long long total, float* out) {
  hzp::ProcessGroup grp;
  for (int r = 0; r < g; ++r) grp.ranks.push_back(r);
  std::vector<hzp::RankTensor<float>> f(g);
  for (int r = 0; r < g; ++r)
    f[r] = {r, -1, hzp::Dtype::FP32,
            std::vector<float>(fulls + r * total, fulls + (r + 1) * total)};
  try {
    auto s = hzp::reduce_scatter(grp, f);
    for (int r = 0; r < g; ++r)
      std::memcpy(out + r * (total / g), s[r].elems.data(), sizeof(float) * (total / g));
    return 0;
  } catch (const hzp::CollectiveError& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  }
}

void ref_all_reduce_f32(const float* ts, int g, long long n, float* out) {
  hzp::ProcessGroup grp;
  for (int r = 0; r < g; ++r) grp.ranks.push_back(r);
  std::vector<hzp::RankTensor<float>> t(g);
  for (int r = 0; r < g; ++r)
    t[r] = {r, -1, hzp::Dtype::FP32, std::vector<float>(ts + r * n, ts + (r + 1) * n)};
  auto o = hzp::all_reduce(grp, t);
  std::memcpy(out, o[0].elems.data(), sizeof(float) * n);
}

// Task graph + simulation (src/sched.cpp:75-387).  Outputs per task:
// kind, layer, microbatch, pass, bytes, start, end, pool_release; deps
// flattened with dep_off[n+1].  Returns task count (or -1 on error; if
// cap < count, only the count is returned).  with_reuse: 0 = default
// one-F-one-B-per-microbatch order; 1 = the CLI's order (build_schedule for
// `rank`) + apply_reuse (hzpsim.cpp:111-126); 2 = that order without reuse.
// recompute != 0 then applies recompute_rule (hzpsim.cpp:127).
struct RefSimOut {
  double makespan, compute_idle, compute_busy;
  long long peak_memory;
  double fragmentation;
  long long peak_grad_buffer_bytes;
  int ag_slot_count, rs_slot_count;
  long long ag_slot_bytes, rs_slot_bytes;
  int r1_eliminated_ag, r2_merged_rs, r3_eliminated_ag;  // ReuseReport (pipeline.hpp:44-49)
  long long extra_cached_bytes;
  // memory_trace / utilization_report (sched.cpp:389-477)
  long long total_static, peak_bytes;
  double utilization;  // peak_flops = device_flops
  int n_samples;
  double sample_time_sum;
  long long sample_bytes_sum;
};

int ref_task_graph(long long layers, long long ppl, long long seq, long long mbsize,
                   long long num_mb, double flops_per_tok_layer, int dp, int z1, int z2,
                   int z3, int pp, int vpp, double intra_bw, double intra_lat,
                   double device_flops, int defer_rs, int rank, int with_reuse, int recompute, int depth,
                   int rs_slots, int vanilla, int cap, int* kind, int* layer, int* mb,
                   int* pass, long long* bytes, double* dur, double* start, double* end,
                   double* pool_release, int* dep_off, int* deps, int dep_cap,
                   RefSimOut* sim) {
  try {
    hzp::ModelSpec spec;
    spec.num_layers = layers;
    spec.params_per_layer = ppl;
    spec.seq_len = seq;
    spec.micro_batch_size = mbsize;
    spec.num_microbatches = num_mb;
    spec.flops_per_token_per_layer = flops_per_tok_layer;
    auto cfg = cfg_of(dp, z1, z2, z3);
    cfg.pp = pp;
    cfg.vpp = vpp;
    hzp::CostModel cost;
    cost.topo.num_nodes = 1;
    cost.topo.ranks_per_node = dp * pp;
    cost.topo.intra_bw = intra_bw;
    cost.topo.inter_bw = intra_bw;
    cost.topo.intra_latency = intra_lat;
    cost.device_flops = device_flops;
    hzp::GraphPolicy pol;
    pol.defer_rs = defer_rs != 0;
    pol.rank = rank;
    hzp::PipeSchedule sched;
    if (with_reuse) {
      sched = hzp::build_schedule(pp, vpp, static_cast<int>(num_mb),
                                  vpp > 1 ? hzp::PipeVariant::Interleaved
                                          : hzp::PipeVariant::OneFOneB);
      pol.order = sched.per_rank[rank];
    }
    auto g = hzp::build_task_graph(spec, cfg, cost, pol);
    hzp::ReuseReport rep;
    if (with_reuse == 1) rep = hzp::apply_reuse(sched, g);
    hzp::recompute_rule(g, recompute != 0);
    const int n = static_cast<int>(g.tasks.size());
    if (n > cap) return n;
    const auto pools = hzp::make_pools(g, depth, rs_slots);
    const auto tl = hzp::simulate(g, pools, vanilla ? hzp::SchedMode::Vanilla
                                                    : hzp::SchedMode::Async);
    const auto mem = hzp::memory_trace(tl, hzp::ledger(spec, cfg), pools);
    int k = 0;
    for (int i = 0; i < n; ++i) {
      const auto& t = g.tasks[i];
      kind[i] = static_cast<int>(t.kind);
      layer[i] = t.layer;
      mb[i] = t.microbatch;
      pass[i] = static_cast<int>(t.pass);
      bytes[i] = t.bytes;
      dur[i] = t.duration;
      start[i] = tl.entries[i].start;
      end[i] = tl.entries[i].end;
      pool_release[i] = tl.entries[i].pool_release;
      dep_off[i] = k;
      for (int d : t.deps) {
        if (k < dep_cap) deps[k] = d;
        ++k;
      }
    }
    dep_off[n] = k;
    sim->makespan = tl.makespan;
    sim->compute_idle = tl.compute_idle;
    sim->compute_busy = tl.compute_busy;
    sim->peak_memory = tl.peak_memory;
    sim->fragmentation = mem.fragmentation;
    sim->peak_grad_buffer_bytes = mem.peak_grad_buffer_bytes;
    sim->ag_slot_count = pools.ag.slot_count;
    sim->rs_slot_count = pools.rs.slot_count;
    sim->ag_slot_bytes = pools.ag.slot_bytes;
    sim->rs_slot_bytes = pools.rs.slot_bytes;
    sim->r1_eliminated_ag = rep.r1_eliminated_ag;
    sim->r2_merged_rs = rep.r2_merged_rs;
    sim->r3_eliminated_ag = rep.r3_eliminated_ag;
    sim->extra_cached_bytes = rep.extra_cached_bytes;
    sim->total_static = hzp::ledger(spec, cfg).total_static;
    sim->peak_bytes = mem.peak_bytes;
    sim->utilization = hzp::utilization_report(tl, spec, device_flops);
    sim->n_samples = static_cast<int>(mem.samples.size());
    sim->sample_time_sum = 0.0;
    sim->sample_bytes_sum = 0;
    for (const auto& [t, b] : mem.samples) {
      sim->sample_time_sum += t;
      sim->sample_bytes_sum += b;
    }
    return n;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_derive_prelaunch_depth(long long layers, long long ppl, int dp, int z1, int z2,
                               int z3, long long free_budget) {
  hzp::ModelSpec spec;
  spec.num_layers = layers;
  spec.params_per_layer = ppl;
  hzp::CostModel cost;
  cost.topo.num_nodes = 1;
  cost.topo.ranks_per_node = dp;
  const auto g = hzp::build_task_graph(spec, cfg_of(dp, z1, z2, z3), cost, {});
  return hzp::derive_prelaunch_depth(g, free_budget);
}

// Wall-clock seconds per train_step_hzp<float> (mixed, bf16 working copy)
// over `steps` steps after one warm-up step — the CPU baseline of the path.
double ref_time_train_step_f32(const int* dims, int nl, int dp, int z1, int z2, int z3,
                               int mbs, int batch, unsigned long long seed, int steps) {
  const auto shape = shape_of(dims, nl);
  const auto cfg = cfg_of(dp, z1, z2, z3);
  auto states = hzp::shard_init<float>(shape, cfg, seed, true);
  const hzp::AdamParams adam;
  const auto b = batches_for<float>(shape, dp, mbs, batch, seed, 0);
  hzp::train_step_hzp(states, shape, cfg, b, batch, adam, true);
  const auto t0 = std::chrono::steady_clock::now();
  for (int s = 0; s < steps; ++s) hzp::train_step_hzp(states, shape, cfg, b, batch, adam, true);
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count() / (steps > 0 ? steps : 1);
}

// The reference's train_step_hzp<float> on `steps` run_case-seeded steps
// (per-(step, rank, mb) batches, train.cpp:501-508, generated before the
// clock starts), fp32 (bf16_working 0) or mixed (1); seconds per step.
// Optionally returns the final per-rank losses.
double ref_time_steps_f32(const int* dims, int nl, int dp, int z1, int z2, int z3, int mbs, int batch,
                          unsigned long long seed, int steps, int bf16_working, float* losses) {
  const auto shape = shape_of(dims, nl);
  const auto cfg = cfg_of(dp, z1, z2, z3);
  auto states = hzp::shard_init<float>(shape, cfg, seed, bf16_working != 0);
  const hzp::AdamParams adam;
  std::vector<hzp::RankBatches<float>> all;
  for (int s = 0; s < steps; ++s) all.push_back(batches_for<float>(shape, dp, mbs, batch, seed, s));
  std::vector<float> l;
  const auto t0 = std::chrono::steady_clock::now();
  for (int s = 0; s < steps; ++s) l = hzp::train_step_hzp(states, shape, cfg, all[s], batch, adam, bf16_working != 0);
  const auto t1 = std::chrono::steady_clock::now();
  if (losses)
    for (int r = 0; r < dp && r < static_cast<int>(l.size()); ++r) losses[r] = l[r];
  return std::chrono::duration<double>(t1 - t0).count() / (steps > 0 ? steps : 1);
}

}  // extern "C"
