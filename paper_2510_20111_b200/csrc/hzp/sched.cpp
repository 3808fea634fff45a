// Scheduler host code: launch order, pools, ring-slot simulation, LaunchPlan.
// Semantics follow /root/reference/proj/src/sched.cpp:75-387 and are checked
// bit-exactly (task list, deps, simulated start/end doubles) against
// tests/golden/sched.json by tests/test_host.py.
#include <array>
#include "hzp/sched.hpp"

#include <algorithm>
#include <map>

namespace hzp {

double collective_cost(CollectiveKind kind, const ProcessGroup& group, std::int64_t bytes,
                       const CostModel& model) {
  const int g = group.size();
  if (g <= 1 || bytes < 0) return 0.0;
  const bool x = group.spans_nodes;
  const double bw = x ? model.topo.inter_bw : model.topo.intra_bw;
  const double lat = x ? model.topo.inter_latency : model.topo.intra_latency;
  const double hops = static_cast<double>(g - 1);
  const double t = hops * (static_cast<double>(bytes) / g) / bw + hops * lat;
  return kind == CollectiveKind::AllReduce ? 2.0 * t : t;
}

const char* to_string(TaskKind kind) {
  static const char* const names[] = {"FWD",    "BWD",    "FWD-recompute", "AG-param",
                                      "RS-grad", "AR-dzp", "OPT-step",      "AG-post-step"};
  const int i = static_cast<int>(kind);
  return (i >= 0 && i < 8) ? names[i] : "?";
}

int TaskGraph::count(TaskKind kind) const {
  return static_cast<int>(std::count_if(tasks.begin(), tasks.end(),
                                        [kind](const Task& t) { return t.kind == kind; }));
}

StreamId stream_of(TaskKind kind) {
  switch (kind) {
    case TaskKind::AgParam:
    case TaskKind::AgPostStep:
      return StreamId::Ag;
    case TaskKind::RsGrad:
    case TaskKind::ArDzp:
      return StreamId::Rs;
    default:
      return StreamId::Compute;  // FWD, BWD, recompute, OPT
  }
}

bool uses_ag_pool(TaskKind kind) {
  return kind == TaskKind::AgParam || kind == TaskKind::AgPostStep;
}

bool is_comm(TaskKind kind) { return stream_of(kind) != StreamId::Compute; }

namespace {

// Emits tasks in issue order; the id of a task is its position.
class GraphWriter {
 public:
  explicit GraphWriter(TaskGraph& g) : g_(g) {}
  int emit(TaskKind kind, int layer, int mb, int vstage, Pass pass, double dur,
           std::int64_t bytes, std::vector<int> deps) {
    Task t;
    t.id = static_cast<int>(g_.tasks.size());
    t.kind = kind;
    t.layer = layer;
    t.microbatch = mb;
    t.virtual_stage = vstage;
    t.pass = pass;
    t.duration = dur;
    t.bytes = bytes;
    t.deps = std::move(deps);
    g_.tasks.push_back(std::move(t));
    return g_.tasks.back().id;
  }

 private:
  TaskGraph& g_;
};

}  // namespace

namespace {

struct SlotRun {  // one F or B slot of the graph: its tasks' layers, in order
  Pass pass;
  int mb, vstage;
  std::vector<int> layers;
};

std::vector<SlotRun> slot_runs(const TaskGraph& g) {
  std::vector<SlotRun> runs;
  for (const Task& t : g.tasks) {
    if (t.kind != TaskKind::Fwd && t.kind != TaskKind::Bwd) continue;
    if (runs.empty() || runs.back().pass != t.pass || runs.back().mb != t.microbatch ||
        runs.back().vstage != t.virtual_stage)
      runs.push_back({t.pass, t.microbatch, t.virtual_stage, {}});
    runs.back().layers.push_back(t.layer);
  }
  return runs;
}

}  // namespace

std::vector<ScheduleSlot> graph_slots(const TaskGraph& graph) {
  std::vector<ScheduleSlot> out;
  for (const SlotRun& r : slot_runs(graph)) out.push_back({r.pass, r.mb, r.vstage});
  return out;
}

ReuseReport apply_reuse(TaskGraph& graph) {
  const std::vector<SlotRun> runs = slot_runs(graph);
  // (pass, mb, vstage, layer) -> AG id;  (mb, vstage, layer) -> RS id
  std::map<std::array<int, 4>, int> ag;
  std::map<std::array<int, 3>, int> rs;
  for (const Task& t : graph.tasks) {
    if (t.kind == TaskKind::AgParam) ag[{int(t.pass), t.microbatch, t.virtual_stage, t.layer}] = t.id;
    if (t.kind == TaskKind::RsGrad) rs[{t.microbatch, t.virtual_stage, t.layer}] = t.id;
  }
  ReuseReport rep;
  std::vector<int> redirect(graph.tasks.size(), -1);  // dropped task -> keeper
  auto drop = [&](int victim, int keeper) {
    if (redirect[victim] >= 0) return false;
    redirect[victim] = keeper;
    return true;
  };
  auto serve_ags = [&](const SlotRun& from, const SlotRun& to) {
    int n = 0;
    for (int layer : to.layers)
      n += drop(ag.at({int(to.pass), to.mb, to.vstage, layer}), ag.at({int(from.pass), from.mb, from.vstage, layer}));
    return n;
  };
  const size_t n = runs.size();
  for (size_t i = 0; i + 1 < n; ++i)  // R1
    if (runs[i].pass == runs[i + 1].pass && runs[i].vstage == runs[i + 1].vstage)
      rep.r1_eliminated_ag += serve_ags(runs[i], runs[i + 1]);
  for (size_t i = 0; i + 2 < n; ++i)  // R3
    if (runs[i].pass == Pass::Forward && runs[i + 1].pass == Pass::Backward &&
        runs[i + 2].pass == Pass::Forward && runs[i].vstage == runs[i + 2].vstage) {
      const int k = serve_ags(runs[i], runs[i + 2]);
      rep.r3_eliminated_ag += k;
      if (k > 0) rep.extra_cached_bytes += std::int64_t(runs[i + 2].layers.size()) * graph.ag_slot_bytes;
    }
  for (size_t i = 0; i < n;) {  // R2
    if (runs[i].pass != Pass::Backward) {
      ++i;
      continue;
    }
    size_t j = i;
    while (j + 1 < n && runs[j + 1].pass == Pass::Backward && runs[j + 1].vstage == runs[i].vstage) ++j;
    for (int layer : runs[j].layers) {
      const int keeper = rs.at({runs[j].mb, runs[j].vstage, layer});
      for (size_t k = i; k < j; ++k) {
        const int victim = rs.at({runs[k].mb, runs[k].vstage, layer});
        if (!drop(victim, keeper)) continue;
        ++rep.r2_merged_rs;
        std::vector<int>& kd = graph.tasks[keeper].deps;
        for (int d : graph.tasks[victim].deps)
          if (std::find(kd.begin(), kd.end(), d) == kd.end()) kd.push_back(d);
      }
    }
    i = j + 1;
  }
  // compact: keep order, renumber, route deps through the (transitive) keepers
  std::vector<int> id_of(graph.tasks.size(), -1);
  std::vector<Task> out;
  for (const Task& t : graph.tasks)
    if (redirect[t.id] < 0) {
      id_of[t.id] = int(out.size());
      out.push_back(t);
    }
  for (Task& t : out) {
    std::vector<int> deps;
    for (int d : t.deps) {
      while (redirect[d] >= 0) d = redirect[d];
      const int nd = id_of[d];
      if (nd >= 0 && std::find(deps.begin(), deps.end(), nd) == deps.end()) deps.push_back(nd);
    }
    t.deps = std::move(deps);
    t.id = id_of[t.id];
  }
  graph.tasks = std::move(out);
  return rep;
}

void recompute_rule(TaskGraph& graph) {
  std::map<int, double> fwd_time;  // last FWD of each layer
  for (const Task& t : graph.tasks)
    if (t.kind == TaskKind::Fwd) fwd_time[t.layer] = t.duration;
  std::vector<int> moved(graph.tasks.size());
  std::vector<Task> out;
  out.reserve(graph.tasks.size() * 3 / 2);
  for (const Task& src : graph.tasks) {
    Task t = src;
    for (int& d : t.deps) d = moved[d];
    if (t.kind == TaskKind::Bwd) {
      Task rc;
      rc.id = int(out.size());
      rc.kind = TaskKind::FwdRecompute;
      rc.layer = t.layer;
      rc.microbatch = t.microbatch;
      rc.virtual_stage = t.virtual_stage;
      rc.pass = Pass::Backward;
      auto it = fwd_time.find(t.layer);
      rc.duration = it != fwd_time.end() ? it->second : t.duration / 2.0;
      rc.deps = t.deps;
      out.push_back(rc);
      std::vector<int> deps;
      for (int d : t.deps)
        if (out[d].kind == TaskKind::AgParam) deps.push_back(d);
      deps.push_back(rc.id);
      t.deps = std::move(deps);
    }
    t.id = int(out.size());
    moved[src.id] = t.id;
    out.push_back(std::move(t));
  }
  graph.tasks = std::move(out);
}

std::vector<ScheduleSlot> pipeline_order(int pp, int vpp, int microbatches, int rank) {
  using E = SchedError::Code;
  if (pp < 1 || vpp < 1 || microbatches < 1) throw SchedError(E::InvalidPolicy, "degrees must be >= 1");
  if (rank < 0 || rank >= pp) throw SchedError(E::InvalidPolicy, "rank out of range");
  if (vpp > 1 && microbatches % pp != 0)
    throw SchedError(E::InvalidPolicy, "interleaved schedule needs microbatches divisible by pp");
  // unit i of the forward stream -> (microbatch, virtual stage); backward
  // units walk the virtual stages in reverse.  vpp == 1 reduces to 1F1B.
  const int units = microbatches * vpp;
  auto fwd = [&](int i) {
    return ScheduleSlot{Pass::Forward, (i / (pp * vpp)) * pp + i % pp, (i / pp) % vpp};
  };
  auto bwd = [&](int i) {
    return ScheduleSlot{Pass::Backward, (i / (pp * vpp)) * pp + i % pp, vpp - 1 - (i / pp) % vpp};
  };
  const int warm = vpp == 1 ? std::min(pp - rank - 1, microbatches)
                            : std::min(2 * (pp - rank - 1) + (vpp - 1) * pp, units);
  std::vector<ScheduleSlot> order;
  int f = 0, b = 0;
  while (f < warm) order.push_back(fwd(f++));
  while (f < units) {
    order.push_back(fwd(f++));
    order.push_back(bwd(b++));
  }
  while (b < units) order.push_back(bwd(b++));
  return order;
}

TaskGraph build_task_graph(const ModelSpec& spec, const ParallelConfig& cfg,
                           const CostModel& cost, const GraphPolicy& policy) {
  using E = SchedError::Code;
  if (cfg.tp != 1) throw SchedError(E::InvalidPolicy, "task graphs model the sharded path; tp must be 1");
  const std::int64_t chunks = std::int64_t(cfg.pp) * cfg.vpp;
  if (spec.num_layers % chunks != 0)
    throw SchedError(E::InvalidPolicy, "num_layers must divide evenly into pp*vpp chunks");
  if (policy.rank < 0 || policy.rank >= cfg.pp) throw SchedError(E::InvalidPolicy, "rank out of range");

  std::vector<ScheduleSlot> order = policy.order;
  if (order.empty()) {
    for (int mb = 0; mb < spec.num_microbatches; ++mb) {
      order.push_back({Pass::Forward, mb, 0});
      order.push_back({Pass::Backward, mb, 0});
    }
  }
  for (const auto& s : order)
    if (s.virtual_stage < 0 || s.virtual_stage >= cfg.vpp || s.microbatch < 0 ||
        s.microbatch >= spec.num_microbatches)
      throw SchedError(E::InvalidPolicy, "schedule slot outside configured ranges");

  const GroupMap groups = build_process_groups(cfg, cost.topo);
  const ProcessGroup& z3 = groups.at(GroupKind::Z3).front();
  const ProcessGroup& z2 = groups.at(GroupKind::Z2).front();
  const ProcessGroup& dzp = groups.at(GroupKind::DzpReplica).front();

  TaskGraph g;
  g.spec = spec;
  g.cfg = cfg;
  g.rank = policy.rank;
  g.ag_slot_bytes = 2 * spec.params_per_layer;   // bf16 working copy of one layer
  g.grad_buf_bytes = 4 * spec.params_per_layer;  // fp32 gradient of one layer
  g.compute_flops_per_sec = cost.device_flops;
  const double t_ag = collective_cost(CollectiveKind::AllGather, z3, g.ag_slot_bytes, cost);
  const double t_rs = collective_cost(CollectiveKind::ReduceScatter, z2, g.grad_buf_bytes, cost);
  const double t_fwd = spec.flops_per_token_per_layer * static_cast<double>(spec.seq_len) *
                       static_cast<double>(spec.micro_batch_size) / cost.device_flops;
  const double t_bwd = 2.0 * t_fwd;

  const std::int64_t per_chunk = spec.num_layers / chunks;
  auto layers_of = [&](int vstage) {
    const std::int64_t c = std::int64_t(vstage) * cfg.pp + policy.rank;
    std::vector<int> ls;
    for (std::int64_t l = c * per_chunk; l < (c + 1) * per_chunk; ++l) ls.push_back(int(l));
    return ls;
  };

  GraphWriter w(g);
  int prev_compute = -1, last_bwd = -1;
  std::vector<int> rs_all;
  std::map<int, std::vector<int>> rs_of_layer;  // ascending layer iteration
  struct Deferred { int layer, mb, vstage, bwd; };
  std::vector<Deferred> deferred;

  auto gathered_compute = [&](TaskKind kind, int l, const ScheduleSlot& s, double dur) {
    const int ag = w.emit(TaskKind::AgParam, l, s.microbatch, s.virtual_stage, s.pass, t_ag,
                          g.ag_slot_bytes, {});
    std::vector<int> deps{ag};
    if (prev_compute >= 0) deps.push_back(prev_compute);
    prev_compute = w.emit(kind, l, s.microbatch, s.virtual_stage, s.pass, dur, 0, std::move(deps));
    return prev_compute;
  };

  for (const auto& s : order) {
    std::vector<int> ls = layers_of(s.virtual_stage);
    if (s.pass == Pass::Forward) {
      for (int l : ls) gathered_compute(TaskKind::Fwd, l, s, t_fwd);
      continue;
    }
    std::reverse(ls.begin(), ls.end());
    for (int l : ls) {
      const int bwd = gathered_compute(TaskKind::Bwd, l, s, t_bwd);
      last_bwd = bwd;
      if (policy.defer_rs) {
        deferred.push_back({l, s.microbatch, s.virtual_stage, bwd});
        continue;
      }
      const int rs = w.emit(TaskKind::RsGrad, l, s.microbatch, s.virtual_stage, Pass::Backward,
                            t_rs, g.grad_buf_bytes, {bwd});
      rs_all.push_back(rs);
      rs_of_layer[l].push_back(rs);
    }
  }
  for (const auto& d : deferred) {
    std::vector<int> deps{d.bwd};
    if (last_bwd >= 0 && last_bwd != d.bwd) deps.push_back(last_bwd);
    const int rs = w.emit(TaskKind::RsGrad, d.layer, d.mb, d.vstage, Pass::Backward, t_rs,
                          g.grad_buf_bytes, std::move(deps));
    rs_all.push_back(rs);
    rs_of_layer[d.layer].push_back(rs);
  }

  // Tail: per-layer DZP all-reduce (only with >1 replica), one optimizer
  // step, per-layer post-step all-gather of the rebuilt working copy.
  std::vector<int> opt_deps = rs_all;
  if (cfg.dp / cfg.z2 > 1) {
    opt_deps.clear();
    const std::int64_t shard_bytes = 4 * shard_elems(spec.params_per_layer, cfg.z2);
    const double t_ar = collective_cost(CollectiveKind::AllReduce, dzp, shard_bytes, cost);
    for (const auto& [layer, ids] : rs_of_layer)
      opt_deps.push_back(
          w.emit(TaskKind::ArDzp, layer, -1, 0, Pass::None, t_ar, shard_bytes, ids));
  }
  const int opt = w.emit(TaskKind::OptStep, -1, -1, 0, Pass::None, 0.0, 0, std::move(opt_deps));
  for (const auto& kv : rs_of_layer)
    w.emit(TaskKind::AgPostStep, kv.first, -1, 0, Pass::None, t_ag, g.ag_slot_bytes, {opt});
  return g;
}

PoolSet make_pools(const TaskGraph& graph, int prelaunch_depth, int rs_slots) {
  PoolSet p;
  p.ag.slot_count = std::max(1, prelaunch_depth);
  p.ag.slot_bytes = graph.ag_slot_bytes;
  p.ag.capacity = p.ag.slot_bytes * p.ag.slot_count;
  p.rs.slot_count = std::max(1, rs_slots);
  p.rs.slot_bytes = graph.grad_buf_bytes;
  p.rs.capacity = p.rs.slot_bytes * p.rs.slot_count;
  return p;
}

int derive_prelaunch_depth(const TaskGraph& graph, std::int64_t free_budget) {
  if (graph.ag_slot_bytes <= 0) return 1;
  const std::int64_t hi = std::max<std::int64_t>(1, graph.spec.num_layers);
  return static_cast<int>(std::clamp<std::int64_t>(free_budget / graph.ag_slot_bytes, 1, hi));
}

namespace {

std::vector<int> first_consumers(const TaskGraph& g) {
  std::vector<int> fc(g.tasks.size(), -1);
  for (const auto& t : g.tasks)
    for (int d : t.deps)
      if (fc[d] < 0) fc[d] = t.id;
  return fc;
}

// The ring rule shared by simulate() and the LaunchPlan: which earlier task
// must finish before task `t` may occupy its pool slot.
struct RingState {
  std::vector<int> ag_order, rs_order;
  int depth, rs_slots;
  const std::vector<int>& fc;
  RingState(int d, int r, const std::vector<int>& f) : depth(d), rs_slots(r), fc(f) {}
  // returns {slot, blocking task whose end frees it (or -1), blocking AG}
  std::pair<int, int> admit(const Task& t, int* ag_blocker) {
    *ag_blocker = -1;
    if (uses_ag_pool(t.kind)) {
      const int k = static_cast<int>(ag_order.size());
      int wait = -1;
      if (k >= depth) {
        const int blocking = ag_order[k - depth];
        *ag_blocker = blocking;
        wait = fc[blocking] >= 0 ? fc[blocking] : blocking;
      }
      ag_order.push_back(t.id);
      return {k % depth, wait};
    }
    if (t.kind == TaskKind::RsGrad) {
      const int k = static_cast<int>(rs_order.size());
      const int wait = k >= rs_slots ? rs_order[k - rs_slots] : -1;
      rs_order.push_back(t.id);
      return {k % rs_slots, wait};
    }
    return {-1, -1};
  }
};

// Interval bookkeeping for the memory sweeps: each hold adds +amount at t0
// and -amount at t1; sweeps visit events by time, equal times in insertion
// order (a stable sort), which fixes how coincident frees and allocations
// count toward a peak.
struct Events {
  std::vector<std::pair<double, std::int64_t>> ev;
  void hold(double t0, double t1, std::int64_t amount) {
    ev.emplace_back(t0, amount);
    ev.emplace_back(t1, -amount);
  }
  void sort() {
    std::stable_sort(ev.begin(), ev.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  }
  std::int64_t peak() {
    sort();
    std::int64_t live = 0, top = 0;
    for (const auto& [t, d] : ev) top = std::max(top, live += d);
    return top;
  }
};

// Everything a timeline derives from its tasks' start / end times: release
// points (an AG's buffer lives until its LAST consumer ends, its pool slot
// until its FIRST consumer ends), makespan, compute busy / idle
// (sched.cpp:341-350) and the dynamic-memory samples (pool slots + the
// unsharded gradients each RS consumes).  `dur` = the busy time per task.
void derive_timeline(const TaskGraph& graph, const PoolSet& pools, const std::vector<double>& dur, Timeline& tl) {
  const int n = static_cast<int>(graph.tasks.size());
  const std::vector<int> fc = first_consumers(graph);
  std::vector<double> last_use(n, 0.0);
  for (const auto& t : graph.tasks)
    for (int d : t.deps) last_use[d] = std::max(last_use[d], tl.entries[t.id].end);
  double last_compute = 0.0;
  for (int id = 0; id < n; ++id) {
    auto& e = tl.entries[id];
    e.buffer_release = std::max(e.end, last_use[id]);
    e.pool_release = fc[id] >= 0 ? tl.entries[fc[id]].end : e.end;
    tl.makespan = std::max(tl.makespan, e.end);
    if (e.stream == StreamId::Compute) {
      tl.compute_busy += dur[id];
      last_compute = std::max(last_compute, e.end);
    }
  }
  tl.compute_idle = last_compute - tl.compute_busy;
  Events mem;
  for (int id = 0; id < n; ++id) {
    const Task& t = graph.tasks[id];
    const auto& e = tl.entries[id];
    if (uses_ag_pool(t.kind)) {
      mem.hold(e.start, e.buffer_release, pools.ag.slot_bytes);
    } else if (t.kind == TaskKind::RsGrad) {
      mem.hold(e.start, e.end, pools.rs.slot_bytes);
      for (int d : t.deps)
        if (graph.tasks[d].kind == TaskKind::Bwd && graph.tasks[d].layer == t.layer)
          mem.hold(tl.entries[d].end, e.end, graph.grad_buf_bytes);
    }
  }
  mem.sort();
  std::int64_t live = 0;
  for (const auto& [t, d] : mem.ev) {
    live += d;
    if (!tl.memory_samples.empty() && tl.memory_samples.back().first == t)
      tl.memory_samples.back().second = std::max(tl.memory_samples.back().second, live);
    else
      tl.memory_samples.emplace_back(t, live);
    tl.peak_memory = std::max(tl.peak_memory, live);
  }
}

}  // namespace

Timeline simulate(const TaskGraph& graph, const PoolSet& pools, SchedMode mode) {
  using E = SchedError::Code;
  if (pools.ag.slot_count < 1 || pools.rs.slot_count < 1)
    throw SchedError(E::InvalidPolicy, "pools need at least one slot each");
  const int n = static_cast<int>(graph.tasks.size());
  const std::vector<int> fc = first_consumers(graph);
  RingState ring(pools.ag.slot_count, pools.rs.slot_count, fc);
  std::vector<double> t0(n, 0.0), t1(n, 0.0);
  double free_at[3] = {0.0, 0.0, 0.0};
  double comm_horizon = 0.0;  // vanilla: compute may not pass issued comm

  Timeline tl;
  tl.mode = mode;
  tl.entries.resize(n);
  for (int id = 0; id < n; ++id) {
    const Task& t = graph.tasks[id];
    const StreamId sid = stream_of(t.kind);
    double at = free_at[int(sid)];
    for (int d : t.deps) {
      if (d >= id) throw SchedError(E::DeadlockDetected, "dependency on a later task in issue order");
      at = std::max(at, t1[d]);
    }
    if (mode == SchedMode::Vanilla && sid == StreamId::Compute) at = std::max(at, comm_horizon);
    int ag_blocker = -1;
    const auto [slot, wait] = ring.admit(t, &ag_blocker);
    (void)slot;
    if (wait >= 0) {
      if (ag_blocker >= 0 && fc[ag_blocker] >= id)
        throw SchedError(E::DeadlockDetected, "pool slot held by an unscheduled consumer");
      at = std::max(at, t1[wait]);
    }
    t0[id] = at;
    t1[id] = at + t.duration;
    free_at[int(sid)] = t1[id];
    if (mode == SchedMode::Vanilla && is_comm(t.kind)) comm_horizon = std::max(comm_horizon, t1[id]);
    auto& e = tl.entries[id];
    e.task_id = id;
    e.kind = t.kind;
    e.layer = t.layer;
    e.microbatch = t.microbatch;
    e.stream = sid;
    e.start = t0[id];
    e.end = t1[id];
    e.bytes = t.bytes;
  }
  std::vector<double> dur(n);
  for (int id = 0; id < n; ++id) dur[id] = graph.tasks[id].duration;
  derive_timeline(graph, pools, dur, tl);
  return tl;
}

void finish_timeline(const TaskGraph& graph, const PoolSet& pools, Timeline& tl) {
  const int n = static_cast<int>(graph.tasks.size());
  if (static_cast<int>(tl.entries.size()) != n) throw std::invalid_argument("timeline / graph size mismatch");
  std::vector<double> dur(n);
  for (int id = 0; id < n; ++id) {
    const Task& t = graph.tasks[id];
    auto& e = tl.entries[id];
    e.task_id = id;
    e.kind = t.kind;
    e.layer = t.layer;
    e.microbatch = t.microbatch;
    e.stream = stream_of(t.kind);
    e.bytes = t.bytes;
    dur[id] = e.end - e.start;
  }
  tl.makespan = tl.compute_busy = tl.compute_idle = 0.0;
  tl.memory_samples.clear();
  tl.peak_memory = 0;
  derive_timeline(graph, pools, dur, tl);
}

MemoryTraceResult memory_trace(const Timeline& timeline, const MemoryLedger& ledger, const PoolSet& pools) {
  MemoryTraceResult out;
  out.peak_bytes = ledger.total_static + timeline.peak_memory;
  out.samples.reserve(timeline.memory_samples.size());
  for (const auto& [t, live] : timeline.memory_samples) out.samples.emplace_back(t, ledger.total_static + live);

  Events ag, rs, grad;
  for (const auto& e : timeline.entries) {
    if (uses_ag_pool(e.kind)) ag.hold(e.start, e.pool_release, pools.ag.slot_bytes);  // ring slot
    else if (e.kind == TaskKind::RsGrad) rs.hold(e.start, e.end, pools.rs.slot_bytes);
  }
  // gradient buffers, counted: BWD(l, mb) end -> end of the RS that consumes it
  std::map<std::pair<int, int>, double> open;  // (layer, mb) -> BWD end
  std::map<int, double> last_rs;               // layer -> latest RS end
  for (const auto& e : timeline.entries) {
    if (e.kind == TaskKind::Bwd) {
      open[{e.layer, e.microbatch}] = e.end;
    } else if (e.kind == TaskKind::RsGrad) {
      const auto it = open.find({e.layer, e.microbatch});
      if (it != open.end()) {
        grad.hold(it->second, e.end, 1);
        open.erase(it);
      }
      last_rs[e.layer] = std::max(last_rs[e.layer], e.end);
    }
  }
  // a BWD whose RS was merged away (reuse R2) holds its buffer until the
  // layer's last RS ends
  for (const auto& [key, t_bwd] : open) {
    const auto it = last_rs.find(key.first);
    if (it != last_rs.end() && it->second > t_bwd) grad.hold(t_bwd, it->second, 1);
  }
  const std::int64_t live_pools =
      std::min(ag.peak(), pools.ag.capacity) + std::min(rs.peak(), pools.rs.capacity);
  const std::int64_t reserved = pools.ag.capacity + pools.rs.capacity;
  out.fragmentation = reserved > 0 ? static_cast<double>(reserved - live_pools) / static_cast<double>(reserved) : 0.0;
  out.peak_grad_buffer_bytes = grad.peak() * pools.rs.slot_bytes;
  return out;
}

double utilization_report(const Timeline& timeline, const ModelSpec& spec, double peak_flops) {
  // forward + backward = 3 x forward FLOPs over every token of every layer
  const double model_flops = 3.0 * spec.flops_per_token_per_layer * static_cast<double>(spec.seq_len) *
                             static_cast<double>(spec.micro_batch_size) *
                             static_cast<double>(spec.num_microbatches) * static_cast<double>(spec.num_layers);
  if (timeline.makespan <= 0.0 || peak_flops <= 0.0) return 0.0;
  return model_flops / (timeline.makespan * peak_flops);
}

LaunchPlan build_launch_plan(const TaskGraph& graph, const PoolSet& pools) {
  const std::vector<int> fc = first_consumers(graph);
  RingState ring(pools.ag.slot_count, pools.rs.slot_count, fc);
  LaunchPlan plan;
  plan.depth = pools.ag.slot_count;
  plan.rs_slots = pools.rs.slot_count;
  plan.entries.reserve(graph.tasks.size());
  for (const Task& t : graph.tasks) {
    PlanEntry e;
    e.id = t.id;
    e.kind = t.kind;
    e.layer = t.layer;
    e.microbatch = t.microbatch;
    e.stream = stream_of(t.kind);
    int ag_blocker = -1;
    const auto [slot, wait] = ring.admit(t, &ag_blocker);
    if (wait >= t.id)
      throw SchedError(SchedError::Code::DeadlockDetected, "pool slot held by an unscheduled consumer");
    e.slot = slot;
    e.ring_wait = wait;
    e.waits = t.deps;
    if (wait >= 0 && std::find(e.waits.begin(), e.waits.end(), wait) == e.waits.end())
      e.waits.push_back(wait);
    plan.entries.push_back(std::move(e));
  }
  return plan;
}

}  // namespace hzp
