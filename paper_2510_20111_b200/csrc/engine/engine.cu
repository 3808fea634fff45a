// Device engine: buffers, P2P wiring, tile tables and the stream/event
// executor that walks the LaunchPlan.
//
// Executor contract:
//  * three CUDA streams per GPU mirror the reference's stream split
//    (sched.cpp:36-51): compute {FWD, BWD, OPT}, ag {AG-param, AG-post},
//    rs {RS-grad, AR-dzp}; comm streams run at high priority;
//  * tasks are issued in task-id order; a task waits (cudaStreamWaitEvent)
//    for every entry of its plan wait-list that ran on another stream, so
//    every event is recorded before it is waited on;
//  * AG-pool slot = k % depth and the ring wait = first consumer of AG-pool
//    task k-depth (the reference's ring rule), RS ring likewise;
//  * the tail AR-dzp(l) + OPT + AG-post(l) collapses into ONE fused kernel
//    (z1_adam: replica pull-reduce + Adam + bf16 P2P store), logged as
//    covering those task ids.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "engine/engine.hpp"
#include "engine/gemm.cuh"

namespace hzp {
namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

Engine::Engine(const hzp_engine_config& c) : cfg(c) {
  if (c.par.dp < 1 || c.par.dp > kMaxRanks) throw std::invalid_argument("dp must be in [1, 64]");
  for (int z : {c.par.z1, c.par.z2, c.par.z3})
    if (z < 1 || c.par.dp % z) throw ValidationError(ValidationError::Code::NonDivisible, "z does not divide dp");
  bf16 = c.precision == HZP_PREC_BF16;
  mcfg.kind = c.model;
  mcfg.bf16 = bf16;
  mcfg.batch = c.batch;
  if (c.model == HZP_MODEL_MLP) {
    if (c.num_dims < 2 || c.num_dims > 32) throw std::invalid_argument("MLP needs 2..32 dims");
    mcfg.dims.assign(c.dims, c.dims + c.num_dims);
    model = make_mlp_model(mcfg);
  } else {
    mcfg.layers = c.gpt_layers;
    mcfg.hidden = c.gpt_hidden;
    mcfg.heads = c.gpt_heads;
    mcfg.ffn = c.gpt_ffn;
    mcfg.vocab = c.gpt_vocab;
    mcfg.seq = c.gpt_seq;
    mcfg.experts = c.gpt_experts;
    mcfg.topk = c.gpt_topk;
    mcfg.capacity = c.gpt_capacity;
    mcfg.recompute = c.recompute;
    if (!bf16) throw std::invalid_argument("the GPT model runs in bf16 only");
    model = make_gpt_model(mcfg);
  }
  HZP_CUDA(cudaSetDevice(c.device));
  const int L = model->num_layers();
  for (int l = 0; l < L; ++l) layers.push_back(model->layer(l));
  geom = ShardGeom(model->param_count(), ParallelConfig{c.par.dp, c.par.z1, c.par.z2, c.par.z3});
  slot_elems = static_cast<int64_t>(align_up(size_t(model->max_layer_size()), 128));
  emulate = c.my_rank < 0;
  depth = std::max(1, c.prelaunch_depth);
  rs_slots = std::max(1, c.rs_slots);
  wslots = std::max(2, c.wgrad_slots);
  direct_grad = geom.z2 == 1;
  zero_copy_ag = geom.z3 == 1;

  // ---- task graph + plan (the drop-in scheduler) ----
  ModelSpec spec;
  spec.num_layers = L;
  spec.params_per_layer = std::max<int64_t>(1, model->max_layer_size());
  spec.num_microbatches = std::max(1, c.num_microbatches);
  spec.seq_len = 1;
  spec.micro_batch_size = 1;
  CostModel cost;
  cost.topo.num_nodes = 1;
  cost.topo.ranks_per_node = c.par.dp;
  graph = build_task_graph(spec, ParallelConfig{c.par.dp, c.par.z1, c.par.z2, c.par.z3}, cost, {});
  if (c.reuse) apply_reuse(graph);
  if (c.recompute) recompute_rule(graph);
  pools = make_pools(graph, depth, rs_slots);
  plan = build_launch_plan(graph, pools);
  {
    const int nt = static_cast<int>(graph.tasks.size());
    auto is_compute = [](TaskKind k) {
      return k == TaskKind::Fwd || k == TaskKind::Bwd || k == TaskKind::FwdRecompute;
    };
    std::vector<int> passes(nt, 0), last_use(nt, -1);
    for (const Task& t : graph.tasks) {
      if (!is_compute(t.kind)) continue;
      if (t.deps.empty() || graph.tasks[t.deps[0]].kind != TaskKind::AgParam)
        throw std::logic_error("compute task without its all-gather as first dependency");
      if (t.kind != TaskKind::FwdRecompute) ++passes[t.deps[0]];
      for (int d : t.deps)
        if (graph.tasks[d].kind == TaskKind::AgParam) last_use[d] = t.id;
    }
    ag_slot.assign(nt, -1);
    param_slot.assign(nt, -1);
    ag_phys_wait.assign(nt, -1);
    std::vector<int> ring;  // AG-pool issue order (plan ring rule)
    for (const Task& t : graph.tasks) {
      if (t.kind == TaskKind::AgParam) {
        // several passes read it (reuse): it outlives its ring slot
        const bool cached = passes[t.id] > 1 && !zero_copy_ag;
        ag_slot[t.id] = cached ? depth + t.layer : plan.entries[t.id].slot;
        if (cached) cache_slots = L;
        // the ring frees a slot at its occupant's FIRST consumer; a later
        // reader (the BWD after its FWD-recompute) must finish before the
        // slot is overwritten on the device
        const int k = static_cast<int>(ring.size());
        if (k >= depth && !cached && !zero_copy_ag) {
          const int prev = ring[k - depth];
          const bool prev_in_ring = ag_slot[prev] < depth;
          if (prev_in_ring && last_use[prev] >= 0 && last_use[prev] != plan.entries[t.id].ring_wait) {
            if (last_use[prev] > t.id) throw std::logic_error("slot reader issued after the AG that overwrites it");
            ag_phys_wait[t.id] = last_use[prev];
          }
        }
      }
      if (uses_ag_pool(t.kind)) ring.push_back(t.id);
      if (is_compute(t.kind)) param_slot[t.id] = -2;
    }
    for (const Task& t : graph.tasks)
      if (param_slot[t.id] == -2) param_slot[t.id] = ag_slot[t.deps[0]];
  }

  // ---- streams / events ----
  int lo = 0, hi = 0;
  HZP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  HZP_CUDA(cudaStreamCreateWithPriority(&st[0], cudaStreamNonBlocking, lo));
  HZP_CUDA(cudaStreamCreateWithPriority(&st[1], cudaStreamNonBlocking, hi));
  HZP_CUDA(cudaStreamCreateWithPriority(&st[2], cudaStreamNonBlocking, hi));
  const int n = static_cast<int>(plan.entries.size());
  done.resize(n);
  for (auto& e : done) HZP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (c.timeline) {
    tev0.resize(n);
    tev1.resize(n);
    for (int i = 0; i < n; ++i) {
      HZP_CUDA(cudaEventCreate(&tev0[i]));
      HZP_CUDA(cudaEventCreate(&tev1[i]));
    }
  }
  HZP_CUDA(cudaEventCreate(&ev_step0));
  HZP_CUDA(cudaEventCreate(&ev_step1));
  HZP_CUDA(cudaEventCreateWithFlags(&ev_opt, cudaEventDisableTiming));

  // ---- per-rank peer-visible arenas ----
  const int es = bf16 ? 2 : 4;
  const size_t p_bytes = align_up(size_t(geom.s3) * es, 256);
  const size_t g_bytes = align_up(size_t(geom.s2) * 4, 256);
  const size_t w_bytes = direct_grad ? 0 : align_up(size_t(wslots) * slot_elems * es, 256);
  const size_t f_bytes = align_up(sizeof(uint64_t) * kNumFlagKinds * kMaxRanks, 256);
  arenas.resize(c.par.dp);
  std::vector<int> mine;
  if (emulate) {
    mine.resize(c.par.dp);
    std::iota(mine.begin(), mine.end(), 0);
  } else {
    if (c.my_rank >= c.par.dp) throw std::invalid_argument("my_rank out of range");
    mine.push_back(c.my_rank);
  }
  for (int r : mine) {
    Arena& a = arenas[r];
    a.bytes = p_bytes + g_bytes + w_bytes + f_bytes;
    HZP_CUDA(cudaMalloc(&a.base, a.bytes));
    HZP_CUDA(cudaMemset(a.base, 0, a.bytes));
    a.owned = true;
  }
  auto carve = [&](Arena& a) {
    char* b = static_cast<char*>(a.base);
    a.param = b;
    a.grad = reinterpret_cast<float*>(b + p_bytes);
    a.wgrad = w_bytes ? b + p_bytes + g_bytes : nullptr;
    a.flags = reinterpret_cast<uint64_t*>(b + p_bytes + g_bytes + w_bytes);
  };
  for (int r : mine) carve(arenas[r]);

  // ---- driven ranks ----
  for (int r : mine) {
    LocalRank lr;
    lr.rank = r;
    HZP_CUDA(cudaMalloc(&lr.ag, size_t(depth + cache_slots) * slot_elems * es));
    HZP_CUDA(cudaMalloc(&lr.master, size_t(geom.s1) * 4));
    HZP_CUDA(cudaMalloc(&lr.mom, size_t(geom.s1) * 4));
    HZP_CUDA(cudaMalloc(&lr.var, size_t(geom.s1) * 4));
    HZP_CUDA(cudaMemset(lr.master, 0, size_t(geom.s1) * 4));
    HZP_CUDA(cudaMemset(lr.mom, 0, size_t(geom.s1) * 4));
    HZP_CUDA(cudaMemset(lr.var, 0, size_t(geom.s1) * 4));
    if (geom.P < (int64_t(1) << 24)) HZP_CUDA(cudaMalloc(&lr.dbg, size_t(geom.s1) * 4));
    lr.mbuf = model->alloc_rank_buffers();
    locals.push_back(lr);
  }
  HZP_CUDA(cudaMallocHost(&hloss, sizeof(float) * locals.size()));
  input_bytes_per_mb = size_t(model->input_elems_per_mb()) * model->input_elem_bytes();
  HZP_CUDA(cudaMalloc(&dinputs, std::max<size_t>(256, input_bytes_per_mb * locals.size() *
                                                         std::max(1, c.num_microbatches))));

  // ---- pointer table ----
  std::memset(&table, 0, sizeof(table));
  for (int r = 0; r < c.par.dp; ++r) {
    table.param[r] = arenas[r].param;
    table.grad[r] = arenas[r].grad;
    table.wgrad[r] = arenas[r].wgrad;
    table.flags[r] = arenas[r].flags;
  }
  for (size_t i = 0; i < locals.size(); ++i) {
    table.ag_slots[i] = locals[i].ag;
    table.master[i] = locals[i].master;
    table.mom[i] = locals[i].mom;
    table.var[i] = locals[i].var;
    table.z1_grad_dbg[i] = locals[i].dbg;
    table.global_rank[i] = locals[i].rank;
  }
  HZP_CUDA(cudaMalloc(&dtable, sizeof(RankTable)));
  HZP_CUDA(cudaMemcpy(dtable, &table, sizeof(RankTable), cudaMemcpyHostToDevice));
  peers_open = emulate || c.par.dp == 1;
  debug_sync = std::getenv("HZP_DEBUG_SYNC") != nullptr;
  if (const char* c = std::getenv("HZP_COMM_CTAS")) comm_ctas = std::max(1, std::atoi(c));  // tuning knob
  if (const char* c = std::getenv("HZP_AG_CE")) ag_ce = std::atoi(c) != 0;
  if (const char* c = std::getenv("HZP_RS_CE")) rs_ce = std::atoi(c) != 0;
  if (const char* c = std::getenv("HZP_Z1_CE")) z1_ce = std::atoi(c) != 0;
  if (const char* c = std::getenv("HZP_RS_CHUNKS")) rs_chunks = std::max(1, std::atoi(c));
  if (const char* c = std::getenv("HZP_RS_PAR")) rs_par = std::atoi(c) != 0;
  if (const char* c = std::getenv("HZP_AG_PAR")) ag_par = std::atoi(c) != 0;
  if (const char* c = std::getenv("HZP_RS_MIN_CHUNK_MB")) rs_min_chunk_bytes = std::max<int64_t>(1, std::atoll(c)) << 20;
  build_tiles();
}

Engine::~Engine() {
  cudaDeviceSynchronize();
  for (auto& l : locals) {
    cudaFree(l.ag);
    cudaFree(l.master);
    cudaFree(l.mom);
    cudaFree(l.var);
    cudaFree(l.dbg);
    model->free_rank_buffers(l.mbuf);
  }
  for (auto& a : arenas) {
    if (a.base && a.owned) cudaFree(a.base);
    else if (a.base) cudaIpcCloseMemHandle(a.base);
  }
  cudaFree(dtable);
  for (auto d : dtable_staged) cudaFree(d);
  for (auto e : rs_ev) cudaEventDestroy(e);
  for (auto& ch : z1_chunks) cudaFree(ch.table);
  for (auto p : z1_stage) cudaFree(p);
  if (z1_copy_stream) cudaStreamDestroy(z1_copy_stream);
  if (rs_red_stream) cudaStreamDestroy(rs_red_stream);
  for (auto st : rs_copy_streams) cudaStreamDestroy(st);
  for (auto st : ag_copy_streams) cudaStreamDestroy(st);
  for (auto e : ag_par_ev) cudaEventDestroy(e);
  for (auto e : rs_par_ev) cudaEventDestroy(e);
  for (auto p : rs_stage) cudaFree(p);
  cudaFree(dtiles);
  cudaFree(dinputs);
  cudaFreeHost(hloss);
  for (auto e : done) cudaEventDestroy(e);
  for (auto e : tev0) cudaEventDestroy(e);
  for (auto e : tev1) cudaEventDestroy(e);
  cudaEventDestroy(ev_step0);
  cudaEventDestroy(ev_step1);
  cudaEventDestroy(ev_opt);
  for (auto s : st) cudaStreamDestroy(s);
}

int Engine::local_index(int rank) const {
  for (size_t i = 0; i < locals.size(); ++i)
    if (locals[i].rank == rank) return int(i);
  return -1;
}

void Engine::build_tiles() {
  std::vector<Range64> lr;
  for (const auto& l : layers) lr.push_back({l.off, l.size});
  std::vector<int> ranks;
  for (const auto& l : locals) ranks.push_back(l.rank);
  TileTables T = build_comm_tiles(geom, lr, ranks, bf16 ? 2 : 4, direct_grad);
  ag_off = T.ag_off;
  rs_off = T.rs_off;
  tiles_host = T.tiles;
  ag_runs.assign(ag_off.size() > 0 ? ag_off.size() - 1 : 0, {});
  for (size_t l = 0; l + 1 < ag_off.size(); ++l)
    for (int i = ag_off[l]; i < ag_off[l + 1]; ++i) {
      const CommTile& t = T.tiles[i];
      auto& runs = ag_runs[l];
      if (!runs.empty()) {
        CopyRun& r = runs.back();
        if (r.local == t.local && r.src == t.src && r.dst_off + r.len == t.a_off && r.src_off + r.len == t.b_off) {
          r.len += t.len;
          continue;
        }
      }
      runs.push_back({t.local, t.src, t.a_off, t.b_off, t.len});
    }
  if (!emulate && locals.size() == 1) {
    // rotate the owners: rank r reads owner r+1 first, r+2 next, ..., its own
    // shard last, so at every moment each owner's egress serves one reader
    // (ascending order would have every rank hit owner 0 first)
    const int me = cfg.my_rank % geom.z3;
    auto phase = [&](const CopyRun& r) { return (r.src % geom.z3 - me - 1 + 2 * geom.z3) % geom.z3; };
    for (auto& runs : ag_runs)
      std::stable_sort(runs.begin(), runs.end(),
                       [&](const CopyRun& a, const CopyRun& b) { return phase(a) < phase(b); });
    if (ag_par && geom.z3 > 2 && ag_copy_streams.empty()) {
      int lo = 0, hi = 0;
      HZP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      ag_copy_streams.resize(geom.z3 - 1);
      for (auto& st : ag_copy_streams) HZP_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
      ag_par_ev.resize(geom.z3);
      for (auto& e : ag_par_ev) HZP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  }
  z1_off = T.z1_off;
  z1_n = T.z1_n;
  if (dtiles) cudaFree(dtiles);
  HZP_CUDA(cudaMalloc(&dtiles, std::max<size_t>(1, T.tiles.size()) * sizeof(CommTile)));
  if (!T.tiles.empty())
    HZP_CUDA(cudaMemcpy(dtiles, T.tiles.data(), T.tiles.size() * sizeof(CommTile), cudaMemcpyHostToDevice));
}

void Engine::ag_layer(int layer, int slot, cudaStream_t s) {
  if (ag_ce && !emulate) {  // multi-process: NVLink leg on the copy engines
    const int es = bf16 ? 2 : 4;
    const bool par = !ag_copy_streams.empty();
    const int me = cfg.my_rank % geom.z3;
    if (par) {  // fork after everything already on s (slot reuse waits included)
      HZP_CUDA(cudaEventRecord(ag_par_ev[0], s));
      for (auto st : ag_copy_streams) HZP_CUDA(cudaStreamWaitEvent(st, ag_par_ev[0], 0));
    }
    for (const CopyRun& r : ag_runs[layer])
      HZP_CUDA(cudaMemcpyAsync(static_cast<char*>(table.ag_slots[r.local]) + (slot * slot_elems + r.dst_off) * es,
                               static_cast<const char*>(table.param[r.src]) + r.src_off * es, r.len * es,
                               cudaMemcpyDeviceToDevice,
                               par && r.src % geom.z3 != me
                                   ? ag_copy_streams[(r.src % geom.z3 - me - 1 + 2 * geom.z3) % geom.z3]
                                   : s));
    if (par)  // join: the AG task ends when every owner's copies have landed
      for (size_t i = 0; i < ag_copy_streams.size(); ++i) {
        HZP_CUDA(cudaEventRecord(ag_par_ev[1 + i], ag_copy_streams[i]));
        HZP_CUDA(cudaStreamWaitEvent(s, ag_par_ev[1 + i], 0));
      }
    ++launches;
    return;
  }
  launch_ag_pull(dtable, dtiles + ag_off[layer], ag_off[layer + 1] - ag_off[layer], slot,
                 slot_elems, bf16, comm_ctas, s);
  ++launches;
}

void Engine::setup_z1_staging() {
  if (emulate || !z1_ce || geom.replicas() <= 1) return;
  const int t_end = z1_off + z1_n;
  // chunk boundaries: whole tiles, <= kZ1ChunkElems elements
  std::vector<std::pair<int, int>> ranges;
  for (int t = z1_off; t < t_end;) {
    int64_t n = 0;
    int u = t;
    while (u < t_end && (u == t || n + tiles_host[u].len <= kZ1ChunkElems)) n += tiles_host[u++].len;
    ranges.push_back({t, u});
    t = u;
  }
  z1_stage.assign(cfg.par.dp, nullptr);
  for (int r = 0; r < cfg.par.dp; ++r)
    if (local_index(r) < 0) {
      // a rank is a remote replica source if some chunk tile reads from it
      bool used = false;
      for (int t = z1_off; t < t_end && !used; ++t)
        for (int b = 1; b < geom.replicas() && !used; ++b) used = tiles_host[t].src + b * geom.z2 == r;
      for (int t = z1_off; t < t_end && !used; ++t) used = tiles_host[t].src == r;
      if (used) HZP_CUDA(cudaMalloc(&z1_stage[r], size_t(2 * kZ1ChunkElems) * 4));
    }
  for (size_t c = 0; c < ranges.size(); ++c) {
    Z1Chunk ch;
    ch.t0 = ranges[c].first;
    ch.t1 = ranges[c].second;
    RankTable t = table;
    for (int r = 0; r < cfg.par.dp; ++r) {
      if (!z1_stage[r]) continue;
      // rank r's grad offsets read by this chunk form one contiguous range
      int64_t lo = INT64_MAX, hi = -1;
      for (int u = ch.t0; u < ch.t1; ++u) {
        const CommTile& x = tiles_host[u];
        bool reads = false;
        for (int b = 0; b < geom.replicas(); ++b) reads = reads || x.src + b * geom.z2 == r;
        if (!reads) continue;
        lo = std::min<int64_t>(lo, x.b_off);
        hi = std::max<int64_t>(hi, x.b_off + x.len);
      }
      if (hi < 0) continue;
      float* buf = static_cast<float*>(z1_stage[r]) + (c & 1) * kZ1ChunkElems;
      t.grad[r] = buf - lo;  // the kernel indexes grad[r] + b_off
      ch.copies.push_back({0, r, 0, lo, hi - lo});
    }
    HZP_CUDA(cudaMalloc(&ch.table, sizeof(RankTable)));
    HZP_CUDA(cudaMemcpy(ch.table, &t, sizeof(RankTable), cudaMemcpyHostToDevice));
    z1_chunks.push_back(ch);
  }
  int lo = 0, hi = 0;
  HZP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  HZP_CUDA(cudaStreamCreateWithPriority(&z1_copy_stream, cudaStreamNonBlocking, hi));
  if (rs_ev.empty()) {
    rs_ev.resize(64);
    for (auto& e : rs_ev) HZP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
}

void Engine::setup_rs_staging() {
  setup_z1_staging();
  if (emulate || direct_grad || geom.z2 <= 1 || !rs_ce) return;
  const int es = bf16 ? 2 : 4;
  const int base = geom.z2_base(cfg.my_rank);
  rs_stage.assign(cfg.par.dp, nullptr);
  for (int q = 0; q < geom.z2; ++q)
    if (base + q != cfg.my_rank) HZP_CUDA(cudaMalloc(&rs_stage[base + q], size_t(slot_elems) * es));
  int lo = 0, hi = 0;
  HZP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  HZP_CUDA(cudaStreamCreateWithPriority(&rs_red_stream, cudaStreamNonBlocking, hi));
  if (rs_ev.empty()) {
    rs_ev.resize(64);
    for (auto& e : rs_ev) HZP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (rs_par) {
    rs_copy_streams.resize(geom.z2 - 1);
    for (auto& st : rs_copy_streams) HZP_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
    rs_par_ev.resize(size_t(geom.z2) * 64);
    for (auto& e : rs_par_ev) HZP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  for (int w = 0; w < int(wslots); ++w) {
    RankTable t = table;
    for (int r = 0; r < cfg.par.dp; ++r)
      if (rs_stage[r]) t.wgrad[r] = static_cast<char*>(rs_stage[r]) - int64_t(w) * slot_elems * es;
    RankTable* d = nullptr;
    HZP_CUDA(cudaMalloc(&d, sizeof(RankTable)));
    HZP_CUDA(cudaMemcpy(d, &t, sizeof(RankTable), cudaMemcpyHostToDevice));
    dtable_staged.push_back(d);
  }
}

void Engine::rs_layer(int layer, int wslot, bool assign, cudaStream_t s) {
  if (!dtable_staged.empty()) {
    const int es = bf16 ? 2 : 4;
    const int t0 = rs_off[layer], t1 = rs_off[layer + 1];
    const int base = geom.z2_base(cfg.my_rank);
    int ev = 0;
    if (rs_par) {  // fork: every copy stream starts after the producer's work on s
      cudaEvent_t f = rs_par_ev[0];
      HZP_CUDA(cudaEventRecord(f, s));
      for (auto st : rs_copy_streams) HZP_CUDA(cudaStreamWaitEvent(st, f, 0));
    }
    // at most rs_chunks chunks per layer and a floor per peer copy: enough to
    // overlap the copies with the reduce, few enough that per-copy overhead
    // stays small.  Floor 8 MB with one peer, 64 MB with several concurrent
    // peer streams (bf16 sweeps: N=2 256 MB layer 399 vs 319 GB/s with the
    // 8 MB floor; N=4 64 MB layer 377 as one chunk vs 327 as two, 1 GB best
    // with 4; profiles/r01_rs_sweep_n4.jsonl, r01_rs_chunk_n2.jsonl)
    const int64_t floor_bytes =
        rs_min_chunk_bytes > 0 ? rs_min_chunk_bytes : (int64_t(rs_par && geom.z2 > 2 ? 64 : 8) << 20);
    const int64_t seg_bytes = t1 <= t0 ? 0 : (tiles_host[t1 - 1].b_off + tiles_host[t1 - 1].len - tiles_host[t0].b_off) * es;
    const int nch = int(std::max<int64_t>(1, std::min<int64_t>(rs_chunks, seg_bytes / floor_bytes)));
    const int chunk = std::max(kRsChunkTiles, (t1 - t0 + nch - 1) / nch);
    for (int c0 = t0; c0 < t1; c0 += chunk, ++ev) {
      const int c1 = std::min(t1, c0 + chunk);
      const int64_t b0 = tiles_host[c0].b_off;
      const int64_t b1 = tiles_host[c1 - 1].b_off + tiles_host[c1 - 1].len;
      for (int j = 1; j < geom.z2; ++j) {  // rotated: peer r+1 first (one reader per owner)
        const int g = base + (cfg.my_rank - base + j) % geom.z2;
        if (!rs_stage[g]) continue;  // this rank's own buffer is read in place
        cudaStream_t cs = rs_par ? rs_copy_streams[j - 1] : s;
        HZP_CUDA(cudaMemcpyAsync(static_cast<char*>(rs_stage[g]) + b0 * es,
                                 static_cast<const char*>(table.wgrad[g]) + (wslot * slot_elems + b0) * es,
                                 (b1 - b0) * es, cudaMemcpyDeviceToDevice, cs));
        if (rs_par) {
          cudaEvent_t pe = rs_par_ev[size_t(geom.z2) * (1 + ev % 63) + j];
          HZP_CUDA(cudaEventRecord(pe, cs));
          HZP_CUDA(cudaStreamWaitEvent(rs_red_stream, pe, 0));
        }
      }
      cudaEvent_t e = rs_ev[ev % rs_ev.size()];
      HZP_CUDA(cudaEventRecord(e, s));
      HZP_CUDA(cudaStreamWaitEvent(rs_red_stream, e, 0));
      launch_rs_pull(dtable_staged[wslot], dtiles + c0, c1 - c0, wslot, slot_elems, geom.z2, bf16, assign,
                     static_cast<float>(cfg.grad_scale), comm_ctas, rs_red_stream, 4);
    }
    cudaEvent_t e = rs_ev[ev % rs_ev.size()];
    HZP_CUDA(cudaEventRecord(e, rs_red_stream));
    HZP_CUDA(cudaStreamWaitEvent(s, e, 0));  // the RS task ends when its last reduce does
    ++launches;
    return;
  }
  launch_rs_pull(dtable, dtiles + rs_off[layer], rs_off[layer + 1] - rs_off[layer], wslot,
                 slot_elems, geom.z2, bf16, assign, static_cast<float>(cfg.grad_scale), comm_ctas, s);
  ++launches;
}

void Engine::z1_adam(cudaStream_t s) {
  // Bias corrections exactly as the reference (train.cpp:179-180 with T=float):
  // (T)1 - (T)std::pow((T)beta, step), std::pow(float, int) promoting to double.
  LocalRank& l0 = locals.front();
  for (auto& l : locals) l.adam_step += 1;
  const int step = l0.adam_step;
  AdamArgs a;
  a.lr = static_cast<float>(cfg.lr);
  a.b1 = static_cast<float>(cfg.beta1);
  a.b2 = static_cast<float>(cfg.beta2);
  a.eps = static_cast<float>(cfg.eps);
  volatile float one = 1.0f;
  a.omb1 = one - a.b1;
  a.omb2 = one - a.b2;
  a.bc1 = one - static_cast<float>(std::pow(static_cast<double>(a.b1), step));
  a.bc2 = one - static_cast<float>(std::pow(static_cast<double>(a.b2), step));
  if (!z1_chunks.empty()) {
    // chunk c's copy (copy engines, z1_copy_stream) overlaps chunk c-1's
    // kernel (s); buffer c & 1 is reused by chunk c+2 only after chunk c's
    // kernel retired
    std::vector<cudaEvent_t> done_k(z1_chunks.size());
    cudaEvent_t e0 = rs_ev[0];
    HZP_CUDA(cudaEventRecord(e0, s));  // grads complete (the caller's barrier)
    HZP_CUDA(cudaStreamWaitEvent(z1_copy_stream, e0, 0));
    for (size_t c = 0; c < z1_chunks.size(); ++c) {
      const Z1Chunk& ch = z1_chunks[c];
      if (c >= 2) HZP_CUDA(cudaStreamWaitEvent(z1_copy_stream, done_k[c - 2], 0));
      for (const CopyRun& r : ch.copies)
        HZP_CUDA(cudaMemcpyAsync(static_cast<float*>(z1_stage[r.src]) + (c & 1) * kZ1ChunkElems,
                                 table.grad[r.src] + r.src_off, size_t(r.len) * 4, cudaMemcpyDeviceToDevice,
                                 z1_copy_stream));
      cudaEvent_t ec = rs_ev[1 + (2 * c) % (rs_ev.size() - 1)];
      HZP_CUDA(cudaEventRecord(ec, z1_copy_stream));
      HZP_CUDA(cudaStreamWaitEvent(s, ec, 0));
      launch_z1_adam(ch.table, dtiles + ch.t0, ch.t1 - ch.t0, geom.z2, geom.replicas(), &a, 1, bf16,
                     l0.dbg != nullptr, 8 * kNumSMs, s);
      done_k[c] = rs_ev[1 + (2 * c + 1) % (rs_ev.size() - 1)];
      HZP_CUDA(cudaEventRecord(done_k[c], s));
    }
    ++launches;
    return;
  }
  launch_z1_adam(dtable, dtiles + z1_off, z1_n, geom.z2, geom.replicas(), &a, 1, bf16,
                 l0.dbg != nullptr, 8 * kNumSMs, s);  // HBM-bound, never beside a GEMM
  ++launches;
}

void Engine::barrier(cudaStream_t s) {
  if (emulate || cfg.par.dp == 1) return;
  ++barrier_epoch;
  launch_signal(dtable, cfg.my_rank, kFlagBarrier, 0, cfg.par.dp, 1, barrier_epoch, kFlagBarrier,
                barrier_epoch, s);
  ++launches;
}

const void* Engine::layer_params(int li, int layer, int slot) const {
  const int es = bf16 ? 2 : 4;
  if (zero_copy_ag)  // z3 == 1: this rank's shard is the whole working copy
    return static_cast<const char*>(arenas[locals[li].rank].param) + layers[layer].off * es;
  return static_cast<const char*>(locals[li].ag) + (int64_t(slot) * slot_elems) * es;
}

GradTarget Engine::grad_target(int li, int layer, int wslot, int mb) const {
  GradTarget t;
  const int r = locals[li].rank;
  if (direct_grad) {  // z2 == 1: the grad shard is the whole flat gradient
    t.ptr = arenas[r].grad + layers[layer].off;
    t.bf16 = 0;
    t.mode = mb == 0 ? kEpiAssign0 : kEpiAccum;
  } else {
    const int es = bf16 ? 2 : 4;
    t.ptr = static_cast<char*>(arenas[r].wgrad) + int64_t(wslot) * slot_elems * es;
    t.bf16 = bf16;
    t.mode = kEpiStore;
  }
  return t;
}

void Engine::step(const void* inputs, bool on_device, float* losses_out) {
  if (!peers_open) throw std::runtime_error("peers not opened (hzp_ctx_open_peers)");
  HZP_CUDA(cudaSetDevice(cfg.device));
  log.clear();
  launches = 0;
  const int nmb = std::max(1, cfg.num_microbatches);
  const size_t in_total = input_bytes_per_mb * locals.size() * nmb;
  cudaStream_t cs = st[0];
  // Step start: the previous step's tail (fused Z1 kernel + barrier) must be
  // complete before any stream touches grads or param shards again.
  HZP_CUDA(cudaEventRecord(ev_step0, cs));
  HZP_CUDA(cudaStreamWaitEvent(st[1], ev_step0, 0));
  HZP_CUDA(cudaStreamWaitEvent(st[2], ev_step0, 0));
  const char* in_dev = static_cast<const char*>(inputs);
  if (!on_device) {
    HZP_CUDA(cudaMemcpyAsync(dinputs, inputs, in_total, cudaMemcpyHostToDevice, cs));
    in_dev = static_cast<const char*>(dinputs);
  }
  for (auto& l : locals) model->begin_step(l.mbuf, cs);

  const int n = static_cast<int>(plan.entries.size());
  std::vector<int> rs_index(n, -1);  // RS sequence index within this step
  {
    int k = 0;
    for (const auto& e : plan.entries)
      if (e.kind == TaskKind::RsGrad) rs_index[e.id] = k++;
  }
  // BWD(l, mb) produces the gradient consumed by RS task rs_of_bwd.
  std::vector<int> rs_of_bwd(n, -1);
  for (const auto& t : graph.tasks)
    if (t.kind == TaskKind::RsGrad)
      for (int d : t.deps)
        if (graph.tasks[d].kind == TaskKind::Bwd && graph.tasks[d].layer == t.layer) rs_of_bwd[d] = t.id;
  std::vector<int> rs_ids;
  for (const auto& e : plan.entries)
    if (e.kind == TaskKind::RsGrad) rs_ids.push_back(e.id);
  const uint64_t seq0 = rs_seq;
  int last_comm_ev[3] = {-1, -1, -1};

  auto rec_log = [&](const PlanEntry& e, int stream, int cov0, int cov1) {
    hzp_launch_rec r{};
    r.task_id = e.id;
    r.kind = static_cast<int>(e.kind);
    r.layer = e.layer;
    r.microbatch = e.microbatch;
    r.stream = stream;
    r.slot = e.slot;
    r.covered_first = cov0;
    r.covered_last = cov1;
    log.push_back(r);
  };
  int opt_id = -1;
  for (const auto& e : plan.entries)
    if (e.kind == TaskKind::OptStep) opt_id = e.id;

  for (const auto& e : plan.entries) {
    cudaStream_t s = st[static_cast<int>(e.stream)];
    for (int w : e.waits)
      if (plan.entries[w].stream != e.stream) HZP_CUDA(cudaStreamWaitEvent(s, done[w], 0));
    if (cfg.mode == HZP_MODE_VANILLA && e.stream == StreamId::Compute) {
      // vanilla: compute may not run past any issued collective (sched.cpp:280-284)
      for (int k = 1; k < 3; ++k)
        if (last_comm_ev[k] >= 0) HZP_CUDA(cudaStreamWaitEvent(s, done[last_comm_ev[k]], 0));
    }
    if (cfg.timeline) HZP_CUDA(cudaEventRecord(tev0[e.id], s));
    switch (e.kind) {
      case TaskKind::AgParam:
        if (zero_copy_ag) {
          rec_log(e, -1, e.id, e.id);  // identity: layers read the shard in place
        } else {
          if (ag_phys_wait[e.id] >= 0) HZP_CUDA(cudaStreamWaitEvent(s, done[ag_phys_wait[e.id]], 0));
          ag_layer(e.layer, ag_slot[e.id], s);
          rec_log(e, int(e.stream), e.id, e.id);
        }
        break;
      case TaskKind::Fwd: {
        const int slot = param_slot[e.id];
        for (size_t li = 0; li < locals.size(); ++li) {
          const char* in = in_dev + (li * nmb + e.microbatch) * input_bytes_per_mb;
          model->fwd(locals[li].mbuf, e.layer, in, layer_params(int(li), e.layer, slot), s);
        }
        launches += int64_t(locals.size()) * model->launches_per_fwd();
        rec_log(e, 0, e.id, e.id);
        break;
      }
      case TaskKind::FwdRecompute: {
        const int slot = param_slot[e.id];
        for (size_t li = 0; li < locals.size(); ++li)
          model->recompute(locals[li].mbuf, e.layer, layer_params(int(li), e.layer, slot), s);
        launches += int64_t(locals.size()) * model->launches_per_recompute(e.layer);
        rec_log(e, 0, e.id, e.id);
        break;
      }
      case TaskKind::Bwd: {
        const int slot = param_slot[e.id];
        const int rs = rs_of_bwd[e.id];
        const int k = rs >= 0 ? rs_index[rs] : 0;
        const int wslot = static_cast<int>((seq0 + k) % wslots);
        if (!direct_grad) {
          // the gradient buffer is free once RS k - wslots finished everywhere
          if (k >= wslots) HZP_CUDA(cudaStreamWaitEvent(s, done[rs_ids[k - wslots]], 0));
          if (!emulate && geom.z2 > 1 && seq0 + k >= uint64_t(wslots)) {
            launch_wait(dtable, cfg.my_rank, kFlagRsDone, geom.z2_base(cfg.my_rank), geom.z2, 1,
                        seq0 + k + 1 - wslots, s);
            ++launches;
          }
        }
        for (size_t li = 0; li < locals.size(); ++li)
          model->bwd(locals[li].mbuf, e.layer, layer_params(int(li), e.layer, slot),
                     grad_target(int(li), e.layer, wslot, e.microbatch), s);
        launches += int64_t(locals.size()) * 3;
        rec_log(e, 0, e.id, e.id);
        break;
      }
      case TaskKind::RsGrad: {
        const int k = rs_index[e.id];
        const uint64_t seq = seq0 + k + 1;  // 1-based sequence number of this RS
        if (direct_grad) {
          rec_log(e, -1, e.id - 1, e.id);  // fused into the BWD's wgrad epilogue
        } else {
          if (!emulate && geom.z2 > 1) {  // publish + wait for every Z2 peer's gradient
            launch_signal(dtable, cfg.my_rank, kFlagRsReady, geom.z2_base(cfg.my_rank), geom.z2, 1,
                          seq, kFlagRsReady, seq, s);
            ++launches;
          }
          rs_layer(e.layer, static_cast<int>((seq - 1) % wslots), e.microbatch == 0, s);
          if (!emulate && geom.z2 > 1) {
            launch_signal(dtable, cfg.my_rank, kFlagRsDone, geom.z2_base(cfg.my_rank), geom.z2, 1,
                          seq, -1, 0, s);
            ++launches;
          }
          rec_log(e, int(e.stream), e.id, e.id);
        }
        break;
      }
      case TaskKind::ArDzp:
        rec_log(e, -1, opt_id, opt_id);  // folded into the fused Z1 kernel
        break;
      case TaskKind::OptStep: {
        barrier(s);  // every rank's RS complete; nobody reads param shards any more
        z1_adam(s);
        barrier(s);  // every push landed, every grad pull done
        int first = e.id, last = e.id;
        for (const auto& x : plan.entries)
          if (x.kind == TaskKind::ArDzp || x.kind == TaskKind::AgPostStep) {
            first = std::min(first, x.id);
            last = std::max(last, x.id);
          }
        rec_log(e, 0, first, last);
        break;
      }
      case TaskKind::AgPostStep:
        rec_log(e, -1, opt_id, opt_id);  // done by the fused kernel's P2P stores
        break;
      default:
        break;
    }
    if (cfg.timeline) HZP_CUDA(cudaEventRecord(tev1[e.id], s));
    HZP_CUDA(cudaEventRecord(done[e.id], s));
    if (e.stream != StreamId::Compute) last_comm_ev[static_cast<int>(e.stream)] = e.id;
    if (debug_sync) {  // HZP_DEBUG_SYNC=1: serialise every task across all ranks
      HZP_CUDA(cudaDeviceSynchronize());
      barrier(cs);
      HZP_CUDA(cudaDeviceSynchronize());
    }
  }
  rs_seq = seq0 + rs_ids.size();
  // join the comm streams back into the compute stream
  for (int k = 1; k < 3; ++k)
    if (last_comm_ev[k] >= 0) HZP_CUDA(cudaStreamWaitEvent(cs, done[last_comm_ev[k]], 0));
  for (size_t li = 0; li < locals.size(); ++li)
    HZP_CUDA(cudaMemcpyAsync(hloss + li, model->loss_device(locals[li].mbuf), sizeof(float),
                             cudaMemcpyDeviceToHost, cs));
  HZP_CUDA(cudaEventRecord(ev_step1, cs));
  if (losses_out) {
    HZP_CUDA(cudaEventSynchronize(ev_step1));
    std::memcpy(losses_out, hloss, sizeof(float) * locals.size());
  }
}

}  // namespace hzp
