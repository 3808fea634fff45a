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

#include <unistd.h>

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
    mcfg.swiglu = c.gpt_swiglu;
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
  // Priorities (numerically lower = scheduled first when an SM frees up):
  // compute highest, so a pending persistent GEMM takes every SM it needs
  // before any queued collective / optimizer CTA (those then fill the space
  // beside the resident GEMM CTAs, one per SM); collectives next; the
  // per-layer optimizer lowest: its grids are thousands of CTAs, and at the
  // collectives' priority a rank's later RS kernels queued behind them, so
  // its GradReady reached the other ranks late (MoE N = 4: 238 K -> 265 K
  // tokens/s at the lowest priority, 7B N = 4: 94.7 K -> 96.1 K;
  // profiles/r02_optprio_*.jsonl).
  const int mid = hi < lo ? std::min(lo, hi + 1) : hi;
  HZP_CUDA(cudaStreamCreateWithPriority(&st[0], cudaStreamNonBlocking, hi));
  HZP_CUDA(cudaStreamCreateWithPriority(&st[1], cudaStreamNonBlocking, mid));
  HZP_CUDA(cudaStreamCreateWithPriority(&st[2], cudaStreamNonBlocking, mid));
  HZP_CUDA(cudaStreamCreateWithPriority(&opt_stream, cudaStreamNonBlocking, lo));
  const int n = static_cast<int>(plan.entries.size());
  done.resize(n);
  for (auto& e : done) HZP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (c.timeline) timeline_events(true);
  HZP_CUDA(cudaEventCreate(&ev_step0));
  HZP_CUDA(cudaEventCreate(&ev_step1));
  HZP_CUDA(cudaEventCreateWithFlags(&ev_opt, cudaEventDisableTiming));
  HZP_CUDA(cudaEventCreateWithFlags(&ev_z1, cudaEventDisableTiming));

  // ---- per-rank peer-visible arenas ----
  const int es = bf16 ? 2 : 4;
  const bool shared = !emulate && c.par.dp > 1;  // one process per GPU: cuMem + NVLS
  const size_t al = shared ? symm_granularity(c.device) : 256;
  lay.param = 0;
  lay.grad = align_up(size_t(geom.s3) * es, 256);
  lay.flags = lay.grad + align_up(size_t(geom.s2) * 4, 256);
  lay.ag = align_up(lay.flags + sizeof(uint64_t) * kNumFlagKinds * kMaxRanks, al);
  lay.ag_bytes = zero_copy_ag ? 0 : align_up(size_t(depth + cache_slots) * slot_elems * es, al);
  lay.wgrad = lay.ag + lay.ag_bytes;
  lay.wgrad_bytes = direct_grad ? 0 : align_up(size_t(wslots) * slot_elems * es, al);
  lay.total = align_up(lay.wgrad + lay.wgrad_bytes, al);
  arenas.resize(c.par.dp);
  std::vector<int> mine;
  if (emulate) {
    mine.resize(c.par.dp);
    std::iota(mine.begin(), mine.end(), 0);
  } else {
    if (c.my_rank >= c.par.dp) throw std::invalid_argument("my_rank out of range");
    mine.push_back(c.my_rank);
  }
  if (shared && (ag_multicast() || rs_multicast()) && !multicast_supported(c.device))
    throw CudaError("groups of >= 3 GPUs need NVLS multicast (NVSwitch); this device has none");
  for (int r : mine) {
    Arena& a = arenas[r];
    if (shared) {
      a.symm = symm_alloc(c.device, lay.total);
      a.base = reinterpret_cast<void*>(a.symm.va);
    } else {
      HZP_CUDA(cudaMalloc(&a.base, lay.total));
      a.cuda_malloc = true;
    }
    a.bytes = lay.total;
    HZP_CUDA(cudaMemset(a.base, 0, a.bytes));
    carve(a);
  }
  if (shared) {  // the group's first rank creates the multicast objects
    if (ag_multicast() && c.my_rank % geom.z3 == 0) ag_mc = mc_create(geom.z3, lay.ag_bytes);
    if (rs_multicast() && c.my_rank % geom.z2 == 0) wg_mc = mc_create(geom.z2, lay.wgrad_bytes);
  }

  // ---- driven ranks ----
  for (int r : mine) {
    LocalRank lr;
    lr.rank = r;
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
    table.ag[r] = arenas[r].ag;
    table.flags[r] = arenas[r].flags;
  }
  for (size_t i = 0; i < locals.size(); ++i) {
    table.master[i] = locals[i].master;
    table.mom[i] = locals[i].mom;
    table.var[i] = locals[i].var;
    table.z1_grad_dbg[i] = locals[i].dbg;
    table.global_rank[i] = locals[i].rank;
  }
  HZP_CUDA(cudaMalloc(&dtable, sizeof(RankTable)));
  HZP_CUDA(cudaMemcpy(dtable, &table, sizeof(RankTable), cudaMemcpyHostToDevice));
  peers_open = !shared;
  debug_sync = std::getenv("HZP_DEBUG_SYNC") != nullptr;  // debugging aid: serialise every task
  build_tiles();
}

void Engine::carve(Arena& a) const {
  char* b = static_cast<char*>(a.base);
  a.param = b + lay.param;
  a.grad = reinterpret_cast<float*>(b + lay.grad);
  a.flags = reinterpret_cast<uint64_t*>(b + lay.flags);
  a.ag = lay.ag_bytes ? b + lay.ag : nullptr;
  a.wgrad = lay.wgrad_bytes ? b + lay.wgrad : nullptr;
}

ShareRecord Engine::share_record() const {
  if (emulate || cfg.par.dp == 1) throw std::invalid_argument("only a multi-process ctx shares its arena");
  ShareRecord r;
  r.magic = kShareMagic;
  r.rank = cfg.my_rank;
  r.pid = static_cast<int32_t>(getpid());
  r.arena_fd = arenas[cfg.my_rank].symm.fd;
  r.arena_bytes = static_cast<int64_t>(lay.total);
  r.ag_mc_fd = ag_mc.fd;
  r.wg_mc_fd = wg_mc.fd;
  r.ag_mc_bytes = static_cast<int64_t>(lay.ag_bytes);
  r.wg_mc_bytes = static_cast<int64_t>(lay.wgrad_bytes);
  return r;
}

void Engine::open_peers(const ShareRecord* rec, int n) {
  if (emulate || cfg.par.dp == 1) return;
  if (peers_open) throw std::invalid_argument("peers already opened");
  if (n != cfg.par.dp) throw std::invalid_argument("need one share record per dp rank");
  for (int r = 0; r < n; ++r)
    if (rec[r].magic != kShareMagic || rec[r].rank != r || rec[r].arena_bytes != int64_t(lay.total))
      throw std::invalid_argument("share record " + std::to_string(r) + " does not match this layout");
  HZP_CUDA(cudaSetDevice(cfg.device));
  const int me = cfg.my_rank;
  for (int r = 0; r < n; ++r) {
    if (r == me) continue;
    Arena& a = arenas[r];
    a.symm = symm_import(cfg.device, rec[r].pid, rec[r].arena_fd, lay.total);
    a.base = reinterpret_cast<void*>(a.symm.va);
    a.bytes = lay.total;
    carve(a);
    table.param[r] = a.param;
    table.grad[r] = a.grad;
    table.wgrad[r] = a.wgrad;
    table.ag[r] = a.ag;
    table.flags[r] = a.flags;
  }
  // bind this rank's AG / gradient regions into its groups' multicast
  // objects (mc_attach blocks until every member has added its device)
  const Arena& mine = arenas[me];
  if (ag_multicast()) {
    const ShareRecord& lead = rec[geom.z3_base(me)];
    if (me != lead.rank) ag_mc = mc_import(lead.pid, lead.ag_mc_fd, lay.ag_bytes);
    mc_attach(ag_mc, cfg.device, mine.symm, lay.ag);
    table.ag_mc = reinterpret_cast<void*>(ag_mc.va);
  }
  if (rs_multicast()) {
    const ShareRecord& lead = rec[geom.z2_base(me)];
    if (me != lead.rank) wg_mc = mc_import(lead.pid, lead.wg_mc_fd, lay.wgrad_bytes);
    mc_attach(wg_mc, cfg.device, mine.symm, lay.wgrad);
    table.wgrad_mc = reinterpret_cast<void*>(wg_mc.va);
  }
  HZP_CUDA(cudaMemcpy(dtable, &table, sizeof(RankTable), cudaMemcpyHostToDevice));
  HZP_CUDA(cudaDeviceSynchronize());
  peers_open = true;
}

void Engine::timeline_events(bool on) {
  const size_t n = plan.entries.size(), nl = layers.size();
  if (!on || tev0.size() == n) return;
  tev0.resize(n);
  tev1.resize(n);
  for (size_t i = 0; i < n; ++i) {
    HZP_CUDA(cudaEventCreate(&tev0[i]));
    HZP_CUDA(cudaEventCreate(&tev1[i]));
  }
  for (auto* v : {&zev_ready, &zev_start, &zev_end}) {
    v->resize(nl);
    for (auto& e : *v) HZP_CUDA(cudaEventCreate(&e));
  }
}

Engine::~Engine() {
  cudaDeviceSynchronize();
  for (auto& l : locals) {
    cudaFree(l.master);
    cudaFree(l.mom);
    cudaFree(l.var);
    cudaFree(l.dbg);
    model->free_rank_buffers(l.mbuf);
  }
  mc_release(ag_mc);
  mc_release(wg_mc);
  for (auto& a : arenas) {
    if (a.cuda_malloc) cudaFree(a.base);
    else if (a.symm.va) symm_release(a.symm);
  }
  cudaFree(dtable);
  cudaFree(dtiles);
  cudaFree(dinputs);
  cudaFreeHost(hloss);
  for (auto e : done) cudaEventDestroy(e);
  for (auto e : tev0) cudaEventDestroy(e);
  for (auto e : tev1) cudaEventDestroy(e);
  for (auto* v : {&zev_ready, &zev_start, &zev_end})
    for (auto e : *v) cudaEventDestroy(e);
  cudaEventDestroy(ev_step0);
  cudaEventDestroy(ev_step1);
  cudaEventDestroy(ev_opt);
  cudaEventDestroy(ev_z1);
  for (auto s : st) cudaStreamDestroy(s);
  if (opt_stream) cudaStreamDestroy(opt_stream);
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
  ag_pull = T.ag_pull;
  rs_off = T.rs_off;
  z1_off = T.z1_off;
  z1_n = T.z1_n;
  z1_layer_off = T.z1_layer_off;
  z1_wait_mask.assign(layers.size(), 0);
  if (!emulate)
    for (size_t l = 0; l < layers.size(); ++l)
      for (int i = z1_layer_off[l]; i < z1_layer_off[l + 1]; ++i) {
        const CommTile& t = T.tiles[i];
        for (int b = 0; b < geom.replicas(); ++b) z1_wait_mask[l] |= 1ull << (t.src + b * geom.z2);
        z1_wait_mask[l] |= t.mask;
        // the owners we push parameters into are read by their whole Z3
        // group (AG pull): those readers must be past this layer too
        for (uint64_t m = t.mask; m; m &= m - 1) {
          const int q = __builtin_ctzll(m);
          z1_wait_mask[l] |= rank_mask(geom.z3_base(q), geom.z3);
        }
      }
  // members of this rank's Z3 group whose shard holds part of each layer
  ag_owners.assign(layers.size(), 0);
  if (!emulate)
    for (size_t l = 0; l < layers.size(); ++l) {
      const int base = geom.z3_base(cfg.my_rank);
      const int j0 = static_cast<int>(layers[l].off / geom.s3);
      const int j1 = static_cast<int>((layers[l].off + layers[l].size - 1) / geom.s3);
      for (int j = j0; j <= j1 && j < geom.z3; ++j) ag_owners[l] |= 1ull << (base + j);
    }
  if (dtiles) cudaFree(dtiles);
  HZP_CUDA(cudaMalloc(&dtiles, std::max<size_t>(1, T.tiles.size()) * sizeof(CommTile)));
  if (!T.tiles.empty())
    HZP_CUDA(cudaMemcpy(dtiles, T.tiles.data(), T.tiles.size() * sizeof(CommTile), cudaMemcpyHostToDevice));
}

// AG task: every member posts "slot free" (its ring wait is already on the
// stream), the owner(s) of the layer multicast their spans once every member
// is ready and post "landed"; every member waits for all the layer's owners.
void Engine::ag_layer(int layer, int slot, cudaStream_t s, bool ready_posted) {
  if (zero_copy_ag) throw std::invalid_argument("z3 == 1: the all-gather is the identity (layers read the shard)");
  const int t0 = ag_off[layer], nt = ag_off[layer + 1] - t0;
  if (emulate || ag_pull) {
    // pull (groups of 2): each reader copies the layer's owner spans into its
    // own slot; its ring wait is already on this stream and the owners'
    // shards do not change during the step, so no cross-GPU rendezvous
    launch_ag_push(dtable, dtiles + t0, nt, slot, slot_elems, geom.z3, bf16, ag_pull ? kAgPull : kAgUnicastPush,
                   FlagGate{}, kCommCtas, s);
    ++launches;
    return;
  }
  // the waits run in single-CTA flag kernels, so the data kernel's CTAs
  // (one per SM, beside the GEMM) never spin
  const int me = cfg.my_rank;
  const uint64_t seq = ++ag_seq;
  const uint64_t grp = rank_mask(geom.z3_base(me), geom.z3);
  launch_flags(dtable, me, kFlagAgReady, ready_posted ? 0 : grp, seq, kFlagAgReady, nt > 0 ? grp : 0, seq, s);
  if (nt > 0)
    launch_ag_push(dtable, dtiles + t0, nt, slot, slot_elems, geom.z3, bf16, kAgMulticast, FlagGate{}, kCommCtas,
                   s);
  launch_flags(dtable, me, kFlagAgDone, nt > 0 ? grp : 0, seq, kFlagAgDone, ag_owners[layer], seq, s);
  launches += nt > 0 ? 3 : 2;
}

// RS task (sequence number seq): every member posts "gradient slot written";
// the owner of (layer ∩ its Z2 segment) waits for all members, reduces; every
// member posts "done" (BWD reuses a slot once every member posted done for
// the RS that read it).
void Engine::rs_layer(int layer, int wslot, bool assign, uint64_t seq, cudaStream_t s) {
  if (direct_grad) throw std::invalid_argument("z2 == 1: the reduce-scatter is fused into the wgrad GEMM");
  const int t0 = rs_off[layer], nt = rs_off[layer + 1] - t0;
  const float scale = static_cast<float>(cfg.grad_scale);
  if (emulate) {
    launch_rs_reduce(dtable, dtiles + t0, nt, wslot, slot_elems, geom.z2, bf16,
                     rs_multicast_group() ? kRsOrderedRound : kRsOrdered, assign, scale, FlagGate{}, kCommCtas, s);
    ++launches;
    return;
  }
  const int me = cfg.my_rank;
  const uint64_t grp = rank_mask(geom.z2_base(me), geom.z2);
  launch_flags(dtable, me, kFlagRsReady, grp, seq, kFlagRsReady, nt > 0 ? grp : 0, seq, s);
  if (nt > 0)
    launch_rs_reduce(dtable, dtiles + t0, nt, wslot, slot_elems, geom.z2, bf16, rs_multicast() ? kRsMulticast : kRsOrdered,
                     assign, scale, FlagGate{}, kCommCtas, s);
  launch_flags(dtable, me, kFlagRsDone, grp, seq, 0, 0, 0, s);
  launches += nt > 0 ? 3 : 2;
}

AdamArgs Engine::next_adam_args() {
  // Bias corrections exactly as the reference (train.cpp:179-180 with T=float):
  // (T)1 - (T)std::pow((T)beta, step), std::pow(float, int) promoting to double.
  for (auto& l : locals) l.adam_step += 1;
  const int step = locals.front().adam_step;
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
  return a;
}

void Engine::z1_adam(cudaStream_t s) {
  const AdamArgs a = next_adam_args();
  launch_z1_adam(dtable, dtiles + z1_off, z1_n, geom.z2, geom.replicas(), &a, 1, bf16,
                 locals.front().dbg != nullptr, kCommCtas, s);  // HBM-bound
  ++launches;
}

void Engine::z1_layer(int layer, const AdamArgs& a, cudaStream_t s, cudaStream_t post) {
  if (!emulate && cfg.par.dp > 1) {
    // announce "layer final here" to every rank from the stream of the task
    // that made it final (not from the optimizer stream, where it would queue
    // behind this rank's earlier layers' Z1 and hold back every rank that
    // waits for it), then wait on the optimizer stream for the ranks this
    // layer's Z1 reads gradients from / pushes parameters into
    const uint64_t seq = ++grad_seq;
    const uint64_t all = rank_mask(0, cfg.par.dp);
    if (post && post != s) {
      launch_flags(dtable, cfg.my_rank, kFlagGradReady, all, seq, 0, 0, 0, post);
      launch_flags(dtable, cfg.my_rank, 0, 0, 0, kFlagGradReady, z1_wait_mask[layer], seq, s);
      launches += 2;
    } else {
      launch_flags(dtable, cfg.my_rank, kFlagGradReady, all, seq, kFlagGradReady, z1_wait_mask[layer], seq, s);
      ++launches;
    }
  }
  if (cfg.timeline && !zev_start.empty()) HZP_CUDA(cudaEventRecord(zev_start[layer], s));
  const int t0 = z1_layer_off[layer], nt = z1_layer_off[layer + 1] - t0;
  launch_z1_adam(dtable, dtiles + t0, nt, geom.z2, geom.replicas(), &a, 1, bf16, locals.front().dbg != nullptr,
                 kCommCtas, s);
  launches += nt > 0;
}

void Engine::barrier(cudaStream_t s) {
  if (emulate || cfg.par.dp == 1) return;
  ++barrier_epoch;
  const uint64_t all = rank_mask(0, cfg.par.dp);
  launch_flags(dtable, cfg.my_rank, kFlagBarrier, all, barrier_epoch, kFlagBarrier, all, barrier_epoch, s);
  ++launches;
}

const void* Engine::layer_params(int li, int layer, int slot) const {
  const int es = bf16 ? 2 : 4;
  if (zero_copy_ag)  // z3 == 1: this rank's shard is the whole working copy
    return static_cast<const char*>(arenas[locals[li].rank].param) + layers[layer].off * es;
  return static_cast<const char*>(arenas[locals[li].rank].ag) + (int64_t(slot) * slot_elems) * es;
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
  HZP_CUDA(cudaStreamWaitEvent(opt_stream, ev_step0, 0));
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
  // async mode: each layer's Z1 (replica reduce + Adam + bf16 push, covering
  // AR-dzp(l) and AG-post-step(l)) is enqueued on the RS stream right after
  // the task that makes the layer's gradient final (its last RS; its last BWD
  // when z2 == 1 fuses the RS into the wgrad GEMM), overlapping the rest of
  // the backward.  Vanilla mode keeps the reference's tail order.
  const bool early_z1 = cfg.mode != HZP_MODE_VANILLA;
  std::vector<int> final_of(n, -1);  // task id -> layer whose gradient it finalises
  if (early_z1) {
    std::vector<int> last(layers.size(), -1);
    for (const auto& t : graph.tasks)
      if ((direct_grad && t.kind == TaskKind::Bwd) || (!direct_grad && t.kind == TaskKind::RsGrad))
        last[t.layer] = std::max(last[t.layer], t.id);
    for (size_t l = 0; l < layers.size(); ++l)
      if (last[l] >= 0) final_of[last[l]] = static_cast<int>(l);
  }
  AdamArgs adam{};
  bool adam_ready = false;
  int z1_issued = 0;
  // multi-process AG: every member posts "slot free" for AG k from its
  // compute stream as soon as the task that releases the slot (the ring wait:
  // first consumer of the slot's previous occupant, or its last reader) ends,
  // so an owner's multicast waits on the members' compute progress only, not
  // on their AG streams.  post_after[t] = AG sequence number to post after
  // compute task t (monotone); AGs with no ring wait are free at step start.
  const bool post_ready_early = !emulate && !zero_copy_ag && !ag_pull && cfg.par.dp > 1;
  std::vector<uint64_t> post_after(n, 0);
  uint64_t post_at_start = 0;
  if (post_ready_early) {
    uint64_t k = ag_seq;
    for (const auto& e : plan.entries) {
      if (e.kind != TaskKind::AgParam) continue;
      const uint64_t q = ++k;
      const int freed = std::max(e.ring_wait, ag_phys_wait[e.id]);
      if (freed < 0) post_at_start = std::max(post_at_start, q);
      else post_after[freed] = std::max(post_after[freed], q);
    }
    uint64_t run = post_at_start;  // keep the posted values monotone in issue order
    for (int t = 0; t < n; ++t)
      if (post_after[t]) post_after[t] = run = std::max(run, post_after[t]);
    if (post_at_start)
      launch_flags(dtable, cfg.my_rank, kFlagAgReady, rank_mask(geom.z3_base(cfg.my_rank), geom.z3), post_at_start,
                   0, 0, 0, cs);
  }

  for (const auto& e : plan.entries) {
    cudaStream_t s = st[static_cast<int>(e.stream)];
    for (int w : e.waits)
      if (plan.entries[w].stream != e.stream) HZP_CUDA(cudaStreamWaitEvent(s, done[w], 0));
    if (cfg.mode == HZP_MODE_VANILLA && e.stream == StreamId::Compute) {
      // vanilla: compute may not run past any issued collective (sched.cpp:280-284)
      for (int k = 1; k < 3; ++k)
        if (last_comm_ev[k] >= 0) HZP_CUDA(cudaStreamWaitEvent(s, done[last_comm_ev[k]], 0));
    }
    if (e.kind == TaskKind::OptStep) {
      // cross-stream / cross-rank waits of the optimizer step happen before
      // its start event: they count as idle (exposed), not as compute
      if (early_z1 && z1_issued) HZP_CUDA(cudaStreamWaitEvent(s, ev_z1, 0));
      barrier(s);  // early: every push landed; tail: every rank's RS complete
    }
    if (cfg.timeline) HZP_CUDA(cudaEventRecord(tev0[e.id], s));
    switch (e.kind) {
      case TaskKind::AgParam:
        if (zero_copy_ag) {
          rec_log(e, -1, e.id, e.id);  // identity: layers read the shard in place
        } else {
          if (ag_phys_wait[e.id] >= 0) HZP_CUDA(cudaStreamWaitEvent(s, done[ag_phys_wait[e.id]], 0));
          ag_layer(e.layer, ag_slot[e.id], s, post_ready_early);
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
            launch_flags(dtable, cfg.my_rank, 0, 0, 0, kFlagRsDone, rank_mask(geom.z2_base(cfg.my_rank), geom.z2),
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
          rs_layer(e.layer, static_cast<int>((seq - 1) % wslots), e.microbatch == 0, seq, s);
          rec_log(e, int(e.stream), e.id, e.id);
        }
        break;
      }
      case TaskKind::ArDzp:
        // folded into the fused Z1 kernel(s): per layer (async) or the tail
        rec_log(e, early_z1 ? 2 : -1, early_z1 ? e.id : opt_id, early_z1 ? e.id : opt_id);
        break;
      case TaskKind::OptStep: {
        if (!early_z1) z1_adam(s);  // the reference's tail order (vanilla)
        int first = e.id, last = e.id;
        for (const auto& x : plan.entries)
          if ((!early_z1 && x.kind == TaskKind::ArDzp) || x.kind == TaskKind::AgPostStep) {
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
    if (post_after[e.id])  // this compute task freed AG ring slots
      launch_flags(dtable, cfg.my_rank, kFlagAgReady, rank_mask(geom.z3_base(cfg.my_rank), geom.z3),
                   post_after[e.id], 0, 0, 0, s);
    if (e.kind == TaskKind::OptStep && !early_z1) barrier(s);  // every push landed, every grad pull done
    if (final_of[e.id] >= 0) {  // this task made a layer's gradient final: its Z1 now
      cudaStream_t zs = opt_stream;  // its own stream: later RSs never queue behind it
      HZP_CUDA(cudaStreamWaitEvent(zs, done[e.id], 0));
      const bool zt = cfg.timeline && !zev_ready.empty();
      if (zt) HZP_CUDA(cudaEventRecord(zev_ready[final_of[e.id]], zs));
      if (!adam_ready) {
        adam = next_adam_args();
        adam_ready = true;
      }
      z1_layer(final_of[e.id], adam, zs, s);
      if (zt) HZP_CUDA(cudaEventRecord(zev_end[final_of[e.id]], zs));
      HZP_CUDA(cudaEventRecord(ev_z1, zs));
      ++z1_issued;
    }
    if (e.stream != StreamId::Compute) last_comm_ev[static_cast<int>(e.stream)] = e.id;
    if (debug_sync) {  // HZP_DEBUG_SYNC=1: serialise every task across all ranks
      HZP_CUDA(cudaDeviceSynchronize());
      barrier(cs);
      HZP_CUDA(cudaDeviceSynchronize());
    }
  }
  rs_seq = seq0 + rs_ids.size();
  z1_timed = cfg.timeline && !zev_ready.empty() && z1_issued == static_cast<int>(layers.size());
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
