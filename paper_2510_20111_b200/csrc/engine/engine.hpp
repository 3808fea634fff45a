// Device engine: one hzp_ctx drives one GPU and either one dp rank (one
// process per GPU; peers' arenas mapped over NVLink/NVSwitch from shared
// cuMem allocations, AG / gradient rings bound to NVLS multicast objects) or
// all dp ranks emulated on that GPU (single-process parity mode: the same
// kernels with unicast stores / ordered loads in place of multimem).
#pragma once

#include <memory>
#include <vector>

#include "hzp/sched.hpp"
#include "hzp_b200.h"
#include "engine/comm.cuh"
#include "engine/model.hpp"
#include "engine/symm.hpp"

namespace hzp {

// One dp rank's peer-visible memory, carved from one allocation:
//   [ param s3 | grad s2 fp32 | flags | AG ring + reuse cache | gradient ring ]
// (multi-process: a cuMem allocation; the AG and gradient regions start at
// multicast-granularity offsets so they can be bound to the group objects).
struct Arena {
  void* base = nullptr;
  size_t bytes = 0;
  SymmBuf symm;        // multi-process: exported (own) or imported (peer) mapping
  bool cuda_malloc = false;
  void* param = nullptr;
  float* grad = nullptr;
  uint64_t* flags = nullptr;
  void* ag = nullptr;     // [depth + cache_slots][slot_elems]: ring, then the reuse cache
  void* wgrad = nullptr;  // [wslots][slot_elems] wire dtype (null when z2 == 1)
};

struct ArenaLayout {
  size_t param = 0, grad = 0, flags = 0, ag = 0, ag_bytes = 0, wgrad = 0, wgrad_bytes = 0, total = 0;
};

struct LocalRank {
  int rank = 0;
  float* master = nullptr;
  float* mom = nullptr;
  float* var = nullptr;
  float* dbg = nullptr;
  void* mbuf = nullptr;  // model buffers
  int adam_step = 0;
};

struct Engine {
  hzp_engine_config cfg{};
  ModelConfig mcfg;
  std::unique_ptr<Model> model;
  ShardGeom geom;
  std::vector<LayerRange> layers;
  int64_t slot_elems = 0;  // padded max layer size
  bool emulate = true;
  bool bf16 = true;
  int depth = 2, rs_slots = 1, wslots = 2;
  bool direct_grad = false;  // z2 == 1: wgrad GEMM accumulates into the grad shard
  bool zero_copy_ag = false; // z3 == 1: layers read straight from the param shard

  TaskGraph graph;
  PoolSet pools;
  LaunchPlan plan;
  // Parameter reuse (cfg.reuse): an AG consumed by more than one FWD/BWD lands
  // in cache slot depth + layer (it outlives its ring slot); param_slot[task]
  // = the AG-buffer slot a FWD/BWD reads, ag_slot[task] = where an AG writes.
  int cache_slots = 0;
  std::vector<int> param_slot, ag_slot;
  std::vector<int> ag_phys_wait;  // AG task -> extra wait (last reader of the slot's occupant)

  cudaStream_t st[3] = {nullptr, nullptr, nullptr};
  cudaStream_t opt_stream = nullptr;  // per-layer Z1 kernels (async mode)
  std::vector<cudaEvent_t> done;
  std::vector<cudaEvent_t> tev0, tev1;
  // per-layer Z1 on the optimizer stream (timeline, async mode): gradient
  // final here / every GradReady wait passed / kernel done
  std::vector<cudaEvent_t> zev_ready, zev_start, zev_end;
  bool z1_timed = false;  // the last step recorded them
  void timeline_events(bool on);
  cudaEvent_t ev_step0 = nullptr, ev_step1 = nullptr, ev_opt = nullptr;

  std::vector<Arena> arenas;  // [dp]
  std::vector<LocalRank> locals;
  RankTable table{};
  RankTable* dtable = nullptr;

  CommTile* dtiles = nullptr;
  std::vector<int> ag_off, rs_off;  // [L + 1] per layer tile ranges
  std::vector<uint64_t> ag_owners;  // [L] Z3 members owning part of layer l (multi-process)
  bool ag_pull = false;             // Z3 groups of 2: readers pull (tiles in pull form)
  int z1_off = 0, z1_n = 0;
  std::vector<int> z1_layer_off;       // [L + 1] Z1 tiles per layer
  std::vector<uint64_t> z1_wait_mask;  // [L] ranks whose GradReady(l) this rank's Z1(l) needs
  cudaEvent_t ev_z1 = nullptr;         // last per-layer Z1 of the step (async mode)
  ArenaLayout lay;
  McGroup ag_mc, wg_mc;  // NVLS objects of this rank's Z3 / Z2 group (multi-process)
  // AG / RS launch one short-lived 128-thread CTA per tile (<= 64 KB, ~10 us):
  // one fits beside a resident persistent GEMM CTA, and a comm CTA that lands
  // on an SM between two GEMMs delays the next GEMM's CTA there by one tile at
  // most (a grid-stride CTA would hold it for the whole collective)
  static constexpr int kCommCtas = 1 << 16;

  void* dinputs = nullptr;
  size_t input_bytes_per_mb = 0;
  float* hloss = nullptr;  // pinned [nlocal]

  uint64_t rs_seq = 0, ag_seq = 0, grad_seq = 0, barrier_epoch = 0;
  std::vector<hzp_launch_rec> log;
  int64_t launches = 0;
  bool peers_open = false;
  bool debug_sync = false;

  explicit Engine(const hzp_engine_config& c);
  ~Engine();

  int local_index(int rank) const;
  void build_tiles();
  // Collective algorithm by group size (both hand-written kernels; chosen by
  // the traffic shape, as NCCL picks ring / NVLS): a layer lies inside one
  // member's shard, so the AG is a broadcast and the RS a reduce at that
  // owner.  With one peer (group of 2) the owner's unicast stores / ordered
  // pull move the layer over its link once at up to ~760 GB/s; with >= 2
  // peers a unicast broadcast / pull would cross the owner's link (z - 1)
  // times, so the NVLS multicast store / in-switch reduce (one crossing,
  // ~470-570 GB/s measured) wins.  Emulation runs the unicast model of the
  // same choice (multicast groups: the sum rounded to bf16 like the switch).
  bool rs_multicast_group() const { return bf16 && !direct_grad && geom.z2 >= 3; }
  bool ag_multicast() const { return !emulate && cfg.par.dp > 1 && !zero_copy_ag && geom.z3 >= 3; }
  // (groups of 2 pull: tiles.hpp ag_pull)
  bool rs_multicast() const { return !emulate && cfg.par.dp > 1 && rs_multicast_group(); }
  void carve(Arena& a) const;
  ShareRecord share_record() const;
  void open_peers(const ShareRecord* records, int n);
  void step(const void* inputs, bool on_device, float* losses_out);
  // ready_posted: the step posted this AG's "slot free" from the compute
  // stream already (at the task that released the slot); else post it here
  void ag_layer(int layer, int slot, cudaStream_t s, bool ready_posted = false);
  void rs_layer(int layer, int wslot, bool assign, uint64_t seq, cudaStream_t s);
  void z1_adam(cudaStream_t s);  // every layer at once (test entry / vanilla mode)
  AdamArgs next_adam_args();     // advances the Adam step of every driven rank
  // Z1 of one layer as soon as its gradient is final everywhere it is read
  // from and its parameters are no longer read anywhere this step
  void z1_layer(int layer, const AdamArgs& a, cudaStream_t s, cudaStream_t post = nullptr);
  void barrier(cudaStream_t s);
  GradTarget grad_target(int li, int layer, int wslot, int mb) const;
  const void* layer_params(int li, int layer, int slot) const;
};

}  // namespace hzp
