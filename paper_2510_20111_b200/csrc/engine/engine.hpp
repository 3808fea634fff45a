// Device engine: one hzp_ctx drives one GPU and either one dp rank (one
// process per GPU, peers reached through CUDA IPC over NVLink/NVSwitch) or
// all dp ranks emulated on that GPU (single-process parity mode).
#pragma once

#include <memory>
#include <vector>

#include "hzp/sched.hpp"
#include "hzp_b200.h"
#include "engine/comm.cuh"
#include "engine/model.hpp"

namespace hzp {

struct Arena {
  void* base = nullptr;
  size_t bytes = 0;
  bool owned = false;  // allocated here (else IPC-mapped)
  void* param = nullptr;
  float* grad = nullptr;
  void* wgrad = nullptr;
  uint64_t* flags = nullptr;
};

struct LocalRank {
  int rank = 0;
  void* ag = nullptr;  // [depth + cache_slots][slot_elems]: ring, then the reuse cache
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
  std::vector<cudaEvent_t> done;
  std::vector<cudaEvent_t> tev0, tev1;
  cudaEvent_t ev_step0 = nullptr, ev_step1 = nullptr, ev_opt = nullptr;

  std::vector<Arena> arenas;  // [dp]
  std::vector<LocalRank> locals;
  RankTable table{};
  RankTable* dtable = nullptr;

  CommTile* dtiles = nullptr;
  std::vector<int> ag_off, rs_off;  // [nlocal_layers + 1] per layer tile ranges
  // AG through the copy engines (no SMs taken from the concurrent GEMMs): the
  // layer's tiles merged into contiguous (owner -> slot) runs
  struct CopyRun {
    int local, src;
    int64_t dst_off, src_off, len;
  };
  std::vector<std::vector<CopyRun>> ag_runs;
  bool ag_ce = true;   // HZP_AG_CE=0 to use the SM pull
  // HZP_AG_PAR=1: each owner's runs on its own copy stream (all owners read at once)
  bool ag_par = false;
  std::vector<cudaStream_t> ag_copy_streams;
  std::vector<cudaEvent_t> ag_par_ev;  // [0] fork, [1 + i] join of stream i
  // RS with the NVLink leg on the copy engines: each remote Z2 member's
  // gradient-buffer segment is copied into a local staging slot, then the
  // (now HBM-local) reduction kernel runs on a table whose remote wgrad
  // entries point at the staging slots (one table per ring slot).
  std::vector<void*> rs_stage;                // [dp] staging slot per remote member (or null)
  std::vector<RankTable*> dtable_staged;      // [wslots]
  // The copy of chunk c+1 overlaps the HBM-local reduce of chunk c: copies
  // on the RS stream, reduces on rs_red_stream, chained by rs_ev.
  std::vector<CommTile> tiles_host;
  cudaStream_t rs_red_stream = nullptr;
  std::vector<cudaEvent_t> rs_ev;
  // each peer's copies on its own stream, all peers pulled at once (HZP_RS_PAR=0:
  // one stream, peers in rotated order; 441 vs 576 GB/s for a 1 GB layer at N=4)
  bool rs_par = true;
  std::vector<cudaStream_t> rs_copy_streams;
  std::vector<cudaEvent_t> rs_par_ev;
  static constexpr int kRsChunkTiles = 128;  // 4 M elements per pipelined chunk
  int64_t rs_min_chunk_bytes = 0;  // per peer copy, 0 = auto (HZP_RS_MIN_CHUNK_MB)
  bool rs_ce = true;
  // Z1 with DZP replicas (R > 1): the remote replicas' gradient segments of
  // this rank's chunk are copied (copy engines) into double-buffered local
  // staging, chunk by chunk, while the fused Z1 kernel consumes the previous
  // chunk through a table whose remote grad entries point at the staging.
  bool z1_ce = false;  // HZP_Z1_CE=1 (7B dp=4: 36.6 vs 31.3 ms SM pull, so off)
  struct Z1Chunk {
    int t0, t1;                       // tile range (within the Z1 tiles)
    RankTable* table;                 // device table for this chunk
    std::vector<CopyRun> copies;      // CopyRun.src = global rank; dst_off into its staging buffer
  };
  std::vector<Z1Chunk> z1_chunks;
  std::vector<void*> z1_stage;        // [dp]: 2 x kZ1ChunkElems fp32 per remote replica rank
  cudaStream_t z1_copy_stream = nullptr;
  static constexpr int64_t kZ1ChunkElems = int64_t(16) << 20;
  void setup_z1_staging();   // HZP_RS_CE=0 to use the SM pull (dp=4: 184.5 -> 160.1 ms with both CE legs)
  void setup_rs_staging();
  int z1_off = 0, z1_n = 0;

  void* dinputs = nullptr;
  size_t input_bytes_per_mb = 0;
  float* hloss = nullptr;  // pinned [nlocal]

  uint64_t rs_seq = 0, barrier_epoch = 0;
  std::vector<hzp_launch_rec> log;
  int64_t launches = 0;
  int comm_ctas = kNumSMs;  // one 256-thread CTA per SM, beside the persistent GEMM
  int rs_chunks = 4;        // copy-engine RS: at most this many pipelined chunks per layer (HZP_RS_CHUNKS)
  bool peers_open = false;
  bool debug_sync = false;

  explicit Engine(const hzp_engine_config& c);
  ~Engine();

  int local_index(int rank) const;
  void build_tiles();
  void step(const void* inputs, bool on_device, float* losses_out);
  void ag_layer(int layer, int slot, cudaStream_t s);
  void rs_layer(int layer, int wslot, bool assign, cudaStream_t s);
  void z1_adam(cudaStream_t s);
  void barrier(cudaStream_t s);
  GradTarget grad_target(int li, int layer, int wslot, int mb) const;
  const void* layer_params(int li, int layer, int slot) const;
};

}  // namespace hzp
