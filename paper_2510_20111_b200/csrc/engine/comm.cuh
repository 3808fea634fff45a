// P2P collective kernels of the hot path (declarations + tile format).
//
//   ag_pull   — layer-wise parameter all-gather within the Z3 group
//               (collective.cpp:44-67 at train.cpp:281-293), pulled from the
//               owners' param shards into this rank's AG ring slot.
//   rs_pull   — gradient reduce-scatter within the Z2 group
//               (collective.cpp:69-97 + train.cpp:306-323): ascending-rank
//               fp32 sum of the peers' gradient ring buffers (bf16->fp32 cast
//               and scale fused), accumulated into the Z2 grad shard.
//   z1_adam   — the ZeRO-1 stage: pull-reduce of the Z1 chunk across DZP
//               replicas (collective.cpp:99-115 at train.cpp:326-350), Adam
//               (train.cpp:171-189), round-to-bf16 and P2P store of the new
//               working copy into every Z3 owner of the Z1 group
//               (train.cpp:361-379).
//
// All three walk a host-built tile table; every tile is a contiguous element
// range that lies inside one owner / segment, flagged vectorisable when all
// of its addresses are 16-byte aligned.
#pragma once

#include <cstdint>

#include "engine/common.cuh"
#include "hzp/tiles.hpp"

namespace hzp {

constexpr int kMaxRanks = 64;

// CommTile: see hzp/tiles.hpp (host-built work table).

// Device-visible pointer table (one per ctx).
struct RankTable {
  void* param[kMaxRanks];   // working-copy shards [s3] of every dp rank
  float* grad[kMaxRanks];   // fp32 grad shards [s2]
  void* wgrad[kMaxRanks];   // gradient ring buffers [wslots][max_layer]
  uint64_t* flags[kMaxRanks];
  // driven (local) ranks only
  void* ag_slots[kMaxRanks];  // [depth][max_layer]
  float* master[kMaxRanks];
  float* mom[kMaxRanks];
  float* var[kMaxRanks];
  float* z1_grad_dbg[kMaxRanks];  // optional reduced-gradient dump [s1]
  int global_rank[kMaxRanks];     // driven-rank index -> global dp rank
};

struct AdamArgs {
  float lr, b1, b2, eps, omb1, omb2, bc1, bc2;  // omb = 1 - b (fp32), bc from (T)pow
};

enum FlagKind { kFlagBarrier = 0, kFlagRsReady = 1, kFlagRsDone = 2, kNumFlagKinds = 3 };

// Launch wrappers (stream-ordered; grid sized by `ctas`).
void launch_ag_pull(const RankTable* dev_table, const CommTile* tiles, int ntiles, int slot,
                    int64_t slot_elems, bool bf16, int ctas, cudaStream_t s);
// split: CTAs per tile (HBM-local reduces of staged gradients use > 1).
void launch_rs_pull(const RankTable* dev_table, const CommTile* tiles, int ntiles, int wslot,
                    int64_t wslot_elems, int z2, bool bf16_wire, bool assign, float scale,
                    int ctas, cudaStream_t s, int split = 1);
void launch_z1_adam(const RankTable* dev_table, const CommTile* tiles, int ntiles, int z2,
                    int replicas, const AdamArgs* per_local, int nlocal, bool bf16_param,
                    bool dbg, int ctas, cudaStream_t s);
// Signals (single CTA): post `value` into flags[kind][me] of every rank in
// [first, first+count) (stride 1), then optionally wait until this rank's
// flags[kind][q] >= wait_value for all q in that range.
void launch_signal(const RankTable* dev_table, int me, int kind, int first, int count,
                   int stride, uint64_t value, int wait_kind, uint64_t wait_value,
                   cudaStream_t s);
void launch_wait(const RankTable* dev_table, int me, int kind, int first, int count, int stride,
                 uint64_t value, cudaStream_t s);

}  // namespace hzp
