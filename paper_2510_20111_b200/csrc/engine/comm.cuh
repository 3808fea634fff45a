// Collective kernels of the hot path (declarations + pointer table).
//
//   ag_push   — layer-wise parameter all-gather within the Z3 group
//               (collective.cpp:44-67 at train.cpp:281-293).  With the flat
//               layout a layer lies (almost always) inside ONE member's Z3
//               shard, so the gather is a broadcast from that owner: the
//               owner stores its span once into the group's NVLS multicast
//               AG slot (multimem.st.v4) and the switch delivers it to every
//               member's slot — the owner's link carries the layer once, not
//               (z3 - 1) times, and the readers spend no SM time.  In a
//               group of 2 the one reader pulls instead (same single link
//               crossing, faster unicast loads, no rendezvous).
//   rs_reduce — gradient reduce-scatter within the Z2 group
//               (collective.cpp:69-97 + train.cpp:306-323): the member that
//               owns (layer ∩ its Z2 segment) reduces it and accumulates
//               into its fp32 grad shard, with the cast / scale fused:
//                 bf16 wire: multimem.ld_reduce (in-switch fp32 accumulate,
//                   bf16 result) over the group's multicast gradient slot;
//                 fp32 wire: ordered pull — fp32 sum of the members'
//                   gradient slots in ascending rank order (bit-exact tier).
//   z1_adam   — the ZeRO-1 stage: pull-reduce of the Z1 chunk across DZP
//               replicas (collective.cpp:99-115 at train.cpp:326-350), Adam
//               (train.cpp:171-189), round-to-bf16 and P2P store of the new
//               working copy into every Z3 owner of the Z1 group
//               (train.cpp:361-379).
//
// With every dp rank emulated on one GPU (parity mode) the same kernels run
// with the NVLink primitive replaced by its unicast equivalent: the owner
// stores to each member's slot; the reducer sums the members' slots in
// ascending order and (bf16 wire) rounds the sum to bf16 as the switch does.
//
// All walk a host-built tile table (hzp/tiles.hpp).
#pragma once

#include <cstdint>

#include "engine/common.cuh"
#include "hzp/tiles.hpp"

namespace hzp {

constexpr int kMaxRanks = 64;

// Device-visible pointer table (one per ctx).  Indexed by GLOBAL dp rank;
// peers' entries are their arenas mapped over NVLink (multi-process) or the
// emulated ranks' buffers (one GPU).
struct RankTable {
  void* param[kMaxRanks];   // working-copy shards [s3] of every dp rank
  float* grad[kMaxRanks];   // fp32 grad shards [s2]
  void* wgrad[kMaxRanks];   // gradient ring buffers [wslots][slot]
  void* ag[kMaxRanks];      // AG ring + reuse cache [depth + cache][slot]
  uint64_t* flags[kMaxRanks];
  // this process's NVLS multicast addresses (multi-process only, else null)
  void* ag_mc;     // Z3 group's AG buffer
  void* wgrad_mc;  // Z2 group's gradient ring (bf16 wire)
  // driven (local) ranks, by local index
  float* master[kMaxRanks];
  float* mom[kMaxRanks];
  float* var[kMaxRanks];
  float* z1_grad_dbg[kMaxRanks];  // optional reduced-gradient dump [s1]
  int global_rank[kMaxRanks];     // driven-rank index -> global dp rank
};

struct AdamArgs {
  float lr, b1, b2, eps, omb1, omb2, bc1, bc2;  // omb = 1 - b (fp32), bc from (T)pow
};

// Monotonic 64-bit flags in every rank's arena: flags[kind * kMaxRanks + q]
// on rank r = the latest value rank q posted to r.
enum FlagKind {
  kFlagBarrier = 0,
  kFlagRsReady = 1,  // gradient slot written (RS sequence number)
  kFlagRsDone = 2,   // RS finished on the poster (its reads of peers' slots too)
  kFlagAgReady = 3,  // AG slot free on the poster (AG sequence number)
  kFlagAgDone = 4,   // owner's span landed in every member's slot
  kFlagGradReady = 5,  // a layer's gradient final on the poster (and its param reads done)
  kNumFlagKinds = 6
};

// Optional in-kernel gate: spin until flags[me][kind][q] >= value for every
// q in mask (multi-process only; 0 = no gate).
struct FlagGate {
  int me = 0, kind = 0;
  uint64_t mask = 0, value = 0;
};

enum RsMode {
  kRsOrdered = 0,       // ascending-rank fp32 sum of unicast loads
  kRsOrderedRound = 1,  // same, sum rounded to bf16 (unicast model of the switch)
  kRsMulticast = 2      // multimem.ld_reduce.add.acc::f32 (bf16 wire, NVLS)
};

enum AgMode {
  kAgUnicastPush = 0,  // owner stores into every member's slot (the unicast model of kAgMulticast)
  kAgMulticast = 1,    // owner: one multimem.st into the group's NVLS slot
  kAgPull = 2          // reader copies the owners' spans into its own slot (pull-form tiles)
};
// AG of one layer into slot `slot`: owner-push tiles (z3 members from
// z3_base(owner)) or reader-pull tiles (tiles.hpp ag_pull).
void launch_ag_push(const RankTable* dev_table, const CommTile* tiles, int ntiles, int slot,
                    int64_t slot_elems, int z3, bool bf16, AgMode mode, FlagGate gate, int ctas,
                    cudaStream_t s);
void launch_rs_reduce(const RankTable* dev_table, const CommTile* tiles, int ntiles, int wslot,
                      int64_t wslot_elems, int z2, bool bf16_wire, RsMode mode, bool assign, float scale,
                      FlagGate gate, int ctas, cudaStream_t s);
void launch_z1_adam(const RankTable* dev_table, const CommTile* tiles, int ntiles, int z2,
                    int replicas, const AdamArgs* per_local, int nlocal, bool bf16_param,
                    bool dbg, int ctas, cudaStream_t s);
// Post `value` into flags[q][post_kind][me] for every q in post_mask, then
// wait until flags[me][wait_kind][q] >= wait_value for every q in wait_mask
// (single CTA; either mask may be 0).
void launch_flags(const RankTable* dev_table, int me, int post_kind, uint64_t post_mask, uint64_t post_value,
                  int wait_kind, uint64_t wait_mask, uint64_t wait_value, cudaStream_t s);

inline uint64_t rank_mask(int first, int count) {
  return (count >= 64 ? ~0ull : ((1ull << count) - 1)) << first;
}

}  // namespace hzp
