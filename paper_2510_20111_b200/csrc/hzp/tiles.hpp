// Host-side work decomposition of the P2P collectives (pure C++, no CUDA):
// every AG / RS / Z1 pass is a table of CommTiles, each a contiguous element
// range inside one owner / segment, flagged vectorisable when all of its
// addresses are 16-byte aligned.  Built once per ctx; the kernels only walk
// the table.  Exposed through the C-ABI (hzp_comm_tiles) so the multi-rank
// coverage properties are testable on the CPU.
#pragma once

#include <cstdint>
#include <vector>

#include "hzp/config.hpp"

namespace hzp {

struct CommTile {
  int64_t a_off;   // AG: slot offset | RS: grad offset | Z1: chunk offset
  int64_t b_off;   // AG: offset in the owner's shard | RS: gradient-buffer offset | Z1: grad-shard offset
  int64_t c_off;   // Z1: param-shard offset
  uint64_t mask;   // Z1: push targets, bit q = global rank q
  int32_t len;     // elements
  int16_t local;   // index of the rank among the ctx's driven ranks (AG push: the owner, AG pull: the reader;
                   // RS / Z1: the destination)
  int16_t src;     // AG: owner rank | RS: Z2 group base | Z1: Z2 segment index j
  int32_t vec;     // 1 = every address 16-byte aligned and len a multiple of the vector
  int32_t pad_;
};

struct TileTables {
  std::vector<CommTile> tiles;
  std::vector<int> ag_off;  // [L + 1]
  bool ag_pull = false;     // AG tiles in reader-pull form (Z3 groups of 2) instead of owner-push
  std::vector<int> rs_off;  // [L + 1]
  int z1_off = 0, z1_n = 0;
  std::vector<int> z1_layer_off;  // [L + 1]: Z1 tiles of layer l (every driven rank)
};

struct Range64 {
  int64_t off, size;
};

// working_bytes: 2 (bf16) or 4 (fp32) for param shards / AG slots / wire.
// direct_grad: z2 == 1, no RS tiles.
TileTables build_comm_tiles(const ShardGeom& g, const std::vector<Range64>& layers,
                            const std::vector<int>& local_ranks, int working_bytes,
                            bool direct_grad);

}  // namespace hzp
