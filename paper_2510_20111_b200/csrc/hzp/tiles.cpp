// Tile tables of the AG / RS / Z1 passes (see tiles.hpp).  Geometry follows
// the reference's flat-vector sharding: element e of the working copy lives
// on Z3 member e / s3 (train.cpp:229-249), rank r's gradient segment is
// [(r%z2)*s2, +s2) and its optimizer chunk [(r%z1)*s1, +s1) (train.cpp:354).
#include "hzp/tiles.hpp"

#include <algorithm>

namespace hzp {
namespace {

// Tile = the work of one short-lived 128-thread CTA (these kernels run beside
// the persistent GEMMs, so a CTA must not hold an SM for long): 32 K elements
// for AG / RS (64 KB of bf16 moved), 4 K for the optimizer (30 B / element of
// HBM traffic, ~120 KB).
constexpr int64_t kTileElems = 1 << 15;
constexpr int64_t kZ1TileElems = 1 << 12;

// Split a contiguous element run whose streams start at offs[] (element
// offsets into 256-byte aligned buffers of elem bytes ebytes[]) into tiles:
// scalar head, vector body (aligned for every stream, multiple of vec
// elements), scalar tail; bodies are cut into pieces of <= kTileElems.
template <typename Emit>
void split_run(const int64_t* offs, const int* ebytes, int nstreams, int64_t len, int vec,
               Emit&& emit, int64_t tile = kTileElems) {
  auto aligned_at = [&](int64_t h) {
    for (int s = 0; s < nstreams; ++s)
      if (((offs[s] + h) * ebytes[s]) % 16 != 0) return false;
    return true;
  };
  int64_t head = -1;
  for (int64_t h = 0; h < 64 && h <= len; ++h)
    if (aligned_at(h)) {
      head = h;
      break;
    }
  if (head < 0 || len - head < vec) {
    for (int64_t p = 0; p < len; p += tile) emit(p, std::min(tile, len - p), false);
    return;
  }
  if (head > 0) emit(0, head, false);
  const int64_t body = (len - head) / vec * vec;
  const int64_t piece = std::max<int64_t>(vec, tile / vec * vec);
  for (int64_t p = 0; p < body; p += piece) emit(head + p, std::min(piece, body - p), true);
  if (head + body < len) emit(head + body, len - head - body, false);
}

uint64_t z1_targets(const ShardGeom& g, int rank, int j3) {
  uint64_t m = 0;
  const int base = g.z1_base(rank);
  for (int q = base; q < base + g.z1; ++q)
    if (q % g.z3 == j3) m |= 1ull << q;
  return m;
}

}  // namespace

TileTables build_comm_tiles(const ShardGeom& g, const std::vector<Range64>& layers,
                            const std::vector<int>& local_ranks, int es, bool direct_grad) {
  TileTables T;
  auto& tiles = T.tiles;
  const int L = static_cast<int>(layers.size());
  // AG (owner push): per layer, per driven rank o, the part of the layer o
  // owns (layer ∩ o's Z3 shard).  o stores it into the AG slot of every
  // member of its Z3 group (one multimem.st on NVLS; the union over the
  // group's owners covers the layer once).
  //
  // AG (reader pull, Z3 groups of 2): per layer, per driven rank r, the
  // layer's spans by owner; r copies them from the owners' shards into its
  // own slot (with one peer the owner's link carries the layer once either
  // way, and a pull needs no rendezvous: the owner's shard does not change
  // during the step).
  T.ag_off.assign(L + 1, 0);
  T.ag_pull = g.z3 == 2;
  for (int l = 0; l < L && T.ag_pull; ++l) {
    T.ag_off[l] = static_cast<int>(tiles.size());
    for (size_t li = 0; li < local_ranks.size(); ++li) {
      const int r = local_ranks[li];
      int64_t e = layers[l].off;
      const int64_t end = layers[l].off + layers[l].size;
      while (e < end) {
        const int j3 = static_cast<int>(e / g.s3);
        const int64_t stop = std::min(end, (j3 + 1) * g.s3);
        const int64_t offs[2] = {e - layers[l].off, e - j3 * g.s3};
        const int eb[2] = {es, es};
        split_run(offs, eb, 2, stop - e, 16 / es, [&](int64_t p, int64_t n, bool v) {
          CommTile t{};
          t.a_off = offs[0] + p;
          t.b_off = offs[1] + p;
          t.len = static_cast<int32_t>(n);
          t.local = static_cast<int16_t>(li);
          t.src = static_cast<int16_t>(g.z3_base(r) + j3);
          t.vec = v;
          tiles.push_back(t);
        });
        e = stop;
      }
    }
  }
  for (int l = 0; l < L && !T.ag_pull; ++l) {
    T.ag_off[l] = static_cast<int>(tiles.size());
    for (size_t li = 0; li < local_ranks.size(); ++li) {
      const int o = local_ranks[li];
      const int i3 = o % g.z3;
      const int64_t e0 = std::max(layers[l].off, i3 * g.s3);
      const int64_t e1 = std::min(layers[l].off + layers[l].size, (i3 + 1) * g.s3);
      if (e0 >= e1) continue;
      const int64_t offs[2] = {e0 - layers[l].off, e0 - i3 * g.s3};
      const int eb[2] = {es, es};
      split_run(offs, eb, 2, e1 - e0, 16 / es, [&](int64_t p, int64_t n, bool v) {
        CommTile t{};
        t.a_off = offs[0] + p;
        t.b_off = offs[1] + p;
        t.len = static_cast<int32_t>(n);
        t.local = static_cast<int16_t>(li);
        t.src = static_cast<int16_t>(o);
        t.vec = v;
        tiles.push_back(t);
      });
    }
  }
  T.ag_off[L] = static_cast<int>(tiles.size());
  // RS: per layer, per driven rank, the layer ∩ its Z2 segment.
  T.rs_off.assign(L + 1, 0);
  for (int l = 0; l < L; ++l) {
    T.rs_off[l] = static_cast<int>(tiles.size());
    if (direct_grad) continue;
    for (size_t li = 0; li < local_ranks.size(); ++li) {
      const int r = local_ranks[li];
      const int i2 = r % g.z2;
      const int64_t e0 = std::max(layers[l].off, i2 * g.s2);
      const int64_t e1 = std::min(layers[l].off + layers[l].size, (i2 + 1) * g.s2);
      if (e0 >= e1) continue;
      const int64_t offs[2] = {e0 - i2 * g.s2, e0 - layers[l].off};
      const int eb[2] = {4, es};
      split_run(offs, eb, 2, e1 - e0, es == 2 ? 8 : 4, [&](int64_t p, int64_t n, bool v) {
        CommTile t{};
        t.a_off = offs[0] + p;
        t.b_off = offs[1] + p;
        t.len = static_cast<int32_t>(n);
        t.local = static_cast<int16_t>(li);
        t.src = static_cast<int16_t>(g.z2_base(r));
        t.vec = v;
        tiles.push_back(t);
      });
    }
  }
  T.rs_off[L] = static_cast<int>(tiles.size());
  // Z1: each driven rank's chunk ∩ [0, P), cut at Z2 and Z3 segment bounds
  // and at layer bounds; grouped by layer (z1_layer_off) so the optimizer
  // step of a layer can run as soon as that layer's gradient is final.
  T.z1_off = static_cast<int>(tiles.size());
  T.z1_layer_off.assign(L + 1, T.z1_off);
  for (int l = 0; l < L; ++l) {
    T.z1_layer_off[l] = static_cast<int>(tiles.size());
    for (size_t li = 0; li < local_ranks.size(); ++li) {
      const int r = local_ranks[li];
      const int i1 = r % g.z1;
      int64_t e = std::max(int64_t(i1) * g.s1, layers[l].off);
      const int64_t end = std::min({int64_t(i1 + 1) * g.s1, g.P, layers[l].off + layers[l].size});
      while (e < end) {
        const int j2 = static_cast<int>(e / g.s2), j3 = static_cast<int>(e / g.s3);
        const int64_t stop = std::min({end, (j2 + 1) * g.s2, (j3 + 1) * g.s3});
        const int64_t offs[3] = {e - i1 * g.s1, e - j2 * g.s2, e - j3 * g.s3};
        // master/m/v and grads are fp32 (16-byte float4); the param stream is
        // stored 4 elements at a time (float4 or 4 x bf16 = 8 bytes), so all
        // three need offset % 4 == 0: model that as 4-byte elements.
        const int eb[3] = {4, 4, 4};
        const uint64_t mask = z1_targets(g, r, j3);
        split_run(offs, eb, 3, stop - e, 4, [&](int64_t p, int64_t n, bool v) {
          CommTile t{};
          t.a_off = offs[0] + p;
          t.b_off = offs[1] + p;
          t.c_off = offs[2] + p;
          t.mask = mask;
          t.len = static_cast<int32_t>(n);
          t.local = static_cast<int16_t>(li);
          t.src = static_cast<int16_t>(j2);
          t.vec = v;
          tiles.push_back(t);
        }, kZ1TileElems);
        e = stop;
      }
    }
  }
  T.z1_layer_off[L] = static_cast<int>(tiles.size());
  T.z1_n = static_cast<int>(tiles.size()) - T.z1_off;
  return T;
}

}  // namespace hzp
