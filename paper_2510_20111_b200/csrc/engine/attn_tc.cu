// Fused causal attention (head dim 128) on tcgen05 (sm_100a).
//
// Forward, attn_fwd2_kernel (used whenever the query-tile count is even; the
// single-tile attn_fwd_kernel below covers odd counts and the optional P
// output): one CTA per (head, sequence, pair of 128-query tiles), 10 warps:
//   warp 0    TMA producer: both Q tiles once, then K_j (3-deep ring) and V_j
//             (2-deep, MN-major 64x64 boxes), 128 keys per tile
//   warp 1    TMEM owner + MMA issuer (one thread), ping-pong per query tile g:
//               S_g = Q_g K_j^T   -> TMEM [g*128, +128)    (M=N=K=128)
//               O_g += P_g V_j    -> TMEM [256 + g*128, +128), A = P_g from TMEM
//   warps 2-9 two softmax warpgroups (one per query tile), one thread per
//             query row (its TMEM lane): row max over S, P = 2^(s c - m) with
//             FFMA2 and 1/4 of the exp2 on the FMA pipe, P (bf16) written back
//             over the consumed S columns, lazy O rescale, final O / l and lse.
// Neither S nor P ever leaves the SM.  The backward (attn_bwd_kernel, further
// down) works per 128-key tile with P^T / dS^T kept in TMEM the same way.
#include <cmath>
#include <type_traits>

#include "engine/gemm.cuh"
#include "engine/tc_ptx.cuh"

namespace hzp {
namespace {

using namespace tc;

#ifndef HZP_ATTN_POLY_FROM
#define HZP_ATTN_POLY_FROM 6  // forward: pairs i % 8 >= this use the FMA-pipe exp2 (2 of 8; swept 3..8 of 8 on B200: 6 best)
#endif
#ifndef HZP_ATTN_BWD_POLY_FROM
#define HZP_ATTN_BWD_POLY_FROM 3  // backward: pairs i % 4 >= this use the FMA-pipe exp2
#endif
constexpr int kHd = 128;    // head dim
constexpr int kBQ = 128;    // query rows per CTA
constexpr int kBK = 128;    // keys per iteration
constexpr int kTileBytes = 128 * kHd * 2;  // 32 KB (Q, K_j, V_j, P_j)
constexpr int kThreads = 192;

struct AttnParams {
  CUtensorMap tmQ, tmK, tmV;  // 4-D views of qkv: {d, s, head, seq}
  CUtensorMap tmV5;           // V as {64 d, s, 2, head, seq}: a 64-key box carries both d halves
  uint16_t* O;                // [b, S, h]
  uint16_t* P;                // [b*nh, S, S] or null
  float* lse;                 // [b*nh, S] or null
  int S, h, nh, nq;
  float scale_log2;           // log2(e) / sqrt(d)
};

// smem map
constexpr int kOffQ = 0;
constexpr int kOffK = kTileBytes;              // 2 stages
constexpr int kOffV = 3 * kTileBytes;          // 2 stages
constexpr int kOffP = 5 * kTileBytes;          // 2 buffers
constexpr int kOffBar = 7 * kTileBytes;
constexpr size_t kSmem = 7 * kTileBytes + 1024 + 1024;

__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;     // [2]
  uint64_t* v_full = bar + 3;     // [2]
  uint64_t* kv_empty = bar + 5;   // [2]
  uint64_t* s_full = bar + 7;     // [2]
  uint64_t* s_free = bar + 9;     // [2]
  uint64_t* p_full = bar + 11;    // [2]
  uint64_t* p_empty = bar + 13;   // [2]
  uint64_t* o_ready = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  // grid (heads, seqs, tiles): the tile index varies slowest, so every head's
  // heavy (late) query tiles are dispatched before any light one (LPT order)
  const int qt = p.nq - 1 - blockIdx.z;
  const int head = blockIdx.x, seq = blockIdx.y;
  const int q0 = qt * kBQ;
  const int nkv = qt + 1;  // causal: key tiles 0..qt

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_empty[i], 1);
    }
    mbar_init(o_ready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S0: cols [0,128), S1: [128,256), O: [256,384)

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, kTileBytes);
      for (int c = 0; c < 2; ++c)
        tma_load_4d(smem + kOffQ + c * 16384, &p.tmQ, q_full, c * 64, q0, head, seq);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&kv_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_4d(smem + kOffK + st * kTileBytes + c * 16384, &p.tmK, &k_full[st], c * 64, j * kBK,
                      head, seq);
        mbar_expect_tx(&v_full[st], kTileBytes);
        for (int kc = 0; kc < 2; ++kc)
          tma_load_5d(smem + kOffV + st * kTileBytes + kc * 16384, &p.tmV5, &v_full[st], 0, j * kBK + kc * 64,
                      0, head, seq);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = make_idesc(128, 128, 0, 0);   // Q K-major, K K-major
      constexpr uint32_t kIdPV = make_idesc(128, 128, 0, 1);  // P K-major, V MN-major
      const uint32_t sq = smem_u32(smem + kOffQ);
      auto issue_pv = [&](int i) {
        const int st = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        mbar_wait(&p_full[st], ph);
        mbar_wait(&v_full[st], ph);
        tc_fence_after();
        const uint32_t sp = smem_u32(smem + kOffP + st * kTileBytes);
        const uint32_t sv = smem_u32(smem + kOffV + st * kTileBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = smem_desc(sp + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = smem_desc(sv + (kk >> 2) * 16384 + (kk & 3) * 2048, 8192, 1024);
          tc_mma(tmem + 256, ad, bd, kIdPV, (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(&p_empty[st]);
        tc_commit(&kv_empty[st]);
        tc_commit(o_ready);
      };
      mbar_wait(q_full, 0);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&k_full[st], ph);
        mbar_wait(&s_free[st], ph ^ 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + kOffK + st * kTileBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = smem_desc(sq + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = smem_desc(sk + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
          tc_mma(tmem + st * 128, ad, bd, kIdS, kk > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[st]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(nkv - 1);
    }
  } else {
    // ---- softmax warps: row = TMEM lane ----
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int q = q0 + row;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const int z = seq * p.nh + head;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      mbar_wait(&s_full[st], ph);
      tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + st * 128 + c * 32, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(r[i]) * p.scale_log2;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[st]);
      if (j == nkv - 1) {  // diagonal tile: keys j*128 + c > q are masked
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c > row) s[c] = -INFINITY;
      }
      float mx = m;
#pragma unroll
      for (int c = 0; c < 128; ++c) mx = fmaxf(mx, s[c]);
      // lazy rescaling (FA4): keep the stale max unless it grew by > 8 (log2
      // units); P <= 2^8 stays well inside fp32 / bf16 range and O, l use the
      // same reference max, so the result is exact up to rounding
      const bool bump = mx > m + 8.f;
      const float mref = bump ? mx : m;
      const float corr = bump ? exp2_fast(m - mx) : 1.f;  // 0 on the first tile (m = -inf)
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        s[c] = exp2_fast(s[c] - mref);
        sum += s[c];
      }
      l = l * corr + sum;
      m = mref;
      // P_j -> smem (K-major SW128 A operand) and global (backward)
      mbar_wait(&p_empty[st], ph ^ 1);
      uint8_t* pb = smem + kOffP + st * kTileBytes;
      uint4* pg = p.P ? reinterpret_cast<uint4*>(p.P + (int64_t(z) * p.S + q) * p.S + int64_t(j) * kBK) : nullptr;
#pragma unroll
      for (int c8 = 0; c8 < 16; ++c8) {
        const uint4 w = pack8f(s + 8 * c8);
        const int kc = c8 >> 3, j8 = c8 & 7;
        *reinterpret_cast<uint4*>(pb + kc * 16384 + row * 128 + ((j8 ^ (row & 7)) * 16)) = w;
        if (pg) pg[c8] = w;
      }
      // O holds P_{<j} V; only a row whose reference max moved needs PV_{j-1}
      // to land before rescaling.  Skipping the wait otherwise is safe: PV_j
      // cannot complete before this warp arrives on p_full[j], so o_ready is
      // never more than one phase ahead of the one waited for.
      if (j >= 1 && __any_sync(0xffffffffu, bump)) {
        mbar_wait(o_ready, (j - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_off + 256 + c * 32, r);
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
          tmem_st32(tmem + lane_off + 256 + c * 32, r);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[st]);
    }
    mbar_wait(o_ready, (nkv - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    uint4* og = reinterpret_cast<uint4*>(p.O + (int64_t(seq) * p.S + q) * p.h + int64_t(head) * kHd);
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + 256 + c * 32, r);
      float o[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r[i]) * inv;
#pragma unroll
      for (int i = 0; i < 4; ++i) og[c * 4 + i] = pack8f(o + 8 * i);
    }
    if (p.lse) p.lse[int64_t(z) * p.S + q] = (m + log2f(l)) * 0.6931471805599453f;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}



// ---------------------------------------------------------------------------
// Forward, two 128-row query tiles per CTA (qt0 = 2i, qt1 = 2i+1) sharing the
// K / V stream; 10 warps: TMA, MMA, and two softmax warpgroups (WG g owns Q
// tile g, TMEM S_g = [g*128, +128), O_g = [256 + g*128, +128)).  The tensor
// core alternates S0_j, S1_j, PV0_{j-1}, PV1_{j-1} so each warpgroup's
// softmax overlaps the other's MMAs.  Q0 skips the last key tile (fully
// masked).  K is double-buffered, V single-buffered.
constexpr int kThreads2 = 320;  // producer, MMA, 2 softmax warpgroups
constexpr int kKSt = 3;  // K_j stages
constexpr int kVSt = 2;  // V_j stages
constexpr int k2OffQ = 0;                               // 2 x 32 KB (both query tiles)
constexpr int k2OffK = 2 * kTileBytes;                  // 3 x 32 KB
constexpr int k2OffV = k2OffK + kKSt * kTileBytes;      // 2 x 32 KB
constexpr int k2OffBar = k2OffV + kVSt * kTileBytes;
constexpr size_t k2Smem = size_t(k2OffBar) + 256 + 1024;
static_assert(k2Smem <= 232448, "attention forward smem budget");

// P_j never touches shared memory: each softmax warpgroup writes it as bf16
// into the first 64 TMEM columns of its own S region, and O += P V_j reads A
// from TMEM.  That frees the smem for a 3-deep K ring and a 2-deep V ring.
__global__ void __launch_bounds__(kThreads2, 1) attn_fwd2_kernel(const __grid_constant__ AttnParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + k2OffBar);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;    // [kKSt]
  uint64_t* k_empty = bar + 4;   // [kKSt]
  uint64_t* v_full = bar + 7;    // [kVSt]
  uint64_t* v_empty = bar + 9;   // [kVSt]
  uint64_t* s_full = bar + 11;   // [g]
  uint64_t* p_full = bar + 13;   // [g]
  uint64_t* o_ready = bar + 15;  // [g]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int pair = (p.nq / 2) - 1 - blockIdx.z;  // heavy pairs first (LPT order)
  const int head = blockIdx.x, seq = blockIdx.y;
  const int qt0 = 2 * pair;
  const int nkv = qt0 + 2;  // key tiles 0..qt1

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < kKSt; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kVSt; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_ready[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S/P [g*128, +128), O [256 + g*128, +128)

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, 2 * kTileBytes);
      for (int g = 0; g < 2; ++g)
        for (int c = 0; c < 2; ++c)
          tma_load_4d(smem + k2OffQ + g * kTileBytes + c * 16384, &p.tmQ, q_full, c * 64,
                      (qt0 + g) * kBQ, head, seq);
      for (int j = 0; j < nkv; ++j) {
        const int ks = j % kKSt, vs = j % kVSt;
        mbar_wait(&k_empty[ks], ((j / kKSt) & 1) ^ 1);
        mbar_expect_tx(&k_full[ks], kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_4d(smem + k2OffK + ks * kTileBytes + c * 16384, &p.tmK, &k_full[ks], c * 64, j * kBK,
                      head, seq);
        mbar_wait(&v_empty[vs], ((j / kVSt) & 1) ^ 1);
        mbar_expect_tx(&v_full[vs], kTileBytes);
        for (int kc = 0; kc < 2; ++kc)
          tma_load_5d(smem + k2OffV + vs * kTileBytes + kc * 16384, &p.tmV5, &v_full[vs], 0, j * kBK + kc * 64,
                      0, head, seq);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = make_idesc(128, 128, 0, 0);
      constexpr uint32_t kIdPV = make_idesc(128, 128, 0, 1);
      // Ping-pong order: as soon as tile g's P_j is in TMEM, O_g += P_j V_j and
      // S_g = Q_g K_{j+1} are issued back to back (the latter overwrites P_j's
      // columns after the former has read them: same-thread MMAs run in
      // order), so each softmax warpgroup's next scores are computed while
      // the other warpgroup runs its softmax.  (Q0 is fully masked on the last
      // key tile: neither product is issued for it.)
      auto issue_s = [&](int g, int j) {
        const uint32_t sq = smem_u32(smem + k2OffQ + g * kTileBytes);
        const uint32_t sk = smem_u32(smem + k2OffK + (j % kKSt) * kTileBytes);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          tc_mma(tmem + g * 128, smem_desc(sq + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                 smem_desc(sk + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), kIdS, kk > 0);
        tc_commit(&s_full[g]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&k_full[0], 0);
      tc_fence_after();
      for (int g = 0; g < 2; ++g)
        if (!(g == 0 && nkv == 1)) issue_s(g, 0);
      tc_commit(&k_empty[0]);
      for (int j = 0; j < nkv; ++j) {
        const bool knext = j + 1 < nkv;
        mbar_wait(&v_full[j % kVSt], (j / kVSt) & 1);
        if (knext) mbar_wait(&k_full[(j + 1) % kKSt], ((j + 1) / kKSt) & 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + k2OffV + (j % kVSt) * kTileBytes);
        for (int g = 0; g < 2; ++g) {
          if (!(g == 0 && j == nkv - 1)) {
            mbar_wait(&p_full[g], j & 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // A = P_j (bf16 pairs, 8 columns per K = 16)
              tc_mma_ts(tmem + 256 + g * 128, tmem + g * 128 + kk * 8,
                        smem_desc(sv + (kk >> 2) * 16384 + (kk & 3) * 2048, 8192, 1024), kIdPV,
                        (j > 0 || kk > 0) ? 1u : 0u);
            tc_commit(&o_ready[g]);
          }
          if (knext && !(g == 0 && j + 1 == nkv - 1)) issue_s(g, j + 1);
        }
        tc_commit(&v_empty[j % kVSt]);
        if (knext) tc_commit(&k_empty[(j + 1) % kKSt]);
      }
    }
  } else {
    const int g = (warp - 2) >> 2;  // softmax warpgroup = query tile
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int qt = qt0 + g;
    const int q = qt * kBQ + row;
    const int nj = qt + 1;  // this tile's key tiles
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint32_t s_col = g * 128, o_col = 256 + g * 128;
    const int z = seq * p.nh + head;
    // m: running row max in log2 units (scores x scale log2 e)
    float m = -INFINITY, l = 0.f;
    const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2);
    for (int j = 0; j < nj; ++j) {
      mbar_wait(&s_full[g], j & 1);
      tc_fence_after();
      // Two passes over the row's 128 scores, read from TMEM once into
      // registers: the row max, then P = 2^(s c - mref) packed to bf16 and
      // stored over S_j's first 64 columns (chunk c's P on [16c, 16c+16)).
      const bool diag = j == nj - 1;
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      uint32_t r[128];  // the row's scores, kept for pass 2 (S is read from TMEM once)
      {  // pass 1: all 128 scores in flight at once, one wait
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32_nw(tmem + lane_off + s_col + c * 32, r + 32 * c);
        tmem_wait_ld32(r);
        tmem_pin32(r + 32);
        tmem_pin32(r + 64);
        tmem_pin32(r + 96);
        if (diag) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i > row) r[i] = 0xff800000u;  // -inf
        }
#pragma unroll
        for (int i = 0; i < 128; i += 8)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mx4[k] = fmaxf(mx4[k], fmaxf(__uint_as_float(r[i + 2 * k]), __uint_as_float(r[i + 2 * k + 1])));
      }
      const float mx = fmaxf(m, fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * p.scale_log2);
      const bool bump = mx > m + 8.f;
      const float mref = bump ? mx : m;
      const float corr = bump ? exp2_fast(m - mx) : 1.f;  // 0 on the first tile (m = -inf)
      // pass 2: P = 2^(s c - mref), FFMA2 per pair; 2 of every 8 pairs' exp2
      // on the FMA pipe so MUFU (16/clk/SM) stops bounding the tile.
      const uint64_t nm2 = f2_pack(-mref, -mref);
      uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t* rc = r + 32 * c;  // (the diagonal mask was applied in pass 1)
        uint32_t pw[16];
#pragma unroll
        for (int ii = 0; ii < 16; ++ii) {
          const int i = c * 16 + ii;
          const uint64_t x = f2_fma(f2_pack(__uint_as_float(rc[2 * ii]), __uint_as_float(rc[2 * ii + 1])), sc2, nm2);
          uint64_t e;
          if ((i & 7) >= HZP_ATTN_POLY_FROM) {
            e = exp2_poly2(x);
          } else {
            float a0, a1;
            f2_unpack(x, a0, a1);
            e = f2_pack(exp2_fast(a0), exp2_fast(a1));
          }
          acc[i & 3] = f2_add(acc[i & 3], e);
          float e0, e1;
          f2_unpack(e, e0, e1);
          pw[ii] = bf16x2(e0, e1);
        }
        tmem_st16_nw(tmem + lane_off + s_col + c * 16, pw);
      }
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float a0, a1;
        f2_unpack(acc[k], a0, a1);
        sum += a0 + a1;
      }
      l = l * corr + sum;
      m = mref;
      tmem_wait_st();
      if (j >= 1 && __any_sync(0xffffffffu, bump)) {
        mbar_wait(&o_ready[g], (j - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_off + o_col + c * 32, r);
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
          tmem_st32(tmem + lane_off + o_col + c * 32, r);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[g]);
    }
    mbar_wait(&o_ready[g], (nj - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    uint4* og = reinterpret_cast<uint4*>(p.O + (int64_t(seq) * p.S + q) * p.h + int64_t(head) * kHd);
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_off + o_col + c * 32, r);
      float o[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r[i]) * inv;
#pragma unroll
      for (int i = 0; i < 4; ++i) og[c * 4 + i] = pack8f(o + 8 * i);
    }
    if (p.lse) p.lse[int64_t(z) * p.S + q] = (m + log2f(l)) * 0.6931471805599453f;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------------------
// Fused causal attention backward for dK, dV (and dS^T for the dQ GEMM).
//
// One CTA per (128-key tile, head, sequence), iterating 64-query sub-tiles
// q >= key tile.  Rows of every TMEM accumulator are KEYS:
//   S^T  = K Q_i^T          TMEM S[b]  (64 cols)  P^T  = exp2(S^T*c - lse2_q)
//   dP^T = V dO_i^T         TMEM dP[b] (64 cols)  dS^T = P^T (dP^T - D_q) / sqrt(d)
//   dV  += P^T dO_i         TMEM [256,384)        (A = P^T from TMEM, dO_i as MN-major B)
//   dK  += dS^T Q_i         TMEM [384,512)        (A = dS^T from TMEM, Q_i as MN-major B)
// The softmax warps write P^T / dS^T as bf16 pairs back over the S^T / dP^T
// columns they read (each warp only over its own), so they never touch
// shared memory.  Q_i / dO_i (+ their lse / D slices, bulk-copied on the same
// barrier) are a 4-deep ring and S / dP double-buffered in TMEM, so the MMAs
// of sub-tile i+1 run while the softmax warps process sub-tile i.  The same
// K-major SW128 smem tile of Q_i / dO_i serves as the K-major B of the first
// products and the MN-major B of the accumulations (64-wide d chunks at LBO =
// 8 KB, 8-row query groups at SBO = 1 KB).  A 128-query variant (M = N = 128
// everywhere, single-buffered S / dP) measured slower: 232 vs 206 us.
constexpr int kBQ2 = 64;  // query rows per backward sub-tile
constexpr int kThreadsB = 320;  // producer, MMA, 8 softmax warps (2 per TMEM lane quarter)
struct AttnBwdParams {
  CUtensorMap tmQ, tmK, tmV, tmdO;
  CUtensorMap tmdS;  // dS^T as {q, key, head, seq}, box {64, 128}, SW128 (TMA store)
  const float* V;    // [2][z][S]: -rowsum(dO * O) / sqrt(d) | -lse log2(e)
  int64_t zS;        // z * S (offset of the second vector)
  uint16_t* dqkv;    // [b, S, 3h]: dK, dV written into the k / v thirds
  uint16_t* dsT;     // [z, S(key), S(q)] bf16, for dQ = dS K
  int S, h, nh, nq;
  float scale_log2, scale;
};

constexpr int kQTile = kBQ2 * kHd * 2;                 // 16 KB
constexpr int kBOffK = 0;                              // 32 KB
constexpr int kBOffV = kTileBytes;                     // 32 KB
// Q_i / dO_i (and their vector slices) are released only when sub-tile i's
// accumulation MMAs retire, i.e. after its softmax; four stages keep the
// next sub-tiles' loads in flight across that (P^T / dS^T live in TMEM, so
// the smem they used to take holds the extra stages).
constexpr int kQStages = 4;
constexpr int kBOffQ = 2 * kTileBytes;                 // 4 x 16 KB
constexpr int kBOffdO = kBOffQ + kQStages * kQTile;    // 4 x 16 KB
constexpr int kBOffVec = kBOffdO + kQStages * kQTile;  // 4 x (-lse log2 e [64] | -D/sqrt(d) [64])
// dS^T of one sub-tile (128 keys x 64 queries bf16, the SW128 image of the
// TMA box) staged for one bulk tensor store: a thread's 64 bytes of a key
// row as direct global stores were 32 rows per warp instruction (~1 K L1
// wavefronts per sub-tile, holding the softmax warps' registers).
constexpr int kBOffDs = kBOffVec + kQStages * 512;      // 16 KB (1024-aligned)
constexpr int kBOffBar = kBOffDs + kQTile;
constexpr size_t kBSmem = size_t(kBOffBar) + 256 + 1024;
static_assert(kBSmem <= 232448, "attention backward smem budget");

__global__ void __launch_bounds__(kThreadsB, 1) attn_bwd_kernel(const __grid_constant__ AttnBwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kBOffBar);
  uint64_t* kv_full = bar + 0;
  uint64_t* qd_full = bar + 1;   // [kQStages]
  uint64_t* qd_empty = bar + 5;  // [kQStages]
  uint64_t* s_full = bar + 9;    // [2]
  uint64_t* p_full = bar + 11;   // [2]
  uint64_t* acc_done = bar + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int kt = blockIdx.z;  // key tile; small kt = most query tiles (launched first)
  const int head = blockIdx.x, seq = blockIdx.y;
  const int k0 = kt * kBK;
  const int nit = (p.S - k0) / kBQ2;
  const int z = seq * p.nh + head;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int i = 0; i < kQStages; ++i) {
      mbar_init(&qd_full[i], 1);
      mbar_init(&qd_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
    }
    mbar_init(acc_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S^T[b] = b*128, dP^T[b] = b*128 + 64, dV 256, dK 384

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * kTileBytes);
      for (int c = 0; c < 2; ++c) {
        tma_load_4d(smem + kBOffK + c * 16384, &p.tmK, kv_full, c * 64, k0, head, seq);
        tma_load_4d(smem + kBOffV + c * 16384, &p.tmV, kv_full, c * 64, k0, head, seq);
      }
      for (int it = 0; it < nit; ++it) {
        const int qs = it % kQStages;
        const uint32_t qph = (it / kQStages) & 1;
        const int q0 = k0 + it * kBQ2;
        mbar_wait(&qd_empty[qs], qph ^ 1);
        mbar_expect_tx(&qd_full[qs], 2 * kQTile + 2 * kBQ2 * 4);
        for (int c = 0; c < 2; ++c) {
          tma_load_4d(smem + kBOffQ + qs * kQTile + c * 8192, &p.tmQ, &qd_full[qs], c * 64, q0, head, seq);
          tma_load_4d(smem + kBOffdO + qs * kQTile + c * 8192, &p.tmdO, &qd_full[qs], c * 64, q0, head, seq);
        }
        float* vec = reinterpret_cast<float*>(smem + kBOffVec + qs * 512);
        bulk_load(vec, p.V + p.zS + int64_t(z) * p.S + q0, kBQ2 * 4, &qd_full[qs]);  // -lse log2 e
        bulk_load(vec + kBQ2, p.V + int64_t(z) * p.S + q0, kBQ2 * 4, &qd_full[qs]);  // -D / sqrt(d)
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = make_idesc(128, 64, 0, 0);    // K/V K-major, Q/dO K-major (N = 64 q)
      constexpr uint32_t kIdAcc = make_idesc(128, 128, 0, 1); // A = P^T / dS^T in TMEM, dO/Q MN-major
      const uint32_t sk = smem_u32(smem + kBOffK), sv = smem_u32(smem + kBOffV);
      auto accumulate = [&](int i) {
        const int b = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        const int qs = i % kQStages;
        mbar_wait(&p_full[b], ph);
        tc_fence_after();
        const uint32_t sq = smem_u32(smem + kBOffQ + qs * kQTile);
        const uint32_t sdo = smem_u32(smem + kBOffdO + qs * kQTile);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // K = 64 queries (16 per step: 8 packed columns)
          const uint32_t ac = b * 128 + (kk >> 1) * 32 + (kk & 1) * 8;
          tc_mma_ts(tmem + 256, tmem + ac, smem_desc(sdo + kk * 2048, 8192, 1024), kIdAcc,
                    (i > 0 || kk > 0) ? 1u : 0u);
          tc_mma_ts(tmem + 384, tmem + 64 + ac, smem_desc(sq + kk * 2048, 8192, 1024), kIdAcc,
                    (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(&qd_empty[qs]);
      };
      mbar_wait(kv_full, 0);
      for (int it = 0; it < nit; ++it) {
        const int b = it & 1;
        const int qs = it % kQStages;
        mbar_wait(&qd_full[qs], (it / kQStages) & 1);
        // region b (S^T / P^T, dP^T / dS^T of it-2) is free: accumulate(it-2)
        // read it and was issued earlier by this thread (in-order MMAs)
        tc_fence_after();
        const uint32_t sq = smem_u32(smem + kBOffQ + qs * kQTile);
        const uint32_t sdo = smem_u32(smem + kBOffdO + qs * kQTile);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 head dims
          const uint32_t ok = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint32_t oq = (kk >> 2) * 8192 + (kk & 3) * 32;
          tc_mma(tmem + b * 128, smem_desc(sk + ok, 16, 1024), smem_desc(sq + oq, 16, 1024), kIdS, kk > 0);
          tc_mma(tmem + b * 128 + 64, smem_desc(sv + ok, 16, 1024), smem_desc(sdo + oq, 16, 1024), kIdS,
                 kk > 0);
        }
        tc_commit(&s_full[b]);
        if (it >= 1) accumulate(it - 1);
      }
      accumulate(nit - 1);
      tc_commit(acc_done);
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;     // which 32 of the sub-tile's 64 queries
    const int row = quarter * 32 + lane;  // key k0 + row
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), dsc2 = f2_pack(p.scale, p.scale);
    for (int it = 0; it < nit; ++it) {
      const int b = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      const int q0 = k0 + it * kBQ2;
      const int qs = it % kQStages;
      mbar_wait(&qd_full[qs], (it / kQStages) & 1);  // -lse log2 e / -D / sqrt(d) slices
      mbar_wait(&s_full[b], ph);
      tc_fence_after();
      uint32_t rs[32], rd[32];
      tmem_ld32_nw(tmem + lane_off + b * 128 + half * 32, rs);
      tmem_ld32_nw(tmem + lane_off + b * 128 + 64 + half * 32, rd);
      tmem_wait_ld32(rs);
      tmem_pin32(rd);
      // P^T = 2^(S^T c - lse log2 e), dS^T = P^T (dP^T / sqrt(d) - D / sqrt(d)):
      // two queries per FFMA2/FMUL2; every 4th pair's exp2 on the FMA pipe
      const uint32_t vs = smem_u32(smem + kBOffVec + qs * 512) + half * 128;
      float nl[32], nd[32];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        lds128(vs + 16 * i, nl + 4 * i);
        lds128(vs + kBQ2 * 4 + 16 * i, nd + 4 * i);
      }
      // queries q0 + half*32 + qc with qc < -lim are masked (key > query);
      // only the diagonal sub-tiles have any, warp-uniformly known
      const int lim = q0 + half * 32 - k0 - row;
      const bool masked = __any_sync(0xffffffffu, lim < 0);
      uint32_t ptw[16], dsw[16];
      auto body = [&](auto mask_tag) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x = f2_fma(f2_pack(__uint_as_float(rs[2 * i]), __uint_as_float(rs[2 * i + 1])), sc2,
                                    f2_pack(nl[2 * i], nl[2 * i + 1]));
          uint64_t e;
          if ((i & 3) >= HZP_ATTN_BWD_POLY_FROM) {
            e = exp2_poly2(x);
          } else {
            float a0, a1;
            f2_unpack(x, a0, a1);
            e = f2_pack(exp2_fast(a0), exp2_fast(a1));
          }
          if (decltype(mask_tag)::value) {
            float e0, e1;
            f2_unpack(e, e0, e1);
            e = f2_pack(2 * i + lim < 0 ? 0.f : e0, 2 * i + 1 + lim < 0 ? 0.f : e1);
          }
          const uint64_t dsv =
              f2_mul(e, f2_fma(f2_pack(__uint_as_float(rd[2 * i]), __uint_as_float(rd[2 * i + 1])), dsc2,
                               f2_pack(nd[2 * i], nd[2 * i + 1])));
          float e0, e1, d0, d1;
          f2_unpack(e, e0, e1);
          f2_unpack(dsv, d0, d1);
          ptw[i] = bf16x2(e0, e1);
          dsw[i] = bf16x2(d0, d1);
        }
      };
      if (masked) body(std::true_type{});
      else body(std::false_type{});
      // P^T / dS^T (bf16 pairs) over the consumed S^T / dP^T columns this
      // warp read: the A operands of dV / dK
      tmem_st16_nw(tmem + lane_off + b * 128 + half * 32, ptw);
      tmem_st16_nw(tmem + lane_off + b * 128 + 64 + half * 32, dsw);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      if (p.dsT) {  // dQ = dS K as a GEMM over dS^T in HBM
        // the previous sub-tile's store has finished reading the buffer
        const bool issuer = warp == 2 && lane == 0;
        if (issuer && it > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const uint32_t rb = smem_u32(smem + kBOffDs) + row * 128;
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4) {
          const uint32_t c = (half * 4 + j4) ^ (row & 7);  // SW128: 16-byte chunk ^ row % 8
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rb + c * 16), "r"(dsw[4 * j4]),
                       "r"(dsw[4 * j4 + 1]), "r"(dsw[4 * j4 + 2]), "r"(dsw[4 * j4 + 3])
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (issuer) {
          tma_store_4d(&p.tmdS, smem + kBOffDs, q0, k0, head, seq);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (p.dsT && warp == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    mbar_wait(acc_done, 0);
    tc_fence_after();
    const int64_t rowbase = (int64_t(seq) * p.S + k0 + row) * (3 * int64_t(p.h)) + int64_t(head) * kHd;
    uint4* dkg = reinterpret_cast<uint4*>(p.dqkv + rowbase + p.h);
    uint4* dvg = reinterpret_cast<uint4*>(p.dqkv + rowbase + 2 * p.h);
#pragma unroll 1
    for (int c = half * 2; c < half * 2 + 2; ++c) {  // each half writes 64 of the 128 dims
      uint32_t r[32];
      float o[32];
      tmem_ld32(tmem + lane_off + 256 + c * 32, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r[i]);
#pragma unroll
      for (int i = 0; i < 4; ++i) dvg[c * 4 + i] = pack8f(o + 8 * i);
      tmem_ld32(tmem + lane_off + 384 + c * 32, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r[i]);
#pragma unroll
      for (int i = 0; i < 4; ++i) dkg[c * 4 + i] = pack8f(o + 8 * i);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------------------
// dQ without dS in HBM: one CTA per (128-query tile, head, sequence), walking
// the 64-key sub-tiles k < query tile end, the key-tile backward's structure
// with the roles of queries and keys swapped (rows of every TMEM accumulator
// are QUERIES):
//   S   = Q K_a^T          TMEM S[b]  (64 cols)  P  = exp2(S c - lse2_q)
//   dP  = dO V_a^T         TMEM dP[b] (64 cols)  dS = P (dP - D_q) / sqrt(d)
//   dQ += dS K_a           TMEM [256,384)        (A = dS from TMEM, K_a as MN-major B)
// P / dS are recomputed from lse (two extra 128x64x128 products per sub-tile
// instead of a [b*nh, S, S] dS^T round trip through HBM).  Q / dO stay in
// smem; K_a / V_a are a 4-deep ring; S / dP double-buffered in TMEM so the
// products of sub-tile a+1 run while the softmax warps process sub-tile a.
// Every query row's -lse log2 e and -D / sqrt(d) are two scalars of its
// thread.  Heaviest query tiles are launched first.
struct AttnDqParams {
  CUtensorMap tmQ, tmdO;  // 128-row boxes
  CUtensorMap tmK, tmV;   // 64-row boxes
  const float* V;         // [2][z][S]: -rowsum(dO * O) / sqrt(d) | -lse log2(e)
  int64_t zS;
  uint16_t* dqkv;         // dQ written into the q third
  int S, h, nh, nq;
  float scale_log2, scale;
};

constexpr int kKTile = kBQ2 * kHd * 2;                 // 16 KB: 64 keys
constexpr int kKStages = 4;
constexpr int kDOffQ = 0;                              // 32 KB
constexpr int kDOffdO = kTileBytes;                    // 32 KB
constexpr int kDOffK = 2 * kTileBytes;                 // 4 x 16 KB
constexpr int kDOffV = kDOffK + kKStages * kKTile;     // 4 x 16 KB
constexpr int kDOffBar = kDOffV + kKStages * kKTile;
constexpr size_t kDSmem = size_t(kDOffBar) + 256 + 1024;
static_assert(kDSmem <= 232448, "attention dQ smem budget");

__global__ void __launch_bounds__(kThreadsB, 1) attn_dq_kernel(const __grid_constant__ AttnDqParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kDOffBar);
  uint64_t* qd_full = bar + 0;
  uint64_t* kv_full = bar + 1;   // [kKStages]
  uint64_t* kv_empty = bar + 5;  // [kKStages]
  uint64_t* s_full = bar + 9;    // [2]
  uint64_t* p_full = bar + 11;   // [2]
  uint64_t* acc_done = bar + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int qt = p.nq - 1 - int(blockIdx.z);  // heaviest (most key tiles) first
  const int head = blockIdx.x, seq = blockIdx.y;
  const int q0 = qt * kBQ;
  const int nit = (q0 + kBQ) / kBQ2;  // 64-key sub-tiles up to the tile's last query
  const int z = seq * p.nh + head;

  if (threadIdx.x == 0) {
    mbar_init(qd_full, 1);
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
    }
    mbar_init(acc_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S[b] = b*128, dP[b] = b*128 + 64, dQ 256

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(qd_full, 2 * kTileBytes);
      for (int c = 0; c < 2; ++c) {
        tma_load_4d(smem + kDOffQ + c * 16384, &p.tmQ, qd_full, c * 64, q0, head, seq);
        tma_load_4d(smem + kDOffdO + c * 16384, &p.tmdO, qd_full, c * 64, q0, head, seq);
      }
      for (int a = 0; a < nit; ++a) {
        const int ks = a % kKStages;
        const uint32_t kph = (a / kKStages) & 1;
        mbar_wait(&kv_empty[ks], kph ^ 1);
        mbar_expect_tx(&kv_full[ks], 2 * kKTile);
        for (int c = 0; c < 2; ++c) {
          tma_load_4d(smem + kDOffK + ks * kKTile + c * 8192, &p.tmK, &kv_full[ks], c * 64, a * kBQ2, head, seq);
          tma_load_4d(smem + kDOffV + ks * kKTile + c * 8192, &p.tmV, &kv_full[ks], c * 64, a * kBQ2, head, seq);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = make_idesc(128, 64, 0, 0);    // Q / dO K-major, K_a / V_a K-major (N = 64 keys)
      constexpr uint32_t kIdAcc = make_idesc(128, 128, 0, 1); // A = dS from TMEM, K_a MN-major
      const uint32_t sq = smem_u32(smem + kDOffQ), sdo = smem_u32(smem + kDOffdO);
      auto accumulate = [&](int i) {
        const int b = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        const int ks = i % kKStages;
        mbar_wait(&p_full[b], ph);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + kDOffK + ks * kKTile);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // K = 64 keys (16 per step: 8 packed columns)
          const uint32_t ac = b * 128 + (kk >> 1) * 32 + (kk & 1) * 8;
          tc_mma_ts(tmem + 256, tmem + ac, smem_desc(sk + kk * 2048, 8192, 1024), kIdAcc,
                    (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(&kv_empty[ks]);
      };
      mbar_wait(qd_full, 0);
      for (int a = 0; a < nit; ++a) {
        const int b = a & 1;
        const int ks = a % kKStages;
        mbar_wait(&kv_full[ks], (a / kKStages) & 1);
        tc_fence_after();  // region b is free: accumulate(a-2) read it, issued earlier (in-order MMAs)
        const uint32_t sk = smem_u32(smem + kDOffK + ks * kKTile);
        const uint32_t sv = smem_u32(smem + kDOffV + ks * kKTile);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 head dims
          const uint32_t oq = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint32_t ok = (kk >> 2) * 8192 + (kk & 3) * 32;
          tc_mma(tmem + b * 128, smem_desc(sq + oq, 16, 1024), smem_desc(sk + ok, 16, 1024), kIdS, kk > 0);
          tc_mma(tmem + b * 128 + 64, smem_desc(sdo + oq, 16, 1024), smem_desc(sv + ok, 16, 1024), kIdS,
                 kk > 0);
        }
        tc_commit(&s_full[b]);
        if (a >= 1) accumulate(a - 1);
      }
      accumulate(nit - 1);
      tc_commit(acc_done);
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;     // which 32 of the sub-tile's 64 keys
    const int row = quarter * 32 + lane;  // query q0 + row
    const int q = q0 + row;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const float nl = p.V[p.zS + int64_t(z) * p.S + q];  // -lse log2 e
    const float nd = p.V[int64_t(z) * p.S + q];         // -D / sqrt(d)
    const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), dsc2 = f2_pack(p.scale, p.scale);
    const uint64_t nl2 = f2_pack(nl, nl), nd2 = f2_pack(nd, nd);
    for (int a = 0; a < nit; ++a) {
      const int b = a & 1;
      const uint32_t ph = (a >> 1) & 1;
      mbar_wait(&s_full[b], ph);
      tc_fence_after();
      uint32_t rs[32], rd[32];
      tmem_ld32_nw(tmem + lane_off + b * 128 + half * 32, rs);
      tmem_ld32_nw(tmem + lane_off + b * 128 + 64 + half * 32, rd);
      tmem_wait_ld32(rs);
      tmem_pin32(rd);
      // keys a*64 + half*32 + c with c > lim lie above the diagonal (masked);
      // only the last two sub-tiles have any, warp-uniformly known
      const int lim = q - (a * kBQ2 + half * 32);
      const bool masked = __any_sync(0xffffffffu, lim < 31);
      uint32_t dsw[16];
      auto body = [&](auto mask_tag) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint64_t x = f2_fma(f2_pack(__uint_as_float(rs[2 * i]), __uint_as_float(rs[2 * i + 1])), sc2, nl2);
          uint64_t e;
          if ((i & 3) >= HZP_ATTN_BWD_POLY_FROM) {
            e = exp2_poly2(x);
          } else {
            float a0, a1;
            f2_unpack(x, a0, a1);
            e = f2_pack(exp2_fast(a0), exp2_fast(a1));
          }
          if (decltype(mask_tag)::value) {
            float e0, e1;
            f2_unpack(e, e0, e1);
            e = f2_pack(2 * i > lim ? 0.f : e0, 2 * i + 1 > lim ? 0.f : e1);
          }
          const uint64_t dsv =
              f2_mul(e, f2_fma(f2_pack(__uint_as_float(rd[2 * i]), __uint_as_float(rd[2 * i + 1])), dsc2, nd2));
          float d0, d1;
          f2_unpack(dsv, d0, d1);
          dsw[i] = bf16x2(d0, d1);
        }
      };
      if (masked) body(std::true_type{});
      else body(std::false_type{});
      // dS (bf16 pairs) over the consumed S columns this warp read: the A of dQ += dS K_a
      tmem_st16_nw(tmem + lane_off + b * 128 + half * 32, dsw);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
    }
    mbar_wait(acc_done, 0);
    tc_fence_after();
    const int64_t rowbase = (int64_t(seq) * p.S + q) * (3 * int64_t(p.h)) + int64_t(head) * kHd;
    uint4* dqg = reinterpret_cast<uint4*>(p.dqkv + rowbase);
#pragma unroll 1
    for (int c = half * 2; c < half * 2 + 2; ++c) {  // each half writes 64 of the 128 dims
      uint32_t r[32];
      float o[32];
      tmem_ld32(tmem + lane_off + 256 + c * 32, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(r[i]);
#pragma unroll
      for (int i = 0; i < 4; ++i) dqg[c * 4 + i] = pack8f(o + 8 * i);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}


}  // namespace

void attention_dq(const uint16_t* qkv, const uint16_t* dsT, uint16_t* dqkv, int b, int nh, int S, int h,
                  cudaStream_t stream) {
  const int64_t h3 = 3 * int64_t(h), SS = int64_t(S) * S;
  // dQ[q, d] = sum_key dS[q, key] K[key, d]: A = dS stored as dSᵀ [key][q]
  // (MN-major), B = K [key][d] (MN-major), K range [0, q tile end).  The
  // product is HBM-bound on dSᵀ (b·nh·S² bf16 read once); the transposed
  // formulation (N = 256 query tiles) measured slower (77 vs 67 us).
  GemmShape sh{S, kHd, S, S, int(h3), 1, 1};
  sh.nh = nh;
  sh.nb = b;
  sh.a_sh = SS;
  sh.a_sb = SS * nh;
  sh.b_sh = kHd;
  sh.b_sb = S * h3;
  sh.c_sh = kHd;
  sh.c_sb = S * h3;
  sh.causal = 2;
  Epilogue e;
  e.ldc = int(h3);
  gemm_tc_bf16(dsT, qkv + h, dqkv, sh, e, stream);
}

// qkv [b, S, 3h] (q | k | v, heads contiguous in each), O [b, S, h].
void attention_fwd_tc(const uint16_t* qkv, uint16_t* O, uint16_t* P, float* lse, int b, int nh,
                      int S, int h, cudaStream_t stream) {
  if (h != nh * kHd || S % kBQ) throw std::invalid_argument("fused attention needs head dim 128, S % 128 == 0");
  static bool attr = false;
  if (!attr) {
    HZP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem)));
    attr = true;
  }
  AttnParams p;
  const int64_t h3 = 3 * int64_t(h);
  p.tmQ = make_tma_map_bf16(qkv, kHd, S, h3, 128, nh, b, kHd, int64_t(S) * h3);
  p.tmK = make_tma_map_bf16(qkv + h, kHd, S, h3, 128, nh, b, kHd, int64_t(S) * h3);
  p.tmV = make_tma_map_bf16(qkv + 2 * h, kHd, S, h3, 64, nh, b, kHd, int64_t(S) * h3);
  if (!make_map_mn5(qkv + 2 * h, kHd, S, h3, nh, b, kHd, int64_t(S) * h3, &p.tmV5))
    throw CudaError("attention: 5-D V tensor map rejected");
  p.O = O;
  p.P = P;
  p.lse = lse;
  p.S = S;
  p.h = h;
  p.nh = nh;
  p.nq = S / kBQ;
  p.scale_log2 = 1.4426950408889634f / std::sqrt(float(kHd));
  if (P == nullptr && (S / kBQ) % 2 == 0) {  // two query tiles per CTA
    static bool attr2 = false;
    if (!attr2) {
      HZP_CUDA(cudaFuncSetAttribute(attn_fwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(k2Smem)));
      attr2 = true;
    }
    dim3 grid(nh, b, S / kBQ / 2);
    attn_fwd2_kernel<<<grid, kThreads2, k2Smem, stream>>>(p);
    HZP_LAUNCH_CHECK();
    return;
  }
  dim3 grid(nh, b, S / kBQ);
  attn_fwd_kernel<<<grid, kThreads, kSmem, stream>>>(p);
  HZP_LAUNCH_CHECK();
}

void attention_dq_tc(const uint16_t* qkv, const uint16_t* dO, const float* D, uint16_t* dqkv, int b, int nh,
                     int S, int h, cudaStream_t stream) {
  if (h != nh * kHd || S % kBQ) throw std::invalid_argument("fused attention needs head dim 128, S % 128 == 0");
  static bool attr = false;
  if (!attr) {
    HZP_CUDA(cudaFuncSetAttribute(attn_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDSmem)));
    attr = true;
  }
  AttnDqParams p;
  const int64_t h3 = 3 * int64_t(h);
  p.tmQ = make_tma_map_bf16(qkv, kHd, S, h3, 128, nh, b, kHd, int64_t(S) * h3);
  p.tmdO = make_tma_map_bf16(dO, kHd, S, h, 128, nh, b, kHd, int64_t(S) * h);
  p.tmK = make_tma_map_bf16(qkv + h, kHd, S, h3, kBQ2, nh, b, kHd, int64_t(S) * h3);
  p.tmV = make_tma_map_bf16(qkv + 2 * h, kHd, S, h3, kBQ2, nh, b, kHd, int64_t(S) * h3);
  p.V = D;
  p.zS = int64_t(b) * nh * S;
  p.dqkv = dqkv;
  p.S = S;
  p.h = h;
  p.nh = nh;
  p.nq = S / kBQ;
  p.scale = 1.f / std::sqrt(float(kHd));
  p.scale_log2 = 1.4426950408889634f * p.scale;
  dim3 grid(nh, b, S / kBQ);
  attn_dq_kernel<<<grid, kThreadsB, kDSmem, stream>>>(p);
  HZP_LAUNCH_CHECK();
}

void attention_bwd_tc(const uint16_t* qkv, const uint16_t* dO, const float* lse, const float* D,
                      uint16_t* dqkv, uint16_t* dsT, int b, int nh, int S, int h, cudaStream_t stream) {
  if (h != nh * kHd || S % kBQ) throw std::invalid_argument("fused attention needs head dim 128, S % 128 == 0");
  static bool attr = false;
  if (!attr) {
    HZP_CUDA(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBSmem)));
    attr = true;
  }
  AttnBwdParams p;
  const int64_t h3 = 3 * int64_t(h);
  p.tmQ = make_tma_map_bf16(qkv, kHd, S, h3, kBQ2, nh, b, kHd, int64_t(S) * h3);
  p.tmK = make_tma_map_bf16(qkv + h, kHd, S, h3, 128, nh, b, kHd, int64_t(S) * h3);
  p.tmV = make_tma_map_bf16(qkv + 2 * h, kHd, S, h3, 128, nh, b, kHd, int64_t(S) * h3);
  p.tmdO = make_tma_map_bf16(dO, kHd, S, h, kBQ2, nh, b, kHd, int64_t(S) * h);
  (void)lse;  // consumed through D (attn_rowdot's -lse log2 e vector)
  p.V = D;
  p.zS = int64_t(b) * nh * S;
  p.dqkv = dqkv;
  p.dsT = dsT;
  if (dsT) p.tmdS = make_tma_map_bf16(dsT, S, S, S, 128, nh, b, int64_t(S) * S, int64_t(S) * S * nh);
  p.S = S;
  p.h = h;
  p.nh = nh;
  p.nq = S / kBQ;
  p.scale = 1.f / std::sqrt(float(kHd));
  p.scale_log2 = 1.4426950408889634f * p.scale;
  dim3 grid(nh, b, S / kBK);
  attn_bwd_kernel<<<grid, kThreadsB, kBSmem, stream>>>(p);
  HZP_LAUNCH_CHECK();
}

}  // namespace hzp
