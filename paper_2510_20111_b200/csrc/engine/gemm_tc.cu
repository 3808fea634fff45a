// tcgen05 GEMM for sm_100a: C = epilogue(A · Bᵀ), bf16 operands, fp32
// accumulation in TMEM.
//
// Structure (persistent, one CTA per SM, 10 warps, warp-specialised):
//   warp 0   : TMA producer — one lane streams A/B k-blocks (128B swizzle)
//              into a STAGES-deep shared-memory ring (mbarrier full/empty).
//   warp 1   : TMEM allocator + MMA issuer — one lane issues tcgen05.mma.
//              Products with >= 2 M tiles run on CTA pairs (cluster of 2,
//              cta_group::2, M = 256 per MMA, each CTA staging its A rows and
//              half of B); the rest on single CTAs (cta_group::1, M = 128).
//   warps 2-9: epilogue — two warps per TMEM lane quarter, alternating 32-column
//              chunks: tcgen05.ld, bias / activation / residual / accumulate,
//              swizzled smem staging, TMA bulk tensor store (or reduce-add).
// Two TMEM accumulators (2 x BN fp32 columns) let the epilogue of tile i
// overlap the MMAs of tile i+1.
//
// Operands may be K-major or MN-major in global memory; MN-major tiles are
// loaded as 64-wide boxes and described to the tensor core with the MN-major
// SW128 canonical layout (LBO = 64-wide block stride, SBO = 8-row K-group
// stride), so dgrad / wgrad never materialise a transpose.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "engine/gemm.cuh"
#include "engine/tc_ptx.cuh"

namespace hzp {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle row of bf16
constexpr int kEpiWarps = 8;  // two per TMEM lane quarter, each owning half the columns
constexpr int kThreadsTC = 64 + 32 * kEpiWarps;
// 4 KB TMA-store staging buffers per epilogue warp.  One buffer (and a
// mainloop stage more) measured 0.5-5% faster than double-buffered staging.
#ifndef HZP_STAGE_BUFS
#define HZP_STAGE_BUFS 1
#endif
constexpr int kStageBufs = HZP_STAGE_BUFS;

int g_sm_budget = kNumSMs;

using namespace tc;

struct TcParams {
  CUtensorMap tmC;    // output (STORE != 0)
  CUtensorMap tmAux;  // GELU pre-activation output (STORE == 1, act == Gelu)
  CUtensorMap tmSide; // side input (SIDE): aux for the *-grad epilogues, else resid
  CUtensorMap tmBh;   // CL == 2, K-major B: half-height boxes (each CTA loads one half)
  CUtensorMap tmBq;   // CL == 2, K-major B: quarter-height boxes (split tail units)
  CUtensorMap tmA5, tmB5;  // MN-major operands as 5-D maps, box = two 64-wide MN chunks
  int a5, b5;              // the 5-D maps are valid (MN extent % 64 == 0)
  int M, N, K;
  int tiles_m, tiles_n, tiles_mn, num_tiles;
  int pairs_m;        // CL == 2: ceil(tiles_m / 2); tile index space = pairs
  int n_fast;         // raster: 1 = N tiles vary fastest (A streamed once, B kept in L2)
  int nfull;          // CL == 2: units [0, nfull) are 256 x BN; the rest are the
                      // last units split into two 256 x BN/2 halves (tail wave)
  int nh, nz, causal;
  int64_t c_sh, c_sb;
  Epilogue e;
  void* C;
};

// Tile t -> (m0, n0, zh, zb); z slowest so concurrent CTAs share operands.
struct TileCoord {
  int m0, n0, zh, zb;
  int w;  // tile width (BN, or BN/2 for a split tail unit)
};
__device__ __forceinline__ TileCoord tile_coord(const TcParams& p, int t, int bn) {
  const int z = t / p.tiles_mn;
  const int r = t - z * p.tiles_mn;
  if (p.n_fast) return {(r / p.tiles_n) * BM, (r % p.tiles_n) * bn, z % p.nh, z / p.nh, bn};
  return {(r % p.tiles_m) * BM, (r / p.tiles_m) * bn, z % p.nh, z / p.nh, bn};
}
// CTA pair along M: unit t is a 256 x bn tile; CTA `rank` owns M rows
// [m0 + 128 rank, +128) (possibly past M: zero fill) and B half `rank`.
// Causal (mode 2) products walk the M pairs heaviest-first (LPT order).
// Units past nfull are halves (alternating left / right) of the last units.
__device__ __forceinline__ TileCoord pair_coord(const TcParams& p, int t, int bn, int rank) {
  int half = -1;
  if (t >= p.nfull) {
    const int h = t - p.nfull;
    t = p.nfull + (h >> 1);
    half = h & 1;
  }
  TileCoord c;
  if (p.causal) {
    const int per_m = p.tiles_n * p.nz;
    const int mp = p.pairs_m - 1 - t / per_m;
    const int r = t - (t / per_m) * per_m;
    const int z = r / p.tiles_n;
    c = {(2 * mp + rank) * BM, (r - z * p.tiles_n) * bn, z % p.nh, z / p.nh, bn};
  } else {
    const int per_z = p.pairs_m * p.tiles_n;
    const int z = t / per_z;
    const int r = t - z * per_z;
    if (p.n_fast)
      c = {(2 * (r / p.tiles_n) + rank) * BM, (r % p.tiles_n) * bn, z % p.nh, z / p.nh, bn};
    else
      c = {(2 * (r % p.pairs_m) + rank) * BM, (r / p.pairs_m) * bn, z % p.nh, z / p.nh, bn};
  }
  if (half >= 0) {
    c.n0 += half * (bn / 2);
    c.w = bn / 2;
  }
  return c;
}
// K-block range of a tile under the causal mode (see GemmShape::causal).  A
// CTA pair shares one range: the union over its 256 rows (mode 2 only; the
// lower CTA then reads A past its diagonal, which the caller keeps zero).
template <int CL>
__device__ __forceinline__ void kb_range(const TcParams& p, int m0, int n0, int& kb0, int& kb1) {
  const int nkb = (p.K + BK - 1) / BK;
  const int span = CL == 2 ? 2 * BM : BM;
  if (CL == 2) m0 &= ~(2 * BM - 1);  // pair base (pairs start at multiples of 256)
  kb0 = 0;
  kb1 = nkb;
  if (p.causal == 1 && n0 >= m0 + span) kb1 = 0;  // fully masked tile: no work
  else if (p.causal == 2) kb1 = min(nkb, (m0 + span + BK - 1) / BK);
  else if (p.causal == 3) kb0 = min(nkb, m0 / BK);
}

template <int BN, int A_MN, int B_MN, int STAGES, int STORE, int SIDE, int CL>
__global__ void __launch_bounds__(kThreadsTC, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ TcParams p) {
  constexpr uint32_t A_BYTES = BM * BK * 2;
  // CL == 2 (CTA pair, cta_group::2): each CTA holds its own 128 A rows and
  // one half of the BN-wide B tile; the leader's MMA (M = 256) reads both.
  constexpr uint32_t B_BYTES = (CL == 2 ? BN / 2 : BN) * BK * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  constexpr uint32_t IDESC = make_idesc(BM * CL, BN, A_MN, B_MN);
  constexpr uint32_t IDESC_H = make_idesc(BM * CL, BN / 2, A_MN, B_MN);  // split tail units

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);  // released by the (leader's) MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * CL);  // CL == 2: both CTAs' epilogues, on the leader
    }
    if (SIDE)
      for (int i = 0; i < 2 * kEpiWarps; ++i)
        mbar_init(reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + 512) + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (CL == 2) cluster_sync_all();  // peers' barriers initialised before any cross-CTA signal
  if (warp == 1) {
    if (CL == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_base_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_base_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  // CL == 2: both CTAs of a cluster walk the same pair sequence
  const int rank = CL == 2 ? int(cluster_rank()) : 0;
  const int unit0 = CL == 2 ? int(blockIdx.x) / 2 : int(blockIdx.x);
  const int ustep = CL == 2 ? int(gridDim.x) / 2 : int(gridDim.x);
  const int nunits = CL == 2 ? 2 * p.pairs_m * p.tiles_n * p.nz - p.nfull : p.num_tiles;
  if (CL == 2) cluster_sync_all();  // both TMEM allocations done

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = unit0; t < nunits; t += ustep) {
        const TileCoord tc = CL == 2 ? pair_coord(p, t, BN, rank) : tile_coord(p, t, BN);
        int kb0, kb1;
        kb_range<CL>(p, tc.m0, tc.n0, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const int k0 = kb * BK;
          if (CL == 2) {  // both CTAs' loads complete on the leader's full barrier
            const uint32_t fb = mapa_shared(smem_u32(&full[stage]), 0);
            const bool split = tc.w != BN;  // tail half-unit: each CTA stages a quarter of B
            if (rank == 0)
              mbar_expect_tx(&full[stage], 2 * (A_BYTES + uint32_t(tc.w / 2) * BK * 2));
            if (A_MN) {
              if (p.a5) {
                tma_load_5d_pair(sa, &p.tmA5, fb, 0, k0, tc.m0 / 64, tc.zh, tc.zb);
              } else {
#pragma unroll
                for (int j = 0; j < BM / 64; ++j)
                  tma_load_4d_pair(sa + j * (BK * 128), &tmA, fb, tc.m0 + 64 * j, k0, tc.zh, tc.zb);
              }
            } else {
              tma_load_4d_pair(sa, &tmA, fb, k0, tc.m0, tc.zh, tc.zb);
            }
            if (B_MN) {
              if (p.b5 && !split) {
                tma_load_5d_pair(sb, &p.tmB5, fb, 0, k0, (tc.n0 + rank * (tc.w / 2)) / 64, tc.zh, tc.zb);
              } else {
                for (int j = 0; j < tc.w / 128; ++j)
                  tma_load_4d_pair(sb + j * (BK * 128), &tmB, fb, tc.n0 + rank * (tc.w / 2) + 64 * j, k0, tc.zh,
                                   tc.zb);
              }
            } else {
              tma_load_4d_pair(sb, split ? &p.tmBq : &p.tmBh, fb, k0, tc.n0 + rank * (tc.w / 2), tc.zh, tc.zb);
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          if (A_MN) {
            if (p.a5) {
              tma_load_5d(sa, &p.tmA5, &full[stage], 0, k0, tc.m0 / 64, tc.zh, tc.zb);
            } else {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_4d(sa + j * (BK * 128), &tmA, &full[stage], tc.m0 + 64 * j, k0, tc.zh, tc.zb);
            }
          } else {
            tma_load_4d(sa, &tmA, &full[stage], k0, tc.m0, tc.zh, tc.zb);
          }
          if (B_MN) {
            if (p.b5) {
#pragma unroll
              for (int j = 0; j < BN / 128; ++j)
                tma_load_5d(sb + j * (2 * BK * 128), &p.tmB5, &full[stage], 0, k0, tc.n0 / 64 + 2 * j, tc.zh,
                            tc.zb);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_4d(sb + j * (BK * 128), &tmB, &full[stage], tc.n0 + 64 * j, k0, tc.zh, tc.zb);
            }
          } else {
            tma_load_4d(sb, &tmB, &full[stage], k0, tc.n0, tc.zh, tc.zb);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // CL == 2: the leader issues the pair's MMAs
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = unit0; t < nunits; t += ustep) {
        const TileCoord tc = CL == 2 ? pair_coord(p, t, BN, rank) : tile_coord(p, t, BN);
        int kb0, kb1;
        kb_range<CL>(p, tc.m0, tc.n0, kb0, kb1);
        if (kb1 <= kb0) continue;  // skipped tile: the epilogue skips it too
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: advance 32 bytes inside the swizzled row; MN-major:
            // advance 16 K-rows = 2 eight-row groups = 2048 bytes.
            const uint64_t ad = A_MN ? smem_desc(sa + k * 2048, BK * 128, 1024)
                                     : smem_desc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc(sb + k * 2048, BK * 128, 1024)
                                     : smem_desc(sb + k * 32, 16, 1024);
            if (CL == 2) tc_mma_pair(d_tmem, ad, bd, tc.w == BN ? IDESC : IDESC_H, (kb > kb0 || k) ? 1u : 0u);
            else tc_mma(d_tmem, ad, bd, IDESC, (kb > kb0 || k) ? 1u : 0u);
          }
          // frees this smem stage (in both CTAs of a pair) when the MMAs retire
          if (CL == 2) tc_commit_pair_mc(&empty[stage], 0x3);
          else tc_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        // accumulator ready for the epilogue(s)
        if (CL == 2) tc_commit_pair_mc(&tfull[acc], 0x3);
        else tc_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---- epilogue warps 2..5: TMEM lane quarter = warp % 4 ----
    // Thread `lane` of warp quarter q owns accumulator row q*32 + lane.  Each
    // 32-column chunk is computed in registers; with STORE != 0 it is staged
    // in the warp's 128B/64B-swizzled smem buffer and written by a single
    // TMA bulk tensor store (reduce-add for fp32 accumulation), so global
    // writes are full-line and coalesced whatever the row pitch.
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;  // 0 | 1: which interleaved 32-column chunks
    const Epilogue& e = p.e;
    // kStageBufs 4 KB staging buffers per warp (chunk parity when 2)
    uint8_t* stage_base = smem + STAGES * STAGE_BYTES + 1024 + (warp - 2) * (kStageBufs * 4096);
    // SIDE: the side input (P / pre-activation / residual) of each 32x32
    // chunk is TMA-loaded into one of two 2 KB SW64 buffers per warp, the next
    // chunk's load issued before the current one is consumed.
    uint8_t* side_base = smem + STAGES * STAGE_BYTES + 1024 + kEpiWarps * (kStageBufs * 4096) + (warp - 2) * 4096;
    uint64_t* side_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + 512) + (warp - 2) * 2;
    uint32_t side_phase = 0;  // bit b = parity of buffer b's next completion
    int side_buf = 0;
    int acc = 0, nchunk = 0;
    uint32_t acc_phase = 0;
    for (int t = unit0; t < nunits; t += ustep) {
      const TileCoord tc = CL == 2 ? pair_coord(p, t, BN, rank) : tile_coord(p, t, BN);
      int kb0, kb1;
      kb_range<CL>(p, tc.m0, tc.n0, kb0, kb1);
      if (kb1 <= kb0) continue;
      const int m0 = tc.m0, n0 = tc.n0;
      const int64_t zoff = int64_t(tc.zh) * p.c_sh + int64_t(tc.zb) * p.c_sb;
      if (SIDE && lane == 0 && n0 + half * 32 < p.N) {  // first chunk's side input
        mbar_expect_tx(&side_bar[side_buf], 2048);
        tma_load_4d(side_base + side_buf * 2048, &p.tmSide, &side_bar[side_buf], n0 + half * 32,
                    m0 + quarter * 32, tc.zh, tc.zb);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int m = m0 + quarter * 32 + lane;
      const bool row_ok = m < p.M;
      float rv = 0.f;
      if (e.act == kActSoftmaxGrad && row_ok)
        rv = e.rowvec[int64_t(tc.zh) * e.rv_sh + int64_t(tc.zb) * e.rv_sb + m];
      const int nch = tc.w / 32;
#pragma unroll 1
      for (int c = half; c < nch; c += 2) {
        uint32_t r[32];
        tmem_ld32(tmem_base + (uint32_t(quarter * 32) << 16) + acc * BN + c * 32, r);
        if (c + 2 >= nch) {  // last read of this accumulator: hand it back to the MMA warp now
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CL == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
            else mbar_arrive(&tempty[acc]);
          }
        }
        const int nb = n0 + c * 32;
        if (nb >= p.N) continue;                 // warp-uniform
        if (STORE == 0 && !row_ok) continue;
        float sd[32];  // side input row (SIDE)
        if (SIDE) {
          const int nx = nb + 64;  // this warp's next chunk
          if (lane == 0 && c + 2 < nch && nx < p.N) {
            mbar_expect_tx(&side_bar[side_buf ^ 1], 2048);
            tma_load_4d(side_base + (side_buf ^ 1) * 2048, &p.tmSide, &side_bar[side_buf ^ 1], nx,
                        m0 + quarter * 32, tc.zh, tc.zb);
          }
          mbar_wait(&side_bar[side_buf], (side_phase >> side_buf) & 1);
          side_phase ^= 1u << side_buf;
          const uint8_t* sb = side_base + side_buf * 2048 + lane * 64;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            unpack8f(*reinterpret_cast<const uint4*>(sb + ((q ^ ((lane >> 1) & 3)) * 16)), sd + 8 * q);
          side_buf ^= 1;
        }
        float v[32];
        if (e.alpha != 1.f) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * e.alpha;
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        }
        const bool full_chunk = nb + 32 <= p.N;
        if (row_ok) {
          if (e.bias_any) {  // same 32 bias values for every lane: 4 broadcast 16-byte loads
            const uint16_t* bp = static_cast<const uint16_t*>(e.bias_any) + int64_t(tc.zh) * e.bias_sh + nb;
            if (full_chunk && (reinterpret_cast<uintptr_t>(bp) & 15) == 0) {
              float bb[32];
#pragma unroll
              for (int q = 0; q < 4; ++q) unpack8f(__ldg(reinterpret_cast<const uint4*>(bp) + q), bb + 8 * q);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += bb[j];
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < p.N) v[j] += bf16_bits_to_f32(bp[j]);
            }
          } else if (e.bias) {
            if (full_chunk && (reinterpret_cast<uintptr_t>(e.bias + nb) & 15) == 0) {
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(e.bias + nb) + q);
                v[4 * q] += b4.x;
                v[4 * q + 1] += b4.y;
                v[4 * q + 2] += b4.z;
                v[4 * q + 3] += b4.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < p.N) v[j] += e.bias[nb + j];
            }
          }
        }
        float pre[32];  // GELU pre-activation (aux output)
        if (e.act == kActTanh) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = tanhf(v[j]);
        } else if (e.act == kActGelu) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            pre[j] = v[j];
            v[j] = gelu_tanh(v[j]);
          }
          if (STORE == 0) {
            uint16_t* aux = static_cast<uint16_t*>(e.aux) + zoff + int64_t(m) * e.ldaux + nb;
            if (full_chunk) {
#pragma unroll
              for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(aux)[q] = pack8f(pre + 8 * q);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < p.N) aux[j] = f32_to_bf16_bits(pre[j]);
            }
          }
        } else if (e.act == kActTanhGrad || e.act == kActGeluGrad || e.act == kActSoftmaxGrad) {
          float a[32];
          if (SIDE) {
#pragma unroll
            for (int j = 0; j < 32; ++j) a[j] = sd[j];
          } else if (row_ok) {
            const int64_t ab = zoff + int64_t(m) * e.ldaux + nb;
            if (e.aux_bf16 && full_chunk) {
              const uint4* ap = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(e.aux) + ab);
#pragma unroll
              for (int q = 0; q < 4; ++q) unpack8f(ap[q], a + 8 * q);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                a[j] = (full_chunk || nb + j < p.N)
                           ? (e.aux_bf16 ? bf16_bits_to_f32(static_cast<const uint16_t*>(e.aux)[ab + j])
                                         : static_cast<const float*>(e.aux)[ab + j])
                           : 0.f;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) a[j] = 0.f;
          }
          if (e.act == kActTanhGrad) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= 1.f - a[j] * a[j];
          } else if (e.act == kActGeluGrad) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= gelu_tanh_grad(a[j]);
          } else {
            // dS = P * (alpha*dP - alpha*D), alpha already applied to acc
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = a[j] * (v[j] - e.alpha * rv);
          }
        }
        if (SIDE && e.resid) {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] += sd[j];
        } else if (e.resid && row_ok) {
          const uint16_t* rp = static_cast<const uint16_t*>(e.resid) + zoff + int64_t(m) * e.ldres + nb;
          if (full_chunk) {
            float rr[32];
#pragma unroll
            for (int q = 0; q < 4; ++q) unpack8f(reinterpret_cast<const uint4*>(rp)[q], rr + 8 * q);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += rr[j];
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nb + j < p.N) v[j] += bf16_bits_to_f32(rp[j]);
          }
        }
        if (STORE != 0) {
          // ---- stage in smem (swizzled) and TMA-store the 32x32 chunk ----
          // buffer nchunk & 1: the store issued two chunks ago must have
          // finished reading it
          uint8_t* buf = stage_base + (kStageBufs == 2 ? (nchunk & 1) * 4096 : 0);
          if (lane == 0) {
            if (kStageBufs == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          __syncwarp();
          if (STORE == 1) {  // bf16: 32 rows x 64 B, SWIZZLE_64B; GELU aux in the 2nd half
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int pc = q ^ ((lane >> 1) & 3);
              *reinterpret_cast<uint4*>(buf + lane * 64 + pc * 16) = pack8f(v + 8 * q);
              if (e.act == kActGelu)
                *reinterpret_cast<uint4*>(buf + 2048 + lane * 64 + pc * 16) = pack8f(pre + 8 * q);
            }
          } else {  // fp32: 32 rows x 128 B, SWIZZLE_128B
            if (e.mode == kEpiAssign0) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(0.f, v[j]);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int pc = q ^ (lane & 7);
              *reinterpret_cast<float4*>(buf + lane * 128 + pc * 16) =
                  make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            const int mr = m0 + quarter * 32;
            if (STORE == 2 && e.mode == kEpiAccum)
              tma_reduce_add_4d(&p.tmC, buf, nb, mr, tc.zh, tc.zb);
            else
              tma_store_4d(&p.tmC, buf, nb, mr, tc.zh, tc.zb);
            if (STORE == 1 && e.act == kActGelu) tma_store_4d(&p.tmAux, buf + 2048, nb, mr, tc.zh, tc.zb);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++nchunk;
          continue;
        }
        // ---- direct stores (fallback for TMA-incompatible C layouts) ----
        const int64_t ci = zoff + int64_t(m) * e.ldc + nb;
        if (e.out_bf16) {
          uint16_t* out = static_cast<uint16_t*>(p.C) + ci;
          if (full_chunk && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) reinterpret_cast<uint4*>(out)[q] = pack8f(v + 8 * q);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (nb + j < p.N) out[j] = f32_to_bf16_bits(v[j]);
          }
        } else {
          float* out = static_cast<float*>(p.C) + ci;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (nb + j >= p.N) continue;
            float w = v[j];
            if (e.mode == kEpiAccum) w += out[j];
            else if (e.mode == kEpiAssign0) w = __fadd_rn(0.f, w);
            out[j] = w;
          }
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (STORE != 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (CL == 2) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    if (CL == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ---- SIMT fallback for shapes TMA cannot describe (unaligned leading dims)
__global__ void gemm_bf16_simt_kernel(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B,
                                      void* C, GemmShape s, Epilogue e) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int m = blockIdx.y;
  if (n >= s.N || m >= s.M) return;
  float acc = 0.f;
  for (int k = 0; k < s.K; ++k) {
    const float a = bf16_bits_to_f32(s.a_mn ? A[int64_t(k) * s.lda + m] : A[int64_t(m) * s.lda + k]);
    const float b = bf16_bits_to_f32(s.b_mn ? B[int64_t(k) * s.ldb + n] : B[int64_t(n) * s.ldb + k]);
    acc += a * b;
  }
  if (e.bias_any) acc += bf16_bits_to_f32(static_cast<const uint16_t*>(e.bias_any)[n]);
  else if (e.bias) acc += e.bias[n];
  acc *= e.alpha;
  float v = acc;
  if (e.act == kActTanh) v = tanhf(acc);
  else if (e.act == kActGelu) {
    static_cast<uint16_t*>(e.aux)[int64_t(m) * e.ldaux + n] = f32_to_bf16_bits(acc);
    v = gelu_tanh(acc);
  } else if (e.act == kActTanhGrad || e.act == kActGeluGrad) {
    const int64_t ai = int64_t(m) * e.ldaux + n;
    const float a = e.aux_bf16 ? bf16_bits_to_f32(static_cast<const uint16_t*>(e.aux)[ai])
                               : static_cast<const float*>(e.aux)[ai];
    v = acc * (e.act == kActTanhGrad ? (1.f - a * a) : gelu_tanh_grad(a));
  }
  const int64_t ci = int64_t(m) * e.ldc + n;
  if (e.out_bf16) {
    static_cast<uint16_t*>(C)[ci] = f32_to_bf16_bits(v);
  } else {
    float* o = static_cast<float*>(C) + ci;
    *o = e.mode == kEpiAccum ? *o + v : (e.mode == kEpiAssign0 ? __fadd_rn(0.f, v) : v);
  }
}

// ---- host side --------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map(const void* base, int64_t inner, int64_t outer, int64_t ld, int box_outer,
                     int nh, int nb, int64_t sh, int64_t sb) {
  return make_tma_map_bf16(base, inner, outer, ld, box_outer, nh, nb, sh, sb);
}

// Output map for the TMA-store epilogue: {N, M, nh, nb}, box {32, 32, 1, 1};
// bf16 rows of 64 B use SWIZZLE_64B, fp32 rows of 128 B SWIZZLE_128B.
CUtensorMap make_out_map(const void* base, bool f32, int64_t N, int64_t M, int64_t ld, int nh, int nb,
                         int64_t sh, int64_t sb) {
  CUtensorMap m;
  const int es = f32 ? 4 : 2;
  if (nh <= 1) sh = ld * M;
  if (nb <= 1) sb = sh * nh;
  cuuint64_t dims[4] = {cuuint64_t(N), cuuint64_t(M), cuuint64_t(nh), cuuint64_t(nb)};
  cuuint64_t strides[3] = {cuuint64_t(ld) * es, cuuint64_t(sh) * es, cuuint64_t(sb) * es};
  cuuint32_t box[4] = {32, 32, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = get_encode()(
      &m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base),
      dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (out) failed: " + std::to_string(int(r)));
  return m;
}

bool aligned16(const void* p, int64_t ld, int64_t sh, int64_t sb, int es) {
  return (reinterpret_cast<uintptr_t>(p) % 16) == 0 && (ld * es) % 16 == 0 && (sh * es) % 16 == 0 &&
         (sb * es) % 16 == 0;
}

// Tail-wave balancing for the persistent CTA-pair kernel: units are dealt
// round-robin to `clusters`; converting the last x units into two half-width
// units each (2x BN/2 work items) shortens the final wave.  Returns the
// number of full units (units - x) minimising the most-loaded cluster's work
// (in half-unit weights, +1 per extra item for its pipeline fill), keeping
// all units whole unless that saves >= 4%.
int split_tail(int units, int clusters, bool allowed) {
  if (!allowed || clusters <= 1 || units % clusters == 0) return units;
  auto makespan = [&](int nfull) {
    std::vector<int> load(clusters, 0);
    const int items = nfull + 2 * (units - nfull);
    for (int i = 0; i < items; ++i) load[i % clusters] += (i < nfull ? 8 : 4) + 1;
    return *std::max_element(load.begin(), load.end());
  };
  int best_n = units, best = makespan(units);
  const int waves = (units + clusters - 1) / clusters;
  for (int w = 0; w < waves; ++w) {  // halves start on a wave boundary
    const int nfull = w * clusters;
    const int m = makespan(nfull);
    if (m < best) { best = m; best_n = nfull; }
  }
  return best * 100 <= makespan(units) * 96 ? best_n : units;
}

template <int BN, int A_MN, int B_MN, int STORE, int SIDE, int CL>
void launch_tc(const void* A, const void* B, void* C, const GemmShape& s, const Epilogue& e,
               cudaStream_t stream) {
  // as many mainloop stages as fit beside the epilogue staging (a side-input
  // epilogue doubles that); a CTA pair holds half a B tile per stage
  constexpr size_t STAGE_B = size_t(BM * BK * 2) + size_t(CL == 2 ? BN / 2 : BN) * BK * 2;
  constexpr size_t FIXED = 1024 + 1024 + size_t(kEpiWarps) * (kStageBufs * 4096 + (SIDE ? 4096 : 0));
  constexpr int STAGES = int((232448 - FIXED) / STAGE_B) > 8 ? 8 : int((232448 - FIXED) / STAGE_B);
  constexpr size_t SMEM = size_t(STAGES) * STAGE_B + FIXED;
  static_assert(SMEM <= 232448, "smem budget");
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, STAGES, STORE, SIDE, CL>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    HZP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM)));
    attr_set = true;
  }
  const CUtensorMap ta = A_MN ? make_map(A, s.M, s.K, s.lda, BK, s.nh, s.nb, s.a_sh, s.a_sb)
                              : make_map(A, s.K, s.M, s.lda, BM, s.nh, s.nb, s.a_sh, s.a_sb);
  const CUtensorMap tb = B_MN ? make_map(B, s.N, s.K, s.ldb, BK, s.nh, s.nb, s.b_sh, s.b_sb)
                              : make_map(B, s.K, s.N, s.ldb, BN, s.nh, s.nb, s.b_sh, s.b_sb);
  TcParams p;
  p.a5 = A_MN && make_map_mn5(A, s.M, s.K, s.lda, s.nh, s.nb, s.a_sh, s.a_sb, &p.tmA5);
  p.b5 = B_MN && make_map_mn5(B, s.N, s.K, s.ldb, s.nh, s.nb, s.b_sh, s.b_sb, &p.tmB5);
  if (STORE != 0) {
    p.tmC = make_out_map(C, STORE == 2, s.N, s.M, e.ldc, s.nh, s.nb, s.c_sh, s.c_sb);
    if (STORE == 1 && e.act == kActGelu)
      p.tmAux = make_out_map(e.aux, false, s.N, s.M, e.ldaux, s.nh, s.nb, s.c_sh, s.c_sb);
  }
  if (SIDE) {
    if (e.resid) p.tmSide = make_out_map(e.resid, false, s.N, s.M, e.ldres, s.nh, s.nb, s.c_sh, s.c_sb);
    else p.tmSide = make_out_map(e.aux, false, s.N, s.M, e.ldaux, s.nh, s.nb, s.c_sh, s.c_sb);
  }
  p.M = s.M;
  p.N = s.N;
  p.K = s.K;
  p.tiles_m = (s.M + BM - 1) / BM;
  p.tiles_n = (s.N + BN - 1) / BN;
  p.tiles_mn = p.tiles_m * p.tiles_n;
  p.num_tiles = p.tiles_mn * s.nh * s.nb;
  p.nh = s.nh;
  p.nz = s.nh * s.nb;
  // Raster order: the units in flight at once cover a band of the faster
  // dimension; vary N fastest when A (M x K) is the larger operand so every
  // A row block is read from HBM once while B stays L2-resident, else M.
  p.n_fast = (int64_t(s.M) * s.K > int64_t(s.N) * s.K) ? 1 : 0;
  p.causal = s.causal;
  p.c_sh = s.c_sh;
  p.c_sb = s.c_sb;
  p.e = e;
  p.C = C;
  if (CL == 2) {
    if (!B_MN) {
      p.tmBh = make_map(B, s.K, s.N, s.ldb, BN / 2, s.nh, s.nb, s.b_sh, s.b_sb);
      p.tmBq = make_map(B, s.K, s.N, s.ldb, BN / 4, s.nh, s.nb, s.b_sh, s.b_sb);
    }
    p.pairs_m = (p.tiles_m + 1) / 2;
    const int units = p.pairs_m * p.tiles_n * p.nz;
    const int clusters = std::min(units, g_sm_budget / 2);
    p.nfull = split_tail(units, clusters, BN == 256 && s.N % BN == 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(kThreadsTC);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HZP_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, p));
    ++launch_counter();
    return;
  }
  p.nfull = p.num_tiles;
  const int grid = p.num_tiles < g_sm_budget ? p.num_tiles : g_sm_budget;
  kern<<<grid, kThreadsTC, SMEM, stream>>>(ta, tb, p);
  HZP_LAUNCH_CHECK();
}

template <int BN, int STORE, int SIDE, int CL>
void dispatch_major(const void* A, const void* B, void* C, const GemmShape& s, const Epilogue& e,
                    cudaStream_t st) {
  if (s.a_mn) {
    if (s.b_mn) launch_tc<BN, 1, 1, STORE, SIDE, CL>(A, B, C, s, e, st);
    else throw std::invalid_argument("A MN-major with B K-major is not instantiated");
  } else {
    if (s.b_mn) launch_tc<BN, 0, 1, STORE, SIDE, CL>(A, B, C, s, e, st);
    else launch_tc<BN, 0, 0, STORE, SIDE, CL>(A, B, C, s, e, st);
  }
}

template <int BN>
void dispatch_store(const void* A, const void* B, void* C, const GemmShape& s, const Epilogue& e,
                    cudaStream_t st) {
  // TMA-store epilogue whenever the output (and GELU aux) layouts are
  // 16-byte describable; kEpiAccum into bf16 has no TMA reduce here.
  const int es = e.out_bf16 ? 2 : 4;
  bool tma = aligned16(C, e.ldc, s.nh > 1 ? s.c_sh : 0, s.nb > 1 ? s.c_sb : 0, es) &&
             !(e.out_bf16 && e.mode == kEpiAccum);
  if (e.act == kActGelu)
    tma = tma && e.out_bf16 && aligned16(e.aux, e.ldaux, s.nh > 1 ? s.c_sh : 0, s.nb > 1 ? s.c_sb : 0, 2);
  // side input through TMA: bf16 grads' aux or the residual, 16-byte layout
  const bool aux_in = e.act == kActTanhGrad || e.act == kActGeluGrad || e.act == kActSoftmaxGrad;
  const int64_t zsh = s.nh > 1 ? s.c_sh : 0, zsb = s.nb > 1 ? s.c_sb : 0;
  const bool side = tma && e.out_bf16 && !(aux_in && e.resid) &&
                    ((aux_in && e.aux_bf16 && aligned16(e.aux, e.ldaux, zsh, zsb, 2)) ||
                     (!aux_in && e.resid && aligned16(e.resid, e.ldres, zsh, zsb, 2)));
  // CTA pairs (cta_group::2, M = 256 per MMA) for every non-causal product
  // with at least two M tiles: each CTA stages half the B tile, halving the
  // per-SM operand traffic and smem per stage (deeper pipeline).  (Pairing
  // the causal dQ product measured slower: 79 vs 67 us — the pair's union K
  // range outweighs the halved B traffic at N = 128.)
  const bool pair = !s.causal && (s.M + BM - 1) / BM >= 2;
  if (!tma) dispatch_major<BN, 0, 0, 1>(A, B, C, s, e, st);
  else if (!e.out_bf16) {
    if (pair) dispatch_major<BN, 2, 0, 2>(A, B, C, s, e, st);
    else dispatch_major<BN, 2, 0, 1>(A, B, C, s, e, st);
  } else if (side) {
    if (pair) dispatch_major<BN, 1, 1, 2>(A, B, C, s, e, st);
    else dispatch_major<BN, 1, 1, 1>(A, B, C, s, e, st);
  } else {
    if (pair) dispatch_major<BN, 1, 0, 2>(A, B, C, s, e, st);
    else dispatch_major<BN, 1, 0, 1>(A, B, C, s, e, st);
  }
}

}  // namespace

// MN-major operand [K rows of MN contiguous elements] as the 5-D map
// {64, K, MN / 64, nh, nb} (box {64, BK, 2, 1, 1}, 128-byte swizzle): one
// instruction loads two 64-wide MN chunks, laid out in smem exactly as two
// 4-D boxes.  Only when MN % 64 == 0 (the chunk dimension then bounds the
// tail exactly); false if the driver rejects the map.
bool make_map_mn5(const void* base, int64_t mn, int64_t K, int64_t ld, int nh, int nb, int64_t sh, int64_t sb,
                  CUtensorMap* out) {
  if (mn % 64 != 0 || ld % 8 != 0) return false;
  if (nh <= 1) sh = ld * K;
  if (nb <= 1) sb = sh * nh;
  cuuint64_t dims[5] = {64, cuuint64_t(K), cuuint64_t(mn / 64), cuuint64_t(nh), cuuint64_t(nb)};
  cuuint64_t strides[4] = {cuuint64_t(ld) * 2, 128, cuuint64_t(sh) * 2, cuuint64_t(sb) * 2};
  cuuint32_t box[5] = {64, cuuint32_t(BK), 2, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  return get_encode()(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
uint64_t& launch_counter() {
  static uint64_t n = 0;
  return n;
}
GemmProfile& gemm_profile() {
  static GemmProfile p;
  return p;
}

// 4-D bf16 tensor map {inner, outer, nh, nb}: row pitch `ld` elements, batch
// strides sh / sb elements, box {64, box_outer, 1, 1}, 128-byte swizzle.
CUtensorMap make_tma_map_bf16(const void* base, int64_t inner, int64_t outer, int64_t ld,
                              int box_outer, int nh, int nb, int64_t sh, int64_t sb) {
  CUtensorMap m;
  if (nh <= 1) sh = ld * outer;
  if (nb <= 1) sb = sh * nh;
  cuuint64_t dims[4] = {cuuint64_t(inner), cuuint64_t(outer), cuuint64_t(nh), cuuint64_t(nb)};
  cuuint64_t strides[3] = {cuuint64_t(ld) * 2, cuuint64_t(sh) * 2, cuuint64_t(sb) * 2};
  cuuint32_t box[4] = {64, cuuint32_t(box_outer), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

void gemm_set_sm_budget(int sms) { g_sm_budget = sms < 1 ? 1 : (sms > kNumSMs ? kNumSMs : sms); }

void gemm_tc_bf16(const void* A, const void* B, void* C, const GemmShape& s, const Epilogue& e,
                  cudaStream_t stream) {
  if (s.M <= 0 || s.N <= 0) return;
  const bool tma_ok = s.K > 0 && (s.lda % 8 == 0) && (s.ldb % 8 == 0) &&
                      (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(B) % 16 == 0);
  if (!tma_ok) {
    if (s.nh * s.nb != 1 || s.causal || e.resid || e.act == kActSoftmaxGrad)
      throw std::invalid_argument("batched/causal GEMMs need TMA-compatible (16-byte) layouts");
    dim3 grid((s.N + 127) / 128, s.M);
    gemm_bf16_simt_kernel<<<grid, 128, 0, stream>>>(static_cast<const uint16_t*>(A),
                                                    static_cast<const uint16_t*>(B), C, s, e);
    HZP_LAUNCH_CHECK();
    return;
  }
  GemmProfile& prof = gemm_profile();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof.on) {
    HZP_CUDA(cudaEventCreate(&e0));
    HZP_CUDA(cudaEventCreate(&e1));
    HZP_CUDA(cudaEventRecord(e0, stream));
  }
  if (s.N > 128) dispatch_store<256>(A, B, C, s, e, stream);
  else dispatch_store<128>(A, B, C, s, e, stream);
  if (prof.on) {
    HZP_CUDA(cudaEventRecord(e1, stream));
    // algorithmic FLOPs: 2MNK per batch; the causal attention products do half
    const double f = 2.0 * s.M * s.N * double(s.K) * s.nh * s.nb * (s.causal ? 0.5 : 1.0);
    prof.ev.emplace_back(e0, e1);
    prof.flops.push_back(f);
    prof.shape.push_back(std::to_string(s.M) + "x" + std::to_string(s.N) + "x" + std::to_string(s.K) +
                         " z" + std::to_string(s.nh * s.nb) + " mn" + std::to_string(s.a_mn) +
                         std::to_string(s.b_mn) + " c" + std::to_string(s.causal) +
                         " act" + std::to_string(e.act) + " bf" + std::to_string(e.out_bf16));
  }
}

}  // namespace hzp
