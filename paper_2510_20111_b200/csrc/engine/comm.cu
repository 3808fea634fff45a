// P2P collective kernels (sm_100a).  See comm.cuh for the contract.
//
// Design notes (B200):
//  * pull, not push: a rank reads what it needs straight out of its peers'
//    HBM through NVLink 5 / NVSwitch (peer pointers are IPC-mapped device
//    addresses), so there is no staging copy and no rendezvous inside a pass.
//  * 16-byte vector loads, UNROLL of them in flight per thread before any
//    use: a peer load costs ~2 us, so bandwidth needs deep memory-level
//    parallelism rather than many threads.
//  * CTA count is bounded (`ctas`) so the comm kernels leave most of the 148
//    SMs to the tcgen05 GEMMs running concurrently on the compute stream.
//  * every reduction sums in ascending rank order in fp32 with IEEE
//    round-to-nearest adds (no FMA contraction), so results are bit-identical
//    to the reference's canonical order.
#include <type_traits>

#include "engine/comm.cuh"

namespace hzp {
namespace {

constexpr int kThreads = 256;  // Z1 / optimizer kernels (run alone)
// AG / RS run beside a persistent tcgen05 GEMM CTA on every SM: 128 threads
// capped at 80 registers (10 K) fit next to the GEMM's 320 x 168 (53.7 K) in
// the 64 K register file, so neither kernel waits for the other to drain.
constexpr int kCommThreads = 128;
constexpr int kCommRegs = 80;
constexpr int kUnroll = 8;    // AG: 16-byte vectors in flight per thread
constexpr int kUnrollRS = 4;  // RS: per source

__device__ __forceinline__ void fadd4(float4& a, const float4& b) {
  a.x = __fadd_rn(a.x, b.x);
  a.y = __fadd_rn(a.y, b.y);
  a.z = __fadd_rn(a.z, b.z);
  a.w = __fadd_rn(a.w, b.w);
}
__device__ __forceinline__ float4 as_f4(uint4 v) {
  return make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z),
                     __uint_as_float(v.w));
}
__device__ __forceinline__ uint4 as_u4(float4 v) {
  return make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z),
                    __float_as_uint(v.w));
}
// 8 bf16 (one uint4) -> two float4
__device__ __forceinline__ void bf8_to_f8(uint4 v, float4& lo, float4& hi) {
  lo = make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xFFFF0000u),
                   __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xFFFF0000u));
  hi = make_float4(__uint_as_float(v.z << 16), __uint_as_float(v.z & 0xFFFF0000u),
                   __uint_as_float(v.w << 16), __uint_as_float(v.w & 0xFFFF0000u));
}

// ---------------------------------------------------------------------------
// AG: copy tile from owner shard to local slot.  Elements are moved as raw
// bits (bit-exact by construction).
template <int kElemBytes>
__global__ void __maxnreg__(kCommRegs) ag_pull_kernel(const RankTable* __restrict__ T,
                                                           const CommTile* __restrict__ tiles,
                                                           int ntiles, int slot,
                                                           int64_t slot_elems) {
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const CommTile t = tiles[ti];
    char* dst = static_cast<char*>(T->ag_slots[t.local]) +
                (slot * slot_elems + t.a_off) * kElemBytes;
    const char* src = static_cast<const char*>(T->param[t.src]) + t.b_off * kElemBytes;
    const int64_t bytes = int64_t(t.len) * kElemBytes;
    if (t.vec) {
      const int64_t nv = bytes / 16;
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      int64_t i = threadIdx.x;
      for (; i + (kUnroll - 1) * kCommThreads < nv; i += kUnroll * kCommThreads) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ld_nc_v4(s4 + i + u * kCommThreads);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) st_v4(d4 + i + u * kCommThreads, v[u]);
      }
      for (; i < nv; i += kCommThreads) st_v4(d4 + i, ld_nc_v4(s4 + i));
    } else {  // unaligned span: element-wise, kUnroll loads in flight per thread
      using E = typename std::conditional<kElemBytes == 2, uint16_t, uint32_t>::type;
      const E* se = reinterpret_cast<const E*>(src);
      E* de = reinterpret_cast<E*>(dst);
      int64_t i = threadIdx.x;
      for (; i + (kUnroll - 1) * kCommThreads < t.len; i += kUnroll * kCommThreads) {
        E v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = se[i + u * kCommThreads];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) de[i + u * kCommThreads] = v[u];
      }
      for (; i < t.len; i += kCommThreads) de[i] = se[i];
    }
  }
}

// ---------------------------------------------------------------------------
// RS: grad[local][a_off + i] (+)= sum_{q=0..z2-1} wire(wgrad[base+q][slot][b_off + i])
template <bool kBf16Wire>
__global__ void __maxnreg__(kCommRegs) rs_pull_kernel(const RankTable* __restrict__ T,
                                                           const CommTile* __restrict__ tiles,
                                                           int ntiles, int wslot,
                                                           int64_t wslot_elems, int z2,
                                                           int assign, float scale, int split) {
  // `split` CTAs share a tile (part = blockIdx % split takes every split-th
  // group of kUnrollRS x kCommThreads vectors): HBM-local reduces want more
  // CTAs in flight than NVLink pulls do.
  constexpr int kEB = kBf16Wire ? 2 : 4;
  const bool do_scale = scale != 1.0f;
  const int part = int(blockIdx.x) % split;
  for (int ti = int(blockIdx.x) / split; ti < ntiles; ti += int(gridDim.x) / split) {
    const CommTile t = tiles[ti];
    float* g = T->grad[T->global_rank[t.local]] + t.a_off;  // local index -> global rank
    const int64_t woff = (int64_t(wslot) * wslot_elems + t.b_off) * kEB;
    if (t.vec) {
      // kUnrollRS 16-byte vectors per thread and source in flight before any
      // use (peer loads are ~2 us away); sources summed in ascending order.
      constexpr int kPer = kBf16Wire ? 8 : 4;  // elements per 16-byte load
      const int64_t nv = t.len / kPer;
      for (int64_t i0 = threadIdx.x + int64_t(part) * kUnrollRS * kCommThreads; i0 < nv;
           i0 += int64_t(kUnrollRS) * kCommThreads * split) {
        float4 lo[kUnrollRS], hi[kUnrollRS];
        uint4 v[kUnrollRS];
        {
          const char* p = static_cast<const char*>(T->wgrad[t.src]) + woff;
#pragma unroll
          for (int u = 0; u < kUnrollRS; ++u) {
            const int64_t i = i0 + int64_t(u) * kCommThreads;
            v[u] = i < nv ? ld_nc_v4(p + i * 16) : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int u = 0; u < kUnrollRS; ++u) {
            if (kBf16Wire) bf8_to_f8(v[u], lo[u], hi[u]);
            else lo[u] = as_f4(v[u]);
          }
        }
        for (int q = 1; q < z2; ++q) {
          const char* p = static_cast<const char*>(T->wgrad[t.src + q]) + woff;
#pragma unroll
          for (int u = 0; u < kUnrollRS; ++u) {
            const int64_t i = i0 + int64_t(u) * kCommThreads;
            v[u] = i < nv ? ld_nc_v4(p + i * 16) : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int u = 0; u < kUnrollRS; ++u) {
            if (kBf16Wire) {
              float4 a, b;
              bf8_to_f8(v[u], a, b);
              fadd4(lo[u], a);
              fadd4(hi[u], b);
            } else {
              fadd4(lo[u], as_f4(v[u]));
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kUnrollRS; ++u) {
          const int64_t i = i0 + int64_t(u) * kCommThreads;
          if (i >= nv) continue;
          if (do_scale) {
            lo[u].x = __fmul_rn(lo[u].x, scale); lo[u].y = __fmul_rn(lo[u].y, scale);
            lo[u].z = __fmul_rn(lo[u].z, scale); lo[u].w = __fmul_rn(lo[u].w, scale);
            if (kBf16Wire) {
              hi[u].x = __fmul_rn(hi[u].x, scale); hi[u].y = __fmul_rn(hi[u].y, scale);
              hi[u].z = __fmul_rn(hi[u].z, scale); hi[u].w = __fmul_rn(hi[u].w, scale);
            }
          }
          float4* g4 = reinterpret_cast<float4*>(g) + i * (kPer / 4);
          float4 acc = assign ? make_float4(0.f, 0.f, 0.f, 0.f) : g4[0];
          fadd4(acc, lo[u]);
          g4[0] = acc;
          if (kBf16Wire) {
            float4 acc2 = assign ? make_float4(0.f, 0.f, 0.f, 0.f) : g4[1];
            fadd4(acc2, hi[u]);
            g4[1] = acc2;
          }
        }
      }
    } else {
      if (part != 0) continue;
      for (int64_t i = threadIdx.x; i < t.len; i += kCommThreads) {
        float s = 0.f;
        for (int q = 0; q < z2; ++q) {
          const char* p = static_cast<const char*>(T->wgrad[t.src + q]) + woff;
          const float v = kBf16Wire ? bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(p)[i])
                                    : reinterpret_cast<const float*>(p)[i];
          s = q == 0 ? v : __fadd_rn(s, v);
        }
        if (do_scale) s = __fmul_rn(s, scale);
        g[i] = __fadd_rn(assign ? 0.f : g[i], s);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Z1 stage: reduce across replicas, Adam, bf16 round, push to Z3 owners.
__device__ __forceinline__ float adam_one(float g, float& m, float& v, float& w,
                                          const AdamArgs& a) {
  m = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(a.omb1, g));
  v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(__fmul_rn(a.omb2, g), g));
  const float mhat = __fdiv_rn(m, a.bc1);
  const float vhat = __fdiv_rn(v, a.bc2);
  w = __fsub_rn(w, __fdiv_rn(__fmul_rn(a.lr, mhat), __fadd_rn(__fsqrt_rn(vhat), a.eps)));
  return w;
}

template <bool kBf16Param>
__global__ void __launch_bounds__(kThreads) z1_adam_kernel(const RankTable* __restrict__ T,
                                                           const CommTile* __restrict__ tiles,
                                                           int ntiles, int z2, int replicas,
                                                           AdamArgs a, int dbg) {
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const CommTile t = tiles[ti];
    float* mw = T->master[t.local] + t.a_off;
    float* mm = T->mom[t.local] + t.a_off;
    float* mv = T->var[t.local] + t.a_off;
    float* gd = dbg ? T->z1_grad_dbg[t.local] + t.a_off : nullptr;
    if (t.vec) {
      // two float4 per thread per pass: all ten 16-byte loads issued before
      // the (IEEE div / sqrt heavy) Adam math
      const int64_t nv = t.len / 4;
      for (int64_t i0 = threadIdx.x; i0 < nv; i0 += 2 * kThreads) {
        float4 g[2], m[2], v[2], w[2];
        bool ok[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t i = i0 + int64_t(u) * kThreads;
          ok[u] = i < nv;
          if (!ok[u]) continue;
          g[u] = as_f4(ld_v4(T->grad[t.src] + t.b_off + 4 * i));
          for (int b = 1; b < replicas; ++b)
            fadd4(g[u], as_f4(ld_v4(T->grad[t.src + b * z2] + t.b_off + 4 * i)));
          m[u] = reinterpret_cast<const float4*>(mm)[i];
          v[u] = reinterpret_cast<const float4*>(mv)[i];
          w[u] = reinterpret_cast<const float4*>(mw)[i];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (!ok[u]) continue;
          const int64_t i = i0 + int64_t(u) * kThreads;
          if (gd) reinterpret_cast<float4*>(gd)[i] = g[u];
          adam_one(g[u].x, m[u].x, v[u].x, w[u].x, a);
          adam_one(g[u].y, m[u].y, v[u].y, w[u].y, a);
          adam_one(g[u].z, m[u].z, v[u].z, w[u].z, a);
          adam_one(g[u].w, m[u].w, v[u].w, w[u].w, a);
          reinterpret_cast<float4*>(mm)[i] = m[u];
          reinterpret_cast<float4*>(mv)[i] = v[u];
          reinterpret_cast<float4*>(mw)[i] = w[u];
          uint64_t targets = t.mask;
          if (kBf16Param) {
            const uint32_t lo = uint32_t(f32_to_bf16_bits(w[u].x)) | (uint32_t(f32_to_bf16_bits(w[u].y)) << 16);
            const uint32_t hi = uint32_t(f32_to_bf16_bits(w[u].z)) | (uint32_t(f32_to_bf16_bits(w[u].w)) << 16);
            while (targets) {
              const int q = __ffsll(targets) - 1;
              targets &= targets - 1;
              uint2* p = reinterpret_cast<uint2*>(static_cast<uint16_t*>(T->param[q]) + t.c_off) + i;
              *p = make_uint2(lo, hi);
            }
          } else {
            while (targets) {
              const int q = __ffsll(targets) - 1;
              targets &= targets - 1;
              reinterpret_cast<float4*>(static_cast<float*>(T->param[q]) + t.c_off)[i] = w[u];
            }
          }
        }
      }
    } else {
      for (int64_t i = threadIdx.x; i < t.len; i += kThreads) {
        float g = T->grad[t.src][t.b_off + i];
        for (int b = 1; b < replicas; ++b) g = __fadd_rn(g, T->grad[t.src + b * z2][t.b_off + i]);
        if (gd) gd[i] = g;
        float m = mm[i], v = mv[i], w = mw[i];
        adam_one(g, m, v, w, a);
        mm[i] = m;
        mv[i] = v;
        mw[i] = w;
        uint64_t targets = t.mask;
        while (targets) {
          const int q = __ffsll(targets) - 1;
          targets &= targets - 1;
          if (kBf16Param)
            static_cast<uint16_t*>(T->param[q])[t.c_off + i] = f32_to_bf16_bits(w);
          else
            static_cast<float*>(T->param[q])[t.c_off + i] = w;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Cross-GPU signals: monotonic 64-bit counters in every rank's peer-visible
// arena, written with st.release.sys, polled with ld.acquire.sys.
__global__ void signal_kernel(const RankTable* __restrict__ T, int me, int kind, int first,
                              int count, int stride, uint64_t value, int wait_kind,
                              uint64_t wait_value) {
  const int q = threadIdx.x;
  if (q < count) {
    const int r = first + q * stride;
    __threadfence_system();
    st_release_sys(T->flags[r] + kind * kMaxRanks + me, value);
  }
  if (wait_kind >= 0 && q < count) {
    const int r = first + q * stride;
    const uint64_t* f = T->flags[me] + wait_kind * kMaxRanks + r;
    while (ld_acquire_sys(f) < wait_value) __nanosleep(64);
  }
  __syncthreads();
}

__global__ void wait_kernel(const RankTable* __restrict__ T, int me, int kind, int first,
                            int count, int stride, uint64_t value) {
  const int q = threadIdx.x;
  if (q < count) {
    const uint64_t* f = T->flags[me] + kind * kMaxRanks + first + q * stride;
    while (ld_acquire_sys(f) < value) __nanosleep(64);
  }
  __syncthreads();
}

int grid_for(int ntiles, int ctas) { return ntiles < ctas ? (ntiles > 0 ? ntiles : 1) : ctas; }

}  // namespace

void launch_ag_pull(const RankTable* T, const CommTile* tiles, int ntiles, int slot,
                    int64_t slot_elems, bool bf16, int ctas, cudaStream_t s) {
  if (ntiles <= 0) return;
  if (bf16)
    ag_pull_kernel<2><<<grid_for(ntiles, ctas), kCommThreads, 0, s>>>(T, tiles, ntiles, slot, slot_elems);
  else
    ag_pull_kernel<4><<<grid_for(ntiles, ctas), kCommThreads, 0, s>>>(T, tiles, ntiles, slot, slot_elems);
  HZP_LAUNCH_CHECK();
}

void launch_rs_pull(const RankTable* T, const CommTile* tiles, int ntiles, int wslot,
                    int64_t wslot_elems, int z2, bool bf16_wire, bool assign, float scale,
                    int ctas, cudaStream_t s, int split) {
  if (ntiles <= 0) return;
  split = split < 1 ? 1 : split;
  const int grid = grid_for(ntiles, ctas) * split;
  if (bf16_wire)
    rs_pull_kernel<true><<<grid, kCommThreads, 0, s>>>(T, tiles, ntiles, wslot, wslot_elems, z2, assign,
                                                       scale, split);
  else
    rs_pull_kernel<false><<<grid, kCommThreads, 0, s>>>(T, tiles, ntiles, wslot, wslot_elems, z2, assign,
                                                        scale, split);
  HZP_LAUNCH_CHECK();
}

void launch_z1_adam(const RankTable* T, const CommTile* tiles, int ntiles, int z2, int replicas,
                    const AdamArgs* a, int /*nlocal*/, bool bf16_param, bool dbg, int ctas,
                    cudaStream_t s) {
  if (ntiles <= 0) return;
  if (bf16_param)
    z1_adam_kernel<true><<<grid_for(ntiles, ctas), kThreads, 0, s>>>(T, tiles, ntiles, z2,
                                                                     replicas, *a, dbg);
  else
    z1_adam_kernel<false><<<grid_for(ntiles, ctas), kThreads, 0, s>>>(T, tiles, ntiles, z2,
                                                                      replicas, *a, dbg);
  HZP_LAUNCH_CHECK();
}

void launch_signal(const RankTable* T, int me, int kind, int first, int count, int stride,
                   uint64_t value, int wait_kind, uint64_t wait_value, cudaStream_t s) {
  signal_kernel<<<1, kMaxRanks, 0, s>>>(T, me, kind, first, count, stride, value, wait_kind,
                                        wait_value);
  HZP_LAUNCH_CHECK();
}

void launch_wait(const RankTable* T, int me, int kind, int first, int count, int stride,
                 uint64_t value, cudaStream_t s) {
  wait_kernel<<<1, kMaxRanks, 0, s>>>(T, me, kind, first, count, stride, value);
  HZP_LAUNCH_CHECK();
}

}  // namespace hzp
