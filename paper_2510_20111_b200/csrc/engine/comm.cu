// Collective kernels (sm_100a).  See comm.cuh for the contract.
//
// Design notes (B200):
//  * AG = owner push through NVLS multicast: the owner reads its span from
//    its own HBM (16-byte ld.global.nc) and issues multimem.st.v4 to the Z3
//    group's multicast AG slot; NVSwitch replicates each store into every
//    member's slot, so the owner's NVLink egress is the layer once (a pull
//    by the z3 - 1 readers moved it z3 - 1 times) and readers stay idle.
//  * RS = reduce at the segment owner: bf16 wire through
//    multimem.ld_reduce.add.acc::f32 (the switch reads every member's slot
//    and returns the fp32-accumulated sum rounded to bf16: the owner's
//    ingress is the layer once), fp32 wire by an ordered pull (ascending rank,
//    __fadd_rn, bit-identical to the reference's canonical order,
//    SPEC.md:208,241).
//  * register-only (no shared memory): these kernels co-reside with the
//    persistent tcgen05 GEMM (which takes ~all of an SM's shared memory) on
//    every SM instead of waiting for it to drain; 128 threads capped at 80
//    registers fit beside the GEMM's 320 x 168.
//  * UNROLL 16-byte vectors in flight per thread before any use (NVLink
//    round trips are ~2 us).
#include <type_traits>

#include "engine/comm.cuh"

namespace hzp {
namespace {

// Z1 / optimizer kernel: it runs beside the backward's persistent GEMMs, so
// it is shaped like the collectives (128 threads, <= 80 registers, one
// short-lived CTA per tile)
constexpr int kThreads = 128;
constexpr int kCommThreads = 128;
constexpr int kCommRegs = 80;
constexpr int kUnroll = 8;    // AG: 16-byte vectors in flight per thread
// Z1: one float4 group per thread per pass at 40 registers — twelve CTAs
// (48 warps) per SM hide the IEEE div / sqrt chains and the loads better
// than two groups at 80 registers (six CTAs): 1.3B N = 1 Z1 8.4 -> 6.8 ms
// (0.95 of its HBM roofline), MoE 51.0 -> 40.9 ms (48 registers: 7.1 / 43.1;
// 32 spills; 4 groups at 128 registers: 11.5 ms).
constexpr int kZ1U = 1;
constexpr int kZ1Regs = 40;
constexpr int kUnrollRS = 4;  // RS: per source
constexpr int kUnrollMC = 4;  // RS through multimem.ld_reduce (+ the fp32 shard's 2 x 16 B each)

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
__device__ __forceinline__ float round_bf16(float f) { return bf16_bits_to_f32(f32_to_bf16_bits(f)); }
__device__ __forceinline__ void round4_bf16(float4& a) {
  a.x = round_bf16(a.x);
  a.y = round_bf16(a.y);
  a.z = round_bf16(a.z);
  a.w = round_bf16(a.w);
}

// NVLS multicast primitives (sm_90+; on B200 through NVSwitch)
__device__ __forceinline__ void mc_st_v4(void* p, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 mc_ld_reduce_bf16x8(const void* p) {
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}

// In-kernel gate (multi-process): wait for the peers' flags before touching
// their slots.
__device__ __forceinline__ void gate_wait(const RankTable* __restrict__ T, const FlagGate& g) {
  if (!g.mask) return;
  const int q = threadIdx.x;
  if (q < kMaxRanks && (g.mask >> q & 1)) {
    const uint64_t* f = T->flags[g.me] + g.kind * kMaxRanks + q;
    while (ld_acquire_sys(f) < g.value) __nanosleep(64);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// AG, kMode: 0 = owner push by unicast stores to every member of the owner's
// Z3 group, 1 = owner push by one multimem.st (NVLS), 2 = reader pull from
// the owner's shard into the reader's own slot.  Raw bits (bit-exact by
// construction).
template <int kEB, int kMode>
__global__ void __maxnreg__(kCommRegs) ag_push_kernel(const RankTable* __restrict__ T,
                                                      const CommTile* __restrict__ tiles, int ntiles,
                                                      int slot, int64_t slot_elems, int z3, FlagGate gate) {
  constexpr bool kMC = kMode == 1;
  gate_wait(T, gate);
  const uint64_t pol = l2_evict_first_policy();
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const CommTile t = tiles[ti];
    const char* src = static_cast<const char*>(T->param[t.src]) + t.b_off * kEB;
    const int64_t dst_off = (slot * slot_elems + t.a_off) * kEB;
    // destination ranks: every member of the owner's group (push), or the reader
    const int base = kMode == 2 ? T->global_rank[t.local] : t.src - t.src % z3;
    const int nd = kMode == 2 ? 1 : z3;
    char* const mc = kMC ? static_cast<char*>(T->ag_mc) + dst_off : nullptr;  // hoisted past the asm clobbers
    if (t.vec) {
      const int64_t nv = int64_t(t.len) * kEB / 16;
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      int64_t i = threadIdx.x;
      for (; i < nv; i += kUnroll * kCommThreads) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int64_t j = i + u * kCommThreads;
          if (j < nv) v[u] = ld_nc_stream_v4(s4 + j, pol);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int64_t j = i + u * kCommThreads;
          if (j >= nv) continue;
          if (kMC) {
            mc_st_v4(mc + j * 16, v[u]);
          } else {
            for (int q = base; q < base + nd; ++q) st_v4(static_cast<char*>(T->ag[q]) + dst_off + j * 16, v[u]);
          }
        }
      }
    } else {  // unaligned head / tail: element-wise unicast stores to every member
      using E = typename std::conditional<kEB == 2, uint16_t, uint32_t>::type;
      const E* se = reinterpret_cast<const E*>(src);
      for (int64_t i = threadIdx.x; i < t.len; i += kCommThreads) {
        const E v = se[i];
        for (int q = base; q < base + nd; ++q)
          reinterpret_cast<E*>(static_cast<char*>(T->ag[q]) + dst_off)[i] = v;
      }
    }
  }
  if (kMC) __threadfence_system();  // stores performed before the owner posts AgDone
}

// ---------------------------------------------------------------------------
// RS at the segment owner:
//   grad[a_off + i] (+)= scale * reduce_{q in Z2 group}(wire(wgrad[q][wslot][b_off + i]))
template <bool kBf16Wire, int kMode>
__global__ void __maxnreg__(kCommRegs) rs_reduce_kernel(const RankTable* __restrict__ T,
                                                        const CommTile* __restrict__ tiles, int ntiles,
                                                        int wslot, int64_t wslot_elems, int z2, int assign,
                                                        float scale, FlagGate gate) {
  constexpr int kEB = kBf16Wire ? 2 : 4;
  constexpr bool kRound = kBf16Wire && kMode != kRsOrdered;
  const bool do_scale = scale != 1.0f;
  gate_wait(T, gate);
  const uint64_t pol = l2_evict_first_policy();
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const CommTile t = tiles[ti];
    float* g = T->grad[T->global_rank[t.local]] + t.a_off;  // local index -> global rank
    const int64_t woff = (int64_t(wslot) * wslot_elems + t.b_off) * kEB;
    const char* const mcw = kMode == kRsMulticast ? static_cast<const char*>(T->wgrad_mc) + woff : nullptr;
    if (kMode == kRsMulticast && t.vec) {
      // one in-switch reduction per 16 bytes: 8 bf16 of every member summed
      // (fp32 accumulate), returned as 8 bf16; kUnrollMC in flight per thread,
      // each with the 32 bytes of the fp32 shard it is added into (issued
      // together: the local read no longer waits for the switch round trip)
      const int64_t nv = t.len / 8;
      for (int64_t i0 = threadIdx.x; i0 < nv; i0 += int64_t(kUnrollMC) * kCommThreads) {
        uint4 v[kUnrollMC];
        float4 ga[kUnrollMC], gb[kUnrollMC];
#pragma unroll
        for (int u = 0; u < kUnrollMC; ++u) {
          const int64_t i = i0 + int64_t(u) * kCommThreads;
          v[u] = i < nv ? mc_ld_reduce_bf16x8(mcw + i * 16) : make_uint4(0u, 0u, 0u, 0u);
          const float4* g4 = reinterpret_cast<const float4*>(g) + i * 2;
          ga[u] = assign || i >= nv ? make_float4(0.f, 0.f, 0.f, 0.f) : as_f4(ld_stream_v4(g4, pol));
          gb[u] = assign || i >= nv ? make_float4(0.f, 0.f, 0.f, 0.f) : as_f4(ld_stream_v4(g4 + 1, pol));
        }
#pragma unroll
        for (int u = 0; u < kUnrollMC; ++u) {
          const int64_t i = i0 + int64_t(u) * kCommThreads;
          if (i >= nv) continue;
          float4 lo, hi;
          bf8_to_f8(v[u], lo, hi);
          if (do_scale) {
            lo.x = __fmul_rn(lo.x, scale); lo.y = __fmul_rn(lo.y, scale);
            lo.z = __fmul_rn(lo.z, scale); lo.w = __fmul_rn(lo.w, scale);
            hi.x = __fmul_rn(hi.x, scale); hi.y = __fmul_rn(hi.y, scale);
            hi.z = __fmul_rn(hi.z, scale); hi.w = __fmul_rn(hi.w, scale);
          }
          float4* g4 = reinterpret_cast<float4*>(g) + i * 2;
          float4 a = ga[u], b = gb[u];
          fadd4(a, lo);
          fadd4(b, hi);
          st_stream_v4(g4, as_u4(a), pol);
          st_stream_v4(g4 + 1, as_u4(b), pol);
        }
      }
    } else if (t.vec) {
      constexpr int kPer = kBf16Wire ? 8 : 4;  // elements per 16-byte load
      const int64_t nv = t.len / kPer;
      for (int64_t i0 = threadIdx.x; i0 < nv; i0 += int64_t(kUnrollRS) * kCommThreads) {
        float4 lo[kUnrollRS], hi[kUnrollRS];
        uint4 v[kUnrollRS];
        {
          // every source's vectors in flight before any use; ascending order
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
          for (int q = 1; q < z2; ++q) {
            const char* pq = static_cast<const char*>(T->wgrad[t.src + q]) + woff;
#pragma unroll
            for (int u = 0; u < kUnrollRS; ++u) {
              const int64_t i = i0 + int64_t(u) * kCommThreads;
              v[u] = i < nv ? ld_nc_v4(pq + i * 16) : make_uint4(0u, 0u, 0u, 0u);
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
          if (kRound) {
#pragma unroll
            for (int u = 0; u < kUnrollRS; ++u) {
              round4_bf16(lo[u]);
              round4_bf16(hi[u]);
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
    } else {  // unaligned head / tail: ordered unicast sum (rounded like the switch)
      for (int64_t i = threadIdx.x; i < t.len; i += kCommThreads) {
        float s = 0.f;
        for (int q = 0; q < z2; ++q) {
          const char* p = static_cast<const char*>(T->wgrad[t.src + q]) + woff;
          const float v = kBf16Wire ? bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(p)[i])
                                    : reinterpret_cast<const float*>(p)[i];
          s = q == 0 ? v : __fadd_rn(s, v);
        }
        if (kRound) s = round_bf16(s);
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
__global__ void __maxnreg__(kZ1Regs) z1_adam_kernel(const RankTable* __restrict__ T,
                                                           const CommTile* __restrict__ tiles,
                                                           int ntiles, int z2, int replicas,
                                                           AdamArgs a, int dbg) {
  const uint64_t pol = l2_evict_first_policy();
  for (int ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
    const CommTile t = tiles[ti];
    float* mw = T->master[t.local] + t.a_off;
    float* mm = T->mom[t.local] + t.a_off;
    float* mv = T->var[t.local] + t.a_off;
    float* gd = dbg ? T->z1_grad_dbg[t.local] + t.a_off : nullptr;
    if (t.vec) {
      // kZ1U float4 per thread per pass, all its 16-byte loads issued before
      // the (IEEE div / sqrt heavy) Adam math
      const int64_t nv = t.len / 4;
      for (int64_t i0 = threadIdx.x; i0 < nv; i0 += kZ1U * kThreads) {
        float4 g[kZ1U], m[kZ1U], v[kZ1U], w[kZ1U];
        bool ok[kZ1U];
#pragma unroll
        for (int u = 0; u < kZ1U; ++u) {
          const int64_t i = i0 + int64_t(u) * kThreads;
          ok[u] = i < nv;
          if (!ok[u]) continue;
          g[u] = as_f4(ld_stream_v4(T->grad[t.src] + t.b_off + 4 * i, pol));
          for (int b = 1; b < replicas; ++b)
            fadd4(g[u], as_f4(ld_stream_v4(T->grad[t.src + b * z2] + t.b_off + 4 * i, pol)));
          m[u] = as_f4(ld_stream_v4(mm + 4 * i, pol));
          v[u] = as_f4(ld_stream_v4(mv + 4 * i, pol));
          w[u] = as_f4(ld_stream_v4(mw + 4 * i, pol));
        }
#pragma unroll
        for (int u = 0; u < kZ1U; ++u) {
          if (!ok[u]) continue;
          const int64_t i = i0 + int64_t(u) * kThreads;
          if (gd) reinterpret_cast<float4*>(gd)[i] = g[u];
          adam_one(g[u].x, m[u].x, v[u].x, w[u].x, a);
          adam_one(g[u].y, m[u].y, v[u].y, w[u].y, a);
          adam_one(g[u].z, m[u].z, v[u].z, w[u].z, a);
          adam_one(g[u].w, m[u].w, v[u].w, w[u].w, a);
          st_stream_v4(mm + 4 * i, as_u4(m[u]), pol);
          st_stream_v4(mv + 4 * i, as_u4(v[u]), pol);
          st_stream_v4(mw + 4 * i, as_u4(w[u]), pol);
          uint64_t targets = t.mask;
          if (kBf16Param) {
            const uint32_t lo = uint32_t(f32_to_bf16_bits(w[u].x)) | (uint32_t(f32_to_bf16_bits(w[u].y)) << 16);
            const uint32_t hi = uint32_t(f32_to_bf16_bits(w[u].z)) | (uint32_t(f32_to_bf16_bits(w[u].w)) << 16);
            while (targets) {
              const int q = __ffsll(targets) - 1;
              targets &= targets - 1;
              st_stream_v2(reinterpret_cast<uint2*>(static_cast<uint16_t*>(T->param[q]) + t.c_off) + i,
                           make_uint2(lo, hi), pol);
            }
          } else {
            while (targets) {
              const int q = __ffsll(targets) - 1;
              targets &= targets - 1;
              st_stream_v4(static_cast<float*>(T->param[q]) + t.c_off + 4 * i, as_u4(w[u]), pol);
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
// Cross-GPU flags: monotonic 64-bit counters in every rank's arena, written
// with st.release.sys, polled with ld.acquire.sys.
__global__ void flags_kernel(const RankTable* __restrict__ T, int me, int post_kind, uint64_t post_mask,
                             uint64_t post_value, int wait_kind, uint64_t wait_mask, uint64_t wait_value) {
  const int q = threadIdx.x;
  if (post_mask >> q & 1) {
    __threadfence_system();
    st_release_sys(T->flags[q] + post_kind * kMaxRanks + me, post_value);
  }
  if (wait_mask >> q & 1) {
    const uint64_t* f = T->flags[me] + wait_kind * kMaxRanks + q;
    while (ld_acquire_sys(f) < wait_value) __nanosleep(64);
  }
  __syncthreads();
}

int grid_for(int ntiles, int ctas) { return ntiles < ctas ? (ntiles > 0 ? ntiles : 1) : ctas; }

}  // namespace

void launch_ag_push(const RankTable* T, const CommTile* tiles, int ntiles, int slot, int64_t slot_elems,
                    int z3, bool bf16, AgMode mode, FlagGate gate, int ctas, cudaStream_t s) {
  if (ntiles <= 0) return;
  const int grid = grid_for(ntiles, ctas);
#define HZP_AG(EB, M) ag_push_kernel<EB, M><<<grid, kCommThreads, 0, s>>>(T, tiles, ntiles, slot, slot_elems, z3, gate)
  if (bf16) {
    if (mode == kAgMulticast) HZP_AG(2, 1);
    else if (mode == kAgPull) HZP_AG(2, 2);
    else HZP_AG(2, 0);
  } else {
    if (mode == kAgMulticast) HZP_AG(4, 1);
    else if (mode == kAgPull) HZP_AG(4, 2);
    else HZP_AG(4, 0);
  }
#undef HZP_AG
  HZP_LAUNCH_CHECK();
}

void launch_rs_reduce(const RankTable* T, const CommTile* tiles, int ntiles, int wslot, int64_t wslot_elems,
                      int z2, bool bf16_wire, RsMode mode, bool assign, float scale, FlagGate gate, int ctas,
                      cudaStream_t s) {
  if (ntiles <= 0) return;
  const int grid = grid_for(ntiles, ctas);
  if (!bf16_wire) {
    if (mode != kRsOrdered) throw std::invalid_argument("fp32 wire reduces in order only (bit-exact tier)");
    rs_reduce_kernel<false, kRsOrdered><<<grid, kCommThreads, 0, s>>>(T, tiles, ntiles, wslot, wslot_elems, z2,
                                                                      assign, scale, gate);
  } else if (mode == kRsMulticast) {
    rs_reduce_kernel<true, kRsMulticast><<<grid, kCommThreads, 0, s>>>(T, tiles, ntiles, wslot, wslot_elems, z2,
                                                                       assign, scale, gate);
  } else if (mode == kRsOrderedRound) {
    rs_reduce_kernel<true, kRsOrderedRound><<<grid, kCommThreads, 0, s>>>(T, tiles, ntiles, wslot, wslot_elems,
                                                                          z2, assign, scale, gate);
  } else {
    rs_reduce_kernel<true, kRsOrdered><<<grid, kCommThreads, 0, s>>>(T, tiles, ntiles, wslot, wslot_elems, z2,
                                                                     assign, scale, gate);
  }
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

void launch_flags(const RankTable* T, int me, int post_kind, uint64_t post_mask, uint64_t post_value,
                  int wait_kind, uint64_t wait_mask, uint64_t wait_value, cudaStream_t s) {
  if (!post_mask && !wait_mask) return;
  flags_kernel<<<1, kMaxRanks, 0, s>>>(T, me, post_kind, post_mask, post_value, wait_kind, wait_mask, wait_value);
  HZP_LAUNCH_CHECK();
}

}  // namespace hzp
