// Non-GEMM kernels of the GPT decoder.  See gpt_ops.cuh.
#include <cmath>

#include <cub/device/device_radix_sort.cuh>

#include "engine/gemm.cuh"
#include "engine/gpt_ops.cuh"
#include "engine/tc_ptx.cuh"

namespace hzp {
namespace {

constexpr int kT = 256;       // threads per row-CTA
constexpr int kMaxVec = 4;    // <= 4 x 8 bf16 per thread  -> h <= 8192

__device__ __forceinline__ void unpack8(uint4 v, float* f) {
  f[0] = __uint_as_float(v.x << 16); f[1] = __uint_as_float(v.x & 0xFFFF0000u);
  f[2] = __uint_as_float(v.y << 16); f[3] = __uint_as_float(v.y & 0xFFFF0000u);
  f[4] = __uint_as_float(v.z << 16); f[5] = __uint_as_float(v.z & 0xFFFF0000u);
  f[6] = __uint_as_float(v.w << 16); f[7] = __uint_as_float(v.w & 0xFFFF0000u);
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 v;
  v.x = uint32_t(f32_to_bf16_bits(f[0])) | (uint32_t(f32_to_bf16_bits(f[1])) << 16);
  v.y = uint32_t(f32_to_bf16_bits(f[2])) | (uint32_t(f32_to_bf16_bits(f[3])) << 16);
  v.z = uint32_t(f32_to_bf16_bits(f[4])) | (uint32_t(f32_to_bf16_bits(f[5])) << 16);
  v.w = uint32_t(f32_to_bf16_bits(f[6])) | (uint32_t(f32_to_bf16_bits(f[7])) << 16);
  return v;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
  return s;
}
__device__ __forceinline__ float block_max(float v, float* red) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = -INFINITY;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) s = fmaxf(s, red[i]);
  return s;
}

__global__ void __launch_bounds__(kT) embed_fwd_kernel(const int* __restrict__ tok,
                                                       const uint16_t* __restrict__ wte,
                                                       const uint16_t* __restrict__ wpe,
                                                       uint16_t* __restrict__ x, int S, int h) {
  const int t = blockIdx.x;
  const int bi = t / S, s = t % S;
  const int id = tok[bi * (S + 1) + s];
  const uint4* a = reinterpret_cast<const uint4*>(wte + int64_t(id) * h);
  const uint4* p = reinterpret_cast<const uint4*>(wpe + int64_t(s) * h);
  uint4* o = reinterpret_cast<uint4*>(x + int64_t(t) * h);
  for (int v = threadIdx.x; v < h / 8; v += blockDim.x) {
    float fa[8], fp[8];
    unpack8(a[v], fa);
    unpack8(p[v], fp);
    for (int j = 0; j < 8; ++j) fa[j] += fp[j];
    o[v] = pack8(fa);
  }
}

__global__ void embed_keys_kernel(const int* __restrict__ tok, int* __restrict__ key, int* __restrict__ val,
                                  int T, int S) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  key[t] = tok[(t / S) * (S + 1) + t % S];
  val[t] = t;
}

// one CTA per sorted position; the first position of each id's run sums the
// run's rows (ascending token order: the sort is stable) into dwte[id]
__global__ void __launch_bounds__(kT) embed_wte_grad_kernel(const int* __restrict__ key,
                                                            const int* __restrict__ val,
                                                            const uint16_t* __restrict__ dx,
                                                            float* __restrict__ dwte, int T, int h) {
  const int i = blockIdx.x;
  const int id = key[i];
  if (i > 0 && key[i - 1] == id) return;
  int end = i + 1;
  while (end < T && key[end] == id) ++end;
  for (int v = threadIdx.x; v < h / 8; v += blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = i; j < end; ++j) {
      float f[8];
      unpack8(reinterpret_cast<const uint4*>(dx + int64_t(val[j]) * h)[v], f);
      for (int q = 0; q < 8; ++q) acc[q] += f[q];
    }
    float4* a = reinterpret_cast<float4*>(dwte + int64_t(id) * h + 8 * v);
    a[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    a[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

__global__ void __launch_bounds__(kT) embed_wpe_grad_kernel(const uint16_t* __restrict__ dx,
                                                            float* __restrict__ dwpe, int b, int S, int h) {
  const int s = blockIdx.x;
  for (int v = threadIdx.x; v < h / 8; v += blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int bi = 0; bi < b; ++bi) {
      float f[8];
      unpack8(reinterpret_cast<const uint4*>(dx + (int64_t(bi) * S + s) * h)[v], f);
      for (int q = 0; q < 8; ++q) acc[q] += f[q];
    }
    float4* p = reinterpret_cast<float4*>(dwpe + int64_t(s) * h + 8 * v);
    p[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    p[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}


__device__ __forceinline__ void write_mode(void* out, int64_t i, float v, int out_bf16, int mode) {
  if (out_bf16) {
    static_cast<uint16_t*>(out)[i] = f32_to_bf16_bits(v);
  } else {
    float* p = static_cast<float*>(out) + i;
    *p = mode == kEpiAccum ? *p + v : (mode == kEpiAssign0 ? __fadd_rn(0.f, v) : v);
  }
}


__global__ void grad_write_kernel(const float* __restrict__ src, int64_t n, void* out, int out_bf16,
                                  int mode) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    write_mode(out, i, src[i], out_bf16, mode);
}


// one warp per (token, head)
// Half a warp per (token, head) row: 16 lanes x 8 bf16 (one uint4 each of dO
// and O) cover head dim 128; hd must be 128.
__global__ void attn_rowdot_kernel(const uint16_t* __restrict__ dO, const uint16_t* __restrict__ O,
                                   const float* __restrict__ lse, float* __restrict__ V, int b, int nh,
                                   int S, int hd, float scale) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / 16;  // (token, head) row
  const int sub = threadIdx.x & 15;
  if (r >= b * S * nh) return;
  const int hh = r % nh, t = r / nh;
  const int bi = t / S, s = t % S;
  const int64_t base = int64_t(t) * nh * hd + int64_t(hh) * hd + sub * 8;
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(dO + base));
  const uint4 c = __ldg(reinterpret_cast<const uint4*>(O + base));
  float fa[8], fc[8];
  tc::unpack8f(a, fa);
  tc::unpack8f(c, fc);
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += fa[i] * fc[i];
  for (int o = 8; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (sub == 0) {
    const int64_t zq = (int64_t(bi) * nh + hh) * S + s;
    V[zq] = -scale * acc;
    V[int64_t(b) * nh * S + zq] = -1.4426950408889634f * lse[zq];
  }
}

// one CTA per token row of the logits
__global__ void __launch_bounds__(kT) cross_entropy_kernel(uint16_t* __restrict__ logits,
                                                           const int* __restrict__ tok, int S,
                                                           int V, float inv_T,
                                                           float* __restrict__ row_loss) {
  __shared__ float red[32];
  const int t = blockIdx.x;
  const int bi = t / S, s = t % S;
  const int target = tok[bi * (S + 1) + s + 1];
  uint16_t* row = logits + int64_t(t) * V;
  const int nv = V / 8;
  const float kL2E = 1.4426950408889634f;
  float mx = -INFINITY, sum = 0.f;  // online softmax per thread
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(row)[v], f);
    float m2 = mx;
    for (int j = 0; j < 8; ++j) m2 = fmaxf(m2, f[j]);
    sum *= exp2f((mx - m2) * kL2E);
    for (int j = 0; j < 8; ++j) sum += exp2f((f[j] - m2) * kL2E);
    mx = m2;
  }
  const float gmax = block_max(mx, red);
  sum = mx == -INFINITY ? 0.f : sum * exp2f((mx - gmax) * kL2E);
  const float gsum = block_sum(sum, red);
  const float lse = gmax + logf(gsum);
  const float xt = bf16_bits_to_f32(row[target]);
  __syncthreads();
  const float inv = 1.f / gsum;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(row)[v], f);
    for (int j = 0; j < 8; ++j) {
      const float p = exp2f((f[j] - gmax) * kL2E) * inv;
      f[j] = (p - ((8 * v + j) == target ? 1.f : 0.f)) * inv_T;
    }
    reinterpret_cast<uint4*>(row)[v] = pack8(f);
  }
  if (threadIdx.x == 0) row_loss[t] = (lse - xt) * inv_T;
}

// *loss += sum of the row losses, in a fixed order (deterministic)
__global__ void __launch_bounds__(1024) loss_sum_kernel(const float* __restrict__ row_loss, int T,
                                                       float* __restrict__ loss) {
  __shared__ float red[32];
  float acc = 0.f;
  for (int t = threadIdx.x; t < T; t += blockDim.x) acc += row_loss[t];
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) *loss += acc;
}


// ---- warp-per-row variants (h <= 4096): no block-wide barriers per row ----
constexpr int kWV = 16;  // max 8-element vectors per lane -> h <= 32*8*16 = 4096

__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256) layernorm_fwd_warp_kernel(
    const uint16_t* __restrict__ x, const uint16_t* __restrict__ g, const uint16_t* __restrict__ be,
    uint16_t* __restrict__ y, float* __restrict__ mu, float* __restrict__ rs, int rows, int h) {
  const int r = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int nv = h / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + int64_t(r) * h);
  float v[kWV][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kWV; ++k) {
    const int i = lane + 32 * k;
    if (i < nv) {
      unpack8(xr[i], v[k]);
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[k][j];
    }
  }
  const float mean = warp_sum(s) / h;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < kWV; ++k)
    if (lane + 32 * k < nv)
      for (int j = 0; j < 8; ++j) {
        const float d = v[k][j] - mean;
        q += d * d;
      }
  const float rstd = rsqrtf(warp_sum(q) / h + 1e-5f);
  if (lane == 0) {
    mu[r] = mean;
    rs[r] = rstd;
  }
  uint4* yr = reinterpret_cast<uint4*>(y + int64_t(r) * h);
#pragma unroll
  for (int k = 0; k < kWV; ++k) {
    const int i = lane + 32 * k;
    if (i < nv) {
      float gg[8], bb[8], o[8];
      unpack8(reinterpret_cast<const uint4*>(g)[i], gg);
      unpack8(reinterpret_cast<const uint4*>(be)[i], bb);
      for (int j = 0; j < 8; ++j) o[j] = (v[k][j] - mean) * rstd * gg[j] + bb[j];
      yr[i] = pack8(o);
    }
  }
}


// ---- LayerNorm / column reductions for h a multiple of 256 -------------------
// NVL = h / 256: 16-byte vectors per lane, so every array below is sized at
// compile time and lives in registers.
// WPR warps per row (h > 2048 uses 2: a warp holding a whole 4096-wide row
// needed 255 registers, one CTA of 8 warps per SM; at h = 2048 two warps per
// row measured no faster: 16 us per launch either way), each
// owning NVL / WPR of the row's 16-byte vectors; the two row sums (mean,
// then the centred square sum) are combined across the row's warps through
// shared memory in a fixed order.
template <int NVL, int WPR = 1>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const uint16_t* __restrict__ x,
                                                     const uint16_t* __restrict__ g,
                                                     const uint16_t* __restrict__ be, uint16_t* __restrict__ y,
                                                     float* __restrict__ mu, float* __restrict__ rs, int rows,
                                                     int h) {
  constexpr int kV = NVL / WPR > 0 ? NVL / WPR : 1;
  __shared__ float red[2][8];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (8 / WPR) + w / WPR, part = w % WPR;
  const bool live = r < rows;
  if (WPR == 1 && !live) return;
  const int rr = live ? r : rows - 1;
  const uint4* xr = reinterpret_cast<const uint4*>(x + int64_t(rr) * h);
  float v[kV][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    unpack8(__ldg(xr + lane + 32 * (part + WPR * k)), v[k]);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[k][j];
  }
  s = warp_sum(s);
  if (WPR > 1) {
    if (lane == 0) red[0][w] = s;
    __syncthreads();
    s = 0.f;
#pragma unroll
    for (int q = 0; q < WPR; ++q) s += red[0][w - part + q];
  }
  const float mean = s / h;
  float q2 = 0.f;
#pragma unroll
  for (int k = 0; k < kV; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float d = v[k][j] - mean;
      q2 += d * d;
    }
  q2 = warp_sum(q2);
  if (WPR > 1) {
    if (lane == 0) red[1][w] = q2;
    __syncthreads();
    q2 = 0.f;
#pragma unroll
    for (int q = 0; q < WPR; ++q) q2 += red[1][w - part + q];
    if (!live) return;
  }
  const float rstd = rsqrtf(q2 / h + 1e-5f);
  if (lane == 0 && part == 0) {
    mu[r] = mean;
    rs[r] = rstd;
  }
  uint4* yr = reinterpret_cast<uint4*>(y + int64_t(r) * h);
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    const int i = lane + 32 * (part + WPR * k);
    float gg[8], bb[8], o[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(g) + i), gg);
    unpack8(__ldg(reinterpret_cast<const uint4*>(be) + i), bb);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (v[k][j] - mean) * rstd * gg[j] + bb[j];
    yr[i] = pack8(o);
  }
}

// Column partial sums over a chunk of rows: part[chunk][c] = sum_r d[r][c]
// (the bias gradients of b_qkv / b_fc1 / the MoE experts).  CTA = 8 warps x
// 256 columns (8 per lane), the warps interleaving the chunk's rows;
// registers, then one smem fold.
__global__ void __launch_bounds__(256) colred_kernel(const uint16_t* __restrict__ d, int rows, int cols,
                                                     float* __restrict__ part, int chunks) {
  __shared__ float red[8][257];
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  const int c0 = blockIdx.x * 256 + lane * 8;
  const int per = (rows + chunks - 1) / chunks;
  const int r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (c0 < cols) {
#pragma unroll 2
    for (int r = r0 + w; r < r1; r += 8) {
      float f[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(d + int64_t(r) * cols + c0)), f);
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] += f[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[w][lane * 8 + j] = a[j];
  __syncthreads();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < cols) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    part[int64_t(blockIdx.y) * cols + c] = t;
  }
}

// LayerNorm backward with its column reductions fused, streamed through
// shared memory.  Persistent CTAs (2 per SM), each owning a contiguous chunk of rows
// and walks it in batches of RB rows; thread t owns the 16-byte column
// vectors t, t + 256, ... of every row and moves them itself with cp.async
// (no register staging) into a 2-stage ring — batch i + 1 is in flight while
// batch i is computed.  Per batch:
// each thread forms its part of mean(dy g) and mean(dy g xhat) per row, one
// CTA reduction (shuffles, then the 8 warps in a fixed order) completes
// them, and a second pass over the thread's own smem vectors writes dx
// (+ resid) and accumulates, in registers, the chunk's column sums
// dgamma = sum dy xhat, dbeta = sum dy and (prev) the sum of the bf16 dx
// written — the bias gradient of the projection whose output gradient dx
// is.  dy, x and resid cross HBM once; no column fold between threads.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <int NV, int RB>
__global__ void __launch_bounds__(256) ln_bwd_fused_kernel(const uint16_t* __restrict__ dy,
                                                           const uint16_t* __restrict__ x,
                                                           const uint16_t* __restrict__ g,
                                                           const float* __restrict__ mu,
                                                           const float* __restrict__ rs,
                                                           const uint16_t* __restrict__ resid,
                                                           uint16_t* __restrict__ dx, int rows, int h, int per,
                                                           float* __restrict__ part, float* __restrict__ prev) {
  extern __shared__ __align__(16) uint8_t lsm[];  // [2 stages][RB rows][3 tensors][h] bf16
  __shared__ float red[2][RB][2][8];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31, t = threadIdx.x;
  const int nvec = h / 8;
  const int rb = blockIdx.x * per, re = min(rows, rb + per);
  const int64_t rowb = int64_t(h) * 2;  // bytes of one row of one tensor
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(lsm));
  auto slot = [&](int st, int q, int ten) -> int64_t { return ((int64_t(st) * RB + q) * 3 + ten) * rowb; };
  auto issue = [&](int r0, int st) {  // this thread's vectors of rows [r0, r0 + RB)
    for (int q = 0; q < RB; ++q) {
      const int r = min(r0 + q, re - 1);
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int v = t + 256 * k;
        if (v >= nvec) continue;
        cp_async16(sbase + uint32_t(slot(st, q, 0)) + v * 16, dy + int64_t(r) * h + 8 * v);
        cp_async16(sbase + uint32_t(slot(st, q, 1)) + v * 16, x + int64_t(r) * h + 8 * v);
        if (resid) cp_async16(sbase + uint32_t(slot(st, q, 2)) + v * 16, resid + int64_t(r) * h + 8 * v);
      }
    }
  };
  float ab[NV][8], ag[NV][8], ap[NV][8], gv[NV][8];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int j = 0; j < 8; ++j) ab[k][j] = ag[k][j] = ap[k][j] = gv[k][j] = 0.f;
    const int v = t + 256 * k;
    if (v < nvec) unpack8(__ldg(reinterpret_cast<const uint4*>(g) + v), gv[k]);
  }
  if (rb < re) issue(rb, 0);
  cp_async_commit();
  int st = 0;
  for (int r0 = rb; r0 < re; r0 += RB, st ^= 1) {
    if (r0 + RB < re) issue(r0 + RB, st ^ 1);  // the next batch streams in meanwhile
    cp_async_commit();
    cp_async_wait1();  // this thread's copies of batch r0 have landed (it reads only those)
    float s1[RB], s2[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const float m = mu[min(r0 + q, re - 1)], rstd = rs[min(r0 + q, re - 1)];
      s1[q] = s2[q] = 0.f;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int v = t + 256 * k;
        if (v >= nvec) continue;
        float d[8], xv[8];
        unpack8(*reinterpret_cast<const uint4*>(lsm + slot(st, q, 0) + v * 16), d);
        unpack8(*reinterpret_cast<const uint4*>(lsm + slot(st, q, 1) + v * 16), xv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xv[j] - m) * rstd, dg = d[j] * gv[k][j];
          s1[q] += dg;
          s2[q] += dg * xh;
        }
      }
      s1[q] = warp_sum(s1[q]);
      s2[q] = warp_sum(s2[q]);
    }
    const int b = (r0 / RB) & 1;  // double-buffered: rewritten only after the next sync
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        red[b][q][0][w] = s1[q];
        red[b][q][1][w] = s2[q];
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int r = r0 + q;
      if (r >= re) continue;
      float t1 = 0.f, t2 = 0.f;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) {  // fixed order: deterministic
        t1 += red[b][q][0][ww];
        t2 += red[b][q][1][ww];
      }
      const float a1 = t1 / h, a2 = t2 / h, m = mu[r], rstd = rs[r];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int v = t + 256 * k;
        if (v >= nvec) continue;
        float d[8], xv[8], o[8];
        unpack8(*reinterpret_cast<const uint4*>(lsm + slot(st, q, 0) + v * 16), d);
        unpack8(*reinterpret_cast<const uint4*>(lsm + slot(st, q, 1) + v * 16), xv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float xh = (xv[j] - m) * rstd;
          o[j] = rstd * (d[j] * gv[k][j] - a1 - xh * a2);
          ab[k][j] += d[j];
          ag[k][j] += d[j] * xh;
        }
        if (resid) {
          float rv[8];
          unpack8(*reinterpret_cast<const uint4*>(lsm + slot(st, q, 2) + v * 16), rv);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += rv[j];
        }
        const uint4 pk = pack8(o);
        reinterpret_cast<uint4*>(dx + int64_t(r) * h)[v] = pk;
        if (prev) {
          float ob[8];
          unpack8(pk, ob);
#pragma unroll
          for (int j = 0; j < 8; ++j) ap[k][j] += ob[j];
        }
      }
    }
  }
  const int64_t cb = int64_t(blockIdx.x) * h, slab = int64_t(gridDim.x) * h;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int v = t + 256 * k;
    if (v >= nvec) continue;
    float4* pg = reinterpret_cast<float4*>(part + cb + 8 * v);
    float4* pb = reinterpret_cast<float4*>(part + slab + cb + 8 * v);
    pg[0] = make_float4(ag[k][0], ag[k][1], ag[k][2], ag[k][3]);
    pg[1] = make_float4(ag[k][4], ag[k][5], ag[k][6], ag[k][7]);
    pb[0] = make_float4(ab[k][0], ab[k][1], ab[k][2], ab[k][3]);
    pb[1] = make_float4(ab[k][4], ab[k][5], ab[k][6], ab[k][7]);
    if (prev) {
      float4* pp = reinterpret_cast<float4*>(prev + cb + 8 * v);
      pp[0] = make_float4(ap[k][0], ap[k][1], ap[k][2], ap[k][3]);
      pp[1] = make_float4(ap[k][4], ap[k][5], ap[k][6], ap[k][7]);
    }
  }
}

// out[c] (mode) = sum_k part[k][c]: 32 columns per CTA, 8 chunk lanes (warp
// w sums chunks w, w + 8, ... of its 32 columns: 128-byte coalesced rows),
// folded in a fixed order.
__global__ void __launch_bounds__(256) colsum_finalize8_kernel(const float* __restrict__ part, int chunks,
                                                               int cols, void* out, int out_bf16, int mode) {
  __shared__ float red[8][32];
  const int cl = threadIdx.x & 31, sub = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  float s = 0.f;
  if (c < cols) {
#pragma unroll 4
    for (int k = sub; k < chunks; k += 8) s += part[int64_t(k) * cols + c];
  }
  red[sub][cl] = s;
  __syncthreads();
  if (sub == 0 && c < cols) {
    float t = red[0][cl];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += red[i][cl];
    write_mode(out, c, t, out_bf16, mode);
  }
}

#define HZP_NVL_SWITCH(nvl, ...)                      \
  switch (nvl) {                                      \
    case 1: { constexpr int NVL = 1; __VA_ARGS__; } break;   \
    case 2: { constexpr int NVL = 2; __VA_ARGS__; } break;   \
    case 3: { constexpr int NVL = 3; __VA_ARGS__; } break;   \
    case 4: { constexpr int NVL = 4; __VA_ARGS__; } break;   \
    case 6: { constexpr int NVL = 6; __VA_ARGS__; } break;   \
    case 8: { constexpr int NVL = 8; __VA_ARGS__; } break;   \
    case 12: { constexpr int NVL = 12; __VA_ARGS__; } break; \
    case 16: { constexpr int NVL = 16; __VA_ARGS__; } break; \
    default: handled = false;                         \
  }

}  // namespace

namespace {

// SwiGLU: one thread per 8 columns (16-byte loads of gate, up, dact);
// silu(x) = x * sigmoid(x), silu'(x) = sigmoid(x) * (1 + x * (1 - sigmoid(x))).
__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + __expf(-x)); }
__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  return uint32_t(f32_to_bf16_bits(a)) | (uint32_t(f32_to_bf16_bits(b)) << 16);
}

__global__ void __launch_bounds__(256) swiglu_fwd_kernel(const uint16_t* __restrict__ pre, uint16_t* __restrict__ act,
                                                         int64_t rows, int f) {
  const int vec = f / 8;
  const int64_t n = rows * vec;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / vec;
    const int c = int(i - r * vec) * 8;
    const uint4 g = *reinterpret_cast<const uint4*>(pre + r * 2 * f + c);
    const uint4 u = *reinterpret_cast<const uint4*>(pre + r * 2 * f + f + c);
    const uint32_t gv[4] = {g.x, g.y, g.z, g.w}, uv[4] = {u.x, u.y, u.z, u.w};
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float g0 = bf_lo(gv[k]), g1 = bf_hi(gv[k]);
      o[k] = pack_bf2(g0 * sigmoid_f(g0) * bf_lo(uv[k]), g1 * sigmoid_f(g1) * bf_hi(uv[k]));
    }
    *reinterpret_cast<uint4*>(act + r * f + c) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void __launch_bounds__(256) swiglu_bwd_kernel(const uint16_t* __restrict__ pre,
                                                         const uint16_t* __restrict__ dact,
                                                         uint16_t* __restrict__ dpre, int64_t rows, int f) {
  const int vec = f / 8;
  const int64_t n = rows * vec;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / vec;
    const int c = int(i - r * vec) * 8;
    const uint4 g = *reinterpret_cast<const uint4*>(pre + r * 2 * f + c);
    const uint4 u = *reinterpret_cast<const uint4*>(pre + r * 2 * f + f + c);
    const uint4 d = *reinterpret_cast<const uint4*>(dact + r * f + c);
    const uint32_t gv[4] = {g.x, g.y, g.z, g.w}, uv[4] = {u.x, u.y, u.z, u.w}, dv[4] = {d.x, d.y, d.z, d.w};
    uint32_t og[4], ou[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float gg[2] = {bf_lo(gv[k]), bf_hi(gv[k])}, uu[2] = {bf_lo(uv[k]), bf_hi(uv[k])},
                  dd[2] = {bf_lo(dv[k]), bf_hi(dv[k])};
      float rg[2], ru[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float sg = sigmoid_f(gg[j]);
        ru[j] = dd[j] * gg[j] * sg;                                 // d up   = dact * silu(gate)
        rg[j] = dd[j] * uu[j] * sg * (1.0f + gg[j] * (1.0f - sg));  // d gate = dact * up * silu'(gate)
      }
      og[k] = pack_bf2(rg[0], rg[1]);
      ou[k] = pack_bf2(ru[0], ru[1]);
    }
    *reinterpret_cast<uint4*>(dpre + r * 2 * f + c) = make_uint4(og[0], og[1], og[2], og[3]);
    *reinterpret_cast<uint4*>(dpre + r * 2 * f + f + c) = make_uint4(ou[0], ou[1], ou[2], ou[3]);
  }
}

}  // namespace

void swiglu_fwd(const uint16_t* pre, uint16_t* act, int64_t rows, int f, cudaStream_t s) {
  if (f % 8) throw std::invalid_argument("swiglu: f % 8 != 0");
  swiglu_fwd_kernel<<<8 * kNumSMs, 256, 0, s>>>(pre, act, rows, f);
  HZP_LAUNCH_CHECK();
}

void swiglu_bwd(const uint16_t* pre, const uint16_t* dact, uint16_t* dpre, int64_t rows, int f, cudaStream_t s) {
  if (f % 8) throw std::invalid_argument("swiglu: f % 8 != 0");
  swiglu_bwd_kernel<<<8 * kNumSMs, 256, 0, s>>>(pre, dact, dpre, rows, f);
  HZP_LAUNCH_CHECK();
}

void embed_fwd(const int* tokens, const uint16_t* wte, const uint16_t* wpe, uint16_t* x, int b, int S,
               int h, cudaStream_t s) {
  embed_fwd_kernel<<<b * S, kT, 0, s>>>(tokens, wte, wpe, x, S, h);
  HZP_LAUNCH_CHECK();
}
namespace {
int key_bits(int V) {
  int bits = 1;
  while ((1 << bits) < V) ++bits;
  return bits;
}
size_t sort_temp_bytes(int T, int V) {
  size_t bytes = 0;
  HZP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const int*>(nullptr),
                                           static_cast<int*>(nullptr), static_cast<const int*>(nullptr),
                                           static_cast<int*>(nullptr), T, 0, key_bits(V)));
  return (bytes + 255) / 256 * 256;
}
}  // namespace

size_t embed_bwd_ws_bytes(int T, int V) {
  const size_t arr = (size_t(T) * 4 + 255) / 256 * 256;
  return 4 * arr + sort_temp_bytes(T, V);
}

void embed_bwd(const int* tokens, const uint16_t* dx, float* dwte, float* dwpe, int b, int S, int h, int V,
               void* ws, cudaStream_t s) {
  const int T = b * S;
  const size_t arr = (size_t(T) * 4 + 255) / 256 * 256;
  char* w = static_cast<char*>(ws);
  int* key_in = reinterpret_cast<int*>(w);
  int* val_in = reinterpret_cast<int*>(w + arr);
  int* key = reinterpret_cast<int*>(w + 2 * arr);
  int* val = reinterpret_cast<int*>(w + 3 * arr);
  size_t temp = sort_temp_bytes(T, V);
  embed_keys_kernel<<<(T + 255) / 256, 256, 0, s>>>(tokens, key_in, val_in, T, S);
  HZP_LAUNCH_CHECK();
  HZP_CUDA(cub::DeviceRadixSort::SortPairs(w + 4 * arr, temp, key_in, key, val_in, val, T, 0, key_bits(V), s));
  embed_wte_grad_kernel<<<T, kT, 0, s>>>(key, val, dx, dwte, T, h);
  HZP_LAUNCH_CHECK();
  embed_wpe_grad_kernel<<<S, kT, 0, s>>>(dx, dwpe, b, S, h);
  HZP_LAUNCH_CHECK();
}
void layernorm_fwd(const uint16_t* x, const uint16_t* g, const uint16_t* beta, uint16_t* y,
                   float* mu, float* rstd, int rows, int h, cudaStream_t s) {
  if (h % 8) throw std::invalid_argument("layernorm: h % 8 != 0");
  bool handled = h % 256 == 0;
  if (handled) {
    if (h / 256 > 8) {  // two warps per row beyond h = 2048 (255 registers with one)
      HZP_NVL_SWITCH(h / 256, (ln_fwd_kernel<NVL, 2><<<(rows + 3) / 4, 256, 0, s>>>(x, g, beta, y, mu, rstd, rows, h)));
    } else {
      HZP_NVL_SWITCH(h / 256, (ln_fwd_kernel<NVL><<<(rows + 7) / 8, 256, 0, s>>>(x, g, beta, y, mu, rstd, rows, h)));
    }
  }
  if (!handled) {
    if (h > 32 * 8 * kWV) throw std::invalid_argument("layernorm: h > 4096 must be 256 x {12, 16}");
    layernorm_fwd_warp_kernel<<<(rows + 7) / 8, 256, 0, s>>>(x, g, beta, y, mu, rstd, rows, h);
  }
  HZP_LAUNCH_CHECK();
}
int layernorm_bwd_chunks(int rows) { return std::max(1, std::min(2 * kNumSMs, (rows + 3) / 4)); }

void layernorm_bwd_fused(const uint16_t* dy, const uint16_t* x, const uint16_t* g, const float* mu,
                         const float* rstd, const uint16_t* resid, uint16_t* dx, float* part, float* prev,
                         int rows, int h, cudaStream_t s) {
  if (h % 8 || h > 2 * 256 * 8) throw std::invalid_argument("layernorm_bwd_fused: h % 8 != 0 or h > 4096");
  const int chunks = layernorm_bwd_chunks(rows);
  const int per = (rows + chunks - 1) / chunks;
  // two persistent CTAs per SM (16 warps hide the per-row latencies; one CTA
  // of 8 warps ran at 54 us, four CTAs at 37 us with a costlier finalize), each
  // a ring of 2 stages x RB rows x (dy, x, resid) in smem
  static bool attr = false;
  if (!attr) {  // both instantiations' ring is at most 2 x 4 x 3 x 2048 bf16
    constexpr int kMaxSmem = 2 * 4 * 3 * 2048 * 2;
    HZP_CUDA(cudaFuncSetAttribute(ln_bwd_fused_kernel<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    HZP_CUDA(cudaFuncSetAttribute(ln_bwd_fused_kernel<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    attr = true;
  }
  auto launch = [&](auto kern, int rb) {
    const size_t smem = size_t(2) * rb * 3 * h * 2;
    kern<<<chunks, 256, smem, s>>>(dy, x, g, mu, rstd, resid, dx, rows, h, per, part, prev);
  };
  if (h <= 256 * 8) launch(ln_bwd_fused_kernel<1, 4>, 4);
  else launch(ln_bwd_fused_kernel<2, 2>, 2);
  HZP_LAUNCH_CHECK();
}

void colsum_partial(const uint16_t* d, int rows, int cols, float* part, int chunks, cudaStream_t s) {
  if (cols % 8) throw std::invalid_argument("colsum: cols % 8 != 0");
  colred_kernel<<<dim3((cols + 255) / 256, chunks), 256, 0, s>>>(d, rows, cols, part, chunks);
  HZP_LAUNCH_CHECK();
}
void colsum_finalize(const float* part, int chunks, int cols, void* out, int out_bf16, int mode,
                     cudaStream_t s) {
  colsum_finalize8_kernel<<<(cols + 31) / 32, 256, 0, s>>>(part, chunks, cols, out, out_bf16, mode);
  HZP_LAUNCH_CHECK();
}
void grad_write(const float* src, int64_t n, void* out, int out_bf16, int mode, cudaStream_t s) {
  grad_write_kernel<<<4 * kNumSMs, 256, 0, s>>>(src, n, out, out_bf16, mode);
  HZP_LAUNCH_CHECK();
}
void attn_rowdot(const uint16_t* dO, const uint16_t* O, const float* lse, float* V, int b, int nh, int S,
                 int hd, cudaStream_t s) {
  if (hd != 128) throw std::invalid_argument("attn_rowdot needs head dim 128");
  const int64_t threads = int64_t(b) * S * nh * 16;
  attn_rowdot_kernel<<<unsigned((threads + 255) / 256), 256, 0, s>>>(dO, O, lse, V, b, nh, S, hd,
                                                                      1.f / sqrtf(float(hd)));
  HZP_LAUNCH_CHECK();
}
void cross_entropy(uint16_t* logits, const int* tokens, int b, int S, int V, float* row_loss, float* loss,
                   cudaStream_t s) {
  if (V % 8) throw std::invalid_argument("vocab must be a multiple of 8");
  cross_entropy_kernel<<<b * S, kT, 0, s>>>(logits, tokens, S, V, 1.f / float(b * S), row_loss);
  HZP_LAUNCH_CHECK();
  loss_sum_kernel<<<1, 1024, 0, s>>>(row_loss, b * S, loss);
  HZP_LAUNCH_CHECK();
}

}  // namespace hzp
