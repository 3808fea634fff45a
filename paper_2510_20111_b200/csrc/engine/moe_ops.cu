// MoE routing kernels.  See moe_ops.cuh.
#include <cmath>

#include "engine/moe_ops.cuh"
#include "engine/tc_ptx.cuh"

namespace hzp {
namespace {

constexpr int kMaxE = 64, kMaxK = 4;

__device__ __forceinline__ float warp_sum32(float v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one thread per token: softmax over E, top-K (ties -> lower expert id)
__global__ void route_kernel(const float* __restrict__ logits, int T, int E, int K, float* __restrict__ probs,
                             int* __restrict__ sel, float* __restrict__ gate) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float p[kMaxE];
  float mx = -INFINITY;
  for (int e = 0; e < E; ++e) {
    p[e] = logits[int64_t(t) * E + e];
    mx = fmaxf(mx, p[e]);
  }
  float s = 0.f;
  for (int e = 0; e < E; ++e) {
    p[e] = expf(p[e] - mx);
    s += p[e];
  }
  const float inv = 1.f / s;
  for (int e = 0; e < E; ++e) {
    p[e] *= inv;
    probs[int64_t(t) * E + e] = p[e];
  }
  int chosen[kMaxK];
  float ps[kMaxK], tot = 0.f;
  for (int k = 0; k < K; ++k) {
    int best = -1;
    for (int e = 0; e < E; ++e) {
      bool taken = false;
      for (int j = 0; j < k; ++j) taken = taken || chosen[j] == e;
      if (!taken && (best < 0 || p[e] > p[best])) best = e;
    }
    chosen[k] = best;
    ps[k] = p[best];
    tot += p[best];
  }
  for (int k = 0; k < K; ++k) {
    sel[int64_t(t) * K + k] = chosen[k];
    gate[int64_t(t) * K + k] = ps[k] / tot;
  }
}

// one CTA per expert: its slots in ascending token order (block scan)
__global__ void __launch_bounds__(1024) dispatch_kernel(const int* __restrict__ sel, int T, int K, int C,
                                                        int* __restrict__ pos, int* __restrict__ slot_tok,
                                                        int* __restrict__ slot_k) {
  __shared__ int warp_tot[32];
  __shared__ int base_sh;
  const int e = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) base_sh = 0;
  __syncthreads();
  for (int t0 = 0; t0 < T; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    int kk = -1;
    if (t < T)
      for (int k = 0; k < K; ++k)
        if (sel[int64_t(t) * K + k] == e) kk = k;
    const int flag = kk >= 0;
    // inclusive warp scan, then across warps
    int v = flag;
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) warp_tot[w] = v;
    __syncthreads();
    if (w == 0) {
      int x = lane < int(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += n;
      }
      warp_tot[lane] = x;  // inclusive prefix over warps
    }
    __syncthreads();
    const int rank = base_sh + (w ? warp_tot[w - 1] : 0) + v - flag;
    if (flag) {
      if (rank < C) {
        pos[int64_t(t) * K + kk] = e * C + rank;
        slot_tok[int64_t(e) * C + rank] = t;
        slot_k[int64_t(e) * C + rank] = kk;
      } else {
        pos[int64_t(t) * K + kk] = -1;  // over capacity: dropped
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) base_sh += warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  for (int r = base_sh + threadIdx.x; r < C; r += blockDim.x) {
    slot_tok[int64_t(e) * C + r] = -1;
    slot_k[int64_t(e) * C + r] = 0;
  }
}

// warp per row (h % 256 == 0 not required: 16-byte vectors, h % 8 == 0)
__global__ void gather_kernel(const uint16_t* __restrict__ x, const int* __restrict__ slot_tok, int slots, int h,
                              uint16_t* __restrict__ xp) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= slots) return;
  const int t = slot_tok[r];
  uint4* o = reinterpret_cast<uint4*>(xp + int64_t(r) * h);
  const uint4* in = t >= 0 ? reinterpret_cast<const uint4*>(x + int64_t(t) * h) : nullptr;
  for (int i = lane; i < h / 8; i += 32) o[i] = in ? __ldg(in + i) : make_uint4(0u, 0u, 0u, 0u);
}

__global__ void combine_kernel(const uint16_t* __restrict__ y, const int* __restrict__ pos,
                               const float* __restrict__ gate, const uint16_t* __restrict__ resid, int T, int K,
                               int h, uint16_t* __restrict__ out) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= T) return;
  for (int i = lane; i < h / 8; i += 32) {
    float acc[8];
    tc::unpack8f(__ldg(reinterpret_cast<const uint4*>(resid + int64_t(t) * h) + i), acc);
    for (int k = 0; k < K; ++k) {
      const int p = pos[int64_t(t) * K + k];
      if (p < 0) continue;
      const float g = gate[int64_t(t) * K + k];
      float v[8];
      tc::unpack8f(__ldg(reinterpret_cast<const uint4*>(y + int64_t(p) * h) + i), v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += g * v[j];
    }
    reinterpret_cast<uint4*>(out + int64_t(t) * h)[i] = tc::pack8f(acc);
  }
}

__global__ void combine_bwd_dy_kernel(const uint16_t* __restrict__ dout, const float* __restrict__ gate,
                                      const int* __restrict__ slot_tok, const int* __restrict__ slot_k, int K,
                                      int slots, int h, uint16_t* __restrict__ dy) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= slots) return;
  const int t = slot_tok[r];
  uint4* o = reinterpret_cast<uint4*>(dy + int64_t(r) * h);
  if (t < 0) {
    for (int i = lane; i < h / 8; i += 32) o[i] = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  const float g = gate[int64_t(t) * K + slot_k[r]];
  for (int i = lane; i < h / 8; i += 32) {
    float v[8];
    tc::unpack8f(__ldg(reinterpret_cast<const uint4*>(dout + int64_t(t) * h) + i), v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] *= g;
    o[i] = tc::pack8f(v);
  }
}

__global__ void combine_bwd_gate_kernel(const uint16_t* __restrict__ dout, const uint16_t* __restrict__ y,
                                        const int* __restrict__ pos, int T, int K, int h,
                                        float* __restrict__ dgate) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= T) return;
  for (int k = 0; k < K; ++k) {
    const int p = pos[int64_t(t) * K + k];
    float s = 0.f;
    if (p >= 0)
      for (int i = lane; i < h / 8; i += 32) {
        float a[8], b[8];
        tc::unpack8f(__ldg(reinterpret_cast<const uint4*>(dout + int64_t(t) * h) + i), a);
        tc::unpack8f(__ldg(reinterpret_cast<const uint4*>(y + int64_t(p) * h) + i), b);
#pragma unroll
        for (int j = 0; j < 8; ++j) s += a[j] * b[j];
      }
    s = warp_sum32(s);
    if (lane == 0) dgate[int64_t(t) * K + k] = s;
  }
}

__global__ void gather_bwd_kernel(const uint16_t* __restrict__ dxp, const int* __restrict__ pos, int T, int K,
                                  int h, uint16_t* __restrict__ dx) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (t >= T) return;
  for (int i = lane; i < h / 8; i += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < K; ++k) {
      const int p = pos[int64_t(t) * K + k];
      if (p < 0) continue;
      float v[8];
      tc::unpack8f(__ldg(reinterpret_cast<const uint4*>(dxp + int64_t(p) * h) + i), v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += v[j];
    }
    reinterpret_cast<uint4*>(dx + int64_t(t) * h)[i] = tc::pack8f(acc);
  }
}

// gate_k = p_k / S over the K selected (S = sum): dp_j = dg_j / S - (sum_k dg_k p_k) / S^2
// for selected j (0 otherwise); softmax: dlogit_e = p_e (dp_e - sum_j p_j dp_j)
__global__ void router_bwd_kernel(const float* __restrict__ probs, const int* __restrict__ sel,
                                  const float* __restrict__ dgate, int T, int E, int K,
                                  uint16_t* __restrict__ dlogits) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float dp[kMaxE];
  for (int e = 0; e < E; ++e) dp[e] = 0.f;
  float S = 0.f, sdg = 0.f;
  for (int k = 0; k < K; ++k) {
    const int e = sel[int64_t(t) * K + k];
    const float p = probs[int64_t(t) * E + e];
    S += p;
    sdg += dgate[int64_t(t) * K + k] * p;
  }
  for (int k = 0; k < K; ++k) {
    const int e = sel[int64_t(t) * K + k];
    dp[e] = dgate[int64_t(t) * K + k] / S - sdg / (S * S);
  }
  float dot = 0.f;
  for (int e = 0; e < E; ++e) dot += probs[int64_t(t) * E + e] * dp[e];
  for (int e = 0; e < E; ++e) {
    const float p = probs[int64_t(t) * E + e];
    dlogits[int64_t(t) * E + e] = f32_to_bf16_bits(p * (dp[e] - dot));
  }
}

}  // namespace

void moe_route(const float* logits, int T, int E, int K, float* probs, int* sel, float* gate, cudaStream_t s) {
  if (E > kMaxE || K > kMaxK || K > E) throw std::invalid_argument("moe: E <= 64, K <= 4, K <= E");
  route_kernel<<<(T + 127) / 128, 128, 0, s>>>(logits, T, E, K, probs, sel, gate);
  HZP_LAUNCH_CHECK();
}
void moe_dispatch(const int* sel, int T, int E, int K, int C, int* pos, int* slot_tok, int* slot_k,
                  cudaStream_t s) {
  dispatch_kernel<<<E, 1024, 0, s>>>(sel, T, K, C, pos, slot_tok, slot_k);
  HZP_LAUNCH_CHECK();
}
void moe_gather(const uint16_t* x, const int* slot_tok, int slots, int h, uint16_t* xp, cudaStream_t s) {
  gather_kernel<<<(slots + 7) / 8, 256, 0, s>>>(x, slot_tok, slots, h, xp);
  HZP_LAUNCH_CHECK();
}
void moe_combine(const uint16_t* y, const int* pos, const float* gate, const uint16_t* resid, int T, int K,
                 int h, uint16_t* out, cudaStream_t s) {
  combine_kernel<<<(T + 7) / 8, 256, 0, s>>>(y, pos, gate, resid, T, K, h, out);
  HZP_LAUNCH_CHECK();
}
void moe_combine_bwd(const uint16_t* dout, const uint16_t* y, const int* pos, const float* gate,
                     const int* slot_tok, const int* slot_k, int T, int K, int slots, int h, uint16_t* dy,
                     float* dgate, cudaStream_t s) {
  combine_bwd_dy_kernel<<<(slots + 7) / 8, 256, 0, s>>>(dout, gate, slot_tok, slot_k, K, slots, h, dy);
  HZP_LAUNCH_CHECK();
  combine_bwd_gate_kernel<<<(T + 7) / 8, 256, 0, s>>>(dout, y, pos, T, K, h, dgate);
  HZP_LAUNCH_CHECK();
}
void moe_gather_bwd(const uint16_t* dxp, const int* pos, int T, int K, int h, uint16_t* dx, cudaStream_t s) {
  gather_bwd_kernel<<<(T + 7) / 8, 256, 0, s>>>(dxp, pos, T, K, h, dx);
  HZP_LAUNCH_CHECK();
}
void moe_router_bwd(const float* probs, const int* sel, const float* dgate, int T, int E, int K,
                    uint16_t* dlogits, cudaStream_t s) {
  router_bwd_kernel<<<(T + 127) / 128, 128, 0, s>>>(probs, sel, dgate, T, E, K, dlogits);
  HZP_LAUNCH_CHECK();
}

}  // namespace hzp
