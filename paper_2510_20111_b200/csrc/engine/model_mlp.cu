// The reference's model family on the GPU: dense tanh MLP with linear output
// and loss sum(y^2) / (2 * B * out)  (/root/reference/proj/src/train.cpp:29-150).
//
// Flat layout per layer (train.cpp:42-53): W (out x in, row-major) then b
// (out).  fp32 mode runs every product on the ordered fp32 GEMM (reference
// summation order); bf16 mode runs them on the tcgen05 GEMM with bf16
// activations and fp32 accumulation.
#include <cmath>

#include "engine/gemm.cuh"
#include "engine/gpt_ops.cuh"
#include "engine/model.hpp"

namespace hzp {
namespace {

// loss += sum(y*y) / denom ; delta = y * scale  (train.cpp:127-131, 137-139).
// ordered (fp32 tier): one thread sums in the reference's (row-major) order.
// Otherwise every block writes the partial sum of its grid-stride elements to
// part[blockIdx.x] and mlp_loss_sum_kernel adds them in a fixed order.
__global__ void mlp_loss_delta_kernel(const float* __restrict__ y, int64_t n, float denom,
                                      float scale, float* __restrict__ loss, void* delta,
                                      int delta_bf16, int ordered, float* __restrict__ part) {
  __shared__ float red[32];
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float d = __fmul_rn(y[i], scale);
    if (delta_bf16) static_cast<uint16_t*>(delta)[i] = f32_to_bf16_bits(d);
    else static_cast<float*>(delta)[i] = d;
  }
  if (ordered) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      float acc = 0.f;
      for (int64_t i = 0; i < n; ++i) acc = __fadd_rn(acc, __fmul_rn(y[i], y[i]));
      *loss = __fadd_rn(*loss, __fdiv_rn(acc, denom));
    }
    return;
  }
  float acc = 0.f;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    acc += y[i] * y[i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

__global__ void mlp_loss_sum_kernel(const float* __restrict__ part, int nparts, float denom,
                                    float* __restrict__ loss) {
  if (threadIdx.x != 0) return;
  float s = 0.f;
  for (int i = 0; i < nparts; ++i) s += part[i];
  *loss += s / denom;
}

// Bias gradient gb[o] = sum_s d[s, o], s ascending (train.cpp:120-123), written
// with the layer's gradient-target mode.
__global__ void colsum_kernel(const void* __restrict__ d, int d_bf16, int rows, int cols,
                              void* out, int out_bf16, int mode) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= cols) return;
  float acc = 0.f;
  for (int s = 0; s < rows; ++s) {
    const int64_t i = int64_t(s) * cols + o;
    const float v = d_bf16 ? bf16_bits_to_f32(static_cast<const uint16_t*>(d)[i])
                           : static_cast<const float*>(d)[i];
    acc = __fadd_rn(acc, v);
  }
  if (out_bf16) {
    static_cast<uint16_t*>(out)[o] = f32_to_bf16_bits(acc);
  } else {
    float* p = static_cast<float*>(out) + o;
    *p = mode == kEpiAccum ? __fadd_rn(*p, acc) : (mode == kEpiAssign0 ? __fadd_rn(0.f, acc) : acc);
  }
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ x, uint16_t* __restrict__ y,
                                     int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = f32_to_bf16_bits(x[i]);
}

constexpr int kColChunks = 64;  // row chunks of the bf16-tier bias column sums

struct MlpBuffers {
  std::vector<void*> acts;  // acts[0..nl-1] working dtype; acts[0] set per microbatch
  float* y = nullptr;       // last layer output, fp32
  void* delta[2] = {nullptr, nullptr};
  int cur = 0;
  float* loss = nullptr;
  void* input_bf16 = nullptr;
  float* part = nullptr;    // bf16 tier: loss partials [256] | bias column partials [64][max dim]
};

class MlpModel final : public Model {
 public:
  explicit MlpModel(const ModelConfig& c) : c_(c) {
    int64_t off = 0;
    for (size_t l = 0; l + 1 < c.dims.size(); ++l) {
      const int64_t n = int64_t(c.dims[l]) * c.dims[l + 1] + c.dims[l + 1];
      ranges_.push_back({off, n});
      off += n;
    }
    P_ = off;
  }
  int num_layers() const override { return int(ranges_.size()); }
  LayerRange layer(int l) const override { return ranges_[l]; }
  int64_t param_count() const override { return P_; }
  int64_t input_elems_per_mb() const override { return int64_t(c_.batch) * c_.dims[0]; }
  int input_elem_bytes() const override { return 4; }
  int64_t tokens_per_mb() const override { return c_.batch; }
  double flops_per_mb() const override {
    double f = 0;
    for (size_t l = 0; l + 1 < c_.dims.size(); ++l) f += 6.0 * c_.batch * c_.dims[l] * c_.dims[l + 1];
    return f;
  }

  void* alloc_rank_buffers() override {
    auto* b = new MlpBuffers();
    const int es = c_.bf16 ? 2 : 4;
    const int nl = num_layers();
    b->acts.assign(nl, nullptr);
    for (int l = 1; l < nl; ++l)
      HZP_CUDA(cudaMalloc(&b->acts[l], size_t(c_.batch) * c_.dims[l] * es));
    if (c_.bf16) HZP_CUDA(cudaMalloc(&b->input_bf16, size_t(c_.batch) * c_.dims[0] * 2));
    HZP_CUDA(cudaMalloc(&b->y, size_t(c_.batch) * c_.dims[nl] * 4));
    int maxd = 0;
    for (int d : c_.dims) maxd = d > maxd ? d : maxd;
    for (auto& d : b->delta) HZP_CUDA(cudaMalloc(&d, size_t(c_.batch) * maxd * es));
    HZP_CUDA(cudaMalloc(&b->loss, sizeof(float)));
    HZP_CUDA(cudaMemset(b->loss, 0, sizeof(float)));
    HZP_CUDA(cudaMalloc(&b->part, (256 + size_t(kColChunks) * maxd) * sizeof(float)));
    return b;
  }
  void free_rank_buffers(void* p) override {
    auto* b = static_cast<MlpBuffers*>(p);
    for (size_t l = 1; l < b->acts.size(); ++l) cudaFree(b->acts[l]);
    cudaFree(b->input_bf16);
    cudaFree(b->y);
    cudaFree(b->delta[0]);
    cudaFree(b->delta[1]);
    cudaFree(b->loss);
    cudaFree(b->part);
    delete b;
  }
  void begin_step(void* p, cudaStream_t s) override {
    HZP_CUDA(cudaMemsetAsync(static_cast<MlpBuffers*>(p)->loss, 0, sizeof(float), s));
  }
  const float* loss_device(void* p) const override { return static_cast<MlpBuffers*>(p)->loss; }

  void fwd(void* p, int l, const void* input_mb, const void* params, cudaStream_t s) override {
    auto* b = static_cast<MlpBuffers*>(p);
    const int nl = num_layers();
    const int in = c_.dims[l], out = c_.dims[l + 1], B = c_.batch;
    if (l == 0) {
      if (c_.bf16) {
        const int64_t n = int64_t(B) * in;
        cast_f32_bf16_kernel<<<int((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0, s>>>(
            static_cast<const float*>(input_mb), static_cast<uint16_t*>(b->input_bf16), n);
        HZP_LAUNCH_CHECK();
        b->acts[0] = b->input_bf16;
      } else {
        b->acts[0] = const_cast<void*>(input_mb);
      }
    }
    const bool last = l + 1 == nl;
    GemmShape sh{B, out, in, in, in, 0, 0};
    Epilogue e;
    e.act = last ? kActNone : kActTanh;
    e.ldc = out;
    e.out_bf16 = (!last && c_.bf16) ? 1 : 0;
    void* C = last ? static_cast<void*>(b->y) : b->acts[l + 1];
    if (c_.bf16) {
      e.bias_any = static_cast<const uint16_t*>(params) + int64_t(in) * out;
      gemm_tc_bf16(b->acts[l], params, C, sh, e, s);
    } else {
      e.bias = static_cast<const float*>(params) + int64_t(in) * out;
      gemm_f32_ordered(static_cast<const float*>(b->acts[l]), static_cast<const float*>(params),
                       static_cast<float*>(C), sh, e, s);
    }
    if (last) {
      const int64_t n = int64_t(B) * out;
      const float scale = 1.0f / (float(B) * float(out));
      const float denom = (2.0f * float(B)) * float(out);
      b->cur = 0;
      const int blocks = int((n + 255) / 256 < 256 ? (n + 255) / 256 : 256);
      mlp_loss_delta_kernel<<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(
          b->y, n, denom, scale, b->loss, b->delta[0], c_.bf16, c_.bf16 ? 0 : 1, b->part);
      HZP_LAUNCH_CHECK();
      if (c_.bf16) {
        mlp_loss_sum_kernel<<<1, 32, 0, s>>>(b->part, blocks < 1 ? 1 : blocks, denom, b->loss);
        HZP_LAUNCH_CHECK();
      }
    }
  }

  void bwd(void* p, int l, const void* params, const GradTarget& g, cudaStream_t s) override {
    auto* b = static_cast<MlpBuffers*>(p);
    const int in = c_.dims[l], out = c_.dims[l + 1], B = c_.batch;
    void* d = b->delta[b->cur];
    // wgrad: dW[out, in] = sum_s d[s, out] x[s, in]
    {
      GemmShape sh{out, in, B, out, in, 1, 1};
      Epilogue e;
      e.mode = g.mode;
      e.out_bf16 = g.bf16;
      e.ldc = in;
      if (c_.bf16) gemm_tc_bf16(d, b->acts[l], g.ptr, sh, e, s);
      else gemm_f32_ordered(static_cast<const float*>(d), static_cast<const float*>(b->acts[l]),
                            static_cast<float*>(g.ptr), sh, e, s);
    }
    // bias grad
    {
      void* gb = g.bf16 ? static_cast<void*>(static_cast<uint16_t*>(g.ptr) + int64_t(in) * out)
                        : static_cast<void*>(static_cast<float*>(g.ptr) + int64_t(in) * out);
      if (c_.bf16 && out % 8 == 0) {  // column partials over row chunks, then a fixed-order sum
        colsum_partial(static_cast<const uint16_t*>(d), B, out, b->part + 256, kColChunks, s);
        colsum_finalize(b->part + 256, kColChunks, out, gb, g.bf16, g.mode, s);
      } else {  // fp32 tier: the reference's ascending-row order
        colsum_kernel<<<(out + 255) / 256, 256, 0, s>>>(d, c_.bf16, B, out, gb, g.bf16, g.mode);
        HZP_LAUNCH_CHECK();
      }
    }
    // dgrad: prev[s, in] = (sum_o d[s, o] W[o, in]) * (1 - a^2), a = acts[l]
    if (l > 0) {
      void* nd = b->delta[b->cur ^ 1];
      GemmShape sh{B, in, out, out, in, 0, 1};
      Epilogue e;
      e.act = kActTanhGrad;
      e.aux = b->acts[l];
      e.aux_bf16 = c_.bf16;
      e.ldaux = in;
      e.ldc = in;
      e.out_bf16 = c_.bf16;
      if (c_.bf16) gemm_tc_bf16(d, params, nd, sh, e, s);
      else gemm_f32_ordered(static_cast<const float*>(d), static_cast<const float*>(params),
                            static_cast<float*>(nd), sh, e, s);
      b->cur ^= 1;
    }
  }

 private:
  ModelConfig c_;
  std::vector<LayerRange> ranges_;
  int64_t P_ = 0;
};

}  // namespace

int64_t Model::max_layer_size() const {
  int64_t m = 0;
  for (int l = 0; l < num_layers(); ++l) m = layer(l).size > m ? layer(l).size : m;
  return m;
}

std::unique_ptr<Model> make_mlp_model(const ModelConfig& c) {
  return std::make_unique<MlpModel>(c);
}

}  // namespace hzp
