// Model interface of the engine: a model is a stack of "layers", each a
// contiguous [offset, offset+size) range of the flat parameter vector (the
// unit of the layer-wise AG / RS tasks), with a forward and a backward that
// run on the compute stream against a gathered copy of that range.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "engine/common.cuh"

namespace hzp {

struct LayerRange {
  int64_t off = 0, size = 0;
};

// Where a backward writes its layer's unsharded gradient.
struct GradTarget {
  void* ptr = nullptr;  // element 0 = the layer's first parameter
  int bf16 = 0;         // dtype of ptr
  int mode = 0;         // EpiMode: store into a ring buffer, or (z2 == 1) accumulate
};                      // straight into the fp32 grad shard

struct ModelBuffers;  // per driven rank, model-owned activations

class Model {
 public:
  virtual ~Model() = default;
  virtual int num_layers() const = 0;
  virtual LayerRange layer(int l) const = 0;
  virtual int64_t param_count() const = 0;
  virtual int64_t max_layer_size() const;
  // Per-microbatch input element count and byte size (fp32 features for the
  // MLP, int32 token ids for the GPT).
  virtual int64_t input_elems_per_mb() const = 0;
  virtual int input_elem_bytes() const = 0;
  virtual double flops_per_mb() const = 0;   // model FLOPs of fwd+bwd of one microbatch
  virtual int64_t tokens_per_mb() const = 0;

  // Per driven rank state.
  virtual void* alloc_rank_buffers() = 0;    // returns opaque ModelBuffers*
  virtual void free_rank_buffers(void* b) = 0;
  virtual void begin_step(void* b, cudaStream_t s) = 0;         // zero loss accumulator
  virtual void fwd(void* b, int layer, const void* input_mb, const void* params,
                   cudaStream_t s) = 0;
  virtual void bwd(void* b, int layer, const void* params, const GradTarget& g,
                   cudaStream_t s) = 0;
  // FWD-recompute of `layer` just before its BWD (recompute_rule,
  // pipeline.cpp:281-318): rebuild the activations the BWD reads from the
  // layer's saved input.  No-op for models / layers that keep them.
  virtual void recompute(void* b, int layer, const void* params, cudaStream_t s) {}
  virtual int64_t launches_per_recompute(int layer) const { return 0; }
  virtual const float* loss_device(void* b) const = 0;          // fp32 summed loss
  virtual int64_t launches_per_fwd() const { return 1; }
};

struct ModelConfig {
  int kind = 0;        // HZP_MODEL_MLP / HZP_MODEL_GPT
  int bf16 = 1;
  std::vector<int> dims;  // MLP widths
  int batch = 1;       // MLP rows / GPT sequences per microbatch
  int layers = 0, hidden = 0, heads = 0, ffn = 0, vocab = 0, seq = 0;
  int experts = 0, topk = 2, capacity = 0;  // GPT MoE feed-forward (experts = 0: dense)
  int swiglu = 0;      // GPT: SwiGLU feed-forward (fc1 [2f, h] gate | up, fc2 [h, f], no FFN biases)
  int recompute = 0;   // GPT: keep only block inputs; blocks share one activation set
};

std::unique_ptr<Model> make_mlp_model(const ModelConfig& c);
std::unique_ptr<Model> make_gpt_model(const ModelConfig& c);

}  // namespace hzp
