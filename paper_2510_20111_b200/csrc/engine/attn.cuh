// Fused attention kernels (tcgen05).
#pragma once

#include <cstdint>

#include "engine/common.cuh"

namespace hzp {

// Causal softmax(Q K^T / sqrt(128)) V over qkv [b, S, 3h] (head dim 128):
// O [b, S, h]; optional P [b*nh, S, S] bf16 (rows zero past the diagonal up
// to the 128-key tile edge) and lse [b*nh, S].
void attention_fwd_tc(const uint16_t* qkv, uint16_t* O, uint16_t* P, float* lse, int b, int nh,
                      int S, int h, cudaStream_t stream);

}  // namespace hzp
