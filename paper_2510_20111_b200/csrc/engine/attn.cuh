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

// Backward for dK, dV (written into the k / v thirds of dqkv [b, S, 3h]) from
// qkv, dO [b, S, h] and the per-query vectors V [2][b*nh][S] of attn_rowdot
// (-D/sqrt(d), -lse log2 e), passed as `D`.  With dsT != null it also writes
// dS^T [b*nh, S(key), S(query)] bf16 for the legacy GEMM dQ (attention_dq).
void attention_bwd_tc(const uint16_t* qkv, const uint16_t* dO, const float* lse, const float* D,
                      uint16_t* dqkv, uint16_t* dsT, int b, int nh, int S, int h, cudaStream_t stream);

// dQ into the q third of dqkv by a query-tile pass that recomputes P / dS in
// TMEM from lse (no dS in HBM): the production path.
void attention_dq_tc(const uint16_t* qkv, const uint16_t* dO, const float* D, uint16_t* dqkv, int b, int nh,
                     int S, int h, cudaStream_t stream);

// Legacy dQ = dS K as one batched causal tcgen05 GEMM over dS^T (kept for A/B
// measurements; reads b*nh*S^2/2 bf16 from HBM).
void attention_dq(const uint16_t* qkv, const uint16_t* dsT, uint16_t* dqkv, int b, int nh, int S, int h,
                  cudaStream_t stream);

}  // namespace hzp
