// Token routing kernels of the MoE feed-forward block (top-k of E experts,
// capacity-bounded dispatch).  Layout conventions:
//   logits / probs  [T, E] fp32 (router output, softmax)
//   sel  [T, K] int32 expert of choice k (descending probability, ties -> lower id)
//   gate [T, K] fp32  p_sel / sum_k p_sel (renormalised over the K choices)
//   pos  [T, K] int32 slot in the expert-major buffer (e * C + rank), -1 = dropped
//   slot_tok [E*C] int32 token of each slot, -1 = empty;  slot_k [E*C] its choice index
// Dispatch is deterministic: an expert's slots are filled in ascending token
// order (a token never selects the same expert twice); tokens past the
// capacity C are dropped (their MoE output is 0 — the residual carries them).
#pragma once

#include <cstdint>

#include "engine/common.cuh"

namespace hzp {

void moe_route(const float* logits, int T, int E, int K, float* probs, int* sel, float* gate,
               cudaStream_t s);
void moe_dispatch(const int* sel, int T, int E, int K, int C, int* pos, int* slot_tok, int* slot_k,
                  cudaStream_t s);
// xp[slot] = x[slot_tok[slot]] (0 for empty slots); rows of h bf16
void moe_gather(const uint16_t* x, const int* slot_tok, int slots, int h, uint16_t* xp, cudaStream_t s);
// out[t] = resid[t] + sum_k gate[t,k] * y[pos[t,k]]
void moe_combine(const uint16_t* y, const int* pos, const float* gate, const uint16_t* resid, int T, int K,
                 int h, uint16_t* out, cudaStream_t s);
// dy[slot] = gate[t,k] * dout[t] (0 for empty); dgate[t,k] = <dout[t], y[pos[t,k]]>
void moe_combine_bwd(const uint16_t* dout, const uint16_t* y, const int* pos, const float* gate,
                     const int* slot_tok, const int* slot_k, int T, int K, int slots, int h, uint16_t* dy,
                     float* dgate, cudaStream_t s);
// dx[t] = sum_k dxp[pos[t,k]]  (deterministic gather, no atomics)
void moe_gather_bwd(const uint16_t* dxp, const int* pos, int T, int K, int h, uint16_t* dx, cudaStream_t s);
// dlogits = softmax' (d probs), d probs from the renormalised top-k gates
void moe_router_bwd(const float* probs, const int* sel, const float* dgate, int T, int E, int K,
                    uint16_t* dlogits, cudaStream_t s);

}  // namespace hzp
