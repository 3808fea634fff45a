// Non-GEMM kernels of the GPT decoder (bf16 activations, fp32 statistics).
// All are HBM-bound row/column passes: 16-byte vector access, one CTA (or
// warp) per row, grids sized in multiples of the 148 SMs.
#pragma once

#include <cstdint>

#include "engine/common.cuh"

namespace hzp {

// x[t] = wte[tok[t]] + wpe[t % S]; tokens laid out [b][S+1] (inputs = [:, :S]).
void embed_fwd(const int* tokens, const uint16_t* wte, const uint16_t* wpe, uint16_t* x, int b, int S,
               int h, cudaStream_t s);
// Embedding gradient, deterministic (no float atomics): tokens are stably
// sorted by id (CUB radix sort) and every id's rows are summed in ascending
// token order; dwpe[s] = sum over sequences in order.  Writes the rows of
// dwte that occur and all of dwpe (the caller zeroes dwte).  ws: a workspace
// of embed_bwd_ws_bytes(b * S, V) bytes.
size_t embed_bwd_ws_bytes(int T, int V);
void embed_bwd(const int* tokens, const uint16_t* dx, float* dwte, float* dwpe, int b, int S, int h, int V,
               void* ws, cudaStream_t s);

// LayerNorm over h (eps 1e-5): y = (x - mu) * rstd * g + beta; saves mu, rstd.
void layernorm_fwd(const uint16_t* x, const uint16_t* g, const uint16_t* beta, uint16_t* y,
                   float* mu, float* rstd, int rows, int h, cudaStream_t s);
// LayerNorm backward: dx = resid + rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat)),
// with the column reductions fused into the one pass over dy / x:
// part [2][chunks][h] = (sum dy xhat, sum dy) per chunk of rows, and, if
// prev != nullptr, prev [chunks][h] = sum of the bf16 dx written (the bias
// gradient of the projection whose output gradient dx is).
// chunks = layernorm_bwd_chunks(rows) (two persistent CTAs per SM); h <= 4096.
int layernorm_bwd_chunks(int rows);
void layernorm_bwd_fused(const uint16_t* dy, const uint16_t* x, const uint16_t* g, const float* mu,
                         const float* rstd, const uint16_t* resid, uint16_t* dx, float* part, float* prev,
                         int rows, int h, cudaStream_t s);

// Column sums of a bf16 [rows, cols] matrix into fp32 partials [chunks][cols].
void colsum_partial(const uint16_t* d, int rows, int cols, float* part, int chunks, cudaStream_t s);
// out[c] (mode, dtype) <- sum over chunks of part[k][c]  (+ optional 2nd slab)
void colsum_finalize(const float* part, int chunks, int cols, void* out, int out_bf16, int mode,
                     cudaStream_t s);
// out[i] (mode, dtype) <- src[i] (fp32 scratch -> gradient target)
void grad_write(const float* src, int64_t n, void* out, int out_bf16, int mode, cudaStream_t s);

// Per-query vectors of the attention backward, V [2][z][q]:
//   V[0] = -scale * sum_d dO[b, q, head, d] * O[b, q, head, d]   (-D / sqrt(d))
//   V[1] = -log2(e) * lse[z][q]
void attn_rowdot(const uint16_t* dO, const uint16_t* O, const float* lse, float* V, int b, int nh, int S,
                 int hd, cudaStream_t s);

// Fused softmax cross-entropy over rows of bf16 logits [T, V]: loss +=
// sum_t (lse - logit[target]) / T (row losses in row_loss [T], summed in a
// fixed order); logits <- (softmax - onehot) / T in place.
void cross_entropy(uint16_t* logits, const int* tokens, int b, int S, int V, float* row_loss, float* loss,
                   cudaStream_t s);

// SwiGLU feed-forward activation over rows of the fc1 output pre [rows, 2f]
// (gate = columns [0, f), up = [f, 2f)):  act[r, j] = silu(gate) * up, bf16.
void swiglu_fwd(const uint16_t* pre, uint16_t* act, int64_t rows, int f, cudaStream_t s);
// Its backward from dact [rows, f]: dpre[r, j] = dact * up * silu'(gate),
// dpre[r, f + j] = dact * silu(gate).
void swiglu_bwd(const uint16_t* pre, const uint16_t* dact, uint16_t* dpre, int64_t rows, int f, cudaStream_t s);

}  // namespace hzp
