// Layer GEMM interface shared by the tcgen05 (bf16) and ordered-fp32 kernels.
//
//   C[m, n] = epilogue( sum_k A[m, k] * B[n, k] )
//
// A is M x K, B is N x K; each is stored K-major (A[m*lda + k]) or MN-major
// (A[k*lda + m]).  The three layer products of a dense layer y = x W^T map to:
//   fwd   y  = x  W^T : A = x (K-major),   B = W (K-major)
//   dgrad dx = dy W   : A = dy (K-major),  B = W (MN-major)
//   wgrad dW = dy^T x : A = dy (MN-major), B = x (MN-major)
// so no transposed copy of any operand is ever materialised.
#pragma once

#include <cstdint>

#include "engine/common.cuh"

namespace hzp {

enum EpiMode : int {
  kEpiStore = 0,    // C = f(acc)
  kEpiAccum = 1,    // C = C + acc       (fp32 C only)
  kEpiAssign0 = 2,  // C = 0.0f + acc    (first microbatch: bit-identical to += into zeros)
};
enum EpiAct : int {
  kActNone = 0,
  kActTanh = 1,       // C = tanh(acc + bias)
  kActGelu = 2,       // C = gelu_tanh(acc + bias), aux <- acc + bias (pre-activation)
  kActTanhGrad = 3,   // C = acc * (1 - a*a), a = aux[m, n]   (MLP dgrad, train.cpp:142-143)
  kActGeluGrad = 4,   // C = acc * gelu'(aux[m, n])           (GPT FC1 dgrad)
  kActSoftmaxGrad = 5,  // C = alpha * aux[m, n] * (acc - rowvec[m])  (attention dS)
};

struct Epilogue {
  int mode = kEpiStore;
  int act = kActNone;
  int out_bf16 = 1;           // C dtype (bf16 bits or fp32)
  int ldc = 0;
  const float* bias = nullptr;  // [N] fp32 (bias-first order in the fp32 kernel)
  const void* bias_any = nullptr;  // [N] in the operand dtype (bf16 path)
  void* aux = nullptr;        // [M, ldaux] pre-activation out (Gelu) / activation in (grads)
  int aux_bf16 = 1;
  int ldaux = 0;
  float alpha = 1.f;          // acc *= alpha before bias / activation
  const void* resid = nullptr;  // bf16 [M, ldres]: C = resid + f(acc)  (residual stream)
  int ldres = 0;
  const float* rowvec = nullptr;  // fp32 per-row vector (softmax-grad D), batch strides below
  int64_t rv_sh = 0, rv_sb = 0;
  int64_t bias_sh = 0;  // batched products: bias_any of head-batch zh starts at + zh * bias_sh (experts)
};

struct GemmShape {
  int M, N, K;
  int lda, ldb;
  int a_mn, b_mn;  // 1 = MN-major storage
  // Batched (attention): z = zb * nh + zh; operand X of batch z starts at
  // X + zh * x_sh + zb * x_sb elements.  C, aux and resid share C's strides.
  int nh = 1, nb = 1;
  int64_t a_sh = 0, a_sb = 0, b_sh = 0, b_sb = 0, c_sh = 0, c_sb = 0;
  // Causal structure of the attention products (M = query or key rows):
  //  1: skip tiles entirely above the diagonal (n0 >= m0 + 128)  S, dP
  //  2: K range [0, m0 + 128)                                      O = PV, dQ
  //  3: K range [m0, K)                                            dV, dK
  int causal = 0;
};

// bf16 x bf16 -> fp32 accumulate on the 5th-gen tensor cores (tcgen05.mma,
// TMA-fed, TMEM accumulator).  Requires 16-byte aligned base pointers and
// leading dimensions that are multiples of 8 elements.
void gemm_tc_bf16(const void* A, const void* B, void* C, const GemmShape& s, const Epilogue& e,
                  cudaStream_t stream);

// fp32 on the CUDA cores with the reference's exact accumulation order:
// acc starts at bias[n] (or 0), then += A[m,k]*B[n,k] for k ascending, each
// product and sum rounded separately (train.cpp:68-79, 118-148).
void gemm_f32_ordered(const float* A, const float* B, float* C, const GemmShape& s,
                      const Epilogue& e, cudaStream_t stream);

// Number of SMs a tcgen05 GEMM launch may use (persistent grid); set by the
// engine when comm kernels reserve some.
void gemm_set_sm_budget(int sms);

}  // namespace hzp
