// Ordered fp32 GEMM on the CUDA cores — the fp32 parity tier (SURVEY §7.4
// tier B).  Each output element accumulates over k in ascending order with
// separately rounded multiply and add, starting from the bias, which is
// exactly the reference's loop (train.cpp:68-79 forward; 118-148 backward),
// and the tanh epilogue is the bit-exact restatement of the host libm's tanhf
// (libm_f32.cuh), so the fp32 step is bitwise the reference's.
// Tiled through shared memory (32x32 outputs, K chunks of 32): tiling along K
// keeps each thread's summation order intact.
#include <cmath>

#include "engine/gemm.cuh"
#include "engine/libm_f32.cuh"

namespace hzp {
namespace {

constexpr int kT = 32;

__device__ __forceinline__ float load_op(const float* P, int ld, int mn, int k, int MN, int K,
                                         int mn_major) {
  if (mn >= MN || k >= K) return 0.f;
  return mn_major ? P[int64_t(k) * ld + mn] : P[int64_t(mn) * ld + k];
}

__global__ void __launch_bounds__(kT* kT) gemm_f32_ordered_kernel(const float* __restrict__ A,
                                                                 const float* __restrict__ B,
                                                                 float* __restrict__ C,
                                                                 GemmShape s, Epilogue e) {
  __shared__ float As[kT][kT + 1];  // [m][k]
  __shared__ float Bs[kT][kT + 1];  // [n][k]
  const int tx = threadIdx.x % kT, ty = threadIdx.x / kT;
  const int m0 = blockIdx.y * kT, n0 = blockIdx.x * kT;
  const int m = m0 + ty, n = n0 + tx;
  float acc = (e.bias && n < s.N) ? e.bias[n] : 0.f;
  for (int k0 = 0; k0 < s.K; k0 += kT) {
    // cooperative loads: for MN-major operands the contiguous index is mn, so
    // map tx to mn; for K-major map tx to k (coalesced either way).
    if (s.a_mn) As[tx][ty] = load_op(A, s.lda, m0 + tx, k0 + ty, s.M, s.K, 1);
    else        As[ty][tx] = load_op(A, s.lda, m0 + ty, k0 + tx, s.M, s.K, 0);
    if (s.b_mn) Bs[tx][ty] = load_op(B, s.ldb, n0 + tx, k0 + ty, s.N, s.K, 1);
    else        Bs[ty][tx] = load_op(B, s.ldb, n0 + ty, k0 + tx, s.N, s.K, 0);
    __syncthreads();
    const int kn = min(kT, s.K - k0);
    for (int k = 0; k < kn; ++k) acc = __fadd_rn(acc, __fmul_rn(As[ty][k], Bs[tx][k]));
    __syncthreads();
  }
  if (m >= s.M || n >= s.N) return;
  const int64_t ci = int64_t(m) * e.ldc + n;
  float v = acc;
  switch (e.act) {
    case kActTanh: v = tanhf_fdlibm(acc); break;
    case kActTanhGrad: {
      const float a = static_cast<const float*>(e.aux)[int64_t(m) * e.ldaux + n];
      v = __fmul_rn(acc, __fsub_rn(1.f, __fmul_rn(a, a)));
      break;
    }
    default: break;
  }
  if (e.mode == kEpiAccum) v = __fadd_rn(C[ci], v);
  else if (e.mode == kEpiAssign0) v = __fadd_rn(0.f, v);
  C[ci] = v;
}

}  // namespace

void gemm_f32_ordered(const float* A, const float* B, float* C, const GemmShape& s,
                      const Epilogue& e, cudaStream_t stream) {
  if (s.M <= 0 || s.N <= 0) return;
  dim3 grid((s.N + kT - 1) / kT, (s.M + kT - 1) / kT);
  gemm_f32_ordered_kernel<<<grid, kT * kT, 0, stream>>>(A, B, C, s, e);
  HZP_LAUNCH_CHECK();
}

}  // namespace hzp
