// GPT-style decoder on the engine (BASELINE configs[1]: 1.3B-class, seq 2048).
//
// Task-graph layers (the unit of layer-wise AG / RS):
//   layer 0        embedding: wte [V, h] | wpe [S, h]
//   layer 1..L     decoder block (pre-LN):
//                  ln1_g ln1_b [h] | w_qkv [3h, h] | b_qkv [3h] | w_o [h, h] | b_o [h] |
//                  ln2_g ln2_b [h] | w_fc1 [f, h] | b_fc1 [f] | w_fc2 [h, f] | b_fc2 [h]
//   layer L+1      head: lnf_g lnf_b [h] | w_head [V, h]  (untied)
// SwiGLU variant (BASELINE configs[2] / [3] dims): the FFN is
//                  w_fc1 [2f, h] (rows [0, f) gate, [f, 2f) up) | w_fc2 [h, f], no biases;
//                  act = silu(gate) * up.
// MoE variant (experts E > 0, BASELINE configs[3]): the FFN part of a block is
//                  ln2_g ln2_b [h] | w_router [E, h] | E x (w_fc1 [f, h] | b_fc1 [f] |
//                  w_fc2 [h, f] | b_fc2 [h])     (SwiGLU: E x (w_fc1 [2f, h] | w_fc2 [h, f]))
// with top-K routing (renormalised gates), capacity-bounded deterministic
// dispatch (moe_ops.cuh) and the E expert products as single batched
// tcgen05 GEMMs over [E, C] slots (per-expert weights via the batch stride).
// Every matrix is row-major [out, in] like the reference's W (train.cpp:42-53),
// so all three products of each linear layer map onto the tcgen05 GEMM
// without transposes (gemm.cuh).  Attention is fused on tcgen05 (attn_tc.cu):
// forward keeps S in TMEM (online softmax, lse saved); backward recomputes P
// per key tile, accumulates dK / dV in TMEM and emits dS^T for dQ = dS K
// (a causal batched GEMM; the alternative query-tile pass recomputing P / dS
// in TMEM, attention_dq_tc, measured slower).
#include <cmath>
#include <vector>

#include "engine/gemm.cuh"
#include "engine/gpt_ops.cuh"
#include "engine/attn.cuh"
#include "engine/model.hpp"
#include "engine/moe_ops.cuh"

namespace hzp {
namespace {

struct BlockOff {  // element offsets inside a block's parameter range
  int64_t ln1_g, ln1_b, w_qkv, b_qkv, w_o, b_o, ln2_g, ln2_b, w_fc1, b_fc1, w_fc2, b_fc2, size;
  int64_t w_router = 0, ex_stride = 0;  // MoE: router, and expert e's tensors at + e * ex_stride
};

struct LayerActs {  // saved activations of one block (one microbatch)
  uint16_t *ln1, *qkv, *attn, *xm, *ln2, *fpre, *fact;
  float *mu1, *rs1, *mu2, *rs2, *lse;  // lse [Z, S]: softmax stats for the backward
  // MoE: router stats and the expert-major slot buffers ([E*C, .] rows)
  float *logits = nullptr, *probs = nullptr, *gate = nullptr;
  int *sel = nullptr, *pos = nullptr, *slot_tok = nullptr, *slot_k = nullptr;
  uint16_t *xp = nullptr, *y = nullptr;
};

struct GptBuffers {
  std::vector<uint16_t*> x;  // x[0..L+1]: x[l] = input of task-layer l (x[1] = embedding out)
  std::vector<LayerActs> acts;  // [L+2] (only 1..L used)
  uint16_t* lnf = nullptr;
  float *muf = nullptr, *rsf = nullptr;
  uint16_t* logits = nullptr;  // [T, V]; dlogits in place after the fused CE
  float* S = nullptr;          // [Z, S, S] fp32 scores
  uint16_t* dS = nullptr;      // [Z, S, S]
  float* D = nullptr;          // [2, Z, S]: attn_rowdot's per-query vectors
  uint16_t* dx[2] = {nullptr, nullptr};
  int cur = 0;
  uint16_t *dln = nullptr, *dqkv = nullptr, *dattn = nullptr, *dfc1 = nullptr, *dxm = nullptr;
  uint16_t* dact = nullptr;  // SwiGLU: grad of the activation [T, f] (dfc1 is [T, 2f])
  float* part = nullptr;       // column-sum partials
  // fused LayerNorm-backward partials, each slab [layernorm_bwd_chunks(T)][h]:
  // 0-1 ln2 (dgamma, dbeta), 2-3 ln1, 4 ln2's dx sum (b_o), 5-6 ln1's / the
  // final LN's dx sum = the next-lower block's b_fc2, by that block's parity
  float* lnpart = nullptr;
  // weight gradients of a block run on a side stream (they are leaves of the
  // backward DAG), so they fill the SMs the dgrad chain's tail waves leave
  // idle; own column-sum partials, fork/join by events.
  cudaStream_t side = nullptr;
  cudaEvent_t ev[12] = {};
  float* part_side = nullptr;
  // MoE backward scratch
  uint16_t *moe_dy = nullptr, *moe_dh = nullptr, *moe_dxp = nullptr, *moe_dlogits = nullptr;
  uint16_t* moe_dact = nullptr;  // SwiGLU experts: [E*C, f]
  float* moe_dgate = nullptr;
  float* emb = nullptr;        // fp32 scratch for the embedding gradient [V*h + S*h]
  void* emb_ws = nullptr;      // embed_bwd's sort workspace
  float* row_loss = nullptr;   // [T] per-token loss (summed in a fixed order)
  float* loss = nullptr;
  const int* tokens = nullptr;  // current microbatch
};

constexpr int kChunks = 64;  // row chunks of the column reductions (bias / LN parameter grads)

class GptModel final : public Model {
 public:
  explicit GptModel(const ModelConfig& c) : c_(c) {
    h_ = c.hidden;
    nh_ = c.heads;
    hd_ = h_ / nh_;
    f_ = c.ffn;
    V_ = c.vocab;
    S_ = c.seq;
    b_ = c.batch;
    T_ = int64_t(b_) * S_;
    L_ = c.layers;
    E_ = c.experts;
    K_ = c.topk > 0 ? c.topk : 2;
    sw_ = c.swiglu != 0;
    f1_ = sw_ ? 2 * f_ : f_;  // fc1 output width
    if (E_ > 0) {
      if (E_ > 64 || K_ > 4 || K_ > E_ || E_ % 8) throw std::invalid_argument("MoE: experts % 8 == 0, <= 64, topk <= 4");
      const int64_t autoc = (int64_t(K_) * T_ * 5 / 4 + E_ - 1) / E_;
      C_ = c.capacity > 0 ? c.capacity : int(autoc);
      C_ = (C_ + 127) / 128 * 128;
    }
    if (h_ % 64 || f_ % 64 || V_ % 64 || S_ % 128 || hd_ != 128 || h_ % nh_)
      throw std::invalid_argument("GPT dims must be multiples of 64, seq of 128, head dim 128");
    int64_t o = 0;
    auto take = [&](int64_t n) {
      const int64_t r = o;
      o += n;
      return r;
    };
    bo_.ln1_g = take(h_);
    bo_.ln1_b = take(h_);
    bo_.w_qkv = take(3 * int64_t(h_) * h_);
    bo_.b_qkv = take(3 * h_);
    bo_.w_o = take(int64_t(h_) * h_);
    bo_.b_o = take(h_);
    bo_.ln2_g = take(h_);
    bo_.ln2_b = take(h_);
    if (E_ > 0) bo_.w_router = take(int64_t(E_) * h_);
    const int64_t ex0 = o;
    bo_.w_fc1 = take(int64_t(f1_) * h_);
    bo_.b_fc1 = sw_ ? -1 : take(f_);
    bo_.w_fc2 = take(int64_t(h_) * f_);
    bo_.b_fc2 = sw_ ? -1 : take(h_);
    if (E_ > 0) {
      bo_.ex_stride = o - ex0;
      o = ex0 + int64_t(E_) * bo_.ex_stride;
    }
    bo_.size = o;
    int64_t off = 0;
    ranges_.push_back({off, int64_t(V_) * h_ + int64_t(S_) * h_});
    off += ranges_.back().size;
    for (int l = 0; l < L_; ++l) {
      ranges_.push_back({off, bo_.size});
      off += bo_.size;
    }
    ranges_.push_back({off, 2 * int64_t(h_) + int64_t(V_) * h_});
    off += ranges_.back().size;
    P_ = off;
  }

  int num_layers() const override { return L_ + 2; }
  LayerRange layer(int l) const override { return ranges_[l]; }
  int64_t param_count() const override { return P_; }
  int64_t input_elems_per_mb() const override { return int64_t(b_) * (S_ + 1); }
  int input_elem_bytes() const override { return 4; }
  int64_t tokens_per_mb() const override { return T_; }
  double flops_per_mb() const override {
    // 6 * dense params * tokens + causal attention (QK^T and PV, fwd + bwd = 3x):
    // 3 * 2 * 2 * S^2/2 * h * b * L
    // MoE: the active parameters per token (K experts + router)
    const double per_ex = (sw_ ? 3.0 : 2.0) * h_ * f_;
    const double ffn = E_ > 0 ? double(K_) * per_ex + double(E_) * h_ : per_ex;
    const double dense = double(L_) * (4.0 * h_ * h_ + ffn) + double(V_) * h_;
    return 6.0 * dense * double(T_) + 6.0 * double(S_) * S_ * h_ * b_ * L_;
  }
  int64_t launches_per_fwd() const override { return 9 + (sw_ ? 1 : 0); }

  void* alloc_rank_buffers() override {
    auto* B = new GptBuffers();
    auto bf = [](int64_t n) {
      uint16_t* p = nullptr;
      HZP_CUDA(cudaMalloc(&p, size_t(n) * 2));
      return p;
    };
    auto f32 = [](int64_t n) {
      float* p = nullptr;
      HZP_CUDA(cudaMalloc(&p, size_t(n) * 4));
      return p;
    };
    auto i32 = [](int64_t n) {
      int* p = nullptr;
      HZP_CUDA(cudaMalloc(&p, size_t(n) * 4));
      return p;
    };
    const int64_t Z = int64_t(b_) * nh_;
    const int64_t SS = Z * S_ * S_;
    B->x.assign(L_ + 2, nullptr);
    for (int l = 1; l <= L_ + 1; ++l) B->x[l] = bf(T_ * h_);
    B->acts.resize(L_ + 2);
    // recompute: one activation set shared by every block (rebuilt from the
    // block's input x[l] by its FWD-recompute before the BWD reads it)
    for (int l = 1; l <= (c_.recompute ? 1 : L_); ++l) {
      LayerActs& a = B->acts[l];
      a.ln1 = bf(T_ * h_);
      a.qkv = bf(T_ * 3 * h_);
      a.lse = f32(int64_t(b_) * nh_ * S_);
      a.attn = bf(T_ * h_);
      a.xm = bf(T_ * h_);
      a.ln2 = bf(T_ * h_);
      const int64_t frows = E_ > 0 ? int64_t(E_) * C_ : T_;
      a.fpre = bf(frows * f1_);
      a.fact = bf(frows * f_);
      if (E_ > 0) {
        a.logits = f32(T_ * E_);
        a.probs = f32(T_ * E_);
        a.gate = f32(T_ * K_);
        a.sel = i32(T_ * K_);
        a.pos = i32(T_ * K_);
        a.slot_tok = i32(int64_t(E_) * C_);
        a.slot_k = i32(int64_t(E_) * C_);
        a.xp = bf(int64_t(E_) * C_ * h_);
        a.y = bf(int64_t(E_) * C_ * h_);
      }
      a.mu1 = f32(T_);
      a.rs1 = f32(T_);
      a.mu2 = f32(T_);
      a.rs2 = f32(T_);
    }
    if (c_.recompute)
      for (int l = 2; l <= L_; ++l) B->acts[l] = B->acts[1];
    B->lnf = bf(T_ * h_);
    B->muf = f32(T_);
    B->rsf = f32(T_);
    B->logits = bf(T_ * V_);
    B->S = nullptr;  // scores stay in TMEM (fused attention)
    B->dS = bf(SS);
    B->D = f32(2 * Z * S_);
    B->dx[0] = bf(T_ * h_);
    B->dx[1] = bf(T_ * h_);
    B->dln = bf(T_ * h_);
    B->dqkv = bf(T_ * 3 * h_);
    B->dattn = bf(T_ * h_);
    B->dfc1 = bf(T_ * f1_);
    if (sw_) B->dact = bf(T_ * f_);
    if (E_ > 0) {
      B->moe_dy = bf(int64_t(E_) * C_ * h_);
      B->moe_dh = bf(int64_t(E_) * C_ * f1_);
      if (sw_) B->moe_dact = bf(int64_t(E_) * C_ * f_);
      B->moe_dxp = bf(int64_t(E_) * C_ * h_);
      B->moe_dlogits = bf(T_ * E_);
      B->moe_dgate = f32(T_ * K_);
    }
    B->dxm = bf(T_ * h_);
    B->part = f32(2 * int64_t(kChunks) * std::max<int64_t>(f_, 3 * int64_t(h_)));
    B->part_side = f32(2 * int64_t(kChunks) * std::max<int64_t>(f_, 3 * int64_t(h_)));
    B->lnpart = f32(7 * lnslab());
    {  // weight-gradient GEMMs: compute, at the compute stream's (highest) priority
      int lo = 0, hi = 0;
      HZP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      HZP_CUDA(cudaStreamCreateWithPriority(&B->side, cudaStreamNonBlocking, hi));
    }
    for (auto& e : B->ev) HZP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    B->emb = f32(int64_t(V_) * h_ + int64_t(S_) * h_);
    HZP_CUDA(cudaMalloc(&B->emb_ws, embed_bwd_ws_bytes(int(T_), V_)));
    B->row_loss = f32(T_);
    B->loss = f32(1);
    HZP_CUDA(cudaMemset(B->loss, 0, 4));
    return B;
  }
  void free_rank_buffers(void* p) override {
    auto* B = static_cast<GptBuffers*>(p);
    for (auto* x : B->x) cudaFree(x);
    for (int l = 0; l < int(B->acts.size()) && !(c_.recompute && l > 1); ++l) {
      const LayerActs& a = B->acts[l];
      for (void* q : {(void*)a.ln1, (void*)a.qkv, (void*)a.lse, (void*)a.attn, (void*)a.xm,
                      (void*)a.ln2, (void*)a.fpre, (void*)a.fact, (void*)a.mu1, (void*)a.rs1,
                      (void*)a.mu2, (void*)a.rs2, (void*)a.logits, (void*)a.probs, (void*)a.gate,
                      (void*)a.sel, (void*)a.pos, (void*)a.slot_tok, (void*)a.slot_k, (void*)a.xp,
                      (void*)a.y})
        cudaFree(q);
    }
    for (void* q : {(void*)B->lnf, (void*)B->muf, (void*)B->rsf, (void*)B->logits, (void*)B->S,
                    (void*)B->dS, (void*)B->D, (void*)B->dx[0], (void*)B->dx[1], (void*)B->dln,
                    (void*)B->dqkv, (void*)B->dattn, (void*)B->dfc1, (void*)B->dxm, (void*)B->part,
                    (void*)B->part_side, (void*)B->lnpart, (void*)B->moe_dy, (void*)B->moe_dh, (void*)B->moe_dxp,
                    (void*)B->moe_dlogits, (void*)B->moe_dgate,
                    (void*)B->emb, B->emb_ws, (void*)B->row_loss, (void*)B->loss})
      cudaFree(q);
    for (auto e : B->ev) cudaEventDestroy(e);
    if (B->side) cudaStreamDestroy(B->side);
    delete B;
  }
  void begin_step(void* p, cudaStream_t s) override {
    HZP_CUDA(cudaMemsetAsync(static_cast<GptBuffers*>(p)->loss, 0, 4, s));
  }
  const float* loss_device(void* p) const override { return static_cast<GptBuffers*>(p)->loss; }

  // ---- helpers ---------------------------------------------------------------
  // y[T, N] (+)= x[T, K] W[N, K]^T with epilogue e
  void linear_fwd(const uint16_t* x, const uint16_t* w, void* y, int N, int K, Epilogue e,
                  cudaStream_t s) const {
    GemmShape sh{int(T_), N, K, K, K, 0, 0};
    e.ldc = N;
    gemm_tc_bf16(x, w, y, sh, e, s);
  }
  // dW[N, K] = dy[T, N]^T x[T, K] -> grad target (+ bias grad colsum(dy) if db_off >= 0)
  void linear_wgrad(const uint16_t* dy, const uint16_t* x, int N, int K, const GradTarget& g,
                    int64_t w_off, int64_t b_off, GptBuffers* B, cudaStream_t s) const {
    float* part = s == B->side ? B->part_side : B->part;
    GemmShape sh{N, K, int(T_), N, K, 1, 1};
    Epilogue e;
    e.mode = g.mode;
    e.out_bf16 = g.bf16;
    e.ldc = K;
    gemm_tc_bf16(dy, x, gptr(g, w_off), sh, e, s);
    if (b_off >= 0) {
      colsum_partial(dy, int(T_), N, part, kChunks, s);
      colsum_finalize(part, kChunks, N, gptr(g, b_off), g.bf16, g.mode, s);
    }
  }
  // dx[T, K] = dy[T, N] W[N, K]   (+ epilogue)
  void linear_dgrad(const uint16_t* dy, const uint16_t* w, uint16_t* dx, int N, int K, Epilogue e,
                    cudaStream_t s) const {
    GemmShape sh{int(T_), K, N, N, K, 0, 1};
    e.ldc = K;
    gemm_tc_bf16(dy, w, dx, sh, e, s);
  }
  static void* gptr(const GradTarget& g, int64_t off) {
    return g.bf16 ? static_cast<void*>(static_cast<uint16_t*>(g.ptr) + off)
                  : static_cast<void*>(static_cast<float*>(g.ptr) + off);
  }
  // fused LayerNorm backward partials (see GptBuffers::lnpart)
  int64_t lnslab() const { return int64_t(layernorm_bwd_chunks(int(T_))) * h_; }
  float* lnp(GptBuffers* B, int slab) const { return B->lnpart + slab * lnslab(); }
  // dense FFN with biases: its b_fc2 gradient is the column sum of the
  // block-output gradient, i.e. of the next block's LN1 (or the final LN) dx
  bool fc2_bias() const { return E_ == 0 && !sw_; }
  float* fc2b_part(GptBuffers* B, int block) const { return lnp(B, 5 + (block & 1)); }
  // LN gamma / beta gradients from layernorm_bwd_fused's partials
  void ln_param_grads(GptBuffers* B, const GradTarget& g, int64_t g_off, int64_t b_off, cudaStream_t s,
                      const float* part) const {
    const int ch = layernorm_bwd_chunks(int(T_));
    colsum_finalize(part, ch, h_, gptr(g, g_off), g.bf16, g.mode, s);
    colsum_finalize(part + lnslab(), ch, h_, gptr(g, b_off), g.bf16, g.mode, s);
  }
  void bias_from_ln(GptBuffers* B, const float* part, const GradTarget& g, int64_t b_off, cudaStream_t s) const {
    colsum_finalize(part, layernorm_bwd_chunks(int(T_)), h_, gptr(g, b_off), g.bf16, g.mode, s);
  }
  // batched attention shapes over z = (sequence b, head)
  GemmShape attn_shape(int M, int N, int K, int lda, int ldb, int a_mn, int b_mn, int64_t a_sh,
                       int64_t a_sb, int64_t b_sh, int64_t b_sb, int64_t c_sh, int64_t c_sb,
                       int causal) const {
    GemmShape sh{M, N, K, lda, ldb, a_mn, b_mn};
    sh.nh = nh_;
    sh.nb = b_;
    sh.a_sh = a_sh;
    sh.a_sb = a_sb;
    sh.b_sh = b_sh;
    sh.b_sb = b_sb;
    sh.c_sh = c_sh;
    sh.c_sb = c_sb;
    sh.causal = causal;
    return sh;
  }

  // ---- MoE feed-forward ---------------------------------------------------------
  // E experts batched in one GEMM: batch index = expert, per-expert slot rows
  // at stride C, per-expert weights at stride ex_stride.
  GemmShape expert_shape(int M, int N, int K, int lda, int ldb, int a_mn, int b_mn, int64_t a_sh,
                         int64_t b_sh, int64_t c_sh) const {
    GemmShape sh{M, N, K, lda, ldb, a_mn, b_mn};
    sh.nh = E_;
    sh.nb = 1;
    sh.a_sh = a_sh;
    sh.b_sh = b_sh;
    sh.c_sh = c_sh;
    return sh;
  }
  void moe_fwd(const LayerActs& a, const uint16_t* W, uint16_t* out, cudaStream_t s) const {
    const BlockOff& o = bo_;
    const int64_t EC = int64_t(E_) * C_;
    {  // router logits [T, E] fp32
      GemmShape sh{int(T_), E_, h_, h_, h_, 0, 0};
      Epilogue e;
      e.out_bf16 = 0;
      e.ldc = E_;
      gemm_tc_bf16(a.ln2, W + o.w_router, a.logits, sh, e, s);
    }
    moe_route(a.logits, int(T_), E_, K_, a.probs, a.sel, a.gate, s);
    moe_dispatch(a.sel, int(T_), E_, K_, C_, a.pos, a.slot_tok, a.slot_k, s);
    moe_gather(a.ln2, a.slot_tok, int(EC), h_, a.xp, s);
    if (sw_) {  // H_e = silu(Xp_e Wg_e^T) * (Xp_e Wu_e^T)  (fc1 output kept for the backward)
      GemmShape sh = expert_shape(C_, f1_, h_, h_, h_, 0, 0, int64_t(C_) * h_, o.ex_stride, int64_t(C_) * f1_);
      Epilogue e;
      e.ldc = f1_;
      gemm_tc_bf16(a.xp, W + o.w_fc1, a.fpre, sh, e, s);
      swiglu_fwd(a.fpre, a.fact, EC, f_, s);
    } else {  // H_e = GELU(Xp_e W1_e^T + b1_e)  (pre-activation kept for the backward)
      GemmShape sh = expert_shape(C_, f_, h_, h_, h_, 0, 0, int64_t(C_) * h_, o.ex_stride, int64_t(C_) * f_);
      Epilogue e;
      e.bias_any = W + o.b_fc1;
      e.bias_sh = o.ex_stride;
      e.act = kActGelu;
      e.aux = a.fpre;
      e.ldaux = f_;
      e.ldc = f_;
      gemm_tc_bf16(a.xp, W + o.w_fc1, a.fact, sh, e, s);
    }
    {  // Y_e = H_e W2_e^T (+ b2_e)
      GemmShape sh = expert_shape(C_, h_, f_, f_, f_, 0, 0, int64_t(C_) * f_, o.ex_stride, int64_t(C_) * h_);
      Epilogue e;
      if (!sw_) {
        e.bias_any = W + o.b_fc2;
        e.bias_sh = o.ex_stride;
      }
      e.ldc = h_;
      gemm_tc_bf16(a.fact, W + o.w_fc2, a.y, sh, e, s);
    }
    moe_combine(a.y, a.pos, a.gate, a.xm, int(T_), K_, h_, out, s);  // + residual
  }
  // Backward of the MoE FFN from dout (grad of the block output); leaves the
  // grad of the ln2 output in B->dattn (scratch here).  Weight gradients run
  // on ws after to_side().
  template <class ToSide>
  void moe_bwd(GptBuffers* B, const LayerActs& a, const uint16_t* W, const GradTarget& g, const uint16_t* dout,
               cudaStream_t s, cudaStream_t ws, ToSide to_side) const {
    const BlockOff& o = bo_;
    const int64_t EC = int64_t(E_) * C_;
    moe_combine_bwd(dout, a.y, a.pos, a.gate, a.slot_tok, a.slot_k, int(T_), K_, int(EC), h_, B->moe_dy,
                    B->moe_dgate, s);
    to_side();
    {  // dW2_e [h, f] = dY_e^T H_e ; db2_e = colsum dY_e
      GemmShape sh = expert_shape(h_, f_, C_, h_, f_, 1, 1, int64_t(C_) * h_, int64_t(C_) * f_, o.ex_stride);
      Epilogue e;
      e.mode = g.mode;
      e.out_bf16 = g.bf16;
      e.ldc = f_;
      gemm_tc_bf16(B->moe_dy, a.fact, gptr(g, o.w_fc2), sh, e, ws);
      for (int x = 0; x < E_ && !sw_; ++x) {
        colsum_partial(B->moe_dy + int64_t(x) * C_ * h_, C_, h_, B->part_side, kChunks, ws);
        colsum_finalize(B->part_side, kChunks, h_, gptr(g, o.b_fc2 + x * o.ex_stride), g.bf16, g.mode, ws);
      }
    }
    if (sw_) {  // dH_e = SwiGLU'(fc1 out) applied to dY_e W2_e
      GemmShape sh = expert_shape(C_, f_, h_, h_, f_, 0, 1, int64_t(C_) * h_, o.ex_stride, int64_t(C_) * f_);
      Epilogue e;
      e.ldc = f_;
      gemm_tc_bf16(B->moe_dy, W + o.w_fc2, B->moe_dact, sh, e, s);
      swiglu_bwd(a.fpre, B->moe_dact, B->moe_dh, EC, f_, s);
    } else {  // dH_e = GELU'(pre) * (dY_e W2_e)
      GemmShape sh = expert_shape(C_, f_, h_, h_, f_, 0, 1, int64_t(C_) * h_, o.ex_stride, int64_t(C_) * f_);
      Epilogue e;
      e.act = kActGeluGrad;
      e.aux = a.fpre;
      e.ldaux = f_;
      e.ldc = f_;
      gemm_tc_bf16(B->moe_dy, W + o.w_fc2, B->moe_dh, sh, e, s);
    }
    to_side();
    {  // dW1_e [f1, h] = dH_e^T Xp_e ; db1_e = colsum dH_e
      GemmShape sh = expert_shape(f1_, h_, C_, f1_, h_, 1, 1, int64_t(C_) * f1_, int64_t(C_) * h_, o.ex_stride);
      Epilogue e;
      e.mode = g.mode;
      e.out_bf16 = g.bf16;
      e.ldc = h_;
      gemm_tc_bf16(B->moe_dh, a.xp, gptr(g, o.w_fc1), sh, e, ws);
      for (int x = 0; x < E_ && !sw_; ++x) {
        colsum_partial(B->moe_dh + int64_t(x) * C_ * f_, C_, f_, B->part_side, kChunks, ws);
        colsum_finalize(B->part_side, kChunks, f_, gptr(g, o.b_fc1 + x * o.ex_stride), g.bf16, g.mode, ws);
      }
    }
    {  // dXp_e = dH_e W1_e
      GemmShape sh = expert_shape(C_, h_, f1_, f1_, h_, 0, 1, int64_t(C_) * f1_, o.ex_stride, int64_t(C_) * h_);
      Epilogue e;
      e.ldc = h_;
      gemm_tc_bf16(B->moe_dh, W + o.w_fc1, B->moe_dxp, sh, e, s);
    }
    moe_gather_bwd(B->moe_dxp, a.pos, int(T_), K_, h_, B->dln, s);  // expert path of d ln2-out
    moe_router_bwd(a.probs, a.sel, B->moe_dgate, int(T_), E_, K_, B->moe_dlogits, s);
    to_side();
    {  // dW_router [E, h] = dlogits^T ln2
      GemmShape sh{E_, h_, int(T_), E_, h_, 1, 1};
      Epilogue e;
      e.mode = g.mode;
      e.out_bf16 = g.bf16;
      e.ldc = h_;
      gemm_tc_bf16(B->moe_dlogits, a.ln2, gptr(g, o.w_router), sh, e, ws);
    }
    {  // d ln2-out = expert path + dlogits W_router
      GemmShape sh{int(T_), h_, E_, E_, h_, 0, 1};
      Epilogue e;
      e.resid = B->dln;
      e.ldres = h_;
      e.ldc = h_;
      gemm_tc_bf16(B->moe_dlogits, W + o.w_router, B->dattn, sh, e, s);
    }
  }

  // ---- forward ---------------------------------------------------------------
  void fwd(void* p, int l, const void* input_mb, const void* params, cudaStream_t s) override {
    auto* B = static_cast<GptBuffers*>(p);
    const auto* W = static_cast<const uint16_t*>(params);
    if (l == 0) {
      B->tokens = static_cast<const int*>(input_mb);
      embed_fwd(B->tokens, W, W + int64_t(V_) * h_, B->x[1], b_, S_, h_, s);
      return;
    }
    if (l == L_ + 1) {
      layernorm_fwd(B->x[l], W, W + h_, B->lnf, B->muf, B->rsf, int(T_), h_, s);
      Epilogue e;
      e.out_bf16 = 1;
      linear_fwd(B->lnf, W + 2 * h_, B->logits, V_, h_, e, s);
      cross_entropy(B->logits, B->tokens, b_, S_, V_, B->row_loss, B->loss, s);
      return;
    }
    block_fwd(B, l, W, true, s);
  }

  void recompute(void* p, int l, const void* params, cudaStream_t s) override {
    if (!c_.recompute || l < 1 || l > L_) return;  // embedding / head keep their outputs
    block_fwd(static_cast<GptBuffers*>(p), l, static_cast<const uint16_t*>(params), false, s);
  }
  int64_t launches_per_recompute(int l) const override {
    return c_.recompute && l >= 1 && l <= L_ ? launches_per_fwd() - (E_ > 0 ? 0 : 1) : 0;
  }

  // One transformer block.  need_out = false (FWD-recompute): only the
  // activations the BWD reads; the dense FFN's output GEMM (x[l+1], already
  // consumed) is skipped.
  void block_fwd(GptBuffers* B, int l, const uint16_t* W, bool need_out, cudaStream_t s) {
    const LayerActs& a = B->acts[l];
    const BlockOff& o = bo_;
    const int64_t h3 = 3 * int64_t(h_);
    layernorm_fwd(B->x[l], W + o.ln1_g, W + o.ln1_b, a.ln1, a.mu1, a.rs1, int(T_), h_, s);
    {
      Epilogue e;
      e.bias_any = W + o.b_qkv;
      linear_fwd(a.ln1, W + o.w_qkv, a.qkv, int(h3), h_, e, s);
    }
    // fused tcgen05 flash attention: S stays in TMEM; P (bf16) kept for the backward
    attention_fwd_tc(a.qkv, a.attn, nullptr, a.lse, b_, nh_, S_, h_, s);
    {
      Epilogue e;
      e.bias_any = W + o.b_o;
      e.resid = B->x[l];
      e.ldres = h_;
      linear_fwd(a.attn, W + o.w_o, a.xm, h_, h_, e, s);
    }
    layernorm_fwd(a.xm, W + o.ln2_g, W + o.ln2_b, a.ln2, a.mu2, a.rs2, int(T_), h_, s);
    if (E_ > 0) {
      moe_fwd(a, W, B->x[l + 1], s);  // recompute rewrites x[l+1] with identical values
      return;
    }
    if (sw_) {
      linear_fwd(a.ln2, W + o.w_fc1, a.fpre, f1_, h_, Epilogue{}, s);
      swiglu_fwd(a.fpre, a.fact, T_, f_, s);
    } else {
      Epilogue e;
      e.bias_any = W + o.b_fc1;
      e.act = kActGelu;
      e.aux = a.fpre;
      e.ldaux = f_;
      linear_fwd(a.ln2, W + o.w_fc1, a.fact, f_, h_, e, s);
    }
    if (need_out) {
      Epilogue e;
      if (!sw_) e.bias_any = W + o.b_fc2;
      e.resid = a.xm;
      e.ldres = h_;
      linear_fwd(a.fact, W + o.w_fc2, B->x[l + 1], h_, f_, e, s);
    }
  }

  // ---- backward --------------------------------------------------------------
  void bwd(void* p, int l, const void* params, const GradTarget& g, cudaStream_t s) override {
    auto* B = static_cast<GptBuffers*>(p);
    const auto* W = static_cast<const uint16_t*>(params);
    if (l == L_ + 1) {  // head: dlogits already in B->logits; dW_head on the side stream
      HZP_CUDA(cudaEventRecord(B->ev[0], s));
      HZP_CUDA(cudaStreamWaitEvent(B->side, B->ev[0], 0));
      linear_wgrad(B->logits, B->lnf, V_, h_, g, 2 * h_, -1, B, B->side);
      Epilogue e;
      linear_dgrad(B->logits, W + 2 * h_, B->dln, V_, h_, e, s);
      B->cur = 0;
      layernorm_bwd_fused(B->dln, B->x[l], W, B->muf, B->rsf, nullptr, B->dx[0], lnp(B, 0),
                          fc2_bias() ? fc2b_part(B, L_) : nullptr, int(T_), h_, s);
      ln_param_grads(B, g, 0, h_, s, lnp(B, 0));
      HZP_CUDA(cudaEventRecord(B->ev[1], B->side));
      HZP_CUDA(cudaStreamWaitEvent(s, B->ev[1], 0));
      return;
    }
    if (l == 0) {
      const int64_t nw = int64_t(V_) * h_, np = int64_t(S_) * h_;
      HZP_CUDA(cudaMemsetAsync(B->emb, 0, size_t(nw) * 4, s));
      embed_bwd(B->tokens, B->dx[B->cur], B->emb, B->emb + nw, b_, S_, h_, V_, B->emb_ws, s);
      grad_write(B->emb, nw + np, g.ptr, g.bf16, g.mode, s);
      return;
    }
    const LayerActs& a = B->acts[l];
    const BlockOff& o = bo_;
    const int64_t h3 = 3 * int64_t(h_);
    uint16_t* dout = B->dx[B->cur];
    uint16_t* din = B->dx[B->cur ^ 1];
    int nev = 0;
    auto to_side = [&] {  // everything issued on s so far is visible to the side stream
      HZP_CUDA(cudaEventRecord(B->ev[nev], s));
      HZP_CUDA(cudaStreamWaitEvent(B->side, B->ev[nev], 0));
      ++nev;
    };
    cudaStream_t ws = B->side;
    if (E_ > 0) {
      moe_bwd(B, a, W, g, dout, s, ws, to_side);
      layernorm_bwd_fused(B->dattn, a.xm, W + o.ln2_g, a.mu2, a.rs2, dout, B->dxm, lnp(B, 0), lnp(B, 4),
                          int(T_), h_, s);
      to_side();  // the LN parameter reductions are leaves too
      ln_param_grads(B, g, o.ln2_g, o.ln2_b, ws, lnp(B, 0));
      bias_from_ln(B, lnp(B, 4), g, o.b_o, ws);
    } else {
    // MLP
    to_side();
    // b_fc2 = column sum of dout, accumulated by the LN backward that made it
    if (fc2_bias()) bias_from_ln(B, fc2b_part(B, l), g, o.b_fc2, ws);
    linear_wgrad(dout, a.fact, h_, f_, g, o.w_fc2, -1, B, ws);
    if (sw_) {
      linear_dgrad(dout, W + o.w_fc2, B->dact, h_, f_, Epilogue{}, s);
      swiglu_bwd(a.fpre, B->dact, B->dfc1, T_, f_, s);
    } else {
      Epilogue e;
      e.act = kActGeluGrad;
      e.aux = a.fpre;
      e.ldaux = f_;
      linear_dgrad(dout, W + o.w_fc2, B->dfc1, h_, f_, e, s);
    }
    to_side();
    linear_wgrad(B->dfc1, a.ln2, f1_, h_, g, o.w_fc1, o.b_fc1, B, ws);
    {
      Epilogue e;
      linear_dgrad(B->dfc1, W + o.w_fc1, B->dln, f1_, h_, e, s);
    }
    layernorm_bwd_fused(B->dln, a.xm, W + o.ln2_g, a.mu2, a.rs2, dout, B->dxm, lnp(B, 0), lnp(B, 4), int(T_),
                        h_, s);
    to_side();  // the LN parameter reductions are leaves too
    ln_param_grads(B, g, o.ln2_g, o.ln2_b, ws, lnp(B, 0));
    bias_from_ln(B, lnp(B, 4), g, o.b_o, ws);  // b_o = column sum of dxm
    }
    // attention output projection
    to_side();
    linear_wgrad(B->dxm, a.attn, h_, h_, g, o.w_o, -1, B, ws);
    {
      Epilogue e;
      linear_dgrad(B->dxm, W + o.w_o, B->dattn, h_, h_, e, s);
    }
    // attention core: fused tcgen05 backward for dK, dV (P recomputed from
    // lse, dS^T emitted), then dQ = dS K as one transposed causal product
    attn_rowdot(B->dattn, a.attn, a.lse, B->D, b_, nh_, S_, hd_, s);
    // dS^T through HBM + one causal GEMM for dQ: measured faster than the
    // query-tile pass that recomputes P / dS in TMEM (attention_dq_tc,
    // 0.290 vs 0.341 ms for the whole backward at b4 / 16 heads / S 2048)
    attention_bwd_tc(a.qkv, B->dattn, a.lse, B->D, B->dqkv, B->dS, b_, nh_, S_, h_, s);
    attention_dq(a.qkv, B->dS, B->dqkv, b_, nh_, S_, h_, s);  // dQ = dS K
    to_side();
    linear_wgrad(B->dqkv, a.ln1, int(h3), h_, g, o.w_qkv, o.b_qkv, B, ws);
    {
      Epilogue e;
      linear_dgrad(B->dqkv, W + o.w_qkv, B->dln, int(h3), h_, e, s);
    }
    // ln1's partials in their own region: the side stream may still be
    // reducing ln2's; its dx sum is block l-1's b_fc2 (consumed at the start
    // of that block's backward, double-buffered by parity)
    float* part1 = lnp(B, 2);
    layernorm_bwd_fused(B->dln, B->x[l], W + o.ln1_g, a.mu1, a.rs1, B->dxm, din, part1,
                        fc2_bias() && l > 1 ? fc2b_part(B, l - 1) : nullptr, int(T_), h_, s);
    to_side();
    ln_param_grads(B, g, o.ln1_g, o.ln1_b, ws, part1);
    // join: the block's task ends when its weight gradients are written (the
    // RS / next block reuse the buffers they read)
    HZP_CUDA(cudaEventRecord(B->ev[nev], ws));
    HZP_CUDA(cudaStreamWaitEvent(s, B->ev[nev], 0));
    B->cur ^= 1;
  }

 private:
  ModelConfig c_;
  int h_, nh_, hd_, f_, V_, S_, b_, L_;
  int E_ = 0, K_ = 2, C_ = 0;  // MoE experts, top-k, slots per expert (E_ = 0: dense FFN)
  bool sw_ = false;            // SwiGLU feed-forward
  int f1_ = 0;                 // fc1 output width (2f for SwiGLU)
  int64_t T_;
  BlockOff bo_;
  std::vector<LayerRange> ranges_;
  int64_t P_ = 0;
};

}  // namespace

std::unique_ptr<Model> make_gpt_model(const ModelConfig& c) { return std::make_unique<GptModel>(c); }

}  // namespace hzp
