/*
 * TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT PATH.
 *
 * CPU restatement (plain C) of the AsyncHZP reference's numerical hot path,
 * used as the parity checker for the B200 kernels.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  Every routine cites the reference function it restates
 * (paths relative to /root/reference/proj).
 *
 * Pinning: tests/test_oracle.py checks every routine here against the
 * reference itself (oracle/_ref/libhzpref.so, compiled from the reference's
 * own sources by oracle/Makefile) and against tests/golden/*.json.
 *
 * Compiled with -O2 -ffp-contract=off and without -mfma so that every float
 * operation rounds exactly where the reference's g++ -O2 build rounds
 * (baseline x86-64 has no FMA, so the reference never contracts).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* mt19937_64 (std::mt19937_64) — used by seeded_uniform, src/train.cpp:17-27 */

typedef struct {
  uint64_t s[312];
  int i;
} orc_mt64;

static void mt64_seed(orc_mt64* m, uint64_t seed) {
  m->s[0] = seed;
  for (int k = 1; k < 312; ++k)
    m->s[k] = 6364136223846793005ULL * (m->s[k - 1] ^ (m->s[k - 1] >> 62)) + (uint64_t)k;
  m->i = 312;
}

static uint64_t mt64_next(orc_mt64* m) {
  if (m->i >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int k = 0; k < 312; ++k) {
      uint64_t x = (m->s[k] & upper) | (m->s[(k + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      m->s[k] = m->s[(k + 156) % 312] ^ xa;
    }
    m->i = 0;
  }
  uint64_t y = m->s[m->i++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* seeded_uniform<T> (src/train.cpp:17-27): (raw >> 11) * 2^-53 - 0.5 */
void orc_seeded_uniform_f64(double* out, size_t n, uint64_t seed) {
  orc_mt64 m;
  mt64_seed(&m, seed);
  for (size_t k = 0; k < n; ++k)
    out[k] = (double)(mt64_next(&m) >> 11) * 0x1p-53 - 0.5;
}

void orc_seeded_uniform_f32(float* out, size_t n, uint64_t seed) {
  orc_mt64 m;
  mt64_seed(&m, seed);
  for (size_t k = 0; k < n; ++k)
    out[k] = (float)((double)(mt64_next(&m) >> 11) * 0x1p-53 - 0.5);
}

/* Per-(step, rank, microbatch) input seed of run_case (src/train.cpp:504-506). */
uint64_t orc_batch_seed(uint64_t seed, int step, int rank, int mb) {
  return seed ^ (0x9E3779B97F4A7C15ULL *
                 ((uint64_t)step * 1024ULL + (uint64_t)rank * 32ULL + (uint64_t)mb + 1ULL));
}

/* ------------------------------------------------------------------------ */
/* bf16 round-to-nearest-even kept in fp32 (include/hzp/kernels.hpp:37-50)   */

float orc_bf16_round(float x) {
  uint32_t b;
  memcpy(&b, &x, 4);
  if ((b & 0x7F800000u) == 0x7F800000u) {
    /* inf stays inf; NaN keeps its payload with the quiet bit forced on */
    if (b & 0x007FFFFFu) b |= 0x00400000u;
  } else {
    b += 0x7FFFu + ((b >> 16) & 1u);
  }
  b &= 0xFFFF0000u;
  float r;
  memcpy(&r, &b, 4);
  return r;
}

void orc_bf16_round_vec(float* v, size_t n) {
  for (size_t k = 0; k < n; ++k) v[k] = orc_bf16_round(v[k]);
}

/* The host libm's tanhf (what the reference's std::tanh on float calls,
 * train.cpp:68-79) over a vector: the checker for the device restatement. */
void orc_tanhf_vec(const float* x, float* y, size_t n) {
  for (size_t k = 0; k < n; ++k) y[k] = tanhf(x[k]);
}

/* shard_elems (src/memory.cpp:13-15): ceil(n / parts) */
int64_t orc_shard_elems(int64_t n, int64_t parts) { return (n + parts - 1) / parts; }

/* ------------------------------------------------------------------------ */
/* Everything below is instantiated for float and double.                   */

#define ORC_DEFINE(T, SFX)                                                           \
                                                                                     \
  /* add_f32/add_f64 (src/kernels.cpp:11-17): acc[i] += src[i] */                   \
  static void add_into_##SFX(T* acc, const T* src, int64_t n) {                      \
    for (int64_t k = 0; k < n; ++k) acc[k] += src[k];                                \
  }                                                                                  \
                                                                                     \
  static int64_t mlp_params_##SFX(const int* dims, int nl) {                         \
    int64_t p = 0;                                                                   \
    for (int l = 0; l < nl; ++l) p += (int64_t)dims[l] * dims[l + 1] + dims[l + 1];  \
    return p;                                                                        \
  }                                                                                  \
                                                                                     \
  /* mlp_loss_grad (src/train.cpp:56-150).  Layer l's view is W (out x in,         \
   * row-major) followed by b (out) at a cumulative offset (train.cpp:42-53).      \
   * grad must hold P zeros on entry.  Returns the loss. */                          \
  T orc_mlp_loss_grad_##SFX(const int* dims, int nl, const T* params,                \
                            const T* inputs, int batch, T* grad) {                   \
    int64_t off[64];                                                                 \
    int64_t tot_act = 0, o = 0;                                                      \
    for (int l = 0; l < nl; ++l) {                                                   \
      off[l] = o;                                                                    \
      o += (int64_t)dims[l] * dims[l + 1] + dims[l + 1];                             \
    }                                                                                \
    for (int l = 0; l <= nl; ++l) tot_act += (int64_t)batch * dims[l];               \
    T* acts = (T*)malloc(sizeof(T) * (size_t)tot_act);                               \
    int64_t aoff[65];                                                                \
    aoff[0] = 0;                                                                     \
    for (int l = 0; l < nl; ++l) aoff[l + 1] = aoff[l] + (int64_t)batch * dims[l];   \
    memcpy(acts, inputs, sizeof(T) * (size_t)batch * dims[0]);                       \
    for (int l = 0; l < nl; ++l) {                                                   \
      const int in = dims[l], out = dims[l + 1];                                     \
      const T* w = params + off[l];                                                  \
      const T* b = w + (int64_t)in * out;                                            \
      const T* x = acts + aoff[l];                                                   \
      T* y = acts + aoff[l + 1];                                                     \
      const int hidden = l + 1 < nl;                                                 \
      for (int s = 0; s < batch; ++s)                                                \
        for (int oo = 0; oo < out; ++oo) {                                           \
          T acc = b[oo];                                                             \
          for (int i = 0; i < in; ++i)                                               \
            acc += w[(int64_t)oo * in + i] * x[(int64_t)s * in + i];                 \
          y[(int64_t)s * out + oo] = hidden ? (T)ORC_TANH_##SFX(acc) : acc;          \
        }                                                                            \
    }                                                                                \
    const int od = dims[nl];                                                         \
    const T* yl = acts + aoff[nl];                                                   \
    const int64_t ny = (int64_t)batch * od;                                          \
    T lacc = (T)0;                                                                   \
    for (int64_t k = 0; k < ny; ++k) lacc += yl[k] * yl[k];                          \
    const T loss = lacc / ((T)2 * (T)batch * (T)od);                                 \
    const T scale = (T)1 / ((T)batch * (T)od);                                       \
    T* delta = (T*)malloc(sizeof(T) * (size_t)ny);                                   \
    for (int64_t k = 0; k < ny; ++k) delta[k] = yl[k] * scale;                       \
    for (int l = nl - 1; l >= 0; --l) {                                              \
      const int in = dims[l], out = dims[l + 1];                                     \
      const T* w = params + off[l];                                                  \
      const T* x = acts + aoff[l];                                                   \
      T* gw = grad + off[l];                                                         \
      T* gb = gw + (int64_t)in * out;                                                \
      for (int s = 0; s < batch; ++s)                                                \
        for (int oo = 0; oo < out; ++oo) {                                           \
          const T d = delta[(int64_t)s * out + oo];                                  \
          gb[oo] += d;                                                               \
          for (int i = 0; i < in; ++i)                                               \
            gw[(int64_t)oo * in + i] += d * x[(int64_t)s * in + i];                  \
        }                                                                            \
      if (l > 0) {                                                                   \
        T* prev = (T*)malloc(sizeof(T) * (size_t)batch * in);                        \
        for (int s = 0; s < batch; ++s)                                              \
          for (int i = 0; i < in; ++i) {                                             \
            T acc = (T)0;                                                            \
            for (int oo = 0; oo < out; ++oo)                                         \
              acc += w[(int64_t)oo * in + i] * delta[(int64_t)s * out + oo];         \
            const T a = x[(int64_t)s * in + i];                                      \
            prev[(int64_t)s * in + i] = acc * ((T)1 - a * a);                        \
          }                                                                          \
        free(delta);                                                                 \
        delta = prev;                                                                \
      }                                                                              \
    }                                                                                \
    free(delta);                                                                     \
    free(acts);                                                                      \
    return loss;                                                                     \
  }                                                                                  \
                                                                                     \
  /* adam_update (src/train.cpp:171-189); bias corrections exactly as             \
   * train.cpp:179-180: (T)pow((T)beta, step) evaluated in double. */              \
  void orc_adam_update_##SFX(T* master, T* m, T* v, const T* g, int64_t n,           \
                             int step, double lr_d, double b1_d, double b2_d,        \
                             double eps_d) {                                         \
    const T lr = (T)lr_d, b1 = (T)b1_d, b2 = (T)b2_d, eps = (T)eps_d;                \
    const T bc1 = (T)1 - (T)pow((double)(T)b1_d, step);                              \
    const T bc2 = (T)1 - (T)pow((double)(T)b2_d, step);                              \
    for (int64_t k = 0; k < n; ++k) {                                                \
      const T gk = g[k];                                                             \
      m[k] = b1 * m[k] + ((T)1 - b1) * gk;                                           \
      v[k] = b2 * v[k] + ((T)1 - b2) * gk * gk;                                      \
      const T mhat = m[k] / bc1;                                                     \
      const T vhat = v[k] / bc2;                                                     \
      master[k] -= lr * mhat / ((T)ORC_SQRT_##SFX(vhat) + eps);                      \
    }                                                                                \
  }                                                                                  \
                                                                                     \
  /* Collectives over flat per-rank buffers (src/collective.cpp:44-115).           \
   * all_gather: out = concat(shard_0..shard_{g-1}).                               \
   * reduce_scatter: sum = full_0; sum += full_r (ascending); rank i keeps seg i.  \
   * all_reduce: same ascending sum, replicated. */                                  \
  void orc_all_gather_##SFX(const T* shards, int g, int64_t per, T* out) {           \
    memcpy(out, shards, sizeof(T) * (size_t)(g * per));                              \
  }                                                                                  \
  int orc_reduce_scatter_##SFX(const T* fulls, int g, int64_t total, T* out) {       \
    if (total % g != 0) return 1; /* CollectiveError::ShapeMismatch */               \
    T* sum = (T*)malloc(sizeof(T) * (size_t)total);                                  \
    memcpy(sum, fulls, sizeof(T) * (size_t)total);                                   \
    for (int r = 1; r < g; ++r) add_into_##SFX(sum, fulls + (int64_t)r * total, total); \
    memcpy(out, sum, sizeof(T) * (size_t)total); /* out[i*seg..] = segment i */      \
    free(sum);                                                                       \
    return 0;                                                                        \
  }                                                                                  \
  void orc_all_reduce_##SFX(const T* ts, int g, int64_t n, T* out) {                 \
    memcpy(out, ts, sizeof(T) * (size_t)n);                                          \
    for (int r = 1; r < g; ++r) add_into_##SFX(out, ts + (int64_t)r * n, n);         \
  }                                                                                  \
                                                                                     \
  /* Sharded state, flat per rank: param[dp][s3], grad[dp][s2],                    \
   * master/mom/var[dp][s1], adam_step[dp] (include/hzp/train.hpp:73-83).          \
   * shard_init (src/train.cpp:224-253). */                                          \
  void orc_shard_init_##SFX(const int* dims, int nl, int dp, int z1, int z2, int z3, \
                            uint64_t seed, int bf16_working, T* param, T* grad,      \
                            T* master, T* mom, T* var, int* adam_step) {             \
    const int64_t p = mlp_params_##SFX(dims, nl);                                    \
    const int64_t s1 = orc_shard_elems(p, z1), s2 = orc_shard_elems(p, z2),          \
                  s3 = orc_shard_elems(p, z3);                                       \
    T* mas = (T*)calloc((size_t)(s1 * z1 > p ? s1 * z1 : p), sizeof(T));             \
    T* wrk = (T*)calloc((size_t)(s3 * z3 > p ? s3 * z3 : p), sizeof(T));             \
    ORC_UNIFORM_##SFX(mas, (size_t)p, seed);                                         \
    memcpy(wrk, mas, sizeof(T) * (size_t)p);                                         \
    ORC_BF16_##SFX(wrk, p, bf16_working);                                            \
    for (int r = 0; r < dp; ++r) {                                                   \
      const int i1 = r % z1, i3 = r % z3;                                            \
      memcpy(master + (int64_t)r * s1, mas + i1 * s1, sizeof(T) * (size_t)s1);       \
      memset(mom + (int64_t)r * s1, 0, sizeof(T) * (size_t)s1);                      \
      memset(var + (int64_t)r * s1, 0, sizeof(T) * (size_t)s1);                      \
      memcpy(param + (int64_t)r * s3, wrk + i3 * s3, sizeof(T) * (size_t)s3);        \
      memset(grad + (int64_t)r * s2, 0, sizeof(T) * (size_t)s2);                     \
      adam_step[r] = 0;                                                              \
    }                                                                                \
    free(mas);                                                                       \
    free(wrk);                                                                       \
  }                                                                                  \
                                                                                     \
  /* train_step_hzp (src/train.cpp:267-381).  inputs[r][mb] is a (batch x dims[0]) \
   * row-major matrix at inputs + (r*num_mb + mb)*batch*dims[0].                   \
   * losses[dp] receives per-rank summed losses.  If per_rank_grads is non-NULL   \
   * it receives each (mb, rank)'s unsharded gradient, padded to s2*z2, at         \
   * [(mb*dp + r)*s2*z2] — the RS inputs, used to drive tier-A kernel parity. */   \
  void orc_train_step_hzp_##SFX(const int* dims, int nl, int dp, int z1, int z2,     \
                                int z3, int num_mb, int batch, const T* inputs,      \
                                double lr, double b1, double b2, double eps,         \
                                int bf16_working, T* param, T* grad, T* master,      \
                                T* mom, T* var, int* adam_step, T* losses,           \
                                T* per_rank_grads) {                                 \
    const int64_t p = mlp_params_##SFX(dims, nl);                                    \
    const int64_t s1 = orc_shard_elems(p, z1), s2 = orc_shard_elems(p, z2),          \
                  s3 = orc_shard_elems(p, z3);                                       \
    const int replicas = dp / z2;                                                    \
    const int64_t in_elems = (int64_t)batch * dims[0];                               \
    /* [AG-Z3] every rank of each contiguous Z3 group gets concat(shards) */        \
    T* full = (T*)malloc(sizeof(T) * (size_t)dp * (size_t)(s3 * z3));                \
    for (int r = 0; r < dp; ++r) {                                                   \
      const int g0 = (r / z3) * z3;                                                  \
      orc_all_gather_##SFX(param + (int64_t)g0 * s3, z3, s3,                         \
                           full + (int64_t)r * s3 * z3);                             \
    }                                                                                \
    for (int r = 0; r < dp; ++r) losses[r] = (T)0;                                   \
    memset(grad, 0, sizeof(T) * (size_t)dp * (size_t)s2);                            \
    T* mbg = (T*)malloc(sizeof(T) * (size_t)dp * (size_t)(s2 * z2));                 \
    T* seg = (T*)malloc(sizeof(T) * (size_t)(s2 * z2));                              \
    for (int mb = 0; mb < num_mb; ++mb) {                                            \
      for (int r = 0; r < dp; ++r) {                                                 \
        T* gr = mbg + (int64_t)r * s2 * z2;                                          \
        memset(gr, 0, sizeof(T) * (size_t)(s2 * z2));                               \
        losses[r] += orc_mlp_loss_grad_##SFX(dims, nl, full + (int64_t)r * s3 * z3,  \
                                             inputs + ((int64_t)r * num_mb + mb) * in_elems, \
                                             batch, gr);                             \
        if (per_rank_grads)                                                          \
          memcpy(per_rank_grads + ((int64_t)mb * dp + r) * s2 * z2, gr,              \
                 sizeof(T) * (size_t)(s2 * z2));                                     \
      }                                                                              \
      /* [RS-Z2] per contiguous Z2 group, then grad_shard += own segment */         \
      for (int g0 = 0; g0 < dp; g0 += z2) {                                          \
        orc_reduce_scatter_##SFX(mbg + (int64_t)g0 * s2 * z2, z2, s2 * z2, seg);     \
        for (int i = 0; i < z2; ++i)                                                 \
          add_into_##SFX(grad + (int64_t)(g0 + i) * s2, seg + (int64_t)i * s2, s2);  \
      }                                                                              \
    }                                                                                \
    /* [DZP] ascending-replica all-reduce of Z2 grad shards {i, i+z2, ...} */       \
    if (replicas > 1) {                                                              \
      T* tmp = (T*)malloc(sizeof(T) * (size_t)replicas * (size_t)s2);                \
      T* red = (T*)malloc(sizeof(T) * (size_t)s2);                                   \
      for (int i = 0; i < z2; ++i) {                                                 \
        for (int b = 0; b < replicas; ++b)                                           \
          memcpy(tmp + (int64_t)b * s2, grad + (int64_t)(i + b * z2) * s2,           \
                 sizeof(T) * (size_t)s2);                                            \
        orc_all_reduce_##SFX(tmp, replicas, s2, red);                                \
        for (int b = 0; b < replicas; ++b)                                           \
          memcpy(grad + (int64_t)(i + b * z2) * s2, red, sizeof(T) * (size_t)s2);    \
      }                                                                              \
      free(tmp);                                                                     \
      free(red);                                                                     \
    }                                                                                \
    /* full gradient from ranks 0..z2-1, truncated to P, padded to s1*z1 */         \
    const int64_t gl = s1 * z1 > s2 * z2 ? s1 * z1 : s2 * z2;                        \
    T* gpad = (T*)calloc((size_t)gl, sizeof(T));                                     \
    for (int i = 0; i < z2; ++i)                                                     \
      memcpy(gpad + (int64_t)i * s2, grad + (int64_t)i * s2, sizeof(T) * (size_t)s2); \
    for (int64_t e = p; e < gl; ++e) gpad[e] = (T)0;                                 \
    /* [ZeRO-1 Adam] each rank on slice (r % z1) */                                 \
    for (int r = 0; r < dp; ++r) {                                                   \
      adam_step[r] += 1;                                                             \
      orc_adam_update_##SFX(master + (int64_t)r * s1, mom + (int64_t)r * s1,         \
                            var + (int64_t)r * s1, gpad + (int64_t)(r % z1) * s1,    \
                            s1, adam_step[r], lr, b1, b2, eps);                      \
    }                                                                                \
    /* [post-step AG] per Z1 group: concat masters, round, recut Z3 shards */       \
    const int64_t wl = s3 * z3 > s1 * z1 ? s3 * z3 : s1 * z1;                        \
    T* wrk = (T*)calloc((size_t)wl, sizeof(T));                                      \
    for (int g0 = 0; g0 < dp; g0 += z1) {                                            \
      memset(wrk, 0, sizeof(T) * (size_t)wl);                                        \
      for (int i = 0; i < z1; ++i)                                                   \
        memcpy(wrk + (int64_t)i * s1, master + (int64_t)(g0 + i) * s1,               \
               sizeof(T) * (size_t)s1);                                              \
      for (int64_t e = p; e < wl; ++e) wrk[e] = (T)0;                                \
      ORC_BF16_##SFX(wrk, p, bf16_working);                                          \
      for (int i = 0; i < z1; ++i) {                                                 \
        const int r = g0 + i;                                                        \
        memcpy(param + (int64_t)r * s3, wrk + (int64_t)(r % z3) * s3,                \
               sizeof(T) * (size_t)s3);                                              \
      }                                                                              \
    }                                                                                \
    free(wrk);                                                                       \
    free(gpad);                                                                      \
    free(seg);                                                                       \
    free(mbg);                                                                       \
    free(full);                                                                      \
  }                                                                                  \
                                                                                     \
  /* train_step_baseline (src/train.cpp:383-420) with ReductionOrder{dp,z2}. */      \
  void orc_train_step_baseline_##SFX(const int* dims, int nl, int dp, int z2,        \
                                     int num_mb, int batch, const T* inputs,         \
                                     double lr, double b1, double b2, double eps,    \
                                     int bf16_working, T* working, T* master,        \
                                     T* mom, T* var, int* adam_step, T* losses) {    \
    const int64_t p = mlp_params_##SFX(dims, nl);                                    \
    const int64_t in_elems = (int64_t)batch * dims[0];                               \
    T* total = (T*)calloc((size_t)p, sizeof(T));                                     \
    T* bacc = (T*)malloc(sizeof(T) * (size_t)p);                                     \
    T* bsum = (T*)malloc(sizeof(T) * (size_t)p);                                     \
    T* g = (T*)malloc(sizeof(T) * (size_t)p);                                        \
    for (int r = 0; r < dp; ++r) losses[r] = (T)0;                                   \
    for (int g0 = 0; g0 < dp; g0 += z2) {                                            \
      memset(bacc, 0, sizeof(T) * (size_t)p);                                        \
      for (int mb = 0; mb < num_mb; ++mb) {                                          \
        memset(bsum, 0, sizeof(T) * (size_t)p);                                      \
        for (int i = 0; i < z2; ++i) {                                               \
          const int r = g0 + i;                                                      \
          memset(g, 0, sizeof(T) * (size_t)p);                                       \
          losses[r] += orc_mlp_loss_grad_##SFX(dims, nl, working,                    \
                                               inputs + ((int64_t)r * num_mb + mb) * in_elems, \
                                               batch, g);                            \
          add_into_##SFX(bsum, g, p);                                                \
        }                                                                            \
        add_into_##SFX(bacc, bsum, p);                                               \
      }                                                                              \
      add_into_##SFX(total, bacc, p);                                                \
    }                                                                                \
    *adam_step += 1;                                                                 \
    orc_adam_update_##SFX(master, mom, var, total, p, *adam_step, lr, b1, b2, eps);  \
    memcpy(working, master, sizeof(T) * (size_t)p);                                  \
    ORC_BF16_##SFX(working, p, bf16_working);                                        \
    free(total);                                                                     \
    free(bacc);                                                                      \
    free(bsum);                                                                      \
    free(g);                                                                         \
  }

#define ORC_TANH_f32 tanhf
#define ORC_TANH_f64 tanh
#define ORC_SQRT_f32 sqrtf
#define ORC_SQRT_f64 sqrt
#define ORC_UNIFORM_f32 orc_seeded_uniform_f32
#define ORC_UNIFORM_f64 orc_seeded_uniform_f64
/* bf16_round_vec (src/train.cpp:155-162): a no-op for double */
#define ORC_BF16_f32(v, n, on) \
  do {                         \
    if (on) orc_bf16_round_vec((v), (size_t)(n)); \
  } while (0)
#define ORC_BF16_f64(v, n, on) \
  do {                         \
    (void)(v);                 \
    (void)(n);                 \
    (void)(on);                \
  } while (0)

ORC_DEFINE(float, f32)
ORC_DEFINE(double, f64)

/* Inputs of one run_case step for all (rank, mb) (src/train.cpp:501-508). */
void orc_make_inputs_f32(const int* dims, int dp, int num_mb, int batch, uint64_t seed,
                         int step, float* out) {
  const int64_t n = (int64_t)batch * dims[0];
  for (int r = 0; r < dp; ++r)
    for (int mb = 0; mb < num_mb; ++mb)
      orc_seeded_uniform_f32(out + ((int64_t)r * num_mb + mb) * n, (size_t)n,
                             orc_batch_seed(seed, step, r, mb));
}

void orc_make_inputs_f64(const int* dims, int dp, int num_mb, int batch, uint64_t seed,
                         int step, double* out) {
  const int64_t n = (int64_t)batch * dims[0];
  for (int r = 0; r < dp; ++r)
    for (int mb = 0; mb < num_mb; ++mb)
      orc_seeded_uniform_f64(out + ((int64_t)r * num_mb + mb) * n, (size_t)n,
                             orc_batch_seed(seed, step, r, mb));
}

/* FNV-1a 64 over raw bytes — the hash used by the golden fixtures. */
uint64_t orc_fnv1a(const void* data, size_t n) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t k = 0; k < n; ++k) {
    h ^= p[k];
    h *= 0x100000001b3ULL;
  }
  return h;
}
