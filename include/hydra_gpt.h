/* hydra_gpt.h — physical layout and synthetic data of the GPT-2 the executor trains.
 *
 * Shared (header-only, C) by the product library and the CPU oracle so both index the
 * same flat fp32 parameter vector and draw the same synthetic tokens and init.
 *
 * Model = the reference cost model's layer chain (model.cpp:165-216):
 *   layer 0          embed : wte [V x d], wpe [T x d]
 *   layer 1..L       block : ln1 g,b [d]; W_qkv [3d x d]; b_qkv [3d]; W_o [d x d]; b_o [d];
 *                            ln2 g,b [d]; W_fc [4d x d]; b_fc [4d]; W_pr [d x 4d]; b_pr [d]
 *   layer L+1        head  : ln_f g,b [d]; logits = ln_f(h) wte^T (tied to layer 0's wte)
 * Weights are [out x in] row-major (y = x W^T + b). Heads: H = max(1, d/64), head dim 64.
 * Each tensor is padded to a multiple of 32 floats; layers are contiguous in layer order
 * so a shard [l0, l1) is one contiguous byte range (one cudaMemcpyAsync per ParamLoad).
 */
#ifndef HYDRA_GPT_H_
#define HYDRA_GPT_H_

#include <math.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HY_VOCAB 50257
#define HY_VOCAB_PAD 50304 /* logits row stride (multiple of 128) */

typedef struct {
  int V, d, L, T, B, H;
} hy_dims;

static inline long hy_pad32(long n) { return (n + 31) / 32 * 32; }

/* tensor slots inside a block layer */
enum {
  HY_LN1_G = 0, HY_LN1_B, HY_WQKV, HY_BQKV, HY_WO, HY_BO, HY_LN2_G, HY_LN2_B, HY_WFC, HY_BFC, HY_WPR, HY_BPR,
  HY_BLOCK_TENSORS
};

static inline long hy_block_tensor_size(int d, int t) {
  switch (t) {
    case HY_WQKV: return 3L * d * d;
    case HY_BQKV: return 3L * d;
    case HY_WO: return (long)d * d;
    case HY_WFC: return 4L * d * d;
    case HY_BFC: return 4L * d;
    case HY_WPR: return 4L * d * d;
    default: return d;
  }
}

static inline long hy_block_tensor_offset(int d, int t) {
  long off = 0;
  for (int i = 0; i < t; ++i) off += hy_pad32(hy_block_tensor_size(d, i));
  return off;
}

static inline long hy_layer_floats(const hy_dims* m, int layer) {
  if (layer == 0) return hy_pad32((long)m->V * m->d) + hy_pad32((long)m->T * m->d);
  if (layer == m->L + 1) return 2 * hy_pad32(m->d);
  return hy_block_tensor_offset(m->d, HY_BLOCK_TENSORS);
}

static inline long hy_layer_offset(const hy_dims* m, int layer) {
  long off = 0;
  for (int l = 0; l < layer; ++l) off += hy_layer_floats(m, l);
  return off;
}

static inline long hy_total_floats(const hy_dims* m) { return hy_layer_offset(m, m->L + 2); }

/* ---- deterministic synthetic data ---------------------------------------------- */
static inline uint64_t hy_mix64(uint64_t x) { /* splitmix64 finalizer */
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* token t of row r (0 <= t <= T) of minibatch mb of job j: inputs use t in [0,T),
 * targets t in [1,T]. Uniform in [0, V). */
static inline int32_t hy_token(uint64_t seed, int job, int mb, int row, int t) {
  uint64_t h = hy_mix64(seed ^ 0x48594452ull);
  h = hy_mix64(h ^ (uint64_t)(uint32_t)job);
  h = hy_mix64(h ^ (uint64_t)(uint32_t)mb);
  h = hy_mix64(h ^ ((uint64_t)(uint32_t)row << 32 | (uint32_t)t));
  return (int32_t)(h % (uint64_t)HY_VOCAB);
}

/* N(0,1) via Box-Muller on two counter-based uniforms. */
static inline float hy_normal(uint64_t key, uint64_t idx) {
  const uint64_t a = hy_mix64(key ^ (idx * 2 + 0x5851F42D4C957F2Dull));
  const uint64_t b = hy_mix64(key ^ (idx * 2 + 1 + 0x14057B7EF767814Full));
  const double u1 = ((double)(a >> 11) + 1.0) * (1.0 / 9007199254740993.0);
  const double u2 = (double)(b >> 11) * (1.0 / 9007199254740992.0);
  return (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}

/* GPT-2 init of one layer's parameters (padding stays 0): N(0, 0.02) for wte/wpe and
 * input projections, N(0, 0.02/sqrt(2L)) for the residual projections W_o, W_pr, LN
 * gains 1, biases 0. `model_key` identifies the model (jobs of one model share init). */
static inline void hy_init_layer(const hy_dims* m, uint64_t model_key, int layer, float* p) {
  const long n = hy_layer_floats(m, layer);
  for (long i = 0; i < n; ++i) p[i] = 0.f;
  const uint64_t key = hy_mix64(model_key ^ ((uint64_t)layer << 20));
  const int d = m->d;
  if (layer == 0) {
    const long nw = (long)m->V * d, np = (long)m->T * d;
    for (long i = 0; i < nw; ++i) p[i] = 0.02f * hy_normal(key, (uint64_t)i);
    float* wpe = p + hy_pad32(nw);
    for (long i = 0; i < np; ++i) wpe[i] = 0.02f * hy_normal(key ^ 0xABCDEFull, (uint64_t)i);
    return;
  }
  if (layer == m->L + 1) {
    for (int i = 0; i < d; ++i) p[i] = 1.f;
    return;
  }
  const float resid = (float)(0.02 / sqrt(2.0 * m->L));
  for (int t = 0; t < HY_BLOCK_TENSORS; ++t) {
    float* q = p + hy_block_tensor_offset(d, t);
    const long sz = hy_block_tensor_size(d, t);
    if (t == HY_LN1_G || t == HY_LN2_G) {
      for (long i = 0; i < sz; ++i) q[i] = 1.f;
    } else if (t == HY_WQKV || t == HY_WFC) {
      for (long i = 0; i < sz; ++i) q[i] = 0.02f * hy_normal(key ^ (uint64_t)t, (uint64_t)i);
    } else if (t == HY_WO || t == HY_WPR) {
      for (long i = 0; i < sz; ++i) q[i] = resid * hy_normal(key ^ (uint64_t)t, (uint64_t)i);
    }
  }
}

#ifdef __cplusplus
}
#endif
#endif /* HYDRA_GPT_H_ */
