/* ORACLE / TEST INFRASTRUCTURE ONLY — see gpt_oracle.h for scope and citations.
 * Plain C: fp32 tensors, every dot product / reduction accumulated in double. */
#include "gpt_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#define LN_EPS 1e-5

int oracle_threads(void) { return omp_get_max_threads(); }

static float* falloc(long n) {
  float* p = (float*)calloc((size_t)(n > 0 ? n : 1), sizeof(float));
  return p;
}

/* C[M,N] (+)= A[M,K] * B[N,K]^T (+ bias[N]) */
static void mm_nt(int M, int N, int K, const float* A, long lda, const float* B, long ldb, float* C, long ldc,
                  const float* bias, int acc) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < M; ++i) {
    const float* a = A + (long)i * lda;
    for (int j = 0; j < N; ++j) {
      const float* b = B + (long)j * ldb;
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += (double)a[k] * (double)b[k];
      if (bias) s += bias[j];
      float* c = C + (long)i * ldc + j;
      *c = acc ? (float)(*c + s) : (float)s;
    }
  }
}

/* C[M,N] (+)= A[M,K] * B[K,N] */
static void mm_nn(int M, int N, int K, const float* A, long lda, const float* B, long ldb, float* C, long ldc,
                  int acc) {
#pragma omp parallel
  {
    double* row = (double*)malloc(sizeof(double) * (size_t)N);
#pragma omp for schedule(static)
    for (int i = 0; i < M; ++i) {
      for (int j = 0; j < N; ++j) row[j] = 0.0;
      const float* a = A + (long)i * lda;
      for (int k = 0; k < K; ++k) {
        const double av = a[k];
        if (av == 0.0) continue;
        const float* b = B + (long)k * ldb;
        for (int j = 0; j < N; ++j) row[j] += av * (double)b[j];
      }
      float* c = C + (long)i * ldc;
      for (int j = 0; j < N; ++j) c[j] = acc ? (float)(c[j] + row[j]) : (float)row[j];
    }
    free(row);
  }
}

/* C[M,N] (+)= A[K,M]^T * B[K,N]  (weight gradients) */
static void mm_tn(int M, int N, int K, const float* A, long lda, const float* B, long ldb, float* C, long ldc,
                  int acc) {
#pragma omp parallel
  {
    double* row = (double*)malloc(sizeof(double) * (size_t)N);
#pragma omp for schedule(static)
    for (int i = 0; i < M; ++i) {
      for (int j = 0; j < N; ++j) row[j] = 0.0;
      for (int k = 0; k < K; ++k) {
        const double av = A[(long)k * lda + i];
        if (av == 0.0) continue;
        const float* b = B + (long)k * ldb;
        for (int j = 0; j < N; ++j) row[j] += av * (double)b[j];
      }
      float* c = C + (long)i * ldc;
      for (int j = 0; j < N; ++j) c[j] = acc ? (float)(c[j] + row[j]) : (float)row[j];
    }
    free(row);
  }
}

static void colsum_acc(int M, int N, const float* X, float* out) {
#pragma omp parallel for schedule(static)
  for (int j = 0; j < N; ++j) {
    double s = 0.0;
    for (int i = 0; i < M; ++i) s += X[(long)i * N + j];
    out[j] = (float)(out[j] + s);
  }
}

static void ln_fwd(int rows, int d, const float* x, const float* g, const float* b, float* y, float* mean,
                   float* rstd) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (long)r * d;
    double mu = 0.0, var = 0.0;
    for (int i = 0; i < d; ++i) mu += xr[i];
    mu /= d;
    for (int i = 0; i < d; ++i) var += (xr[i] - mu) * (xr[i] - mu);
    var /= d;
    const double rs = 1.0 / sqrt(var + LN_EPS);
    float* yr = y + (long)r * d;
    for (int i = 0; i < d; ++i) yr[i] = (float)((xr[i] - mu) * rs * g[i] + b[i]);
    mean[r] = (float)mu;
    rstd[r] = (float)rs;
  }
}

/* dx += LN backward; dg, db += column sums */
static void ln_bwd(int rows, int d, const float* x, const float* g, const float* mean, const float* rstd,
                   const float* dy, float* dx, float* dg, float* db) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (long)r * d;
    const float* dyr = dy + (long)r * d;
    const double mu = mean[r], rs = rstd[r];
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < d; ++i) {
      const double xh = (xr[i] - mu) * rs, gy = (double)dyr[i] * g[i];
      s1 += gy;
      s2 += gy * xh;
    }
    s1 /= d;
    s2 /= d;
    float* dxr = dx + (long)r * d;
    for (int i = 0; i < d; ++i) {
      const double xh = (xr[i] - mu) * rs, gy = (double)dyr[i] * g[i];
      dxr[i] = (float)(dxr[i] + rs * (gy - s1 - xh * s2));
    }
  }
#pragma omp parallel for schedule(static)
  for (int i = 0; i < d; ++i) {
    double a = 0.0, c = 0.0;
    for (int r = 0; r < rows; ++r) {
      const double xh = (x[(long)r * d + i] - mean[r]) * (double)rstd[r];
      a += (double)dy[(long)r * d + i] * xh;
      c += dy[(long)r * d + i];
    }
    dg[i] = (float)(dg[i] + a);
    db[i] = (float)(db[i] + c);
  }
}

static double gelu(double x) { return 0.5 * x * (1.0 + tanh(0.7978845608028654 * (x + 0.044715 * x * x * x))); }
static double gelu_grad(double x) {
  const double k0 = 0.7978845608028654, k1 = 0.044715;
  const double t = tanh(k0 * (x + k1 * x * x * x));
  return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * k0 * (1.0 + 3.0 * k1 * x * x);
}

/* causal attention; qkv [B*T, 3D]; out [B*T, D] */
static void attn_fwd(const hy_dims* m, const float* qkv, float* out) {
  const int B = m->B, T = m->T, H = m->H, D = m->d, hd = D / H;
  const double scale = 1.0 / sqrt((double)hd);
#pragma omp parallel
  {
    double* p = (double*)malloc(sizeof(double) * (size_t)T);
#pragma omp for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b) {
      for (int h = 0; h < H; ++h) {
        for (int i = 0; i < T; ++i) {
          const float* q = qkv + ((long)b * T + i) * 3 * D + h * hd;
          double mx = -1e300;
          for (int j = 0; j <= i; ++j) {
            const float* k = qkv + ((long)b * T + j) * 3 * D + D + h * hd;
            double s = 0.0;
            for (int c = 0; c < hd; ++c) s += (double)q[c] * k[c];
            p[j] = s * scale;
            if (p[j] > mx) mx = p[j];
          }
          double z = 0.0;
          for (int j = 0; j <= i; ++j) {
            p[j] = exp(p[j] - mx);
            z += p[j];
          }
          float* o = out + ((long)b * T + i) * D + h * hd;
          for (int c = 0; c < hd; ++c) {
            double s = 0.0;
            for (int j = 0; j <= i; ++j) s += p[j] * qkv[((long)b * T + j) * 3 * D + 2 * D + h * hd + c];
            o[c] = (float)(s / z);
          }
        }
      }
    }
    free(p);
  }
}

/* dqkv (overwritten) from dout; recomputes probabilities */
static void attn_bwd(const hy_dims* m, const float* qkv, const float* dout, float* dqkv) {
  const int B = m->B, T = m->T, H = m->H, D = m->d, hd = D / H;
  const double scale = 1.0 / sqrt((double)hd);
  memset(dqkv, 0, sizeof(float) * (size_t)B * T * 3 * D);
#pragma omp parallel
  {
    double* p = (double*)malloc(sizeof(double) * (size_t)T);
    double* dp = (double*)malloc(sizeof(double) * (size_t)T);
    double* dq = (double*)malloc(sizeof(double) * (size_t)hd);
    double* dkv = (double*)malloc(sizeof(double) * (size_t)T * 2 * hd);
#pragma omp for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b) {
      for (int h = 0; h < H; ++h) {
        memset(dkv, 0, sizeof(double) * (size_t)T * 2 * hd);
        for (int i = 0; i < T; ++i) {
          const float* q = qkv + ((long)b * T + i) * 3 * D + h * hd;
          const float* go = dout + ((long)b * T + i) * D + h * hd;
          double mx = -1e300;
          for (int j = 0; j <= i; ++j) {
            const float* k = qkv + ((long)b * T + j) * 3 * D + D + h * hd;
            double s = 0.0;
            for (int c = 0; c < hd; ++c) s += (double)q[c] * k[c];
            p[j] = s * scale;
            if (p[j] > mx) mx = p[j];
          }
          double z = 0.0;
          for (int j = 0; j <= i; ++j) {
            p[j] = exp(p[j] - mx);
            z += p[j];
          }
          double delta = 0.0;
          for (int j = 0; j <= i; ++j) {
            p[j] /= z;
            const float* v = qkv + ((long)b * T + j) * 3 * D + 2 * D + h * hd;
            double s = 0.0;
            for (int c = 0; c < hd; ++c) s += (double)go[c] * v[c];
            dp[j] = s;
            delta += p[j] * s;
          }
          for (int c = 0; c < hd; ++c) dq[c] = 0.0;
          for (int j = 0; j <= i; ++j) {
            const double ds = p[j] * (dp[j] - delta) * scale;
            const float* k = qkv + ((long)b * T + j) * 3 * D + D + h * hd;
            double* dk = dkv + (long)j * 2 * hd;
            double* dv = dk + hd;
            for (int c = 0; c < hd; ++c) {
              dq[c] += ds * k[c];
              dk[c] += ds * q[c];
              dv[c] += p[j] * go[c];
            }
          }
          float* dqr = dqkv + ((long)b * T + i) * 3 * D + h * hd;
          for (int c = 0; c < hd; ++c) dqr[c] = (float)dq[c];
        }
        for (int j = 0; j < T; ++j) {
          float* dkr = dqkv + ((long)b * T + j) * 3 * D + D + h * hd;
          float* dvr = dkr + D;
          for (int c = 0; c < hd; ++c) {
            dkr[c] = (float)dkv[(long)j * 2 * hd + c];
            dvr[c] = (float)dkv[(long)j * 2 * hd + hd + c];
          }
        }
      }
    }
    free(p);
    free(dp);
    free(dq);
    free(dkv);
  }
}

typedef struct {
  float *ln1, *mean1, *rstd1, *qkv, *att, *hmid, *ln2, *mean2, *rstd2, *fc, *act;
} block_cache;

static void cache_alloc(const hy_dims* m, block_cache* c) {
  const long R = (long)m->B * m->T, d = m->d;
  c->ln1 = falloc(R * d);
  c->mean1 = falloc(R);
  c->rstd1 = falloc(R);
  c->qkv = falloc(R * 3 * d);
  c->att = falloc(R * d);
  c->hmid = falloc(R * d);
  c->ln2 = falloc(R * d);
  c->mean2 = falloc(R);
  c->rstd2 = falloc(R);
  c->fc = falloc(R * 4 * d);
  c->act = falloc(R * 4 * d);
}
static void cache_free(block_cache* c) {
  free(c->ln1); free(c->mean1); free(c->rstd1); free(c->qkv); free(c->att); free(c->hmid);
  free(c->ln2); free(c->mean2); free(c->rstd2); free(c->fc); free(c->act);
}

#define BT(p, t) ((p) + hy_block_tensor_offset(d, (t)))

/* h_out = block(h_in); fills the cache */
static void block_fwd(const hy_dims* m, const float* w, const float* h_in, float* h_out, block_cache* c) {
  const int R = m->B * m->T, d = m->d;
  ln_fwd(R, d, h_in, BT(w, HY_LN1_G), BT(w, HY_LN1_B), c->ln1, c->mean1, c->rstd1);
  mm_nt(R, 3 * d, d, c->ln1, d, BT(w, HY_WQKV), d, c->qkv, 3 * d, BT(w, HY_BQKV), 0);
  attn_fwd(m, c->qkv, c->att);
  mm_nt(R, d, d, c->att, d, BT(w, HY_WO), d, c->hmid, d, BT(w, HY_BO), 0);
  for (long i = 0; i < (long)R * d; ++i) c->hmid[i] += h_in[i];
  ln_fwd(R, d, c->hmid, BT(w, HY_LN2_G), BT(w, HY_LN2_B), c->ln2, c->mean2, c->rstd2);
  mm_nt(R, 4 * d, d, c->ln2, d, BT(w, HY_WFC), d, c->fc, 4 * d, BT(w, HY_BFC), 0);
  for (long i = 0; i < (long)R * 4 * d; ++i) c->act[i] = (float)gelu(c->fc[i]);
  mm_nt(R, d, 4 * d, c->act, 4 * d, BT(w, HY_WPR), 4 * d, h_out, d, BT(w, HY_BPR), 0);
  for (long i = 0; i < (long)R * d; ++i) h_out[i] += c->hmid[i];
}

/* dh (in: dL/dh_out, out: dL/dh_in); g: this block's gradient slice (+=) */
static void block_bwd(const hy_dims* m, const float* w, float* g, const float* h_in, const block_cache* c, float* dh) {
  const int R = m->B * m->T, d = m->d;
  const long n = (long)R * d;
  float* dact = falloc((long)R * 4 * d);
  float* dhm = falloc(n);
  float* dln = falloc(n);
  float* datt = falloc(n);
  float* dqkv = falloc((long)R * 3 * d);
  /* MLP: h_out = hmid + act W_pr^T + b_pr */
  mm_tn(d, 4 * d, R, dh, d, c->act, 4 * d, BT(g, HY_WPR), 4 * d, 1);
  colsum_acc(R, d, dh, BT(g, HY_BPR));
  mm_nn(R, 4 * d, d, dh, d, BT(w, HY_WPR), 4 * d, dact, 4 * d, 0);
  for (long i = 0; i < (long)R * 4 * d; ++i) dact[i] = (float)(dact[i] * gelu_grad(c->fc[i]));
  mm_tn(4 * d, d, R, dact, 4 * d, c->ln2, d, BT(g, HY_WFC), d, 1);
  colsum_acc(R, 4 * d, dact, BT(g, HY_BFC));
  mm_nn(R, d, 4 * d, dact, 4 * d, BT(w, HY_WFC), d, dln, d, 0);
  memcpy(dhm, dh, sizeof(float) * (size_t)n);
  ln_bwd(R, d, c->hmid, BT(w, HY_LN2_G), c->mean2, c->rstd2, dln, dhm, BT(g, HY_LN2_G), BT(g, HY_LN2_B));
  /* attention: hmid = h_in + att W_o^T + b_o */
  mm_tn(d, d, R, dhm, d, c->att, d, BT(g, HY_WO), d, 1);
  colsum_acc(R, d, dhm, BT(g, HY_BO));
  mm_nn(R, d, d, dhm, d, BT(w, HY_WO), d, datt, d, 0);
  attn_bwd(m, c->qkv, datt, dqkv);
  mm_tn(3 * d, d, R, dqkv, 3 * d, c->ln1, d, BT(g, HY_WQKV), d, 1);
  colsum_acc(R, 3 * d, dqkv, BT(g, HY_BQKV));
  mm_nn(R, d, 3 * d, dqkv, 3 * d, BT(w, HY_WQKV), d, dln, d, 0);
  memcpy(dh, dhm, sizeof(float) * (size_t)n);
  ln_bwd(R, d, h_in, BT(w, HY_LN1_G), c->mean1, c->rstd1, dln, dh, BT(g, HY_LN1_G), BT(g, HY_LN1_B));
  free(dact); free(dhm); free(dln); free(datt); free(dqkv);
}

/* head: loss of ln_f(h) wte^T; if dh != NULL also backward (dh written, grads +=) */
static double head_fwd_bwd(const hy_dims* m, const float* params, float* grads, const float* h,
                           const int32_t* targets, float* dh) {
  const int R = m->B * m->T, d = m->d, V = m->V;
  const float* wte = params;
  const float* lnf = params + hy_layer_offset(m, m->L + 1);
  float* z = falloc((long)R * d);
  float* mean = falloc(R);
  float* rstd = falloc(R);
  ln_fwd(R, d, h, lnf, lnf + hy_pad32(d), z, mean, rstd);
  const int CH = 64;
  float* logits = falloc((long)CH * V);
  float* dz = dh ? falloc((long)R * d) : NULL;
  double loss = 0.0;
  for (int r0 = 0; r0 < R; r0 += CH) {
    const int rows = R - r0 < CH ? R - r0 : CH;
    mm_nt(rows, V, d, z + (long)r0 * d, d, wte, d, logits, V, NULL, 0);
    for (int r = 0; r < rows; ++r) {
      float* l = logits + (long)r * V;
      double mx = -1e300, s = 0.0;
      for (int j = 0; j < V; ++j) if (l[j] > mx) mx = l[j];
      for (int j = 0; j < V; ++j) s += exp(l[j] - mx);
      const int t = targets[r0 + r];
      loss += log(s) + mx - l[t];
      if (dh) {
        for (int j = 0; j < V; ++j) l[j] = (float)((exp(l[j] - mx) / s - (j == t ? 1.0 : 0.0)) / R);
      }
    }
    if (dh) {
      mm_nn(rows, d, V, logits, V, wte, d, dz + (long)r0 * d, d, 0);
      mm_tn(V, d, rows, logits, V, z + (long)r0 * d, d, grads, d, 1); /* dwte += dlogits^T z */
    }
  }
  if (dh) {
    float* lnf_g = grads + hy_layer_offset(m, m->L + 1);
    memset(dh, 0, sizeof(float) * (size_t)R * d);
    ln_bwd(R, d, h, lnf, mean, rstd, dz, dh, lnf_g, lnf_g + hy_pad32(d));
    free(dz);
  }
  free(z); free(mean); free(rstd); free(logits);
  return loss / R;
}

static void embed_fwd(const hy_dims* m, const float* params, const int32_t* tok, float* h) {
  const int R = m->B * m->T, d = m->d;
  const float* wte = params;
  const float* wpe = params + hy_pad32((long)m->V * d);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < d; ++c) h[(long)r * d + c] = wte[(long)tok[r] * d + c] + wpe[(long)(r % m->T) * d + c];
}

static void embed_bwd(const hy_dims* m, float* grads, const int32_t* tok, const float* dh) {
  const int R = m->B * m->T, d = m->d;
  float* gwte = grads;
  float* gwpe = grads + hy_pad32((long)m->V * d);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < d; ++c) {
      gwte[(long)tok[r] * d + c] += dh[(long)r * d + c];
      gwpe[(long)(r % m->T) * d + c] += dh[(long)r * d + c];
    }
}

int oracle_shard_fwd(const hy_dims* m, const float* params, int l0, int l1, const int32_t* tokens,
                     const int32_t* targets, const float* act_in, float* act_out, double* loss) {
  const long n = (long)m->B * m->T * m->d;
  float* h = falloc(n);
  float* tmp = falloc(n);
  block_cache c;
  cache_alloc(m, &c);
  if (l0 > 0) memcpy(h, act_in, sizeof(float) * (size_t)n);
  for (int l = l0; l < l1; ++l) {
    if (l == 0) {
      embed_fwd(m, params, tokens, h);
    } else if (l <= m->L) {
      block_fwd(m, params + hy_layer_offset(m, l), h, tmp, &c);
      memcpy(h, tmp, sizeof(float) * (size_t)n);
    } else {
      *loss = head_fwd_bwd(m, params, NULL, h, targets, NULL);
    }
  }
  if (l1 <= m->L + 1 && act_out) memcpy(act_out, h, sizeof(float) * (size_t)n);
  cache_free(&c);
  free(h);
  free(tmp);
  return 0;
}

int oracle_shard_bwd(const hy_dims* m, const float* params, float* grads, int l0, int l1, const int32_t* tokens,
                     const int32_t* targets, const float* act_in, const float* grad_out, float* grad_in) {
  const long n = (long)m->B * m->T * m->d;
  const int nl = l1 - l0;
  /* recompute: inputs of every layer in the shard */
  float** inp = (float**)calloc((size_t)nl, sizeof(float*));
  float* h = falloc(n);
  block_cache c;
  cache_alloc(m, &c);
  if (l0 > 0) memcpy(h, act_in, sizeof(float) * (size_t)n);
  for (int l = l0; l < l1; ++l) {
    inp[l - l0] = falloc(n);
    memcpy(inp[l - l0], h, sizeof(float) * (size_t)n);
    if (l == 0) {
      embed_fwd(m, params, tokens, h);
    } else if (l <= m->L) {
      float* out = falloc(n);
      block_fwd(m, params + hy_layer_offset(m, l), h, out, &c);
      memcpy(h, out, sizeof(float) * (size_t)n);
      free(out);
    }
  }
  float* dh = falloc(n);
  if (l1 <= m->L + 1) memcpy(dh, grad_out, sizeof(float) * (size_t)n);
  for (int l = l1 - 1; l >= l0; --l) {
    if (l == m->L + 1) {
      head_fwd_bwd(m, params, grads, inp[l - l0], targets, dh);
    } else if (l >= 1) {
      block_fwd(m, params + hy_layer_offset(m, l), inp[l - l0], h, &c);
      block_bwd(m, params + hy_layer_offset(m, l), grads + hy_layer_offset(m, l), inp[l - l0], &c, dh);
    } else {
      embed_bwd(m, grads, tokens, dh);
    }
  }
  if (l0 > 0 && grad_in) memcpy(grad_in, dh, sizeof(float) * (size_t)n);
  for (int i = 0; i < nl; ++i) free(inp[i]);
  free(inp);
  free(h);
  free(dh);
  cache_free(&c);
  return 0;
}

/* round-to-nearest-even to bfloat16, kept in a float */
static float bf16_rne(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  u &= 0xFFFF0000u;
  memcpy(&x, &u, 4);
  return x;
}

void oracle_adam_state(long n, float* p, const float* g, float* m, float* v, float lr, float beta1, float beta2,
                       float eps, float weight_decay, int step, int bf16_state) {
  const float bc1 = (float)(1.0 - pow((double)beta1, step));
  const float bc2 = (float)(1.0 - pow((double)beta2, step));
  const float c1 = 1.f - beta1, c2 = 1.f - beta2;
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    const float mi = beta1 * m[i] + c1 * g[i];
    const float vi = beta2 * v[i] + c2 * g[i] * g[i];
    const float upd = (mi / bc1) / (sqrtf(vi / bc2) + eps);
    p[i] = p[i] - lr * (upd + weight_decay * p[i]);
    m[i] = bf16_state ? bf16_rne(mi) : mi;
    v[i] = bf16_state ? bf16_rne(vi) : vi;
  }
}

void oracle_adam(long n, float* p, const float* g, float* m, float* v, float lr, float beta1, float beta2, float eps,
                 float weight_decay, int step) {
  const float bc1 = (float)(1.0 - pow((double)beta1, step));
  const float bc2 = (float)(1.0 - pow((double)beta2, step));
  const float c1 = 1.f - beta1, c2 = 1.f - beta2;
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    m[i] = beta1 * m[i] + c1 * g[i];
    v[i] = beta2 * v[i] + c2 * g[i] * g[i];
    const float upd = (m[i] / bc1) / (sqrtf(v[i] / bc2) + eps);
    p[i] = p[i] - lr * (upd + weight_decay * p[i]);
  }
}

double oracle_train_step(const hy_dims* m, float* params, float* mom, float* var, int step, float lr,
                         const int32_t* tokens, const int32_t* targets) {
  const long total = hy_total_floats(m);
  float* grads = falloc(total);
  double loss = 0.0;
  oracle_shard_fwd(m, params, 0, m->L + 2, tokens, targets, NULL, NULL, &loss);
  oracle_shard_bwd(m, params, grads, 0, m->L + 2, tokens, targets, NULL, NULL, NULL);
  oracle_adam(total, params, grads, mom, var, lr, 0.9f, 0.999f, 1e-8f, 0.f, step);
  free(grads);
  return loss;
}

void oracle_init_params(const hy_dims* m, uint64_t model_key, float* params) {
  for (int l = 0; l < m->L + 2; ++l) hy_init_layer(m, model_key, l, params + hy_layer_offset(m, l));
}

void oracle_make_tokens(const hy_dims* m, uint64_t seed, int job, int mb, int32_t* tokens, int32_t* targets) {
  for (int r = 0; r < m->B; ++r)
    for (int t = 0; t < m->T; ++t) {
      tokens[r * m->T + t] = hy_token(seed, job, mb, r, t);
      targets[r * m->T + t] = hy_token(seed, job, mb, r, t + 1);
    }
}
