/* ORACLE / TEST INFRASTRUCTURE ONLY — see gpt_oracle.h for scope and citations.
 * Plain C: fp32 tensors, every dot product / reduction accumulated in double. */
#include "gpt_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>
#include <immintrin.h>

#define LN_EPS 1e-5

int oracle_threads(void) { return omp_get_max_threads(); }

static float* falloc(long n) {
  float* p = (float*)calloc((size_t)(n > 0 ? n : 1), sizeof(float));
  return p;
}

/* Blocked GEMM for the oracle: operands packed into fp64 panels (192 x 256 of A, 256 x 256
 * of B), 8 x 16 register micro-tiles (AVX-512 when the host has it, else plain C), every
 * output accumulated in double over the whole K (the per-tile accumulator is double; the
 * k-blocks add into it). Same arithmetic contract as a plain fp64 dot product of the fp32
 * inputs (exactly representable in double); only the summation order differs. */
#define MR 8
#define NR 16
#define MB 192
#define NB 256
#define KC 256

__attribute__((target("avx512f")))
static void ukern_avx512(int kc, const double* restrict a, const double* restrict b, double* restrict c, int ldc) {
  __m512d c00 = _mm512_setzero_pd(), c01 = _mm512_setzero_pd(), c10 = _mm512_setzero_pd(), c11 = _mm512_setzero_pd(),
          c20 = _mm512_setzero_pd(), c21 = _mm512_setzero_pd(), c30 = _mm512_setzero_pd(), c31 = _mm512_setzero_pd(),
          c40 = _mm512_setzero_pd(), c41 = _mm512_setzero_pd(), c50 = _mm512_setzero_pd(), c51 = _mm512_setzero_pd(),
          c60 = _mm512_setzero_pd(), c61 = _mm512_setzero_pd(), c70 = _mm512_setzero_pd(), c71 = _mm512_setzero_pd();
  for (int k = 0; k < kc; ++k) {
    const __m512d b0 = _mm512_load_pd(b + k * NR), b1 = _mm512_load_pd(b + k * NR + 8);
    const double* ak = a + k * MR;
    __m512d av;
    av = _mm512_set1_pd(ak[0]); c00 = _mm512_fmadd_pd(av, b0, c00); c01 = _mm512_fmadd_pd(av, b1, c01);
    av = _mm512_set1_pd(ak[1]); c10 = _mm512_fmadd_pd(av, b0, c10); c11 = _mm512_fmadd_pd(av, b1, c11);
    av = _mm512_set1_pd(ak[2]); c20 = _mm512_fmadd_pd(av, b0, c20); c21 = _mm512_fmadd_pd(av, b1, c21);
    av = _mm512_set1_pd(ak[3]); c30 = _mm512_fmadd_pd(av, b0, c30); c31 = _mm512_fmadd_pd(av, b1, c31);
    av = _mm512_set1_pd(ak[4]); c40 = _mm512_fmadd_pd(av, b0, c40); c41 = _mm512_fmadd_pd(av, b1, c41);
    av = _mm512_set1_pd(ak[5]); c50 = _mm512_fmadd_pd(av, b0, c50); c51 = _mm512_fmadd_pd(av, b1, c51);
    av = _mm512_set1_pd(ak[6]); c60 = _mm512_fmadd_pd(av, b0, c60); c61 = _mm512_fmadd_pd(av, b1, c61);
    av = _mm512_set1_pd(ak[7]); c70 = _mm512_fmadd_pd(av, b0, c70); c71 = _mm512_fmadd_pd(av, b1, c71);
  }
#define ST(r, x0, x1) \
  _mm512_storeu_pd(c + r * ldc, _mm512_add_pd(_mm512_loadu_pd(c + r * ldc), x0)); \
  _mm512_storeu_pd(c + r * ldc + 8, _mm512_add_pd(_mm512_loadu_pd(c + r * ldc + 8), x1));
  ST(0, c00, c01) ST(1, c10, c11) ST(2, c20, c21) ST(3, c30, c31)
  ST(4, c40, c41) ST(5, c50, c51) ST(6, c60, c61) ST(7, c70, c71)
#undef ST
}

static void ukern_generic(int kc, const double* restrict a, const double* restrict b, double* restrict c, int ldc) {
  double acc[MR][NR];
  for (int r = 0; r < MR; ++r) for (int j = 0; j < NR; ++j) acc[r][j] = 0.0;
  for (int k = 0; k < kc; ++k)
    for (int r = 0; r < MR; ++r)
      for (int j = 0; j < NR; ++j) acc[r][j] += a[k * MR + r] * b[k * NR + j];
  for (int r = 0; r < MR; ++r) for (int j = 0; j < NR; ++j) c[r * ldc + j] += acc[r][j];
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

/* "bf16" precision (oracle_set_bf16): the transformer blocks' GEMM operands are rounded to bf16
 * (RNE) as they are packed — the operands the GPU's bf16 block path stores as bf16 (weights, LN
 * outputs, attention output, GELU output, dh, dact, dqkv); accumulation stays fp64. g_round is
 * set only inside block_fwd / block_bwd, so the head GEMMs and attention are unrounded, as on
 * the GPU (paper_2110_08633_b200/csrc/exec/gpt_runner.cpp, block_forward_bf16). */
static int g_bf16 = 0;
static int g_round = 0;
void oracle_set_bf16(int on) { g_bf16 = on != 0; }
static inline double rd(float x) { return g_round ? (double)bf16_rne(x) : (double)x; }

/* pack rows [0,n) x k [0,kc) of X (element (r,k) at X[r*sr + k*sk]) into panels of P rows:
 * out[(p*KC + k)*P + r], zero-padded to a multiple of P */
static void pack(int n, int kc, const float* X, long sr, long sk, int P, int npanels, double* out) {
  for (int p = 0; p < npanels; ++p) {
    double* o = out + (long)p * KC * P;
    if (sk == 1) {
      for (int r = 0; r < P; ++r) {
        const int i = p * P + r;
        if (i < n) { const float* x = X + (long)i * sr; for (int k = 0; k < kc; ++k) o[k * P + r] = rd(x[k]); }
        else for (int k = 0; k < kc; ++k) o[k * P + r] = 0.0;
      }
    } else {
      for (int k = 0; k < kc; ++k) {
        const float* x = X + (long)k * sk;
        for (int r = 0; r < P; ++r) { const int i = p * P + r; o[k * P + r] = i < n ? rd(x[(long)i * sr]) : 0.0; }
      }
    }
  }
}

static void gemm64(int M, int N, int K, const float* A, long sam, long sak, const float* B, long sbk, long sbn,
            float* C, long ldc, const float* bias, int acc) {
  const int mt = (M + MB - 1) / MB, nt = (N + NB - 1) / NB;
  const int avx512 = __builtin_cpu_supports("avx512f");
#pragma omp parallel
  {
    double* ap = (double*)aligned_alloc(64, sizeof(double) * MB * KC);
    double* bp = (double*)aligned_alloc(64, sizeof(double) * NB * KC);
    double* ct = (double*)aligned_alloc(64, sizeof(double) * MB * NB);
#pragma omp for schedule(dynamic) collapse(2)
    for (int tj = 0; tj < nt; ++tj)
      for (int ti = 0; ti < mt; ++ti) {
        const int i0 = ti * MB, j0 = tj * NB;
        const int mb = M - i0 < MB ? M - i0 : MB, nb = N - j0 < NB ? N - j0 : NB;
        const int pm = (mb + MR - 1) / MR, pn = (nb + NR - 1) / NR;
        memset(ct, 0, sizeof(double) * MB * NB);
        for (int k0 = 0; k0 < K; k0 += KC) {
          const int kc = K - k0 < KC ? K - k0 : KC;
          pack(mb, kc, A + (long)i0 * sam + (long)k0 * sak, sam, sak, MR, pm, ap);
          pack(nb, kc, B + (long)j0 * sbn + (long)k0 * sbk, sbn, sbk, NR, pn, bp);
          for (int q = 0; q < pn; ++q)
            for (int p = 0; p < pm; ++p) {
              if (avx512) ukern_avx512(kc, ap + (long)p * KC * MR, bp + (long)q * KC * NR, ct + p * MR * NB + q * NR, NB);
              else ukern_generic(kc, ap + (long)p * KC * MR, bp + (long)q * KC * NR, ct + p * MR * NB + q * NR, NB);
            }
        }
        for (int i = 0; i < mb; ++i) {
          float* c = C + (long)(i0 + i) * ldc + j0;
          for (int j = 0; j < nb; ++j) {
            double s = ct[i * NB + j] + (bias ? bias[j0 + j] : 0.0);
            c[j] = acc ? (float)(c[j] + s) : (float)s;
          }
        }
      }
    free(ap); free(bp); free(ct);
  }
}

/* C[M,N] (+)= A[M,K] * B[N,K]^T (+ bias[N]) */
static void mm_nt(int M, int N, int K, const float* A, long lda, const float* B, long ldb, float* C, long ldc,
                  const float* bias, int acc) {
  gemm64(M, N, K, A, lda, 1, B, 1, ldb, C, ldc, bias, acc);
}

/* C[M,N] (+)= A[M,K] * B[K,N] */
static void mm_nn(int M, int N, int K, const float* A, long lda, const float* B, long ldb, float* C, long ldc,
                  int acc) {
  gemm64(M, N, K, A, lda, 1, B, ldb, 1, C, ldc, NULL, acc);
}

/* C[M,N] (+)= A[K,M]^T * B[K,N]  (weight gradients) */
static void mm_tn(int M, int N, int K, const float* A, long lda, const float* B, long ldb, float* C, long ldc,
                  int acc) {
  gemm64(M, N, K, A, 1, lda, B, ldb, 1, C, ldc, NULL, acc);
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

/* one (batch, head) slice of qkv as contiguous double [T][hd] arrays */
static void head_slices(const hy_dims* m, const float* qkv, int b, int h, double* q, double* k, double* v,
                        double* kt, double* vt) {
  const int T = m->T, D = m->d, hd = D / m->H;
  for (int i = 0; i < T; ++i) {
    const float* row = qkv + ((long)b * T + i) * 3 * D + h * hd;
    for (int c = 0; c < hd; ++c) {
      q[i * hd + c] = row[c];
      k[i * hd + c] = row[D + c];
      v[i * hd + c] = row[2 * D + c];
      kt[(long)c * T + i] = row[D + c];
      vt[(long)c * T + i] = row[2 * D + c];
    }
  }
}

/* s[j] = scale * q . k_j for j <= i: each score is a fp64 dot product over c in order
 * (vectorised across keys through the transposed K) */
static void scores(int i, int T, int hd, const double* qi, const double* kt, double scale, double* s) {
  for (int j = 0; j <= i; ++j) s[j] = 0.0;
  for (int c = 0; c < hd; ++c) {
    const double qc = qi[c];
    const double* kc = kt + (long)c * T;
    for (int j = 0; j <= i; ++j) s[j] += qc * kc[j];
  }
  for (int j = 0; j <= i; ++j) s[j] *= scale;
}

/* causal attention; qkv [B*T, 3D]; out [B*T, D] */
static void attn_fwd(const hy_dims* m, const float* qkv, float* out) {
  const int B = m->B, T = m->T, H = m->H, D = m->d, hd = D / H;
  const double scale = 1.0 / sqrt((double)hd);
#pragma omp parallel
  {
    double* p = (double*)malloc(sizeof(double) * (size_t)T);
    double* q = (double*)malloc(sizeof(double) * (size_t)T * hd * 5);
    double* k = q + (long)T * hd;
    double* v = k + (long)T * hd;
    double* kt = v + (long)T * hd;
    double* vt = kt + (long)T * hd;
    double* o = (double*)malloc(sizeof(double) * (size_t)hd);
#pragma omp for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b) {
      for (int h = 0; h < H; ++h) {
        head_slices(m, qkv, b, h, q, k, v, kt, vt);
        for (int i = 0; i < T; ++i) {
          const double* qi = q + (long)i * hd;
          scores(i, T, hd, qi, kt, scale, p);
          double mx = -1e300;
          for (int j = 0; j <= i; ++j) mx = p[j] > mx ? p[j] : mx;
          double z = 0.0;
          for (int j = 0; j <= i; ++j) {
            p[j] = exp(p[j] - mx);
            z += p[j];
          }
          for (int c = 0; c < hd; ++c) o[c] = 0.0;
          for (int j = 0; j <= i; ++j) {
            const double* vj = v + (long)j * hd;
            for (int c = 0; c < hd; ++c) o[c] += p[j] * vj[c];
          }
          float* orow = out + ((long)b * T + i) * D + h * hd;
          for (int c = 0; c < hd; ++c) orow[c] = (float)(o[c] / z);
        }
      }
    }
    free(p);
    free(q);
    free(o);
  }
}

/* dqkv (overwritten) from dout; recomputes probabilities */
static void attn_bwd(const hy_dims* m, const float* qkv, const float* dout, float* dqkv) {
  const int B = m->B, T = m->T, H = m->H, D = m->d, hd = D / H;
  const double scale = 1.0 / sqrt((double)hd);
#pragma omp parallel
  {
    double* p = (double*)malloc(sizeof(double) * (size_t)T);
    double* dp = (double*)malloc(sizeof(double) * (size_t)T);
    double* dq = (double*)malloc(sizeof(double) * (size_t)hd);
    double* go = (double*)malloc(sizeof(double) * (size_t)hd);
    double* q = (double*)malloc(sizeof(double) * (size_t)T * hd * 7);
    double* k = q + (long)T * hd;
    double* v = k + (long)T * hd;
    double* kt = v + (long)T * hd;
    double* vt = kt + (long)T * hd;
    double* dk = vt + (long)T * hd;
    double* dv = dk + (long)T * hd;
#pragma omp for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b) {
      for (int h = 0; h < H; ++h) {
        head_slices(m, qkv, b, h, q, k, v, kt, vt);
        memset(dk, 0, sizeof(double) * (size_t)T * hd * 2);
        for (int i = 0; i < T; ++i) {
          const double* qi = q + (long)i * hd;
          const float* gor = dout + ((long)b * T + i) * D + h * hd;
          for (int c = 0; c < hd; ++c) go[c] = gor[c];
          scores(i, T, hd, qi, kt, scale, p);
          double mx = -1e300;
          for (int j = 0; j <= i; ++j) mx = p[j] > mx ? p[j] : mx;
          double z = 0.0;
          for (int j = 0; j <= i; ++j) {
            p[j] = exp(p[j] - mx);
            z += p[j];
          }
          scores(i, T, hd, go, vt, 1.0, dp); /* dp[j] = dO_i . v_j */
          double delta = 0.0;
          for (int j = 0; j <= i; ++j) {
            p[j] /= z;
            delta += p[j] * dp[j];
          }
          for (int c = 0; c < hd; ++c) dq[c] = 0.0;
          for (int j = 0; j <= i; ++j) {
            const double ds = p[j] * (dp[j] - delta) * scale;
            const double* kj = k + (long)j * hd;
            double* dkj = dk + (long)j * hd;
            double* dvj = dv + (long)j * hd;
            for (int c = 0; c < hd; ++c) {
              dq[c] += ds * kj[c];
              dkj[c] += ds * qi[c];
              dvj[c] += p[j] * go[c];
            }
          }
          float* dqr = dqkv + ((long)b * T + i) * 3 * D + h * hd;
          for (int c = 0; c < hd; ++c) dqr[c] = (float)dq[c];
        }
        for (int j = 0; j < T; ++j) {
          float* dkr = dqkv + ((long)b * T + j) * 3 * D + D + h * hd;
          float* dvr = dkr + D;
          for (int c = 0; c < hd; ++c) {
            dkr[c] = (float)dk[(long)j * hd + c];
            dvr[c] = (float)dv[(long)j * hd + c];
          }
        }
      }
    }
    free(p);
    free(dp);
    free(dq);
    free(go);
    free(q);
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
  g_round = g_bf16;
  ln_fwd(R, d, h_in, BT(w, HY_LN1_G), BT(w, HY_LN1_B), c->ln1, c->mean1, c->rstd1);
  mm_nt(R, 3 * d, d, c->ln1, d, BT(w, HY_WQKV), d, c->qkv, 3 * d, BT(w, HY_BQKV), 0);
  attn_fwd(m, c->qkv, c->att);
  mm_nt(R, d, d, c->att, d, BT(w, HY_WO), d, c->hmid, d, BT(w, HY_BO), 0);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < (long)R * d; ++i) c->hmid[i] += h_in[i];
  ln_fwd(R, d, c->hmid, BT(w, HY_LN2_G), BT(w, HY_LN2_B), c->ln2, c->mean2, c->rstd2);
  mm_nt(R, 4 * d, d, c->ln2, d, BT(w, HY_WFC), d, c->fc, 4 * d, BT(w, HY_BFC), 0);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < (long)R * 4 * d; ++i) c->act[i] = (float)gelu(c->fc[i]);
  mm_nt(R, d, 4 * d, c->act, 4 * d, BT(w, HY_WPR), 4 * d, h_out, d, BT(w, HY_BPR), 0);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < (long)R * d; ++i) h_out[i] += c->hmid[i];
  g_round = 0;
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
  g_round = g_bf16;
  /* MLP: h_out = hmid + act W_pr^T + b_pr */
  mm_tn(d, 4 * d, R, dh, d, c->act, 4 * d, BT(g, HY_WPR), 4 * d, 1);
  colsum_acc(R, d, dh, BT(g, HY_BPR));
  mm_nn(R, 4 * d, d, dh, d, BT(w, HY_WPR), 4 * d, dact, 4 * d, 0);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < (long)R * 4 * d; ++i) {
    const float v = (float)(dact[i] * gelu_grad(c->fc[i]));
    dact[i] = g_bf16 ? bf16_rne(v) : v; /* the GPU stores dact as bf16; the bias grad sums those */
  }
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
  g_round = 0;
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
  const int CH = 2048;
  float* logits = falloc((long)CH * V);
  float* dz = dh ? falloc((long)R * d) : NULL;
  double loss = 0.0;
  for (int r0 = 0; r0 < R; r0 += CH) {
    const int rows = R - r0 < CH ? R - r0 : CH;
    mm_nt(rows, V, d, z + (long)r0 * d, d, wte, d, logits, V, NULL, 0);
    double* rl = (double*)malloc(sizeof(double) * (size_t)rows);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r) {
      float* l = logits + (long)r * V;
      double mx = -1e300, s = 0.0;
      for (int j = 0; j < V; ++j) if (l[j] > mx) mx = l[j];
      for (int j = 0; j < V; ++j) s += exp(l[j] - mx);
      const int t = targets[r0 + r];
      rl[r] = log(s) + mx - l[t];
      if (dh) {
        for (int j = 0; j < V; ++j) l[j] = (float)((exp(l[j] - mx) / s - (j == t ? 1.0 : 0.0)) / R);
      }
    }
    for (int r = 0; r < rows; ++r) loss += rl[r]; /* row order: deterministic */
    free(rl);
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
  /* recompute (strategies.cpp:771-776: B(s) re-runs the shard forward from its checkpoint):
   * the input of every layer plus each block's intermediates, kept for the backward */
  float** inp = (float**)calloc((size_t)nl, sizeof(float*));
  block_cache* cs = (block_cache*)calloc((size_t)nl, sizeof(block_cache));
  float* h = falloc(n);
  if (l0 > 0) memcpy(h, act_in, sizeof(float) * (size_t)n);
  for (int l = l0; l < l1; ++l) {
    inp[l - l0] = falloc(n);
    memcpy(inp[l - l0], h, sizeof(float) * (size_t)n);
    if (l == 0) {
      embed_fwd(m, params, tokens, h);
    } else if (l <= m->L) {
      cache_alloc(m, &cs[l - l0]);
      block_fwd(m, params + hy_layer_offset(m, l), inp[l - l0], h, &cs[l - l0]);
    }
  }
  float* dh = falloc(n);
  if (l1 <= m->L + 1) memcpy(dh, grad_out, sizeof(float) * (size_t)n);
  for (int l = l1 - 1; l >= l0; --l) {
    if (l == m->L + 1) {
      head_fwd_bwd(m, params, grads, inp[l - l0], targets, dh);
    } else if (l >= 1) {
      block_bwd(m, params + hy_layer_offset(m, l), grads + hy_layer_offset(m, l), inp[l - l0], &cs[l - l0], dh);
      cache_free(&cs[l - l0]);
    } else {
      embed_bwd(m, grads, tokens, dh);
    }
  }
  if (l0 > 0 && grad_in) memcpy(grad_in, dh, sizeof(float) * (size_t)n);
  for (int i = 0; i < nl; ++i) free(inp[i]);
  free(inp);
  free(cs);
  free(h);
  free(dh);
  return 0;
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
#pragma omp parallel for schedule(dynamic)
  for (int l = 0; l < m->L + 2; ++l) hy_init_layer(m, model_key, l, params + hy_layer_offset(m, l));
}

void oracle_make_tokens(const hy_dims* m, uint64_t seed, int job, int mb, int32_t* tokens, int32_t* targets) {
  for (int r = 0; r < m->B; ++r)
    for (int t = 0; t < m->T; ++t) {
      tokens[r * m->T + t] = hy_token(seed, job, mb, r, t);
      targets[r * m->T + t] = hy_token(seed, job, mb, r, t + 1);
    }
}
