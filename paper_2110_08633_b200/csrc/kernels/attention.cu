// Causal multi-head attention, head dim 64, fp32 — flash-style (online softmax, no T x T
// matrix in HBM). CUDA-core FFMA version: K/V (or Q/dO) tiles of 64 rows staged in shared
// memory and broadcast to all threads; one thread (fwd) or one thread pair (bwd) per row.
// Reads the fused QKV projection in place ([B*T, 3*H*64]) and writes dQKV in the same layout.
#include <cfloat>

#include "launch_count.cuh"
#include "ops.cuh"

namespace hy {
namespace {

constexpr int HD = 64;
constexpr int TILE = 64;
constexpr float kScale = 0.125f;  // 1/sqrt(64), exact in fp32

__device__ __forceinline__ void load_tile(float (*dst)[HD], const float* __restrict__ base, long ld, int row0, int T,
                                          int nthreads) {
  for (int idx = threadIdx.x; idx < TILE * (HD / 4); idx += nthreads) {
    const int r = idx >> 4, c4 = idx & 15;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row0 + r < T) v = reinterpret_cast<const float4*>(base + static_cast<long>(row0 + r) * ld)[c4];
    reinterpret_cast<float4*>(&dst[r][0])[c4] = v;
  }
}

__global__ void __launch_bounds__(TILE) attn_fwd_kernel(int T, int H, const float* __restrict__ qkv,
                                                         float* __restrict__ out, float* __restrict__ lse) {
  __shared__ __align__(16) float Ks[TILE][HD];
  __shared__ __align__(16) float Vs[TILE][HD];
  const int D = H * HD;
  const long ld = 3L * D;
  const int qt = gridDim.x - 1 - blockIdx.x;  // heavy (late) tiles first
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int i = qt * TILE + threadIdx.x;
  const bool valid = i < T;
  const float* base = qkv + static_cast<long>(b) * T * ld;
  float q[HD], o[HD];
  {
    const float4* qr = reinterpret_cast<const float4*>(base + static_cast<long>(valid ? i : 0) * ld + h * HD);
#pragma unroll
    for (int c = 0; c < HD / 4; ++c) {
      const float4 v = qr[c];
      q[4 * c] = v.x * kScale;
      q[4 * c + 1] = v.y * kScale;
      q[4 * c + 2] = v.z * kScale;
      q[4 * c + 3] = v.w * kScale;
    }
  }
#pragma unroll
  for (int c = 0; c < HD; ++c) o[c] = 0.f;
  float m = -FLT_MAX, l = 0.f;
  for (int kt = 0; kt <= qt; ++kt) {
    __syncthreads();
    load_tile(Ks, base + D + h * HD, ld, kt * TILE, T, TILE);
    load_tile(Vs, base + 2 * D + h * HD, ld, kt * TILE, T, TILE);
    __syncthreads();
    const int jmax = min(TILE, T - kt * TILE);
    for (int jg = 0; jg < jmax; jg += 16) {
      float s[16];
      float gmax = -FLT_MAX;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int j = jg + u;
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < HD / 4; ++c) {
          const float4 kv = reinterpret_cast<const float4*>(&Ks[j][0])[c];
          acc = fmaf(q[4 * c], kv.x, acc);
          acc = fmaf(q[4 * c + 1], kv.y, acc);
          acc = fmaf(q[4 * c + 2], kv.z, acc);
          acc = fmaf(q[4 * c + 3], kv.w, acc);
        }
        const bool ok = j < jmax && kt * TILE + j <= i;
        s[u] = ok ? acc : -FLT_MAX;
        gmax = fmaxf(gmax, s[u]);
      }
      if (gmax == -FLT_MAX) continue;
      const float m_new = fmaxf(m, gmax);
      const float corr = __expf(m - m_new);
      l *= corr;
#pragma unroll
      for (int c = 0; c < HD; ++c) o[c] *= corr;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float p = s[u] == -FLT_MAX ? 0.f : __expf(s[u] - m_new);
        l += p;
        const int j = jg + u;
#pragma unroll
        for (int c = 0; c < HD / 4; ++c) {
          const float4 vv = reinterpret_cast<const float4*>(&Vs[j][0])[c];
          o[4 * c] = fmaf(p, vv.x, o[4 * c]);
          o[4 * c + 1] = fmaf(p, vv.y, o[4 * c + 1]);
          o[4 * c + 2] = fmaf(p, vv.z, o[4 * c + 2]);
          o[4 * c + 3] = fmaf(p, vv.w, o[4 * c + 3]);
        }
      }
      m = m_new;
    }
  }
  if (!valid) return;
  const float inv = 1.f / l;
  float4* orow = reinterpret_cast<float4*>(out + static_cast<long>(b * T + i) * D + h * HD);
#pragma unroll
  for (int c = 0; c < HD / 4; ++c) orow[c] = make_float4(o[4 * c] * inv, o[4 * c + 1] * inv, o[4 * c + 2] * inv, o[4 * c + 3] * inv);
  lse[(static_cast<long>(b) * H + h) * T + i] = m + logf(l);
}

// delta[b,h,i] = sum_c dout[i, h, c] * out[i, h, c]
__global__ void attn_delta_kernel(int BT, int H, int T, const float* __restrict__ out, const float* __restrict__ dout,
                                  float* __restrict__ delta) {
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long>(BT) * H) return;
  const int row = static_cast<int>(idx / H), h = static_cast<int>(idx % H);
  const long off = static_cast<long>(row) * H * HD + h * HD;
  const float4* a = reinterpret_cast<const float4*>(out + off);
  const float4* g = reinterpret_cast<const float4*>(dout + off);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < HD / 4; ++c) {
    const float4 x = a[c], y = g[c];
    s += x.x * y.x + x.y * y.y + x.z * y.z + x.w * y.w;
  }
  const int b = row / T, i = row % T;
  delta[(static_cast<long>(b) * H + h) * T + i] = s;
}

// dK, dV: thread pair per key row j (each thread owns 32 of the 64 dims).
__global__ void __launch_bounds__(2 * TILE) attn_bwd_kv_kernel(int T, int H, const float* __restrict__ qkv,
                                                                const float* __restrict__ dout,
                                                                const float* __restrict__ lse,
                                                                const float* __restrict__ delta,
                                                                float* __restrict__ dqkv) {
  __shared__ __align__(16) float Qs[TILE][HD];
  __shared__ __align__(16) float Gs[TILE][HD];
  __shared__ float Ls[TILE], Ds[TILE];
  const int D = H * HD;
  const long ld = 3L * D;
  const int kt = blockIdx.x;
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int j = kt * TILE + (threadIdx.x >> 1);
  const int half = threadIdx.x & 1;
  const bool valid = j < T;
  const float* base = qkv + static_cast<long>(b) * T * ld;
  const float* gbase = dout + static_cast<long>(b) * T * D;
  const float* lrow = lse + (static_cast<long>(b) * H + h) * T;
  const float* drow = delta + (static_cast<long>(b) * H + h) * T;
  float k[32], v[32], dk[32], dv[32];
  {
    const long r = static_cast<long>(valid ? j : 0) * ld;
    const float4* kr = reinterpret_cast<const float4*>(base + r + D + h * HD + half * 32);
    const float4* vr = reinterpret_cast<const float4*>(base + r + 2 * D + h * HD + half * 32);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 a = kr[c], bb = vr[c];
      k[4 * c] = a.x; k[4 * c + 1] = a.y; k[4 * c + 2] = a.z; k[4 * c + 3] = a.w;
      v[4 * c] = bb.x; v[4 * c + 1] = bb.y; v[4 * c + 2] = bb.z; v[4 * c + 3] = bb.w;
    }
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    dk[c] = 0.f;
    dv[c] = 0.f;
  }
  const int n_qt = (T + TILE - 1) / TILE;
  for (int qt = kt; qt < n_qt; ++qt) {
    __syncthreads();
    load_tile(Qs, base + h * HD, ld, qt * TILE, T, 2 * TILE);
    load_tile(Gs, gbase + h * HD, D, qt * TILE, T, 2 * TILE);
    for (int r = threadIdx.x; r < TILE; r += 2 * TILE) {
      const int qi = qt * TILE + r;
      Ls[r] = qi < T ? lrow[qi] : 0.f;
      Ds[r] = qi < T ? drow[qi] : 0.f;
    }
    __syncthreads();
    const int imax = min(TILE, T - qt * TILE);
    for (int ii = 0; ii < imax; ++ii) {
      const int qi = qt * TILE + ii;
      const float* qrow = &Qs[ii][half * 32];
      const float* grow = &Gs[ii][half * 32];
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        s = fmaf(qrow[c], k[c], s);
        dp = fmaf(grow[c], v[c], dp);
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      dp += __shfl_xor_sync(0xffffffffu, dp, 1);
      const bool ok = valid && qi >= j;
      const float p = ok ? __expf(s * kScale - Ls[ii]) : 0.f;
      const float ds = p * (dp - Ds[ii]) * kScale;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        dv[c] = fmaf(p, grow[c], dv[c]);
        dk[c] = fmaf(ds, qrow[c], dk[c]);
      }
    }
  }
  if (!valid) return;
  float* out = dqkv + (static_cast<long>(b) * T + j) * ld;
  float4* dkr = reinterpret_cast<float4*>(out + D + h * HD + half * 32);
  float4* dvr = reinterpret_cast<float4*>(out + 2 * D + h * HD + half * 32);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    dkr[c] = make_float4(dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]);
    dvr[c] = make_float4(dv[4 * c], dv[4 * c + 1], dv[4 * c + 2], dv[4 * c + 3]);
  }
}

// dQ: thread pair per query row i.
__global__ void __launch_bounds__(2 * TILE) attn_bwd_q_kernel(int T, int H, const float* __restrict__ qkv,
                                                               const float* __restrict__ dout,
                                                               const float* __restrict__ lse,
                                                               const float* __restrict__ delta,
                                                               float* __restrict__ dqkv) {
  __shared__ __align__(16) float Ks[TILE][HD];
  __shared__ __align__(16) float Vs[TILE][HD];
  const int D = H * HD;
  const long ld = 3L * D;
  const int qt = gridDim.x - 1 - blockIdx.x;
  const int b = blockIdx.y / H, h = blockIdx.y % H;
  const int i = qt * TILE + (threadIdx.x >> 1);
  const int half = threadIdx.x & 1;
  const bool valid = i < T;
  const float* base = qkv + static_cast<long>(b) * T * ld;
  float q[32], g[32], dq[32];
  {
    const long r = static_cast<long>(valid ? i : 0);
    const float4* qr = reinterpret_cast<const float4*>(base + r * ld + h * HD + half * 32);
    const float4* gr = reinterpret_cast<const float4*>(dout + (static_cast<long>(b) * T + r) * D + h * HD + half * 32);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 a = qr[c], bb = gr[c];
      q[4 * c] = a.x; q[4 * c + 1] = a.y; q[4 * c + 2] = a.z; q[4 * c + 3] = a.w;
      g[4 * c] = bb.x; g[4 * c + 1] = bb.y; g[4 * c + 2] = bb.z; g[4 * c + 3] = bb.w;
    }
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) dq[c] = 0.f;
  const float L = valid ? lse[(static_cast<long>(b) * H + h) * T + i] : 0.f;
  const float Dl = valid ? delta[(static_cast<long>(b) * H + h) * T + i] : 0.f;
  for (int kt = 0; kt <= qt; ++kt) {
    __syncthreads();
    load_tile(Ks, base + D + h * HD, ld, kt * TILE, T, 2 * TILE);
    load_tile(Vs, base + 2 * D + h * HD, ld, kt * TILE, T, 2 * TILE);
    __syncthreads();
    const int jmax = min(TILE, T - kt * TILE);
    for (int jj = 0; jj < jmax; ++jj) {
      const int kj = kt * TILE + jj;
      const float* krow = &Ks[jj][half * 32];
      const float* vrow = &Vs[jj][half * 32];
      float s = 0.f, dp = 0.f;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        s = fmaf(q[c], krow[c], s);
        dp = fmaf(g[c], vrow[c], dp);
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      dp += __shfl_xor_sync(0xffffffffu, dp, 1);
      const bool ok = valid && kj <= i;
      const float p = ok ? __expf(s * kScale - L) : 0.f;
      const float ds = p * (dp - Dl) * kScale;
#pragma unroll
      for (int c = 0; c < 32; ++c) dq[c] = fmaf(ds, krow[c], dq[c]);
    }
  }
  if (!valid) return;
  float4* dqr = reinterpret_cast<float4*>(dqkv + (static_cast<long>(b) * T + i) * ld + h * HD + half * 32);
#pragma unroll
  for (int c = 0; c < 8; ++c) dqr[c] = make_float4(dq[4 * c], dq[4 * c + 1], dq[4 * c + 2], dq[4 * c + 3]);
}

}  // namespace

cudaError_t attention_fwd(cudaStream_t s, int B, int T, int H, const float* qkv, float* out, float* lse) {
  dim3 grid((T + TILE - 1) / TILE, B * H);
  count_launch();
  attn_fwd_kernel<<<grid, TILE, 0, s>>>(T, H, qkv, out, lse);
  return cudaGetLastError();
}

cudaError_t attention_bwd(cudaStream_t s, int B, int T, int H, const float* qkv, const float* out, const float* dout,
                          const float* lse, float* dqkv, float* ws) {
  const long n = static_cast<long>(B) * T * H;
  count_launch();
  attn_delta_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(B * T, H, T, out, dout, ws);
  dim3 grid((T + TILE - 1) / TILE, B * H);
  count_launch();
  attn_bwd_kv_kernel<<<grid, 2 * TILE, 0, s>>>(T, H, qkv, dout, lse, ws, dqkv);
  count_launch();
  attn_bwd_q_kernel<<<grid, 2 * TILE, 0, s>>>(T, H, qkv, dout, lse, ws, dqkv);
  return cudaGetLastError();
}

}  // namespace hy
