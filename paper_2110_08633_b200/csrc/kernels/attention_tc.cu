// Causal multi-head attention on the tcgen05 tensor cores (kind::tf32).
//
// The [T x T] score matrix of each (batch, head) is materialised in HBM in the workspace
// the reference cost model budgets for it (workspace_bytes = b * (d/64) * s^2 * bpp,
// model.cpp:193), processed in (batch, head) chunks that fit the region the caller hands
// in. Every contraction is a batched call of the persistent tcgen05 GEMM, reading Q/K/V
// and dO in place from the fused projections through 4-D TMA maps (batch, head, row, col):
//   fwd:  S = Q K^T (upper tiles skipped) -> P = causal softmax(S/8) -> O = P V (K <= diag)
//   bwd:  recompute P;  dP = dO V^T;  dS = P (dP - rowsum(P dP));
//         dQ = dS K / 8 (K <= diag);  dK = dS^T Q / 8 and dV = P^T dO (K >= diag)
// Row-wise softmax kernels are one warp per row (128-bit loads, warp-shuffle reductions);
// they write exact zeros right of the diagonal inside the diagonal 128-tile band so the
// K-range-limited GEMMs never read stale scores.
#include <cfloat>

#include "gemm.cuh"
#include "launch_count.cuh"
#include "ops.cuh"

namespace hy {
namespace {

constexpr int HD = 64;
constexpr int TILE = 128;  // GEMM BM = BN
constexpr float kScale = 0.125f;

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// rows of a [n_mats][T][T] stack; row r -> query index i = r % T. Softmax over j <= i of
// S/8, zeros for i < j < band end, columns beyond the band untouched.
template <int kMaxPerLane>
__global__ void causal_softmax_fwd_kernel(long n_rows, int T, float* __restrict__ S) {
  const long row = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const int i = static_cast<int>(row % T);
  const int band = min(T, (i / TILE + 1) * TILE);
  float* s = S + row * T;
  float v[kMaxPerLane];
  float mx = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < kMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    v[k] = (j <= i) ? s[j] * kScale : -FLT_MAX;
    mx = fmaxf(mx, v[k]);
  }
  mx = warp_max(mx);
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < kMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    v[k] = (j <= i) ? __expf(v[k] - mx) : 0.f;
    sum += v[k];
  }
  const float inv = 1.f / warp_sum(sum);
#pragma unroll
  for (int k = 0; k < kMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    if (j < band) s[j] = v[k] * inv;
  }
}

// dS = P * (dP - sum_j P dP), in place over dP; zeros right of the diagonal in the band.
template <int kMaxPerLane>
__global__ void causal_softmax_bwd_kernel(long n_rows, int T, const float* __restrict__ P, float* __restrict__ dP) {
  const long row = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const int i = static_cast<int>(row % T);
  const int band = min(T, (i / TILE + 1) * TILE);
  const float* p = P + row * T;
  float* g = dP + row * T;
  float pv[kMaxPerLane], gv[kMaxPerLane];
  float dot = 0.f;
#pragma unroll
  for (int k = 0; k < kMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    pv[k] = (j <= i) ? p[j] : 0.f;
    gv[k] = (j <= i) ? g[j] : 0.f;
    dot += pv[k] * gv[k];
  }
  dot = warp_sum(dot);
#pragma unroll
  for (int k = 0; k < kMaxPerLane; ++k) {
    const int j = lane + 32 * k;
    if (j < band) g[j] = pv[k] * (gv[k] - dot);
  }
}

cudaError_t softmax_launch(cudaStream_t s, long rows, int T, float* S, const float* P, bool bwd) {
  const int threads = 256;
  const long blocks = (rows * 32 + threads - 1) / threads;
  count_launch();
  if (T <= 256) {
    if (bwd) causal_softmax_bwd_kernel<8><<<blocks, threads, 0, s>>>(rows, T, P, S);
    else causal_softmax_fwd_kernel<8><<<blocks, threads, 0, s>>>(rows, T, S);
  } else if (T <= 512) {
    if (bwd) causal_softmax_bwd_kernel<16><<<blocks, threads, 0, s>>>(rows, T, P, S);
    else causal_softmax_fwd_kernel<16><<<blocks, threads, 0, s>>>(rows, T, S);
  } else if (T <= 1024) {
    if (bwd) causal_softmax_bwd_kernel<32><<<blocks, threads, 0, s>>>(rows, T, P, S);
    else causal_softmax_fwd_kernel<32><<<blocks, threads, 0, s>>>(rows, T, S);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

struct Chunk {
  int b0, nb, h0, nh;
};

// (batch, head) chunks of at most `mats` score matrices: whole batches when they fit,
// otherwise head groups of one batch.
template <class F>
cudaError_t for_chunks(int B, int H, long mats, F&& f) {
  if (mats < 1) return cudaErrorInvalidValue;
  if (mats >= H) {
    const int per = static_cast<int>(mats / H);
    for (int b0 = 0; b0 < B; b0 += per) {
      const cudaError_t e = f(Chunk{b0, per < B - b0 ? per : B - b0, 0, H});
      if (e != cudaSuccess) return e;
    }
  } else {
    const int per = static_cast<int>(mats);
    for (int b = 0; b < B; ++b) {
      for (int h0 = 0; h0 < H; h0 += per) {
        const cudaError_t e = f(Chunk{b, 1, h0, per < H - h0 ? per : H - h0});
        if (e != cudaSuccess) return e;
      }
    }
  }
  return cudaSuccess;
}

// Batched GEMM helper: batch (z1 over batches, z2 over heads).
cudaError_t bgemm(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool amn, long a_s1, long a_s2,
                  const float* B, long ldb, bool bmn, long b_s1, long b_s2, float* C, long ldc, long c_s1, long c_s2,
                  const Chunk& c, int causal, float alpha) {
  GemmEpilogue e;
  e.C = C;
  e.ldc = ldc;
  e.alpha = alpha;
  GemmBatch bt;
  bt.nb1 = c.nb;
  bt.nb2 = c.nh;
  bt.a_s1 = a_s1;
  bt.a_s2 = a_s2;
  bt.b_s1 = b_s1;
  bt.b_s2 = b_s2;
  bt.c_s1 = c_s1;
  bt.c_s2 = c_s2;
  bt.causal = causal;
  return gemm_tf32(st, M, N, K, A, lda, amn, B, ldb, bmn, e, &bt);
}

}  // namespace

cudaError_t attention_fwd_tc(cudaStream_t st, int B, int T, int H, const float* qkv, float* out, float* work,
                             long work_floats) {
  const long D = static_cast<long>(H) * HD, ld = 3 * D, TT = static_cast<long>(T) * T;
  return for_chunks(B, H, work_floats / TT, [&](const Chunk& c) -> cudaError_t {
    const float* q = qkv + static_cast<long>(c.b0) * T * ld + c.h0 * HD;
    const float* k = q + D;
    const float* v = q + 2 * D;
    const long s1 = static_cast<long>(c.nh) * TT;  // score-stack batch stride
    cudaError_t e = bgemm(st, T, T, HD, q, ld, false, T * ld, HD, k, ld, false, T * ld, HD, work, T, s1, TT, c,
                          kCausalSkipUpper, 1.f);
    if (e != cudaSuccess) return e;
    e = softmax_launch(st, static_cast<long>(c.nb) * c.nh * T, T, work, nullptr, false);
    if (e != cudaSuccess) return e;
    float* o = out + static_cast<long>(c.b0) * T * D + c.h0 * HD;
    return bgemm(st, T, HD, T, work, T, false, s1, TT, v, ld, true, T * ld, HD, o, D, T * D, HD, c, kCausalKLower,
                 1.f);
  });
}

cudaError_t attention_bwd_tc(cudaStream_t st, int B, int T, int H, const float* qkv, const float* dout, float* dqkv,
                             float* work, long work_floats) {
  const long D = static_cast<long>(H) * HD, ld = 3 * D, TT = static_cast<long>(T) * T;
  return for_chunks(B, H, work_floats / (2 * TT), [&](const Chunk& c) -> cudaError_t {
    const long off = static_cast<long>(c.b0) * T * ld + c.h0 * HD;
    const float* q = qkv + off;
    const float* k = q + D;
    const float* v = q + 2 * D;
    const float* go = dout + static_cast<long>(c.b0) * T * D + c.h0 * HD;
    float* dq = dqkv + off;
    float* dk = dq + D;
    float* dv = dq + 2 * D;
    const long nmat = static_cast<long>(c.nb) * c.nh;
    float* P = work;
    float* G = work + nmat * TT;
    const long s1 = static_cast<long>(c.nh) * TT;
    cudaError_t e = bgemm(st, T, T, HD, q, ld, false, T * ld, HD, k, ld, false, T * ld, HD, P, T, s1, TT, c,
                          kCausalSkipUpper, 1.f);
    if (e != cudaSuccess) return e;
    if ((e = softmax_launch(st, nmat * T, T, P, nullptr, false)) != cudaSuccess) return e;
    e = bgemm(st, T, T, HD, go, D, false, T * D, HD, v, ld, false, T * ld, HD, G, T, s1, TT, c, kCausalSkipUpper, 1.f);
    if (e != cudaSuccess) return e;
    if ((e = softmax_launch(st, nmat * T, T, G, P, true)) != cudaSuccess) return e;
    // dQ = dS K / 8
    e = bgemm(st, T, HD, T, G, T, false, s1, TT, k, ld, true, T * ld, HD, dq, ld, T * ld, HD, c, kCausalKLower, kScale);
    if (e != cudaSuccess) return e;
    // dK = dS^T Q / 8
    e = bgemm(st, T, HD, T, G, T, true, s1, TT, q, ld, true, T * ld, HD, dk, ld, T * ld, HD, c, kCausalKUpper, kScale);
    if (e != cudaSuccess) return e;
    // dV = P^T dO
    return bgemm(st, T, HD, T, P, T, true, s1, TT, go, D, true, T * D, HD, dv, ld, T * ld, HD, c, kCausalKUpper, 1.f);
  });
}

}  // namespace hy
