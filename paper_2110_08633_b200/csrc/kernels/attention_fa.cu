// Fused causal attention (head dim 64) on the tcgen05 tensor cores, kind::tf32 — one kernel
// per direction instead of materialising the T x T score matrices in HBM (attention_tc.cu,
// the 3xTF32 "fp32" path, still does that).
//
// Forward, one CTA per (batch, head, 128-query tile), 4 warps, thread t owns query row t:
//   TMA: Q tile [128 x 64] (K-major, 128B swizzle), K tile [64 keys x 64] (K-major),
//        V tile [64 keys x 64] (MN-major B operand, 32B-atom swizzle) — K/V of the next key
//        tile are in flight while the current one is processed
//   S  = Q K^T  -> TMEM (64 fp32 columns), one elected thread issues 8 x tcgen05.mma (K=8)
//   online softmax in registers (tcgen05.ld 32x32b: lane = query row), P written to shared
//        memory in the K-major 128B-swizzle layout the next MMA reads as its A operand
//   PV = P V    -> TMEM (64 columns); O = O * alpha + PV in registers
//   out = O / l ; lse2 = m + log2(l) (log2 domain, kept for the backward)
// Backward (FA2 split, deterministic: no atomics):
//   attn_dkdv_kernel: one CTA per (batch, head, 128-key tile), thread = key row;
//     S^T = K Q^T, dP^T = V dO^T, P^T = exp2(S^T c - lse2), dS^T = P^T (dP^T - Di);
//     dV += P^T dO, dK += dS^T Q / 8   (accumulated in TMEM over the query tiles)
//   attn_dq_kernel: one CTA per (batch, head, 128-query tile), thread = query row;
//     S = Q K^T, dP = dO V^T, dS = P (dP - Di); dQ += dS K / 8 (TMEM)
//   Di = rowsum(dO * O) per (query, head) from a small warp-per-row kernel.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <mutex>

#include "launch_count.cuh"
#include "ops.cuh"
#include "ptx.cuh"

namespace hy {
namespace {

constexpr int HD = 64;
constexpr float kScaleLog2 = 0.125f * 1.4426950408889634f;  // softmax(S/8) in the exp2 domain

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
  });
  return fn;
}

// 2-D fp32 map over a row-major [rows][ld] matrix: box {32 floats, box_rows}; mn_major
// selects the 32B-atom 128B swizzle of MN-major UMMA operands, else plain 128B swizzle.
bool map2d(CUtensorMap* map, const float* ptr, long cols, long rows, long ld, int box_rows, bool mn_major) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// K-major operand, 128B swizzle, rows of 32 fp32 per k-block (k-block stride kb_bytes):
// descriptor of the K=8 slice kk (0..7 for K = 64).
__device__ __forceinline__ uint64_t desc_k(const uint8_t* base, int kk, int kb_bytes) {
  return smem_desc_sw128(smem_u32(base) + (kk >> 2) * kb_bytes + (kk & 3) * 32, 16, 1024);
}
// MN-major operand (N = 64 as two 32-wide atoms 4 KB apart), k-blocks of 32 rows 8 KB apart.
__device__ __forceinline__ uint64_t desc_mn(const uint8_t* base, int kk) {
  return smem_desc_sw128_b32(smem_u32(base) + (kk >> 2) * 8192 + (kk & 3) * 1024, 4096, 512);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Row r (of a K-major 128B-swizzled operand with k-block stride kb_bytes) <- 64 floats,
// rounded to TF32 (nearest, ties away) — the tensor core would otherwise truncate them.
__device__ __forceinline__ void store_row64(uint8_t* base, int r, int kb_bytes, const float (&x)[64]) {
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const int kb = c >> 3, chunk = c & 7;
    float4* dst = reinterpret_cast<float4*>(base + kb * kb_bytes + r * 128 + ((chunk ^ (r & 7)) << 4));
    *dst = make_float4(tf32_rna(x[4 * c]), tf32_rna(x[4 * c + 1]), tf32_rna(x[4 * c + 2]), tf32_rna(x[4 * c + 3]));
  }
}

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&x)[64]) {
  float a[32], b[32];
  tmem_ld_32x32b_x32(taddr, a);
  tmem_ld_32x32b_x32(taddr + 32, b);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    x[i] = a[i];
    x[32 + i] = b[i];
  }
}

__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int kFwdSmem = 32768 + 16384 + 16384 + 32768 + 256 + 1024;

__global__ void __launch_bounds__(128) attn_fwd_kernel(const __grid_constant__ CUtensorMap mq,
                                                       const __grid_constant__ CUtensorMap mk,
                                                       const __grid_constant__ CUtensorMap mv, int T, int H,
                                                       float* __restrict__ out, float* __restrict__ lse2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = align1024(smem_raw);
  uint8_t* sK = sQ + 32768;
  uint8_t* sV = sK + 16384;
  uint8_t* sP = sV + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + 32768);  // q, k, v, s, pv
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 8);
  const int tid = threadIdx.x;
  const int nqt = (T + 127) / 128;
  const int bh = blockIdx.x / nqt;
  const int qt = nqt - 1 - blockIdx.x % nqt;  // longest (most keys) tiles first
  const int b = bh / H, h = bh % H;
  const int q0 = qt * 128, D = H * HD, row0 = b * T;
  const int nkt = min((T + 63) / 64, (q0 + 128) / 64);
  if (tid == 0) {
    tma_prefetch_desc(&mq);
    tma_prefetch_desc(&mk);
    tma_prefetch_desc(&mv);
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc<128>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tS = *tslot, tPV = *tslot + 64;
  const uint32_t lane_off = static_cast<uint32_t>((tid & ~31) << 16);
  if (tid == 0) {
    mbar_expect_tx(&bar[0], 32768);
    tma_load_2d(sQ, &mq, &bar[0], h * HD, row0 + q0);
    tma_load_2d(sQ + 16384, &mq, &bar[0], h * HD + 32, row0 + q0);
    mbar_expect_tx(&bar[1], 16384);
    tma_load_2d(sK, &mk, &bar[1], D + h * HD, row0);
    tma_load_2d(sK + 8192, &mk, &bar[1], D + h * HD + 32, row0);
    mbar_expect_tx(&bar[2], 16384);
    for (int kb = 0; kb < 2; ++kb)
      for (int jn = 0; jn < 2; ++jn) tma_load_2d(sV + kb * 8192 + jn * 4096, &mv, &bar[2], 2 * D + h * HD + 32 * jn, row0 + 32 * kb);
  }
  constexpr uint32_t idS = idesc_tf32(128, 64, false, false);
  constexpr uint32_t idPV = idesc_tf32(128, 64, false, true);
  float o[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) o[i] = 0.f;
  float m_run = -FLT_MAX, l_run = 0.f;
  const int q = q0 + tid;
  uint32_t ph = 0;
  for (int j = 0; j < nkt; ++j, ph ^= 1) {
    const int k0 = j * 64;
    if (tid == 0) {
      if (j == 0) mbar_wait(&bar[0], 0);
      mbar_wait(&bar[1], ph);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tS, desc_k(sQ, kk, 16384), desc_k(sK, kk, 8192), idS, kk > 0);
      mma_commit(&bar[3]);
    }
    mbar_wait(&bar[3], ph);
    tc_fence_after();
    if (tid == 0 && j + 1 < nkt) {  // S consumed K: fetch the next key tile
      mbar_expect_tx(&bar[1], 16384);
      tma_load_2d(sK, &mk, &bar[1], D + h * HD, row0 + k0 + 64);
      tma_load_2d(sK + 8192, &mk, &bar[1], D + h * HD + 32, row0 + k0 + 64);
    }
    float s[64];
    tmem_ld64(tS + lane_off, s);
    float mx = m_run;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      s[i] = (k0 + i <= q) ? s[i] * kScaleLog2 : -FLT_MAX;
      mx = fmaxf(mx, s[i]);
    }
    const float alpha = exp2f(m_run - mx);
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      s[i] = (k0 + i <= q) ? exp2f(s[i] - mx) : 0.f;
      sum += s[i];
    }
    l_run = l_run * alpha + sum;
    m_run = mx;
    store_row64(sP, tid, 16384, s);
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      mbar_wait(&bar[2], ph);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tPV, desc_k(sP, kk, 16384), desc_mn(sV, kk), idPV, kk > 0);
      mma_commit(&bar[4]);
    }
    mbar_wait(&bar[4], ph);
    tc_fence_after();
    if (tid == 0 && j + 1 < nkt) {  // PV consumed V
      mbar_expect_tx(&bar[2], 16384);
      for (int kb = 0; kb < 2; ++kb)
        for (int jn = 0; jn < 2; ++jn)
          tma_load_2d(sV + kb * 8192 + jn * 4096, &mv, &bar[2], 2 * D + h * HD + 32 * jn, row0 + k0 + 64 + 32 * kb);
    }
    float pv[64];
    tmem_ld64(tPV + lane_off, pv);
#pragma unroll
    for (int i = 0; i < 64; ++i) o[i] = o[i] * alpha + pv[i];
  }
  if (q < T) {
    const float inv = 1.f / l_run;
    float4* dst = reinterpret_cast<float4*>(out + static_cast<long>(row0 + q) * D + h * HD);
#pragma unroll
    for (int c = 0; c < 16; ++c) dst[c] = make_float4(o[4 * c] * inv, o[4 * c + 1] * inv, o[4 * c + 2] * inv, o[4 * c + 3] * inv);
    lse2[static_cast<long>(bh) * T + q] = m_run + log2f(l_run);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc<128>(*tslot);
  }
}

// Di[bh*T + q] = sum_c dO[q, h*64 + c] * O[q, h*64 + c]; one warp per (row, head).
__global__ void attn_di_kernel(long n, int T, int H, const float* __restrict__ out, const float* __restrict__ dout,
                               float* __restrict__ Di) {
  const long w = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const long row = w / H;
  const int h = static_cast<int>(w % H);
  const long D = static_cast<long>(H) * HD;
  const float2 a = reinterpret_cast<const float2*>(out + row * D + h * HD)[lane];
  const float2 g = reinterpret_cast<const float2*>(dout + row * D + h * HD)[lane];
  float v = a.x * g.x + a.y * g.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) {
    const long b = row / T, q = row % T;
    Di[(b * H + h) * T + q] = v;
  }
}

// dK, dV of one (batch, head, 128-key tile); thread t owns key row k0 + t.
constexpr int kDkvSmem = 32768 * 2 + 16384 * 4 + 32768 * 2 + 256 + 1024;

__global__ void __launch_bounds__(128) attn_dkdv_kernel(
    const __grid_constant__ CUtensorMap mkv128, const __grid_constant__ CUtensorMap mq64,
    const __grid_constant__ CUtensorMap mqmn, const __grid_constant__ CUtensorMap mdo64,
    const __grid_constant__ CUtensorMap mdomn, int T, int H, const float* __restrict__ lse2,
    const float* __restrict__ Di, float* __restrict__ dqkv) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sK = align1024(smem_raw);
  uint8_t* sV = sK + 32768;
  uint8_t* sQk = sV + 32768;   // Q tile, K-major B (S^T = K Q^T)
  uint8_t* sQm = sQk + 16384;  // Q tile, MN-major B (dK += dS^T Q)
  uint8_t* sGk = sQm + 16384;  // dO tile, K-major B (dP^T = V dO^T)
  uint8_t* sGm = sGk + 16384;  // dO tile, MN-major B (dV += P^T dO)
  uint8_t* sP = sGm + 16384;   // P^T  [128 keys x 64 q], K-major A
  uint8_t* sS = sP + 32768;    // dS^T [128 keys x 64 q], K-major A
  uint64_t* bar = reinterpret_cast<uint64_t*>(sS + 32768);  // kv, q, mma1, mma2
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 8);
  const int tid = threadIdx.x;
  const int nkt = (T + 127) / 128;
  const int bh = blockIdx.x / nkt;
  const int kt = blockIdx.x % nkt;  // tiles near the start see the most queries: schedule them first
  const int b = bh / H, h = bh % H;
  const int k0 = kt * 128, D = H * HD, row0 = b * T;
  const int nq = (T - k0 + 63) / 64;
  if (tid == 0) {
    tma_prefetch_desc(&mkv128);
    tma_prefetch_desc(&mq64);
    tma_prefetch_desc(&mqmn);
    tma_prefetch_desc(&mdo64);
    tma_prefetch_desc(&mdomn);
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tS = *tslot, tP = *tslot + 64, tdV = *tslot + 128, tdK = *tslot + 192;
  const uint32_t lane_off = static_cast<uint32_t>((tid & ~31) << 16);
  auto load_q = [&](int q0) {
    mbar_expect_tx(&bar[1], 4 * 16384);
    for (int kb = 0; kb < 2; ++kb) {
      tma_load_2d(sQk + kb * 8192, &mq64, &bar[1], h * HD + 32 * kb, row0 + q0);
      tma_load_2d(sGk + kb * 8192, &mdo64, &bar[1], h * HD + 32 * kb, row0 + q0);
      for (int jn = 0; jn < 2; ++jn) {
        tma_load_2d(sQm + kb * 8192 + jn * 4096, &mqmn, &bar[1], h * HD + 32 * jn, row0 + q0 + 32 * kb);
        tma_load_2d(sGm + kb * 8192 + jn * 4096, &mdomn, &bar[1], h * HD + 32 * jn, row0 + q0 + 32 * kb);
      }
    }
  };
  if (tid == 0) {
    mbar_expect_tx(&bar[0], 65536);
    for (int kb = 0; kb < 2; ++kb) {
      tma_load_2d(sK + kb * 16384, &mkv128, &bar[0], D + h * HD + 32 * kb, row0 + k0);
      tma_load_2d(sV + kb * 16384, &mkv128, &bar[0], 2 * D + h * HD + 32 * kb, row0 + k0);
    }
    load_q(k0);
  }
  constexpr uint32_t idT = idesc_tf32(128, 64, false, false);   // S^T, dP^T
  constexpr uint32_t idG = idesc_tf32(128, 64, false, true);    // dV, dK (B MN-major)
  const int key = k0 + tid;
  const float* lse_bh = lse2 + static_cast<long>(bh) * T;
  const float* di_bh = Di + static_cast<long>(bh) * T;
  uint32_t ph = 0;
  for (int i = 0; i < nq; ++i, ph ^= 1) {
    const int q0 = k0 + 64 * i;
    if (tid == 0) {
      if (i == 0) mbar_wait(&bar[0], 0);
      mbar_wait(&bar[1], ph);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tS, desc_k(sK, kk, 16384), desc_k(sQk, kk, 8192), idT, kk > 0);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tP, desc_k(sV, kk, 16384), desc_k(sGk, kk, 8192), idT, kk > 0);
      mma_commit(&bar[2]);
    }
    mbar_wait(&bar[2], ph);
    tc_fence_after();
    float s[64], dp[64];
    tmem_ld64(tS + lane_off, s);
    tmem_ld64(tP + lane_off, dp);
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const int q = q0 + c;
      const bool valid = q >= key && q < T;
      const float p = valid ? exp2f(s[c] * kScaleLog2 - lse_bh[q]) : 0.f;
      s[c] = p;
      dp[c] = valid ? p * (dp[c] - di_bh[q]) * 0.125f : 0.f;
    }
    store_row64(sP, tid, 16384, s);
    store_row64(sS, tid, 16384, dp);
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tdV, desc_k(sP, kk, 16384), desc_mn(sGm, kk), idG, (i | kk) > 0);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tdK, desc_k(sS, kk, 16384), desc_mn(sQm, kk), idG, (i | kk) > 0);
      mma_commit(&bar[3]);
      mbar_wait(&bar[3], ph);  // operands free: fetch the next query tile
      if (i + 1 < nq) load_q(q0 + 64);
    }
    mbar_wait(&bar[3], ph);
    tc_fence_after();
  }
  float dv[64], dk[64];
  tmem_ld64(tdV + lane_off, dv);
  tmem_ld64(tdK + lane_off, dk);
  if (key < T) {
    float4* gk = reinterpret_cast<float4*>(dqkv + static_cast<long>(row0 + key) * 3 * D + D + h * HD);
    float4* gv = reinterpret_cast<float4*>(dqkv + static_cast<long>(row0 + key) * 3 * D + 2 * D + h * HD);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      gk[c] = make_float4(dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]);
      gv[c] = make_float4(dv[4 * c], dv[4 * c + 1], dv[4 * c + 2], dv[4 * c + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc<256>(*tslot);
  }
}

// dQ of one (batch, head, 128-query tile); thread t owns query row q0 + t.
constexpr int kDqSmem = 32768 * 2 + 16384 * 3 + 32768 + 256 + 1024;

__global__ void __launch_bounds__(128) attn_dq_kernel(
    const __grid_constant__ CUtensorMap mq128, const __grid_constant__ CUtensorMap mdo128,
    const __grid_constant__ CUtensorMap mk64, const __grid_constant__ CUtensorMap mkmn, int T, int H,
    const float* __restrict__ lse2, const float* __restrict__ Di, float* __restrict__ dqkv) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = align1024(smem_raw);
  uint8_t* sG = sQ + 32768;    // dO tile, K-major A
  uint8_t* sKk = sG + 32768;   // K tile, K-major B (S = Q K^T)
  uint8_t* sKm = sKk + 16384;  // K tile, MN-major B (dQ += dS K)
  uint8_t* sVk = sKm + 16384;  // V tile, K-major B (dP = dO V^T)
  uint8_t* sS = sVk + 16384;   // dS [128 q x 64 keys], K-major A
  uint64_t* bar = reinterpret_cast<uint64_t*>(sS + 32768);  // q, kv, mma1, mma2
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 8);
  const int tid = threadIdx.x;
  const int nqt = (T + 127) / 128;
  const int bh = blockIdx.x / nqt;
  const int qt = nqt - 1 - blockIdx.x % nqt;
  const int b = bh / H, h = bh % H;
  const int q0 = qt * 128, D = H * HD, row0 = b * T;
  const int nkt = min((T + 63) / 64, (q0 + 128) / 64);
  if (tid == 0) {
    tma_prefetch_desc(&mq128);
    tma_prefetch_desc(&mdo128);
    tma_prefetch_desc(&mk64);
    tma_prefetch_desc(&mkmn);
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (tid < 32) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tS = *tslot, tP = *tslot + 64, tdQ = *tslot + 128;
  const uint32_t lane_off = static_cast<uint32_t>((tid & ~31) << 16);
  auto load_kv = [&](int k0) {
    mbar_expect_tx(&bar[1], 3 * 16384);
    for (int kb = 0; kb < 2; ++kb) {
      tma_load_2d(sKk + kb * 8192, &mk64, &bar[1], D + h * HD + 32 * kb, row0 + k0);
      tma_load_2d(sVk + kb * 8192, &mk64, &bar[1], 2 * D + h * HD + 32 * kb, row0 + k0);
      for (int jn = 0; jn < 2; ++jn)
        tma_load_2d(sKm + kb * 8192 + jn * 4096, &mkmn, &bar[1], D + h * HD + 32 * jn, row0 + k0 + 32 * kb);
    }
  };
  if (tid == 0) {
    mbar_expect_tx(&bar[0], 65536);
    for (int kb = 0; kb < 2; ++kb) {
      tma_load_2d(sQ + kb * 16384, &mq128, &bar[0], h * HD + 32 * kb, row0 + q0);
      tma_load_2d(sG + kb * 16384, &mdo128, &bar[0], h * HD + 32 * kb, row0 + q0);
    }
    load_kv(0);
  }
  constexpr uint32_t idS = idesc_tf32(128, 64, false, false);
  constexpr uint32_t idQ = idesc_tf32(128, 64, false, true);
  const int q = q0 + tid;
  const long li = static_cast<long>(bh) * T + min(q, T - 1);
  const float my_lse = lse2[li], my_di = Di[li];
  uint32_t ph = 0;
  for (int j = 0; j < nkt; ++j, ph ^= 1) {
    const int k0 = 64 * j;
    if (tid == 0) {
      if (j == 0) mbar_wait(&bar[0], 0);
      mbar_wait(&bar[1], ph);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tS, desc_k(sQ, kk, 16384), desc_k(sKk, kk, 8192), idS, kk > 0);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tP, desc_k(sG, kk, 16384), desc_k(sVk, kk, 8192), idS, kk > 0);
      mma_commit(&bar[2]);
    }
    mbar_wait(&bar[2], ph);
    tc_fence_after();
    float s[64], dp[64];
    tmem_ld64(tS + lane_off, s);
    tmem_ld64(tP + lane_off, dp);
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      const bool valid = k0 + c <= q;
      const float p = valid ? exp2f(s[c] * kScaleLog2 - my_lse) : 0.f;
      s[c] = valid ? p * (dp[c] - my_di) * 0.125f : 0.f;
    }
    store_row64(sS, tid, 16384, s);
    proxy_fence();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_tf32(tdQ, desc_k(sS, kk, 16384), desc_mn(sKm, kk), idQ, (j | kk) > 0);
      mma_commit(&bar[3]);
      mbar_wait(&bar[3], ph);
      if (j + 1 < nkt) load_kv(k0 + 64);
    }
    mbar_wait(&bar[3], ph);
    tc_fence_after();
  }
  float dq[64];
  tmem_ld64(tdQ + lane_off, dq);
  if (q < T) {
    float4* g = reinterpret_cast<float4*>(dqkv + static_cast<long>(row0 + q) * 3 * D + h * HD);
#pragma unroll
    for (int c = 0; c < 16; ++c) g[c] = make_float4(dq[4 * c], dq[4 * c + 1], dq[4 * c + 2], dq[4 * c + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc<256>(*tslot);
  }
}

}  // namespace

cudaError_t attention_fwd_fa(cudaStream_t st, int B, int T, int H, const float* qkv, float* out, float* lse2) {
  if (B <= 0 || T <= 0 || H <= 0) return cudaSuccess;
  const long D = static_cast<long>(H) * HD, rows = static_cast<long>(B) * T;
  CUtensorMap mq, mk, mv;
  if (!map2d(&mq, qkv, 3 * D, rows, 3 * D, 128, false) || !map2d(&mk, qkv, 3 * D, rows, 3 * D, 64, false) ||
      !map2d(&mv, qkv, 3 * D, rows, 3 * D, 32, true)) {
    return cudaErrorInvalidValue;
  }
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int grid = B * H * ((T + 127) / 128);
  count_launch();
  attn_fwd_kernel<<<grid, 128, kFwdSmem, st>>>(mq, mk, mv, T, H, out, lse2);
  return cudaGetLastError();
}

cudaError_t attention_bwd_fa(cudaStream_t st, int B, int T, int H, const float* qkv, const float* out,
                             const float* dout, const float* lse2, float* dqkv, float* Di) {
  if (B <= 0 || T <= 0 || H <= 0) return cudaSuccess;
  const long D = static_cast<long>(H) * HD, rows = static_cast<long>(B) * T;
  CUtensorMap mkv128, mq64, mqmn, mdo64, mdomn, mq128, mdo128, mk64, mkmn;
  if (!map2d(&mkv128, qkv, 3 * D, rows, 3 * D, 128, false) || !map2d(&mq64, qkv, 3 * D, rows, 3 * D, 64, false) ||
      !map2d(&mqmn, qkv, 3 * D, rows, 3 * D, 32, true) || !map2d(&mdo64, dout, D, rows, D, 64, false) ||
      !map2d(&mdomn, dout, D, rows, D, 32, true) || !map2d(&mq128, qkv, 3 * D, rows, 3 * D, 128, false) ||
      !map2d(&mdo128, dout, D, rows, D, 128, false) || !map2d(&mk64, qkv, 3 * D, rows, 3 * D, 64, false) ||
      !map2d(&mkmn, qkv, 3 * D, rows, 3 * D, 32, true)) {
    return cudaErrorInvalidValue;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_dkdv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDkvSmem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(attn_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDqSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long n = rows * H;
  count_launch();
  attn_di_kernel<<<static_cast<int>((n * 32 + 255) / 256), 256, 0, st>>>(n, T, H, out, dout, Di);
  const int tiles = (T + 127) / 128;
  count_launch();
  attn_dkdv_kernel<<<B * H * tiles, 128, kDkvSmem, st>>>(mkv128, mq64, mqmn, mdo64, mdomn, T, H, lse2, Di, dqkv);
  count_launch();
  attn_dq_kernel<<<B * H * tiles, 128, kDqSmem, st>>>(mq128, mdo128, mk64, mkmn, T, H, lse2, Di, dqkv);
  return cudaGetLastError();
}

}  // namespace hy
