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
//     dV += P^T dO, dK += dS^T Q   (accumulated in TMEM over the query tiles; the softmax
//     scale 1/8 is applied once to dK at the end — exact, a power of two)
//   attn_dq_kernel: one CTA per (batch, head, 128-query tile), thread = query row;
//     S = Q K^T, dP = dO V^T, dS = P (dP - Di); dQ += dS K (TMEM), dQ / 8 at the end
//   Di = rowsum(dO * O) per (query, head) from a small warp-per-row kernel.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <mutex>

#include "launch_count.cuh"
#include "ops.cuh"
#include "ptx.cuh"
#include "pdl.cuh"

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

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp; the TF32 path's probabilities are rounded to TF32
// afterwards anyway); exp2f's range fix-ups cost more than the exponential itself here.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// The same rounding (to nearest, ties away from zero, on the 10-bit TF32 mantissa) as one
// integer add: the tensor core drops the low 13 bits the add has carried into. Finite inputs
// only (softmax probabilities and dS values here).
__device__ __forceinline__ float tf32_round_add(float x) { return __uint_as_float(__float_as_uint(x) + 0x1000u); }

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

// Non-blocking mbarrier phase test (the MMA warp's event loop polls several barriers).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// TMEM <- registers: 32 lanes x 32 columns (thread t of the warp writes its lane's 32 values).
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem: 128 lanes x 8 fp32 columns] * B[smem]^T, kind::tf32 (A K-major).
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Forward: a persistent, warp-specialised kernel. Work units are (batch, head, 128-query tile),
// longest (most key tiles) first, dealt to the CTAs in snake order; each CTA streams the key
// tiles of all its units through one pipeline, so the next unit's Q / K / V loads and its first
// S = Q K^T overlap the current unit's last softmax and epilogue (a CTA per unit paid a cold
// TMA + TMEM start per 2-8 tiles of work).
//   warp 5 (one lane): TMA loads — Q of each unit (single buffer, reloaded once the unit's last
//     S has been computed), K(g) / V(g) double-buffered over the CTA's global tile sequence g;
//   warp 4 (one lane): tcgen05.mma issue from an event loop — S(g) = Q K(g)^T as soon as its
//     buffer is read out (up to two tiles ahead of the softmax), O += P(g) V(g) with P from
//     TMEM once the softmax warps have stored it;
//   warps 0-3 (thread = query row): online softmax in registers. The running max used by the
//     exponentials is only raised when a row's max exceeds it by more than 2^8 (lazy rescale:
//     O and l are multiplied in place then, warp-uniformly, after the previous PV has landed);
//     P <= 2^8 stays well inside fp32 / TF32 range. Max and sum use four accumulators each.
// smem: Q 32 KB + K 2 x 16 KB + V 2 x 16 KB (two CTAs per SM); TMEM: S 2 x 64, P 64, O 64.
constexpr int kFwdSmem = 32768 + 2 * 16384 + 2 * 16384 + 128 + 1024;
constexpr float kRescaleLog2 = 8.0f;

#ifdef HY_ATTN_TRACE  // diagnostics build (tools/attn_trace.cu): per-tile timestamps of CTA 0
__device__ unsigned long long g_attn_trace[8][256];
#define ATTN_TRACE(slot, g)                                                 \
  do {                                                                      \
    if (blockIdx.x == 0 && (g) < 256) g_attn_trace[slot][g] = clock64(); \
  } while (0)
#else
#define ATTN_TRACE(slot, g) \
  do {                      \
  } while (0)
#endif

struct FwdUnits {
  int nqt, BH, U, G;  // query tiles per (b, h), batch*heads, units, CTAs
  // unit -> (bh, qt): longest tiles first
  __device__ __forceinline__ void unit(int u, int& bh, int& qt) const {
    qt = nqt - 1 - u / BH;
    bh = u % BH;
  }
  // r-th unit of CTA c in snake order (-1 past the end)
  __device__ __forceinline__ int nth(int c, int r) const {
    const int u = r * G + ((r & 1) ? G - 1 - c : c);
    return u < U ? u : -1;
  }
};

__global__ void __launch_bounds__(192, 2) attn_fwd_kernel(const __grid_constant__ CUtensorMap mq,
                                                          const __grid_constant__ CUtensorMap mk,
                                                          const __grid_constant__ CUtensorMap mv, int T, int H,
                                                          int B, float* __restrict__ out, float* __restrict__ lse2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = align1024(smem_raw);
  uint8_t* sK0 = sQ + 32768;
  uint8_t* sV0 = sK0 + 2 * 16384;
  // barriers: 0 q, 1-2 kfull, 3-4 vfull, 5-6 sdone, 7-8 pvdone, 9 pready (4 arrivals),
  // 10-11 sfree (4 arrivals: the softmax warps have read S out of that buffer)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV0 + 2 * 16384);
  uint64_t *bq = bar, *bk = bar + 1, *bv = bar + 3, *bs = bar + 5, *bpv = bar + 7, *bp = bar + 9, *bsf = bar + 10;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 12);
  const int tid = threadIdx.x, warp = tid >> 5;
  FwdUnits W;
  W.nqt = (T + 127) / 128;
  W.BH = B * H;
  W.U = W.nqt * W.BH;
  W.G = static_cast<int>(gridDim.x);
  const int c = static_cast<int>(blockIdx.x);
  const int D = H * HD;
  auto nkt_of = [&](int qt) { return min((T + 63) / 64, (qt * 128 + 128) / 64); };
  if (tid == 0) {
    tma_prefetch_desc(&mq);
    tma_prefetch_desc(&mk);
    tma_prefetch_desc(&mv);
    for (int i = 0; i < 12; ++i) mbar_init(&bar[i], i >= 9 ? 4 : 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait_and_trigger();
  const uint32_t tbase = *tslot;
  const uint32_t tP = tbase + 128, tO = tbase + 192;
  if (warp == 5) {
    // two independent loader lanes: lane 0 streams Q and K (K(g) once S(g-2) has read its
    // buffer), lane 1 streams V (V(g) once PV(g-2) has) — one lane for both made every K wait
    // behind the previous V's PV, which left S(g+2) without its K (tools/attn_trace.cu)
    const int ln = lane_id();
    if (ln < 2) {
      int g = 0;
      for (int r = 0;; ++r) {
        const int u = W.nth(c, r);
        if (u < 0) break;
        int bh, qt;
        W.unit(u, bh, qt);
        const int b = bh / H, h = bh % H, row0 = b * T;
        if (ln == 0) {
          if (g > 0) mbar_wait(&bs[(g - 1) & 1], ((g - 1) >> 1) & 1);  // previous unit's last S: Q free
          mbar_expect_tx(bq, 32768);
          tma_load_2d(sQ, &mq, bq, h * HD, row0 + qt * 128);
          tma_load_2d(sQ + 16384, &mq, bq, h * HD + 32, row0 + qt * 128);
        }
        const int nkt = nkt_of(qt);
        for (int j = 0; j < nkt; ++j, ++g) {
          const int s = g & 1;
          if (ln == 0) {
            if (g >= 2) mbar_wait(&bs[s], ((g - 2) >> 1) & 1);  // S(g-2) read K(g-2)
            uint8_t* dk = sK0 + s * 16384;
            mbar_expect_tx(&bk[s], 16384);
            tma_load_2d(dk, &mk, &bk[s], D + h * HD, row0 + j * 64);
            tma_load_2d(dk + 8192, &mk, &bk[s], D + h * HD + 32, row0 + j * 64);
          } else {
            if (g >= 2) mbar_wait(&bpv[s], ((g - 2) >> 1) & 1);  // PV(g-2) read V(g-2)
            uint8_t* dv = sV0 + s * 16384;
            mbar_expect_tx(&bv[s], 16384);
            for (int kb = 0; kb < 2; ++kb)
              for (int jn = 0; jn < 2; ++jn)
                tma_load_2d(dv + kb * 8192 + jn * 4096, &mv, &bv[s], 2 * D + h * HD + 32 * jn, row0 + j * 64 + 32 * kb);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    if (lane_id() == 0) {  // MMA issuer: an event loop over two cursors, S ahead of PV
      constexpr uint32_t idS = idesc_tf32(128, 64, false, false);
      constexpr uint32_t idPV = idesc_tf32(128, 64, false, true);
      // cursor over this CTA's tile sequence: global tile g, unit ordinal r, tile j of nkt
      struct Cur {
        int g, r, j, nkt;
      };
      auto start = [&](Cur& x) {
        x.g = 0;
        x.r = 0;
        x.j = 0;
        const int u = W.nth(c, 0);
        int bh, qt;
        if (u >= 0) W.unit(u, bh, qt);
        x.nkt = u >= 0 ? nkt_of(qt) : 0;
      };
      auto advance = [&](Cur& x) {
        ++x.g;
        if (++x.j == x.nkt) {
          x.j = 0;
          ++x.r;
          const int u = W.nth(c, x.r);
          int bh, qt;
          if (u >= 0) W.unit(u, bh, qt);
          x.nkt = u >= 0 ? nkt_of(qt) : 0;
        }
      };
      Cur cs, cp;
      start(cs);
      start(cp);
      // S(g) = Q K(g)^T may run two tiles ahead of the softmax: it needs K(g) and its unit's Q
      // landed and the softmax warps to have read S(g-2) out of the buffer (sfree), so it is
      // issued while softmax(g-1) still runs, ahead of PV(g-1) in the tensor pipe when it can be.
      // PV(g) needs P(g) stored (pready) and V(g) landed.
      while (cp.nkt > 0) {
        bool progressed = false;
        if (cs.nkt > 0) {
          const int g = cs.g, sb = g & 1;
          if ((g < 2 || mbar_test(&bsf[sb], ((g - 2) >> 1) & 1)) && mbar_test(bq, cs.r & 1) &&
              mbar_test(&bk[sb], (g >> 1) & 1)) {
            tc_fence_after();
            const uint32_t tS = tbase + sb * 64;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_tf32(tS, desc_k(sQ, kk, 16384), desc_k(sK0 + sb * 16384, kk, 8192), idS, kk > 0);
            mma_commit(&bs[sb]);
            ATTN_TRACE(0, g);
            advance(cs);
            progressed = true;
          }
        }
        {
          const int g = cp.g, sb = g & 1;
          if (cp.g < cs.g && mbar_test(bp, g & 1) && mbar_test(&bv[sb], (g >> 1) & 1)) {
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma_tf32_ts(tO, tP + kk * 8, desc_mn(sV0 + sb * 16384, kk), idPV, (cp.j | kk) > 0);
            mma_commit(&bpv[sb]);
            ATTN_TRACE(1, g);
            advance(cp);
            progressed = true;
          }
        }
        if (!progressed) __nanosleep(20);
      }
    }
    __syncwarp();
  } else {
    const uint32_t lane_off = static_cast<uint32_t>((tid & ~31) << 16);
    int g = 0;
    for (int r = 0;; ++r) {
      const int u = W.nth(c, r);
      if (u < 0) break;
      int bh, qt;
      W.unit(u, bh, qt);
      const int b = bh / H, h = bh % H, row0 = b * T, q0 = qt * 128;
      const int nkt = nkt_of(qt);
      const int q = q0 + tid;
      float m_used = -FLT_MAX, l_run = 0.f;  // m_used: scaled (log2-domain) max the exponentials use
      for (int j = 0; j < nkt; ++j, ++g) {
        const int k0 = j * 64, s_ = g & 1;
        if (tid == 0) ATTN_TRACE(2, g);
        mbar_wait(&bs[s_], (g >> 1) & 1);
        if (tid == 0) ATTN_TRACE(3, g);
        tc_fence_after();
        float s[64];
        tmem_ld64(tbase + s_ * 64 + lane_off, s);
        if (tid == 0) ATTN_TRACE(4, g);
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&bsf[s_]);  // S buffer free for S(g+2)
        if (k0 + 63 > q0) {  // diagonal tile: mask keys past the row (CTA-uniform test)
#pragma unroll
          for (int i = 0; i < 64; ++i) s[i] = (k0 + i <= q) ? s[i] : -FLT_MAX;
        }
        float mx4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
        for (int i = 4; i < 64; i += 4) {
#pragma unroll
          for (int v = 0; v < 4; ++v) mx4[v] = fmaxf(mx4[v], s[i + v]);
        }
        const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * kScaleLog2;
        float alpha = 1.f;
        if (mx > m_used + kRescaleLog2 || j == 0) {
          alpha = fast_exp2(m_used - mx);  // 0 on the first tile (m_used = -FLT_MAX)
          m_used = mx;
        }
        float sum4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const float p = fast_exp2(fmaf(s[i + v], kScaleLog2, -m_used));  // masked: 2^-huge = 0
            sum4[v] += p;
            s[i + v] = tf32_round_add(p);
          }
        }
        l_run = l_run * alpha + ((sum4[0] + sum4[1]) + (sum4[2] + sum4[3]));
        if (tid == 0) ATTN_TRACE(5, g);
        if (j > 0) {  // PV(g-1) landed: P free, O final up to tile j-1
          mbar_wait(&bpv[(g - 1) & 1], ((g - 1) >> 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {  // lazy rescale of this warp's O rows
            float o[64];
            tmem_ld64(tO + lane_off, o);
#pragma unroll
            for (int i = 0; i < 64; ++i) o[i] *= alpha;
            tmem_st_x32(tO + lane_off, o);
            tmem_st_x32(tO + lane_off + 32, o + 32);
          }
        }
        if (tid == 0) ATTN_TRACE(6, g);
        tmem_st_x32(tP + lane_off, s);
        tmem_st_x32(tP + lane_off + 32, s + 32);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(bp);
        if (tid == 0) ATTN_TRACE(7, g);
      }
      // unit epilogue: O / l once the last PV has landed (the next unit's first PV, which
      // overwrites O, is only issued after these rows have stored its P, i.e. after this read)
      mbar_wait(&bpv[(g - 1) & 1], ((g - 1) >> 1) & 1);
      tc_fence_after();
      float o[64];
      tmem_ld64(tO + lane_off, o);
      if (q < T) {
        const float inv = 1.f / l_run;
        float4* dst = reinterpret_cast<float4*>(out + static_cast<long>(row0 + q) * D + h * HD);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          dst[i] = make_float4(o[4 * i] * inv, o[4 * i + 1] * inv, o[4 * i + 2] * inv, o[4 * i + 3] * inv);
        lse2[static_cast<long>(bh) * T + q] = m_used + log2f(l_run);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(*tslot);
  }
}

// Di[bh*T + q] = sum_c dO[q, h*64 + c] * O[q, h*64 + c]; 16 lanes per (row, head), one
// float4 of O and of dO each (fully coalesced 256-byte head slices), then a 16-lane shuffle sum.
__global__ void attn_di_kernel(long n, int T, int H, const float* __restrict__ out, const float* __restrict__ dout,
                               float* __restrict__ Di) {
  pdl_wait_and_trigger();
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long w = t >> 4;  // (row, head) pair
  const int sub = static_cast<int>(t & 15);
  float v = 0.f;
  if (w < n) {
    const long row = w / H;
    const int h = static_cast<int>(w % H);
    const long off = row * static_cast<long>(H) * HD + h * HD + 4 * sub;
    const float4 a = __ldg(reinterpret_cast<const float4*>(out + off));
    const float4 g = __ldg(reinterpret_cast<const float4*>(dout + off));
    v = (a.x * g.x + a.y * g.y) + (a.z * g.z + a.w * g.w);
  }
#pragma unroll
  for (int m = 8; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  if (w < n && sub == 0) {
    const long row = w / H;
    const int h = static_cast<int>(w % H);
    const long b = row / T, q = row % T;
    Di[(b * H + h) * T + q] = v;
  }
}

// dK, dV, persistent and warp-specialised: units (batch, head, 128-key tile), those near the
// start of the sequence (the most query tiles) first, in snake order over one CTA per SM; the
// query tiles of all a CTA's units stream through one pipeline (global tile index g):
//   warp 5 (one lane): TMA — K and V of each unit (reloaded once its last S^T / dP^T landed),
//     Q and dO of tile g in both majors into stage g & 1;
//   warp 4 (one lane): tcgen05.mma from an event loop — S^T(g) = K Q(g)^T and dP^T(g) = V dO(g)^T
//     into TMEM buffer g & 1 once the compute warps have read it out, then dV += P^T(g) dO(g) and
//     dK += dS^T(g) Q(g) with P^T, dS^T from TMEM once they are stored;
//   warps 0-3 (thread = key row): P^T = exp2(S^T c - lse2), dS^T = P^T (dP^T - Di), TF32-rounded
//     (the softmax scale 1/8 is applied to dK once at the end).
// smem: K, V 32 KB each + 2 stages x (Q k, Q mn, dO k, dO mn) 64 KB = 192 KB;
// TMEM: S^T 2 x 64, dP^T 2 x 64, P^T 64, dS^T 64, dV 64, dK 64 columns.
constexpr int kDkvSmem = 32768 * 2 + 2 * 65536 + 256 + 1024 + 1024;  // + lse / Di staging

struct KvUnits {
  int nkt, BH, U, G;
  // unit -> (bh, kt): key tiles near the start (most queries) first
  __device__ __forceinline__ void unit(int u, int& bh, int& kt) const {
    kt = u / BH;
    bh = u % BH;
  }
  __device__ __forceinline__ int nth(int c, int r) const {
    const int u = r * G + ((r & 1) ? G - 1 - c : c);
    return u < U ? u : -1;
  }
};

__global__ void __launch_bounds__(192, 1) attn_dkdv_kernel(
    const __grid_constant__ CUtensorMap mkv128, const __grid_constant__ CUtensorMap mq64,
    const __grid_constant__ CUtensorMap mqmn, const __grid_constant__ CUtensorMap mdo64,
    const __grid_constant__ CUtensorMap mdomn, int T, int H, int B, const float* __restrict__ lse2,
    const float* __restrict__ Di, float* __restrict__ dqkv) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sK = align1024(smem_raw);
  uint8_t* sV = sK + 32768;
  uint8_t* sQG = sV + 32768;  // stage s: Q k at +0, Q mn at +16K, dO k at +32K, dO mn at +48K
  // barriers: 0 kv, 1-2 qg, 3-4 spdone, 5-6 sfree (4), 7 pds (4), 8-9 gdone
  uint64_t* bar = reinterpret_cast<uint64_t*>(sQG + 2 * 65536);
  uint64_t *bkv = bar, *bqg = bar + 1, *bsp = bar + 3, *bsf = bar + 5, *bpd = bar + 7, *bgd = bar + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 10);
  float* sLD = reinterpret_cast<float*>(bar + 16);  // [2][lse 64 | Di 64] per query tile
  const int tid = threadIdx.x, warp = tid >> 5;
  KvUnits W;
  W.nkt = (T + 127) / 128;
  W.BH = B * H;
  W.U = W.nkt * W.BH;
  W.G = static_cast<int>(gridDim.x);
  const int c = static_cast<int>(blockIdx.x);
  const int D = H * HD;
  auto nq_of = [&](int kt) { return (T - kt * 128 + 63) / 64; };
  if (tid == 0) {
    tma_prefetch_desc(&mkv128);
    tma_prefetch_desc(&mq64);
    tma_prefetch_desc(&mqmn);
    tma_prefetch_desc(&mdo64);
    tma_prefetch_desc(&mdomn);
    for (int i = 0; i < 10; ++i) mbar_init(&bar[i], (i >= 5 && i <= 7) ? 4 : 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait_and_trigger();
  // S^T: tb + 64s, dP^T: tb + 128 + 64s, P^T: tb + 256, dS^T: tb + 320, dV: tb + 384, dK: tb + 448
  const uint32_t tb = *tslot;
  const uint32_t tPT = tb + 256, tDST = tb + 320, tdV = tb + 384, tdK = tb + 448;
  if (warp == 5) {
    if (lane_id() == 0) {  // loader
      int g = 0;
      for (int r = 0;; ++r) {
        const int u = W.nth(c, r);
        if (u < 0) break;
        int bh, kt;
        W.unit(u, bh, kt);
        const int b = bh / H, h = bh % H, row0 = b * T, k0 = kt * 128;
        if (g > 0) mbar_wait(&bsp[(g - 1) & 1], ((g - 1) >> 1) & 1);  // last S^T / dP^T of the previous unit
        mbar_expect_tx(bkv, 65536);
        for (int kb = 0; kb < 2; ++kb) {
          tma_load_2d(sK + kb * 16384, &mkv128, bkv, D + h * HD + 32 * kb, row0 + k0);
          tma_load_2d(sV + kb * 16384, &mkv128, bkv, 2 * D + h * HD + 32 * kb, row0 + k0);
        }
        const int nq = nq_of(kt);
        for (int i = 0; i < nq; ++i, ++g) {
          const int sb = g & 1;
          if (g >= 2) mbar_wait(&bgd[sb], ((g - 2) >> 1) & 1);  // dV / dK(g-2) read stage sb
          uint8_t* st = sQG + sb * 65536;
          const int q0 = k0 + 64 * i;
          mbar_expect_tx(&bqg[sb], 4 * 16384);
          for (int kb = 0; kb < 2; ++kb) {
            tma_load_2d(st + kb * 8192, &mq64, &bqg[sb], h * HD + 32 * kb, row0 + q0);
            tma_load_2d(st + 32768 + kb * 8192, &mdo64, &bqg[sb], h * HD + 32 * kb, row0 + q0);
            for (int jn = 0; jn < 2; ++jn) {
              tma_load_2d(st + 16384 + kb * 8192 + jn * 4096, &mqmn, &bqg[sb], h * HD + 32 * jn, row0 + q0 + 32 * kb);
              tma_load_2d(st + 49152 + kb * 8192 + jn * 4096, &mdomn, &bqg[sb], h * HD + 32 * jn, row0 + q0 + 32 * kb);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    if (lane_id() == 0) {  // MMA issuer: S^T / dP^T ahead of dV / dK
      constexpr uint32_t idT = idesc_tf32(128, 64, false, false);  // S^T, dP^T
      constexpr uint32_t idG = idesc_tf32(128, 64, false, true);   // dV, dK (B MN-major)
      struct Cur {
        int g, r, j, n;
      };
      auto set_unit = [&](Cur& x) {
        const int u = W.nth(c, x.r);
        int bh, kt;
        if (u >= 0) W.unit(u, bh, kt);
        x.n = u >= 0 ? nq_of(kt) : 0;
      };
      auto advance = [&](Cur& x) {
        ++x.g;
        if (++x.j == x.n) {
          x.j = 0;
          ++x.r;
          set_unit(x);
        }
      };
      Cur cs{0, 0, 0, 0}, cp{0, 0, 0, 0};
      set_unit(cs);
      set_unit(cp);
      while (cp.n > 0) {
        bool progressed = false;
        if (cs.n > 0) {
          const int g = cs.g, sb = g & 1;
          if ((g < 2 || mbar_test(&bsf[sb], ((g - 2) >> 1) & 1)) && mbar_test(bkv, cs.r & 1) &&
              mbar_test(&bqg[sb], (g >> 1) & 1)) {
            tc_fence_after();
            uint8_t* st = sQG + sb * 65536;
            const uint32_t tS = tb + sb * 64, tP = tb + 128 + sb * 64;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_tf32(tS, desc_k(sK, kk, 16384), desc_k(st, kk, 8192), idT, kk > 0);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_tf32(tP, desc_k(sV, kk, 16384), desc_k(st + 32768, kk, 8192), idT, kk > 0);
            mma_commit(&bsp[sb]);
            advance(cs);
            progressed = true;
          }
        }
        {
          const int g = cp.g, sb = g & 1;
          if (cp.g < cs.g && mbar_test(bpd, g & 1)) {
            tc_fence_after();
            uint8_t* st = sQG + sb * 65536;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_tf32_ts(tdV, tPT + kk * 8, desc_mn(st + 49152, kk), idG, (cp.j | kk) > 0);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_tf32_ts(tdK, tDST + kk * 8, desc_mn(st + 16384, kk), idG, (cp.j | kk) > 0);
            mma_commit(&bgd[sb]);
            advance(cp);
            progressed = true;
          }
        }
        if (!progressed) __nanosleep(20);
      }
    }
    __syncwarp();
  } else {
    const uint32_t lane_off = static_cast<uint32_t>((tid & ~31) << 16);
    int g = 0;
    for (int r = 0;; ++r) {
      const int u = W.nth(c, r);
      if (u < 0) break;
      int bh, kt;
      W.unit(u, bh, kt);
      const int b = bh / H, h = bh % H, row0 = b * T, k0 = kt * 128;
      const int nq = nq_of(kt);
      const int key = k0 + tid;
      const float* lse_bh = lse2 + static_cast<long>(bh) * T;
      const float* di_bh = Di + static_cast<long>(bh) * T;
      for (int i = 0; i < nq; ++i, ++g) {
        const int q0 = k0 + 64 * i, sb = g & 1;
        // the tile's 64 lse / Di values, one per compute thread, staged for broadcast reads
        float* ld = sLD + sb * 128;
        {
          const int q = q0 + (tid & 63);
          ld[tid] = q < T ? (tid < 64 ? lse_bh[q] : di_bh[q]) : 0.f;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        mbar_wait(&bsp[sb], (g >> 1) & 1);
        tc_fence_after();
        float s[64], dp[64];
        tmem_ld64(tb + sb * 64 + lane_off, s);
        tmem_ld64(tb + 128 + sb * 64 + lane_off, dp);
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&bsf[sb]);  // S^T / dP^T buffer free for g + 2
        const bool full = q0 >= k0 + 127 && q0 + 63 < T;  // no masked (query, key) pair in the tile
        if (full) {
#pragma unroll
          for (int cc = 0; cc < 64; ++cc) {
            const float p = fast_exp2(fmaf(s[cc], kScaleLog2, -ld[cc]));
            s[cc] = tf32_round_add(p);
            dp[cc] = tf32_round_add(p * (dp[cc] - ld[64 + cc]));  // the 1/8 of dS is applied to dK
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < 64; ++cc) {
            const int q = q0 + cc;
            const bool valid = q >= key && q < T;
            const float p = valid ? fast_exp2(fmaf(s[cc], kScaleLog2, -ld[cc])) : 0.f;
            s[cc] = tf32_round_add(p);
            dp[cc] = valid ? tf32_round_add(p * (dp[cc] - ld[64 + cc])) : 0.f;
          }
        }
        if (g >= 1) mbar_wait(&bgd[(g - 1) & 1], ((g - 1) >> 1) & 1);  // P^T, dS^T(g-1) consumed
        tmem_st_x32(tPT + lane_off, s);
        tmem_st_x32(tPT + lane_off + 32, s + 32);
        tmem_st_x32(tDST + lane_off, dp);
        tmem_st_x32(tDST + lane_off + 32, dp + 32);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(bpd);
      }
      // unit epilogue (the next unit's first dV / dK MMAs overwrite them only after these rows
      // have stored that unit's first P^T / dS^T, i.e. after this read)
      mbar_wait(&bgd[(g - 1) & 1], ((g - 1) >> 1) & 1);
      tc_fence_after();
      float dv[64], dk[64];
      tmem_ld64(tdV + lane_off, dv);
      tmem_ld64(tdK + lane_off, dk);
      if (key < T) {
        float4* gk = reinterpret_cast<float4*>(dqkv + static_cast<long>(row0 + key) * 3 * D + D + h * HD);
        float4* gv = reinterpret_cast<float4*>(dqkv + static_cast<long>(row0 + key) * 3 * D + 2 * D + h * HD);
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) {
          gk[cc] = make_float4(0.125f * dk[4 * cc], 0.125f * dk[4 * cc + 1], 0.125f * dk[4 * cc + 2], 0.125f * dk[4 * cc + 3]);
          gv[cc] = make_float4(dv[4 * cc], dv[4 * cc + 1], dv[4 * cc + 2], dv[4 * cc + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(*tslot);
  }
}

// dQ, persistent and warp-specialised like the forward: units (batch, head, 128-query tile),
// longest first in snake order over one CTA per SM; the key tiles of all a CTA's units stream
// through one pipeline (global tile index g):
//   warp 5 (one lane): TMA — Q and dO of each unit (reloaded once its last S / dP landed),
//     K (K-major), V (K-major), K (MN-major) of tile g into stage g & 1;
//   warp 4 (one lane): tcgen05.mma from an event loop — S(g) = Q K(g)^T and dP(g) = dO V(g)^T
//     into TMEM buffer g & 1 as soon as the softmax warps have read that buffer out, and
//     dQ += dS(g) K(g) (dS from TMEM) once dS(g) is stored;
//   warps 0-3 (thread = query row): dS = P (dP - Di), P = exp2(S c - lse2), TF32-rounded.
// smem: Q, dO 32 KB each + 2 stages x (K k, V k, K mn) 48 KB = 160 KB;
// TMEM: S 2 x 64, dP 2 x 64, dS 2 x 64, dQ 64 columns.
constexpr int kDqSmem = 32768 * 2 + 2 * 49152 + 256 + 1024;

__global__ void __launch_bounds__(192, 1) attn_dq_kernel(
    const __grid_constant__ CUtensorMap mq128, const __grid_constant__ CUtensorMap mdo128,
    const __grid_constant__ CUtensorMap mk64, const __grid_constant__ CUtensorMap mkmn, int T, int H, int B,
    const float* __restrict__ lse2, const float* __restrict__ Di, float* __restrict__ dqkv) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = align1024(smem_raw);
  uint8_t* sG = sQ + 32768;
  uint8_t* sKV = sG + 32768;  // stage s: Kk at +0, Vk at +16K, Km at +32K
  // barriers: 0 q/do, 1-2 kv, 3-4 spdone, 5-6 sfree (4), 7-8 dsready (4), 9-10 dqdone
  uint64_t* bar = reinterpret_cast<uint64_t*>(sKV + 2 * 49152);
  uint64_t *bq = bar, *bkv = bar + 1, *bsp = bar + 3, *bsf = bar + 5, *bds = bar + 7, *bdq = bar + 9;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 12);
  const int tid = threadIdx.x, warp = tid >> 5;
  FwdUnits W;
  W.nqt = (T + 127) / 128;
  W.BH = B * H;
  W.U = W.nqt * W.BH;
  W.G = static_cast<int>(gridDim.x);
  const int c = static_cast<int>(blockIdx.x);
  const int D = H * HD;
  auto nkt_of = [&](int qt) { return min((T + 63) / 64, (qt * 128 + 128) / 64); };
  if (tid == 0) {
    tma_prefetch_desc(&mq128);
    tma_prefetch_desc(&mdo128);
    tma_prefetch_desc(&mk64);
    tma_prefetch_desc(&mkmn);
    for (int i = 0; i < 11; ++i) mbar_init(&bar[i], (i >= 5 && i <= 8) ? 4 : 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait_and_trigger();
  const uint32_t tb = *tslot;  // S: tb + 64s, dP: tb + 128 + 64s, dS: tb + 256 + 64s, dQ: tb + 384
  const uint32_t tdQ = tb + 384;
  if (warp == 5) {
    if (lane_id() == 0) {  // loader
      int g = 0;
      for (int r = 0;; ++r) {
        const int u = W.nth(c, r);
        if (u < 0) break;
        int bh, qt;
        W.unit(u, bh, qt);
        const int b = bh / H, h = bh % H, row0 = b * T, q0 = qt * 128;
        if (g > 0) mbar_wait(&bsp[(g - 1) & 1], ((g - 1) >> 1) & 1);  // last S / dP of the previous unit
        mbar_expect_tx(bq, 65536);
        for (int kb = 0; kb < 2; ++kb) {
          tma_load_2d(sQ + kb * 16384, &mq128, bq, h * HD + 32 * kb, row0 + q0);
          tma_load_2d(sG + kb * 16384, &mdo128, bq, h * HD + 32 * kb, row0 + q0);
        }
        const int nkt = nkt_of(qt);
        for (int j = 0; j < nkt; ++j, ++g) {
          const int s = g & 1;
          if (g >= 2) mbar_wait(&bdq[s], ((g - 2) >> 1) & 1);  // dQ(g-2) read stage s (after S / dP did)
          uint8_t* st = sKV + s * 49152;
          const int k0 = 64 * j;
          mbar_expect_tx(&bkv[s], 3 * 16384);
          for (int kb = 0; kb < 2; ++kb) {
            tma_load_2d(st + kb * 8192, &mk64, &bkv[s], D + h * HD + 32 * kb, row0 + k0);
            tma_load_2d(st + 16384 + kb * 8192, &mk64, &bkv[s], 2 * D + h * HD + 32 * kb, row0 + k0);
            for (int jn = 0; jn < 2; ++jn)
              tma_load_2d(st + 32768 + kb * 8192 + jn * 4096, &mkmn, &bkv[s], D + h * HD + 32 * jn, row0 + k0 + 32 * kb);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    if (lane_id() == 0) {  // MMA issuer: S / dP ahead of dQ
      constexpr uint32_t idS = idesc_tf32(128, 64, false, false);
      constexpr uint32_t idQ = idesc_tf32(128, 64, false, true);
      struct Cur {
        int g, r, j, nkt;
      };
      auto set_unit = [&](Cur& x) {
        const int u = W.nth(c, x.r);
        int bh, qt;
        if (u >= 0) W.unit(u, bh, qt);
        x.nkt = u >= 0 ? nkt_of(qt) : 0;
      };
      auto advance = [&](Cur& x) {
        ++x.g;
        if (++x.j == x.nkt) {
          x.j = 0;
          ++x.r;
          set_unit(x);
        }
      };
      Cur cs{0, 0, 0, 0}, cp{0, 0, 0, 0};
      set_unit(cs);
      set_unit(cp);
      while (cp.nkt > 0) {
        bool progressed = false;
        if (cs.nkt > 0) {
          const int g = cs.g, sb = g & 1;
          if ((g < 2 || mbar_test(&bsf[sb], ((g - 2) >> 1) & 1)) && mbar_test(bq, cs.r & 1) &&
              mbar_test(&bkv[sb], (g >> 1) & 1)) {
            tc_fence_after();
            uint8_t* st = sKV + sb * 49152;
            const uint32_t tS = tb + sb * 64, tP = tb + 128 + sb * 64;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_tf32(tS, desc_k(sQ, kk, 16384), desc_k(st, kk, 8192), idS, kk > 0);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_tf32(tP, desc_k(sG, kk, 16384), desc_k(st + 16384, kk, 8192), idS, kk > 0);
            mma_commit(&bsp[sb]);
            advance(cs);
            progressed = true;
          }
        }
        {
          const int g = cp.g, sb = g & 1;
          if (cp.g < cs.g && mbar_test(&bds[sb], (g >> 1) & 1)) {
            tc_fence_after();
            const uint32_t tdS = tb + 256 + sb * 64;
            uint8_t* km = sKV + sb * 49152 + 32768;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) mma_tf32_ts(tdQ, tdS + kk * 8, desc_mn(km, kk), idQ, (cp.j | kk) > 0);
            mma_commit(&bdq[sb]);
            advance(cp);
            progressed = true;
          }
        }
        if (!progressed) __nanosleep(20);
      }
    }
    __syncwarp();
  } else {
    const uint32_t lane_off = static_cast<uint32_t>((tid & ~31) << 16);
    int g = 0;
    for (int r = 0;; ++r) {
      const int u = W.nth(c, r);
      if (u < 0) break;
      int bh, qt;
      W.unit(u, bh, qt);
      const int b = bh / H, h = bh % H, row0 = b * T, q0 = qt * 128;
      const int nkt = nkt_of(qt);
      const int q = q0 + tid;
      const long li = static_cast<long>(bh) * T + min(q, T - 1);
      const float my_lse = lse2[li], my_di = Di[li];
      for (int j = 0; j < nkt; ++j, ++g) {
        const int k0 = 64 * j, sb = g & 1;
        mbar_wait(&bsp[sb], (g >> 1) & 1);
        tc_fence_after();
        float s[64], dp[64];
        tmem_ld64(tb + sb * 64 + lane_off, s);
        tmem_ld64(tb + 128 + sb * 64 + lane_off, dp);
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&bsf[sb]);  // S / dP buffer free for S(g+2) / dP(g+2)
        if (k0 + 63 <= q0) {  // whole tile visible (CTA-uniform)
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const float p = fast_exp2(fmaf(s[i], kScaleLog2, -my_lse));
            s[i] = tf32_round_add(p * (dp[i] - my_di));  // the 1/8 of dS is applied to dQ
          }
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const bool valid = k0 + i <= q;
            const float p = valid ? fast_exp2(fmaf(s[i], kScaleLog2, -my_lse)) : 0.f;
            s[i] = valid ? tf32_round_add(p * (dp[i] - my_di)) : 0.f;
          }
        }
        if (g >= 2) mbar_wait(&bdq[sb], ((g - 2) >> 1) & 1);  // dQ(g-2) read this dS buffer
        const uint32_t tdS = tb + 256 + sb * 64 + lane_off;
        tmem_st_x32(tdS, s);
        tmem_st_x32(tdS + 32, s + 32);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&bds[sb]);
      }
      // unit epilogue (the next unit's first dQ MMA overwrites dQ only after these rows have
      // stored that unit's first dS, i.e. after this read)
      mbar_wait(&bdq[(g - 1) & 1], ((g - 1) >> 1) & 1);
      tc_fence_after();
      float dq[64];
      tmem_ld64(tdQ + lane_off, dq);
      if (q < T) {
        float4* gq = reinterpret_cast<float4*>(dqkv + static_cast<long>(row0 + q) * 3 * D + h * HD);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          gq[i] = make_float4(0.125f * dq[4 * i], 0.125f * dq[4 * i + 1], 0.125f * dq[4 * i + 2], 0.125f * dq[4 * i + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(*tslot);
  }
}

int attn_sm_count() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v > 0 ? v : 148;
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
  {
    const cudaError_t e = ensure_smem_limit(attn_fwd_kernel, kFwdSmem);
    if (e != cudaSuccess) return e;
  }
  const int units = B * H * ((T + 127) / 128);
  const int grid = std::min(units, 2 * attn_sm_count());  // persistent: two CTAs per SM
  count_launch();
  return launch_pdl(attn_fwd_kernel, dim3(grid), dim3(192), kFwdSmem, st, mq, mk, mv, T, H, B, out, lse2);
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
  {
    cudaError_t e = ensure_smem_limit(attn_dkdv_kernel, kDkvSmem);
    if (e == cudaSuccess) e = ensure_smem_limit(attn_dq_kernel, kDqSmem);
    if (e != cudaSuccess) return e;
  }
  const long n = rows * H;
  count_launch();
  {
    const cudaError_t e = launch_pdl(attn_di_kernel, dim3(static_cast<unsigned>((16 * n + 255) / 256)), dim3(256), 0, st, n, T, H, out, dout, Di);
    if (e != cudaSuccess) return e;
  }
  const int tiles = (T + 127) / 128;
  count_launch();
  {
    const int grid = std::min(B * H * tiles, attn_sm_count());  // persistent: one CTA per SM
    const cudaError_t e = launch_pdl(attn_dkdv_kernel, dim3(grid), dim3(192), kDkvSmem, st, mkv128, mq64, mqmn, mdo64, mdomn, T, H, B, static_cast<const float*>(lse2), static_cast<const float*>(Di), dqkv);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  {
    const int grid = std::min(B * H * tiles, attn_sm_count());  // persistent: one CTA per SM
    const cudaError_t e = launch_pdl(attn_dq_kernel, dim3(grid), dim3(192), kDqSmem, st, mq128, mdo128, mk64, mkmn, T, H, B, static_cast<const float*>(lse2), static_cast<const float*>(Di), dqkv);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace hy
