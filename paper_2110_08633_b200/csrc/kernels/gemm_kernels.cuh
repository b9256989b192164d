#pragma once
// Kernel templates of the GEMM (included by gemm_m{0,1,2}.cu, one TU per epilogue mode so the
// instantiations compile in parallel).
//
// Persistent warp-specialised tcgen05 GEMM for sm_100a (kind::tf32, fp32 in HBM).
//
//   warp 0      TMA producer (one elected lane): A/B tiles -> 4-stage smem ring (128B swizzle)
//   warp 1      MMA issuer  (one elected lane): tcgen05.mma 128xBNx8 into TMEM, commit -> mbarriers
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> bias / residual / GELU / GELU' -> st.global
//
// Operands may be K-major or MN-major in global memory (the UMMA descriptor major bit),
// so forward (X W^T), data-grad (dY W) and weight-grad (dY^T X) GEMMs all read their
// inputs in place with no transposes.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "gemm.cuh"
#include "launch_count.cuh"
#include "ptx.cuh"
#include "pdl.cuh"

namespace hy {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // one 128-byte swizzle atom of fp32
constexpr int kStages = 4;
constexpr int kThreads = 256;

using bf16 = __nv_bfloat16;

// Operand element type: fp32 (kind::tf32, 8-deep MMAs) or bf16 (kind::f16, 16-deep MMAs). A stage
// row is one 128-byte swizzle atom either way (32 fp32 / 64 bf16 of K), so stage bytes, the
// K-major descriptors and their 32-byte per-MMA advance are shared; MN-major operands are staged
// in 128-byte MN chunks (32 fp32 with the 32-byte-atom swizzle, 64 bf16 with the plain 128B one).
template <typename T>
struct Elem {
  static constexpr bool kBf16 = sizeof(T) == 2;
  static constexpr int BK = 128 / static_cast<int>(sizeof(T));  // K per stage
  static constexpr int CW = BK;                                 // MN-major chunk width (128 B)
  static constexpr int kMmaK = kBf16 ? 16 : 8;
  static constexpr int kMmas = BK / kMmaK;  // 4 MMAs per stage
};

// UMMA smem descriptor of MMA kk (0..3) of a stage operand at `base`. K-major: 8-row groups of
// 128 B (SBO 1024), advance 32 B of K. MN-major: LBO = one chunk (BK k-rows x 128 B), SBO = the
// swizzle atom's k-rows (4 for the fp32 32-byte atom, 8 for bf16), advance kMmaK k-rows.
template <typename T, bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int kk) {
  constexpr int BKT = Elem<T>::BK;
  if constexpr (!MN) {
    return smem_desc_sw128(base + kk * 32, 16, 1024);
  } else if constexpr (Elem<T>::kBf16) {
    return smem_desc_sw128(base + kk * 2048, BKT * 128, 1024);
  } else {
    return smem_desc_sw128_b32(base + kk * 1024, BKT * 128, 512);
  }
}
template <typename T>
__host__ __device__ constexpr uint32_t idesc_of(int M, int N, bool a_mn, bool b_mn) {
  return Elem<T>::kBf16 ? idesc_bf16(M, N, a_mn, b_mn) : idesc_tf32(M, N, a_mn, b_mn);
}
template <typename T>
__device__ __forceinline__ void mma_one(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (Elem<T>::kBf16) mma_bf16(d, a, b, idesc, acc);
  else mma_tf32(d, a, b, idesc, acc);
}
template <typename T>
__device__ __forceinline__ void mma_two(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (Elem<T>::kBf16) mma_bf16_pair(d, a, b, idesc, acc);
  else mma_tf32_pair(d, a, b, idesc, acc);
}

// P3 (3xTF32, "fp32" precision): every stage also holds the low parts A_lo, B_lo
// (x = hi + lo, hi = tf32_rna(x)); D += A_lo B_hi + A_hi B_lo + A_hi B_hi.
template <int BN, bool P3 = false>
struct Smem {
  static constexpr int kStagesN = P3 ? 3 : kStages;
  static constexpr int kABytes = BM * BK * 4;
  static constexpr int kBBytes = BN * BK * 4;
  static constexpr int kOpBytes = kABytes + kBBytes;
  static constexpr int kStageBytes = P3 ? 2 * kOpBytes : kOpBytes;
  static constexpr int kRing = kStagesN * kStageBytes;
  static constexpr int kEpi = 4 * 32 * 36 * 4;  // per epilogue warp: 32x32 transpose tile, row stride 36
  static constexpr int kTotal = kRing + kEpi + 1024 /*align slack*/ + 256 /*barriers*/;
};

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// gelu_new (tanh form) through the logistic identity 0.5 (1 + tanh u) = 1 / (1 + e^{-2u}):
// one __expf and one fast reciprocal instead of tanhf (relative error ~1e-6, inside
// the 3xTF32 "fp32" tolerances). d/dx: s + 2 x s (1 - s) k0 (1 + 3 k1 x^2), s = sigmoid(2u).
__device__ __forceinline__ float gelu_sig(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float u = k0 * fmaf(k1 * x, x * x, x);
  // exponent clamped so the denominator stays below 2^126 (__fdividef's range)
  return __fdividef(1.f, 1.f + __expf(fminf(-2.f * u, 80.f)));
}
__device__ __forceinline__ float gelu_tanh(float x) { return x * gelu_sig(x); }
// gelu'(x) from the sigmoid gelu_tanh already computed (the forward epilogue stores it for the
// backward, whose GELU' epilogue is then one multiply: no second sigmoid, measured 2.2x a plain
// store at the XL fc shape when it evaluated gelu' itself).
__device__ __forceinline__ float gelu_grad_s(float x, float sg) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return fmaf(2.f * x * sg * (1.f - sg), k0 * fmaf(3.f * k1, x * x, 1.f), sg);
}

// Programmatic dependent launch (pdl.cuh): the prologue (barrier init, TMEM allocation,
// descriptor prefetch) overlaps the previous kernel's tail. The grid is persistent (every CTA
// resident from the start), so letting the next GEMM launch right away only lets its CTAs take
// SMs as ours retire.
struct TileInfo {
  int m0, n0, z1, z2;
  int kb0, nkb;  // first k-block, number of k-blocks
  bool skip;     // tile not computed (causal upper)
};

template <int BN, int BKT = BK>
__device__ __forceinline__ TileInfo tile_info(int tile, int tiles_m, int tiles_n, int M, int N, int K, int nb2,
                                              int causal, int nb1 = 1) {
  TileInfo t;
  const int per_batch = tiles_m * tiles_n;
  const int z = tile / per_batch;
  const int r = tile - z * per_batch;
  t.z1 = z / nb2;
  t.z2 = z - t.z1 * nb2;
  t.m0 = (r % tiles_m) * BM;
  t.n0 = (r / tiles_m) * BN;
  const int kb_all = (K + BKT - 1) / BKT;
  t.kb0 = 0;
  t.nkb = kb_all;
  t.skip = false;
  if (causal == kCausalSkipUpper) {
    t.skip = t.n0 >= t.m0 + BM;
  } else if (causal == kCausalKLower) {
    const int kend = min(K, t.m0 + BM);
    t.nkb = (kend + BKT - 1) / BKT;
  } else if (causal == kCausalKUpper) {
    t.kb0 = t.m0 / BKT;
    t.nkb = max(0, kb_all - t.kb0);
  } else if (causal == kSplitK) {
    // z1 indexes the K slice; the operands themselves are not batched (TMA z = 0)
    const int per = (kb_all + nb1 - 1) / nb1;
    t.kb0 = t.z1 * per;
    t.nkb = max(0, min(per, kb_all - t.kb0));
  }
  (void)M;
  (void)N;
  return t;
}

// L2 prefetch of the global operands a tile's epilogue reads (the residual R, GELU's
// pre-activation Hin, C when beta != 0): each epilogue warp issues one bulk prefetch per lane
// for its 32 rows as soon as it is waiting for the tile's accumulator, so the loads hit L2
// instead of HBM once the main loop is done.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
               : "memory");
}
template <int BN, int MODE>
__device__ __forceinline__ void prefetch_epilogue_rows(const GemmEpilogue& epi, const GemmBatch& bat,
                                                       const TileInfo& ti, int row, int M, int N) {
  if (row >= M) return;
  const int cols = min(BN, N - ti.n0);
  const uint32_t bytes = static_cast<uint32_t>(cols * 4) & ~15u;
  if (cols <= 0 || bytes == 0) return;
  if (MODE == kEpiGeluBwd && epi.Hin) bulk_prefetch_l2(epi.Hin + static_cast<long>(row) * epi.ldhi + ti.n0, bytes);
  if (MODE == kEpiStore && epi.R) bulk_prefetch_l2(epi.R + static_cast<long>(row) * epi.ldr + ti.n0, bytes);
  if (MODE == kEpiStore && epi.beta != 0.f) {
    const float* c = epi.C + ti.z1 * bat.c_s1 + ti.z2 * bat.c_s2;
    bulk_prefetch_l2(c + static_cast<long>(row) * epi.ldc + ti.n0, bytes);
  }
}

__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void tmem_ld_x32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Epilogue of one accumulator tile, run by epilogue warp q (TMEM lane quarter q), specialised
// per mode at compile time (no per-element mode branches): TMEM -> registers (thread = row,
// the next 32-column chunk's tcgen05.ld in flight while this one is processed) -> smem
// transpose -> each lane takes 4 consecutive columns of a row (8 lanes per 32-column row, 4
// rows per instruction), so bias / residual / GELU operands and the stores move as coalesced
// 128-bit accesses.
struct EpiCtx {
  uint32_t lane, st_base;
  float* stile;
  int row0, nrows, sub_r, sub_c;
  float* Cb;
  const float* src;
  long lds;
  bool use_beta;
  bool c16;  // C is bf16 (GemmEpilogue::c16)
  const float* bias;
};

__device__ __forceinline__ void st_bf16x4(bf16* p, float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = u;
}

// One 32-column chunk (v: this thread's row, 32 accumulator columns).
template <int MODE>
__device__ __forceinline__ void epilogue_chunk(const EpiCtx& x0, const uint32_t (&v)[32], int col0,
                                               const GemmEpilogue& epi, int N) {
  const uint32_t lane = x0.lane;
  if (x0.nrows <= 0 || col0 >= N) return;  // warp-uniform
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    sts128(x0.st_base + (lane * 36 + 4 * k) * 4,
           make_float4(__uint_as_float(v[4 * k]), __uint_as_float(v[4 * k + 1]), __uint_as_float(v[4 * k + 2]),
                       __uint_as_float(v[4 * k + 3])));
  }
  __syncwarp();
  const float alpha = epi.alpha;
  const int col = col0 + x0.sub_c;
  if (col0 + 32 <= N) {
    const bool full_rows = x0.nrows == 32;
    float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (x0.bias) bv = *reinterpret_cast<const float4*>(x0.bias + col);
    const float* be = &bv.x;
    // rows in groups; every global operand of a group is in flight before its first use and
    // loaded before any of the group's stores (which may alias later loads as far as the
    // compiler knows, and would serialise them). GELU' reads the pre-activation for every
    // element, so its 8 rows go out at once; the other modes keep groups of 4 (registers).
    constexpr int kG = MODE == kEpiGeluBwd ? 8 : 4;
#pragma unroll
    for (int g = 0; g < 8 / kG; ++g) {
      float4 xv[kG], av[kG], pv[kG];
#pragma unroll
      for (int i = 0; i < kG; ++i) {
        const int r = (g * kG + i) * 4 + x0.sub_r;
        const bool ok = full_rows || r < x0.nrows;
        const long grow = x0.row0 + r;
        av[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        pv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (x0.src && ok) av[i] = *reinterpret_cast<const float4*>(x0.src + grow * x0.lds + col);
        if (MODE == kEpiStore && x0.use_beta && ok) pv[i] = *reinterpret_cast<const float4*>(x0.Cb + grow * epi.ldc + col);
      }
#pragma unroll
      for (int i = 0; i < kG; ++i) xv[i] = lds128(x0.st_base + (((g * kG + i) * 4 + x0.sub_r) * 36 + x0.sub_c) * 4);
#pragma unroll
      for (int i = 0; i < kG; ++i) {
        const int r = (g * kG + i) * 4 + x0.sub_r;
        if (!full_rows && r >= x0.nrows) continue;
        const long grow = x0.row0 + r;
        float* xe = &xv[i].x;
        const float* ae = &av[i].x;
        if constexpr (MODE == kEpiGeluBwd) {
#pragma unroll
          for (int e = 0; e < 4; ++e) xe[e] = xe[e] * alpha * ae[e];
        } else if constexpr (MODE == kEpiGelu) {
#pragma unroll
          for (int e = 0; e < 4; ++e) xe[e] = gelu_tanh(xe[e] * alpha + be[e]);
        } else if constexpr (MODE == kEpiGeluSave) {
          float4 gd;
          float* ge = &gd.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float h = xe[e] * alpha + be[e];
            const float sg = gelu_sig(h);
            xe[e] = h * sg;
            ge[e] = gelu_grad_s(h, sg);
          }
          *reinterpret_cast<float4*>(epi.Hout + grow * epi.ldho + col) = gd;
        } else {
          const float* pe = &pv[i].x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float y = xe[e] * alpha + be[e];
            if (x0.src) y += ae[e];
            if (x0.use_beta) y += epi.beta * pe[e];
            xe[e] = y;
          }
        }
        if (x0.c16) st_bf16x4(reinterpret_cast<bf16*>(epi.C) + grow * epi.ldc + col, xv[i]);
        else *reinterpret_cast<float4*>(x0.Cb + grow * epi.ldc + col) = xv[i];
      }
    }
  } else {
    // ragged last chunk (N not a multiple of 32): scalar path, lanes over columns
    const int colx = col0 + static_cast<int>(lane);
    if (colx < N) {
      const float bias_v = x0.bias ? x0.bias[colx] : 0.f;
      for (int r = 0; r < x0.nrows; ++r) {
        const long grow = x0.row0 + r;
        float y = x0.stile[r * 36 + lane] * alpha;
        if constexpr (MODE == kEpiGeluBwd) {
          y *= epi.Hin[grow * epi.ldhi + colx];
        } else if constexpr (MODE == kEpiGelu || MODE == kEpiGeluSave) {
          y += bias_v;
          const float sg = gelu_sig(y);
          if (MODE == kEpiGeluSave) epi.Hout[grow * epi.ldho + colx] = gelu_grad_s(y, sg);
          y *= sg;
        } else {
          y += bias_v;
          if (epi.R) y += epi.R[grow * epi.ldr + colx];
          if (epi.beta != 0.f) y += epi.beta * x0.Cb[grow * epi.ldc + colx];
        }
        if (x0.c16) reinterpret_cast<bf16*>(epi.C)[grow * epi.ldc + colx] = __float2bfloat16_rn(y);
        else x0.Cb[grow * epi.ldc + colx] = y;
      }
    }
  }
  __syncwarp();
}

// TMA-store epilogue of one 32-column chunk (CTA-pair kernel; modes with no per-element global
// operand: store with optional bias and beta = 0, GELU, GELU + gelu'): thread = row finishes its
// 32 values in registers (the bias chunk is one broadcast load per 4 columns), writes them to the
// warp's staging tile in the store map's swizzled layout (128B swizzle for 32 fp32, 64B for 32
// bf16: conflict-free 16-byte stores) and one lane issues the bulk tensor store — no shared-memory
// transpose back, no per-lane address math, ragged edges clipped by the TMA unit.
struct TmaEpi {
  const CUtensorMap* map_c;
  uint8_t* stage;     // this warp's staging tile (1024-aligned, 4 KB)
  const float* sbias;  // this warp's bias columns in shared memory (nullptr: no bias), from col_base
  int col_base;
  int slice;          // split-K slice (the map's third coordinate)
};
template <int MODE>
__device__ __forceinline__ void epilogue_chunk_tma(const TmaEpi& t, const uint32_t (&v)[32], int col0, int row0,
                                                   const GemmEpilogue& epi, int N) {
  if (col0 >= N) return;  // warp-uniform
  const uint32_t lane = lane_id();
  const float alpha = epi.alpha;
  float y[32];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t.sbias) b = lds128(smem_u32(t.sbias + (col0 - t.col_base) + 4 * k));  // broadcast
    y[4 * k] = __uint_as_float(v[4 * k]) * alpha + b.x;
    y[4 * k + 1] = __uint_as_float(v[4 * k + 1]) * alpha + b.y;
    y[4 * k + 2] = __uint_as_float(v[4 * k + 2]) * alpha + b.z;
    y[4 * k + 3] = __uint_as_float(v[4 * k + 3]) * alpha + b.w;
  }
  if constexpr (MODE == kEpiGelu) {
#pragma unroll
    for (int i = 0; i < 32; ++i) y[i] = gelu_tanh(y[i]);
  }
  if (lane == 0) bulk_wait_read0();  // the previous chunk's store has read the staging tile
  __syncwarp();
  if (epi.c16) {  // 32 bf16 = 64 B per row, 64B swizzle
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h2[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(y[8 * j + 2 * e], y[8 * j + 2 * e + 1]);
      const uint4 u = *reinterpret_cast<const uint4*>(h2);
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                       smem_u32(t.stage + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4))),
                   "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
                   : "memory");
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sts128(smem_u32(t.stage + lane * 128 + ((j ^ (lane & 7)) << 4)),
             make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(t.map_c, t.stage, col0, row0, t.slice);
    bulk_commit();
  }
}

// Epilogue of one accumulator tile, run by epilogue warp q (TMEM lane quarter q), specialised
// per mode at compile time (no per-element mode branches): TMEM -> registers (thread = row,
// the next 32-column chunk's tcgen05.ld in flight while this one is processed) -> smem
// transpose -> each lane takes 4 consecutive columns of a row (8 lanes per 32-column row, 4
// rows per instruction), so bias / residual / GELU operands and the stores move as coalesced
// 128-bit accesses. With `tma` (CTA-pair kernel, bat.c_tma): epilogue_chunk_tma instead.
template <int BN, int MODE>
__device__ __forceinline__ void epilogue_tile_m(const TileInfo& ti, int acc, uint32_t q, uint32_t tmem_base,
                                                float* epi_smem, const GemmEpilogue& epi, const GemmBatch& bat,
                                                int M, int N, int c_begin = 0, int c_end = BN / 32, int slot = -1,
                                                const TmaEpi* tma = nullptr) {
  EpiCtx x;
  x.lane = lane_id();
  x.stile = epi_smem + (slot < 0 ? static_cast<int>(q) : slot) * (32 * 36);
  x.st_base = smem_u32(x.stile);
  x.row0 = ti.m0 + static_cast<int>(q * 32);
  x.nrows = min(32, M - x.row0);
  x.Cb = epi.C + ti.z1 * bat.c_s1 + ti.z2 * bat.c_s2;
  x.sub_r = static_cast<int>(x.lane >> 3);
  x.sub_c = static_cast<int>(x.lane & 7) * 4;
  x.src = MODE == kEpiGeluBwd ? epi.Hin : (MODE == kEpiStore ? epi.R : nullptr);
  x.lds = MODE == kEpiGeluBwd ? epi.ldhi : epi.ldr;
  x.use_beta = MODE == kEpiStore && epi.beta != 0.f;
  x.c16 = epi.c16 != 0;
  x.bias = MODE == kEpiGeluBwd ? nullptr : epi.bias;
  const uint32_t tbase = tmem_base + ((q * 32) << 16) + acc * BN;
  uint32_t b0[32], b1[32];
  if (ti.nkb > 0) {
    tmem_ld_x32_issue(tbase + c_begin * 32, b0);
#pragma unroll 1
    for (int c = c_begin; c < c_end; c += 2) {
      tmem_ld_wait();
      const bool two = c + 1 < c_end;
      if (two) tmem_ld_x32_issue(tbase + (c + 1) * 32, b1);
      if constexpr (MODE == kEpiStore || MODE == kEpiGelu) {
        if (tma) epilogue_chunk_tma<MODE>(*tma, b0, ti.n0 + c * 32, x.row0, epi, N);
        else epilogue_chunk<MODE>(x, b0, ti.n0 + c * 32, epi, N);
      } else {
        epilogue_chunk<MODE>(x, b0, ti.n0 + c * 32, epi, N);
      }
      if (!two) break;
      tmem_ld_wait();
      if (c + 2 < c_end) tmem_ld_x32_issue(tbase + (c + 2) * 32, b0);
      if constexpr (MODE == kEpiStore || MODE == kEpiGelu) {
        if (tma) epilogue_chunk_tma<MODE>(*tma, b1, ti.n0 + (c + 1) * 32, x.row0, epi, N);
        else epilogue_chunk<MODE>(x, b1, ti.n0 + (c + 1) * 32, epi, N);
      } else {
        epilogue_chunk<MODE>(x, b1, ti.n0 + (c + 1) * 32, epi, N);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) b0[i] = 0u;
#pragma unroll 1
    for (int c = c_begin; c < c_end; ++c) {
      if constexpr (MODE == kEpiStore || MODE == kEpiGelu) {
        if (tma) {
          epilogue_chunk_tma<MODE>(*tma, b0, ti.n0 + c * 32, x.row0, epi, N);
          continue;
        }
      }
      epilogue_chunk<MODE>(x, b0, ti.n0 + c * 32, epi, N);
    }
  }
}

template <typename T, int BN, bool A_MN, bool B_MN, bool P3, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tf32_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, int M,
                 int N, int K, GemmEpilogue epi, GemmBatch bat) {
  using L = Smem<BN, P3>;
  using E = Elem<T>;
  static_assert(!(P3 && E::kBf16), "3xTF32 is an fp32-operand mode");
  constexpr int kStages = L::kStagesN;
  constexpr int BKT = E::BK, CW = E::CW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_smem = reinterpret_cast<float*>(smem + L::kRing);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kRing + L::kEpi);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* conv = tempty + 2;  // P3: hi/lo split of the stage done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv + kStages);

  const uint32_t warp = warp_id();
  const int tiles_m = (M + BM - 1) / BM;
  const int tiles_n = (N + BN - 1) / BN;
  const int n_tiles = tiles_m * tiles_n * bat.nb1 * bat.nb2;

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 64);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait_and_trigger();

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        TileInfo ti = tile_info<BN, BKT>(tile, tiles_m, tiles_n, M, N, K, bat.nb2, bat.causal, bat.nb1);
        if (ti.skip) continue;
        if (bat.causal == kSplitK) ti.z1 = ti.z2 = 0;  // K slices read the same operands
        for (int kb = ti.kb0; kb < ti.kb0 + ti.nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          mbar_expect_tx(&full[stage], L::kOpBytes);
          const int k0 = kb * BKT;
          if constexpr (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / CW; ++j) {
              if (bat.a_perm) tma_load_4d(sa + j * (BKT * 128), &map_a, &full[stage], ti.m0 + CW * j, ti.z2, k0, ti.z1);
              else tma_load_4d(sa + j * (BKT * 128), &map_a, &full[stage], ti.m0 + CW * j, k0, ti.z2, ti.z1);
            }
          } else {
            if (bat.a_perm) tma_load_4d(sa, &map_a, &full[stage], k0, ti.z2, ti.m0, ti.z1);
            else tma_load_4d(sa, &map_a, &full[stage], k0, ti.m0, ti.z2, ti.z1);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / CW; ++j) {
              if (bat.b_perm) tma_load_4d(sb + j * (BKT * 128), &map_b, &full[stage], ti.n0 + CW * j, ti.z2, k0, ti.z1);
              else tma_load_4d(sb + j * (BKT * 128), &map_b, &full[stage], ti.n0 + CW * j, k0, ti.z2, ti.z1);
            }
          } else {
            if (bat.b_perm) tma_load_4d(sb, &map_b, &full[stage], k0, ti.z2, ti.n0, ti.z1);
            else tma_load_4d(sb, &map_b, &full[stage], k0, ti.n0, ti.z2, ti.z1);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_of<T>(BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const TileInfo ti = tile_info<BN, BKT>(tile, tiles_m, tiles_n, M, N, K, bat.nb2, bat.causal, bat.nb1);
      if (ti.skip) continue;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ++local;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      if (ti.nkb == 0) {
        if (elect_one()) mbar_arrive(&tfull[acc]);
        __syncwarp();
        continue;
      }
      for (int kb = 0; kb < ti.nkb; ++kb) {
        if constexpr (P3) {
          mbar_wait(&conv[stage], phase);
        } else {
          mbar_wait(&full[stage], phase);
        }
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + stage * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
#pragma unroll
          for (int kk = 0; kk < E::kMmas; ++kk) {
            if constexpr (P3) {
              const uint32_t la = sa + L::kOpBytes, lb = sb + L::kOpBytes;
              const uint64_t dah = A_MN ? smem_desc_sw128_b32(sa + kk * 1024, BK * 128, 512)
                                        : smem_desc_sw128(sa + kk * 32, 16, 1024);
              const uint64_t dbh = B_MN ? smem_desc_sw128_b32(sb + kk * 1024, BK * 128, 512)
                                        : smem_desc_sw128(sb + kk * 32, 16, 1024);
              const uint64_t dal = A_MN ? smem_desc_sw128_b32(la + kk * 1024, BK * 128, 512)
                                        : smem_desc_sw128(la + kk * 32, 16, 1024);
              const uint64_t dbl = B_MN ? smem_desc_sw128_b32(lb + kk * 1024, BK * 128, 512)
                                        : smem_desc_sw128(lb + kk * 32, 16, 1024);
              mma_tf32(d_tmem, dal, dbh, idesc, (kb | kk) != 0 ? 1u : 0u);
              mma_tf32(d_tmem, dah, dbl, idesc, 1u);
              mma_tf32(d_tmem, dah, dbh, idesc, 1u);
              continue;
            }
            mma_one<T>(d_tmem, op_desc<T, A_MN>(sa, kk), op_desc<T, B_MN>(sb, kk), idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          mma_commit(&empty[stage]);
          if (kb == ti.nkb - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (P3 && (warp == 2 || warp == 3)) {
    // Split each landed stage into tf32 hi (in place) + lo (second half of the stage).
    const int tid = static_cast<int>(threadIdx.x) - 64;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const TileInfo ti = tile_info<BN, BKT>(tile, tiles_m, tiles_n, M, N, K, bat.nb2, bat.causal, bat.nb1);
      if (ti.skip) continue;
      for (int kb = 0; kb < ti.nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        float4* hi = reinterpret_cast<float4*>(smem + stage * L::kStageBytes);
        float4* lo = reinterpret_cast<float4*>(smem + stage * L::kStageBytes + L::kOpBytes);
        for (int i = tid; i < L::kOpBytes / 16; i += 64) {
          float4 x = hi[i];
          float4 h, l;
          h.x = __uint_as_float(tf32_rna(x.x));
          h.y = __uint_as_float(tf32_rna(x.y));
          h.z = __uint_as_float(tf32_rna(x.z));
          h.w = __uint_as_float(tf32_rna(x.w));
          l.x = x.x - h.x;
          l.y = x.y - h.y;
          l.z = x.z - h.z;
          l.w = x.w - h.w;
          hi[i] = h;
          lo[i] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&conv[stage]);
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp - 4;  // TMEM lane quarter this warp may access
    int local = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const TileInfo ti = tile_info<BN, BKT>(tile, tiles_m, tiles_n, M, N, K, bat.nb2, bat.causal, bat.nb1);
      if (ti.skip) continue;
      const int acc = local & 1;
      prefetch_epilogue_rows<BN, MODE>(epi, bat, ti, ti.m0 + static_cast<int>(q * 32 + lane_id()), M, N);
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      ++local;
      tc_fence_after();
      epilogue_tile_m<BN, MODE>(ti, acc, q, tmem_base, epi_smem, epi, bat, M, N);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ---- CTA-pair variant (cta_group::2) ------------------------------------------------
// A cluster of two CTAs on one TPC computes a 256 x BN tile: each CTA stages its own 128
// rows of A and half (BN/2 rows) of B, the even CTA issues tcgen05.mma.cta_group::2 with
// M = 256 over both CTAs' shared memory, and each CTA's TMEM receives its 128 rows of the
// accumulator. Per SM, a 128 x BN x 32 stage now moves 16 KB of A + BN/2 x 128 B of B from
// L2 (vs BN x 128 B of B alone before): the shared-memory / L2 operand traffic per MMA
// flop drops by a third at BN = 256, the bound that held the 1-CTA kernel near 0.6 of the
// library GEMM on the workload's short-K shapes.
// 12 warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4-11 epilogue — two warps
// per TMEM lane quarter, each taking half of the tile's 32-column chunks. The short-K block GEMMs
// (K = 768 at d768: ~2.5 us of bf16 MMA per 256-row tile) were bound by a 4-warp epilogue.
constexpr int kPairEpiWarps = 8;
constexpr int kPairThreads = 128 + 32 * kPairEpiWarps;
template <int BN>
struct SmemPair {
  static constexpr int kABytes = BM * BK * 4;
  static constexpr int kBBytes = (BN / 2) * BK * 4;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // per epilogue warp (1024-aligned): the 32 x 36 transpose tile, or the TMA staging tile (4 KB
  // at +0) and the warp's bias columns (<= 128 floats at +4096)
  static constexpr int kEpiWarp = 5120;
  static constexpr int kEpi = kPairEpiWarps * kEpiWarp;
  static constexpr int kBudget = 232448 - kEpi - 1024 - 256;  // 227 KB of dynamic smem per CTA
  static constexpr int kStagesN = kBudget / kStageBytes > 8 ? 8 : kBudget / kStageBytes;
  static constexpr int kRing = kStagesN * kStageBytes;
  static constexpr int kTotal = kRing + kEpi + 1024 + 256;
};

template <typename T, int BN, bool A_MN, bool B_MN, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
gemm_tf32_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      const __grid_constant__ CUtensorMap map_c, int M,
                      int N, int K, GemmEpilogue epi, GemmBatch bat) {
  using L = SmemPair<BN>;
  using E = Elem<T>;
  constexpr int kStages = L::kStagesN;
  constexpr int BKT = E::BK, CW = E::CW;
  static_assert(!B_MN || (BN / 2) % CW == 0, "MN-major B half-tile in whole 128-byte chunks");
  constexpr int BM2 = 2 * BM;
  constexpr int kHalfChunks = (BN / 32 + 1) / 2;  // epilogue warp 4+q: chunks [0, kHalf); warp 8+q: the rest
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kRing + L::kEpi);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int tiles_m = (M + BM2 - 1) / BM2;
  const int tiles_n = (N + BN - 1) / BN;
  const int n_tiles = tiles_m * tiles_n * bat.nb1 * bat.nb2;
  const int pair = static_cast<int>(cluster_id_x());
  const int n_pairs = static_cast<int>(nclusters_x());

  if (warp == 0 && elect_one()) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    if (bat.c_tma) tma_prefetch_desc(&map_c);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kPairEpiWarps);  // epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  constexpr uint32_t kTmemCols = 2 * BN <= 256 ? 256 : 512;
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait_and_trigger();

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = pair; tile < n_tiles; tile += n_pairs) {
        TileInfo ti = tile_info<BN, BKT>(tile, tiles_m, tiles_n, M, N, K, bat.nb2, bat.causal, bat.nb1);
        // tile_info counts 128-row tiles; rescale to this CTA's half of the 256-row pair tile
        ti.m0 = ti.m0 * 2 + static_cast<int>(rank) * BM;
        if (bat.causal == kSplitK) ti.z1 = ti.z2 = 0;
        const int nb0 = ti.n0 + static_cast<int>(rank) * (BN / 2);
        for (int kb = ti.kb0; kb < ti.kb0 + ti.nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          if (leader) mbar_expect_tx(&full[stage], 2 * L::kStageBytes);
          const int k0 = kb * BKT;
          if constexpr (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / CW; ++j) {
              if (bat.a_perm) tma_load_4d_pair(sa + j * (BKT * 128), &map_a, &full[stage], ti.m0 + CW * j, ti.z2, k0, ti.z1);
              else tma_load_4d_pair(sa + j * (BKT * 128), &map_a, &full[stage], ti.m0 + CW * j, k0, ti.z2, ti.z1);
            }
          } else {
            if (bat.a_perm) tma_load_4d_pair(sa, &map_a, &full[stage], k0, ti.z2, ti.m0, ti.z1);
            else tma_load_4d_pair(sa, &map_a, &full[stage], k0, ti.m0, ti.z2, ti.z1);
          }
          if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < (BN / 2) / CW; ++j) {
              if (bat.b_perm) tma_load_4d_pair(sb + j * (BKT * 128), &map_b, &full[stage], nb0 + CW * j, ti.z2, k0, ti.z1);
              else tma_load_4d_pair(sb + j * (BKT * 128), &map_b, &full[stage], nb0 + CW * j, k0, ti.z2, ti.z1);
            }
          } else {
            if (bat.b_perm) tma_load_4d_pair(sb, &map_b, &full[stage], k0, ti.z2, nb0, ti.z1);
            else tma_load_4d_pair(sb, &map_b, &full[stage], k0, nb0, ti.z2, ti.z1);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = idesc_of<T>(BM2, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = pair; tile < n_tiles; tile += n_pairs) {
        const TileInfo ti = tile_info<BN, BKT>(tile, tiles_m, tiles_n, M, N, K, bat.nb2, bat.causal, bat.nb1);
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        ++local;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        if (ti.nkb == 0) {
          if (elect_one()) {
            mbar_arrive_cluster(&tfull[acc], 0);
            mbar_arrive_cluster(&tfull[acc], 1);
          }
          __syncwarp();
          continue;
        }
        for (int kb = 0; kb < ti.nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(smem + stage * L::kStageBytes);
            const uint32_t sb = sa + L::kABytes;
#pragma unroll
            for (int kk = 0; kk < E::kMmas; ++kk) {
              mma_two<T>(d_tmem, op_desc<T, A_MN>(sa, kk), op_desc<T, B_MN>(sb, kk), idesc, (kb | kk) != 0 ? 1u : 0u);
            }
            mma_commit_pair(&empty[stage], 0x3);
            if (kb == ti.nkb - 1) mma_commit_pair(&tfull[acc], 0x3);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (static_cast<int>(warp) - 4) >> 2;
    const int c0 = half ? kHalfChunks : 0, c1 = half ? BN / 32 : kHalfChunks;
    uint8_t* wsm = smem + L::kRing + (static_cast<int>(warp) - 4) * L::kEpiWarp;
    TmaEpi te{&map_c, wsm, nullptr, 0, 0};
    float* sbias = reinterpret_cast<float*>(wsm + 4096);
    int local = 0;
    for (int tile = pair; tile < n_tiles; tile += n_pairs) {
      TileInfo ti = tile_info<BN, BKT>(tile, tiles_m, tiles_n, M, N, K, bat.nb2, bat.causal, bat.nb1);
      ti.m0 = ti.m0 * 2 + static_cast<int>(rank) * BM;
      const int acc = local & 1;
      if (half == 0) prefetch_epilogue_rows<BN, MODE>(epi, bat, ti, ti.m0 + static_cast<int>(q * 32 + lane_id()), M, N);
      te.slice = bat.causal == kSplitK ? ti.z1 : 0;
      if (bat.c_tma && epi.bias) {  // this warp's bias columns -> shared memory (read as broadcasts),
        te.col_base = ti.n0 + c0 * 32;  // loaded while the accumulator is still being computed
        __syncwarp();  // the previous tile's chunks have read the old values
        for (int i = static_cast<int>(lane_id()); i < (c1 - c0) * 32; i += 32) {
          const int col = te.col_base + i;
          sbias[i] = col < N ? epi.bias[col] : 0.f;
        }
        __syncwarp();
        te.sbias = sbias;
      }
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      ++local;
      tc_fence_after();
      epilogue_tile_m<BN, MODE>(ti, acc, q, tmem_base, reinterpret_cast<float*>(wsm), epi, bat, M, N, c0, c1, 0,
                                bat.c_tma ? &te : nullptr);
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) {
        if (leader) mbar_arrive(&tempty[acc]);
        else mbar_arrive_cluster(&tempty[acc], 0);
      }
    }
    if (bat.c_tma && lane_id() == 0) bulk_wait0();  // this warp's stores complete before exit
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<kTmemCols>(tmem_base);
  }
}

// ---- host side -------------------------------------------------------------------

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

// 4-D tensor map (fp32 or bf16 elements) over {inner, outer, b2, b1}: row stride ld, batch
// strides s2, s1 (elements). Dimensions are ordered by increasing stride: {inner, outer, b2, b1},
// or {inner, b2, outer, b1} when b2's stride is below the row stride (*perm = 1).
template <typename T>
bool make_map(CUtensorMap* map, const T* ptr, long inner, long outer, long ld, int box_inner, int box_outer,
              bool mn_major, long nb2 = 1, long s2 = 0, long nb1 = 1, long s1 = 0, int* perm = nullptr) {
  auto fn = encode_fn();
  if (!fn) return false;
  constexpr long es = sizeof(T);
  const long st2 = s2 > 0 ? s2 : ld * outer;
  const long st1 = s1 > 0 ? s1 : st2 * nb2;
  const bool swap = nb2 > 1 && st2 < ld;
  if (perm) *perm = swap ? 1 : 0;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(swap ? nb2 : outer),
                        static_cast<cuuint64_t>(swap ? outer : nb2), static_cast<cuuint64_t>(nb1)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(swap ? st2 : ld) * es, static_cast<cuuint64_t>(swap ? ld : st2) * es,
                           static_cast<cuuint64_t>(st1) * es};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(box_inner), swap ? 1u : static_cast<cuuint32_t>(box_outer),
                       swap ? static_cast<cuuint32_t>(box_outer) : 1u, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const bool b16 = Elem<T>::kBf16;
  CUresult r = fn(map, b16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                  const_cast<T*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  (mn_major && !b16) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int sm_count() {
  // every GPU of a node is the same part; initialised once, thread-safe (magic static)
  static const int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Operand maps: K-major boxes are {BK, rows} (one 128-byte row of K per tile row), MN-major
// boxes {CW, BK} (one 128-byte MN chunk per k-row).
template <typename T>
bool make_operand_maps(CUtensorMap* ma, CUtensorMap* mb, GemmBatch& b, int M, int N, int K, const T* A, long lda,
                       bool a_mn, const T* B, long ldb, bool b_mn, int b_rows) {
  constexpr int BKT = Elem<T>::BK, CW = Elem<T>::CW;
  const long mb1 = b.causal == kSplitK ? 1 : b.nb1;  // K slices share the (unbatched) operands
  const bool ok_a = a_mn ? make_map(ma, A, M, K, lda, CW, BKT, true, b.nb2, b.a_s2, mb1, b.a_s1, &b.a_perm)
                         : make_map(ma, A, K, M, lda, BKT, BM, false, b.nb2, b.a_s2, mb1, b.a_s1, &b.a_perm);
  const bool ok_b = b_mn ? make_map(mb, B, N, K, ldb, CW, BKT, true, b.nb2, b.b_s2, mb1, b.b_s1, &b.b_perm)
                         : make_map(mb, B, K, N, ldb, BKT, b_rows, false, b.nb2, b.b_s2, mb1, b.b_s1, &b.b_perm);
  return ok_a && ok_b;
}

template <typename T, int BN, bool A_MN, bool B_MN, bool P3, int MODE>
cudaError_t launch(cudaStream_t stream, int M, int N, int K, const T* A, long lda, const T* B, long ldb,
                   const GemmEpilogue& epi, const GemmBatch& bat) {
  CUtensorMap ma, mb;
  GemmBatch b = bat;
  if (!make_operand_maps(&ma, &mb, b, M, N, K, A, lda, A_MN, B, ldb, B_MN, BN)) return cudaErrorInvalidValue;
  auto kern = gemm_tf32_kernel<T, BN, A_MN, B_MN, P3, MODE>;
  {
    const cudaError_t e = ensure_smem_limit(kern, Smem<BN, P3>::kTotal);
    if (e != cudaSuccess) return e;
  }
  const long tiles = static_cast<long>((M + BM - 1) / BM) * ((N + BN - 1) / BN) * bat.nb1 * bat.nb2;
  const int grid = static_cast<int>(tiles < sm_count() ? tiles : sm_count());
  count_launch();
  return launch_pdl(kern, dim3(grid), dim3(kThreads), Smem<BN, P3>::kTotal, stream, ma, mb, M, N, K, epi, b);
}

// Store map of C [slices][rows][ld] for the TMA epilogue: box 32 columns x 32 rows x 1 slice,
// 128B swizzle for fp32 (128-byte box rows), 64B for bf16; split-K partials are the slices (each
// clips at its own last row).
bool make_store_map(CUtensorMap* map, void* ptr, long cols, long rows, long ld, long slices, bool c16) {
  auto fn = encode_fn();
  if (!fn) return false;
  const long es = c16 ? 2 : 4;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(slices)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * es), static_cast<cuuint64_t>(ld * rows * es)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, c16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, c16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_store_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HY_GEMM_TMA_STORE");  // experiments: 0 = per-lane global stores
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename T, int BN, bool A_MN, bool B_MN, int MODE>
cudaError_t launch_pair(cudaStream_t stream, int M, int N, int K, const T* A, long lda, const T* B, long ldb,
                        const GemmEpilogue& epi, const GemmBatch& bat) {
  CUtensorMap ma, mb, mc;
  GemmBatch b = bat;
  if (!make_operand_maps(&ma, &mb, b, M, N, K, A, lda, A_MN, B, ldb, B_MN, BN / 2)) return cudaErrorInvalidValue;
  // TMA-store epilogue: store (bias allowed; no residual, beta = 0) and GELU without the gelu'
  // store, unbatched (split-K partials are the map's slices), 16-byte aligned rows. The residual,
  // beta != 0, GELU' and the gelu' store keep the transposed path (a thread-per-row residual read
  // measured slower: C2 o_proj bf16 18.7 -> 24.4 us, profiles/r02_epilogue/residual_tma.json).
  const long es = epi.c16 ? 2 : 4;
  const bool split = b.causal == kSplitK;
  bool tma = tma_store_enabled() && (MODE == kEpiStore || MODE == kEpiGelu) && !epi.R && epi.beta == 0.f &&
             b.nb2 == 1 && (b.causal == kCausalNone || split) && (b.nb1 == 1 || split) && M >= 32 && N >= 32 &&
             (reinterpret_cast<uintptr_t>(epi.C) & 15) == 0 && (epi.ldc * es) % 16 == 0 &&
             (!split || b.c_s1 == static_cast<long>(M) * epi.ldc);
  if (tma) tma = make_store_map(&mc, epi.C, N, M, epi.ldc, split ? b.nb1 : 1, epi.c16 != 0);
  b.c_tma = tma ? 1 : 0;
  if (!tma) mc = ma;  // unused
  using L = SmemPair<BN>;
  auto kern = gemm_tf32_pair_kernel<T, BN, A_MN, B_MN, MODE>;
  {
    const cudaError_t e = ensure_smem_limit(kern, L::kTotal);
    if (e != cudaSuccess) return e;
  }
  const long tiles = static_cast<long>((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN) * bat.nb1 * bat.nb2;
  const long pairs = std::min<long>(tiles, sm_count() / 2);
  count_launch();
  return launch_pdl(kern, dim3(static_cast<unsigned>(2 * pairs)), dim3(kPairThreads), L::kTotal, stream, ma, mb, mc,
                    M, N, K, epi, b);
}

template <typename T, int BN, int MODE>
cudaError_t dispatch_pair(cudaStream_t st, int M, int N, int K, const T* A, long lda, bool a_mn, const T* B,
                          long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat) {
  if (!a_mn && !b_mn) return launch_pair<T, BN, false, false, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
  if (a_mn && !b_mn) return launch_pair<T, BN, true, false, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
  if constexpr (Elem<T>::kBf16 && (BN / 2) % Elem<T>::CW != 0) {
    return cudaErrorInvalidValue;  // pick_bn_pair never picks this (96-wide bf16 MN-major halves)
  } else {
    if (!a_mn && b_mn) return launch_pair<T, BN, false, true, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
    return launch_pair<T, BN, true, true, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
  }
}

// CTA-pair tile width (256 x BN pair tiles): the widest tile whose wave count is not worse.
// bf16 MN-major B needs whole 64-wide chunks per CTA half: BN 128 or 256.
int pick_bn_pair(int M, int N, long batches, bool no192 = false) {
  static const int forced = [] {
    const char* e = std::getenv("HY_GEMM_BN");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 128 || forced == 256 || (forced == 192 && !no192)) return forced;
  static const int kBN[3] = {128, 192, 256};
  static const double kCost[3] = {128 / 0.62, 192 / 0.70, 256 / 0.76};
  const long tm = (M + 2 * BM - 1) / (2 * BM);
  const long pairs = sm_count() / 2;
  int best = 128;
  double best_t = 1e300;
  for (int i = 0; i < 3; ++i) {
    if (kBN[i] > 128 && N <= 128) break;
    if (kBN[i] == 192 && no192) continue;
    const long tiles = tm * ((N + kBN[i] - 1) / kBN[i]) * batches;
    const double t = static_cast<double>((tiles + pairs - 1) / pairs) * kCost[i];
    if (t < best_t - 1e-9) {
      best_t = t;
      best = kBN[i];
    }
  }
  return best;
}

bool use_pairs() {
  static const bool on = [] {
    const char* e = std::getenv("HY_GEMM_PAIR");  // experiments: 0 = one-CTA tiles only
    return !e || std::atoi(e) != 0;
  }();
  return on;
}

template <typename T, int BN, int MODE>
cudaError_t dispatch_bn(cudaStream_t st, int M, int N, int K, const T* A, long lda, bool a_mn, const T* B,
                        long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat) {
  if (!a_mn && !b_mn) return launch<T, BN, false, false, false, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
  if (!a_mn && b_mn) return launch<T, BN, false, true, false, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
  if (a_mn && !b_mn) return launch<T, BN, true, false, false, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
  return launch<T, BN, true, true, false, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
}

// Output tile width: wider tiles cut the shared-memory traffic per MMA (the TF32 pipe is
// smem-bound at BN=128), but fewer tiles can leave SMs idle in the last wave. Pick the
// width minimising waves x relative per-tile cost.
int pick_bn(int M, int N, long batches) {
  static const int forced = [] {
    const char* e = std::getenv("HY_GEMM_BN");  // experiments only
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 128 || forced == 192 || forced == 256) return forced;
  static const int kBN[3] = {128, 192, 256};
  static const double kCost[3] = {128 / 0.50, 192 / 0.60, 256 / 0.66};  // relative time per tile
  const long tm = (M + BM - 1) / BM;
  int best = 128;
  double best_t = 1e300;
  for (int i = 0; i < 3; ++i) {
    if (kBN[i] > 128 && N <= 128) break;
    const long tiles = tm * ((N + kBN[i] - 1) / kBN[i]) * batches;
    const double t = static_cast<double>((tiles + sm_count() - 1) / sm_count()) * kCost[i];
    if (t < best_t - 1e-9) {
      best_t = t;
      best = kBN[i];
    }
  }
  return best;
}

template <typename T, int MODE>
cudaError_t dispatch_mode(cudaStream_t st, int M, int N, int K, const T* A, long lda, bool a_mn, const T* B,
                          long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3) {
  if (!prec3 && (bat.causal == kCausalNone || bat.causal == kSplitK) && M > BM && use_pairs()) {
    const int bn = pick_bn_pair(M, N, static_cast<long>(bat.nb1) * bat.nb2, Elem<T>::kBf16 && b_mn);
    if (bn == 256) return dispatch_pair<T, 256, MODE>(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
    if (bn == 192) return dispatch_pair<T, 192, MODE>(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
    return dispatch_pair<T, 128, MODE>(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
  }
  if (!prec3 && bat.causal == kCausalNone) {
    const int bn = pick_bn(M, N, static_cast<long>(bat.nb1) * bat.nb2);
    if (bn == 256) return dispatch_bn<T, 256, MODE>(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
    if (bn == 192) return dispatch_bn<T, 192, MODE>(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
  }
  if constexpr (!Elem<T>::kBf16) {
    if (prec3) {
      if (!a_mn && !b_mn) return launch<T, 128, false, false, true, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
      if (!a_mn && b_mn) return launch<T, 128, false, true, true, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
      if (a_mn && !b_mn) return launch<T, 128, true, false, true, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
      return launch<T, 128, true, true, true, MODE>(st, M, N, K, A, lda, B, ldb, e, bat);
    }
  }
  return dispatch_bn<T, 128, MODE>(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
}

}  // namespace
}  // namespace hy
