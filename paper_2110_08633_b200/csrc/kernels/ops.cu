// HBM-bound kernels: one warp per row for row reductions (128-bit loads, warp shuffles),
// grid-stride float4 loops for elementwise work, two-stage deterministic column sums.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <cfloat>

#include "launch_count.cuh"
#include "ops.cuh"
#include "pdl.cuh"

namespace hy {
namespace {

// a failed launch_pdl leaves its error in the thread's last-error state, which the wrappers
// return (cudaGetLastError) exactly as for <<<>>> launches
inline void check_launch(cudaError_t e) { (void)e; }


constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

int sms() {
  // every GPU of a node is the same part; initialised once, thread-safe (magic static)
  static const int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// ---- LayerNorm -----------------------------------------------------------------
// One warp per row; the row lives in registers (d <= 32 * 4 * kMaxVec).
constexpr int kMaxVecAll = 32;  // d <= 4096

// Row split over kSplit warps (<= kVec float4 per lane held in registers between the two
// reductions), the parts' sums meeting in shared memory in a fixed order: more warps per SM
// than a whole row per warp (8192 x 1600: 24.6 -> 22.5 us, L2-cold).
// 4 consecutive values as fp32 or as bf16 (the bf16 precision's GEMM operands).
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void st4(__nv_bfloat16* p, float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = u;
}
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

template <int kVec, int kSplit, typename Y = float>
__global__ void __launch_bounds__(256) ln_fwd_kernel(int rows, int d, const float* __restrict__ x,
                                                     const float* __restrict__ g, const float* __restrict__ b,
                                                     Y* __restrict__ y, float* __restrict__ mean_out,
                                                     float* __restrict__ rstd_out) {
  constexpr int kRows = kWarpsPerBlock / kSplit;
  __shared__ float red[2][kWarpsPerBlock];
  pdl_wait_and_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kRows + warp / kSplit;
  const int part = warp % kSplit, first = (warp / kSplit) * kSplit;
  const bool live = row < rows;
  const int nv = d >> 2;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long>(row) * d);
  float4 buf[kVec];
  float s = 0.f;
  if (live) {
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      const int i = part * 32 + lane + 32 * kSplit * k;
      if (i < nv) {
        buf[k] = xr[i];
        s += (buf[k].x + buf[k].y) + (buf[k].z + buf[k].w);
      }
    }
  }
  s = warp_sum(s);
  if (lane == 0) red[0][warp] = s;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int p = 0; p < kSplit; ++p) t += red[0][first + p];
  const float mu = t / d;
  float q = 0.f;
  if (live) {
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      const int i = part * 32 + lane + 32 * kSplit * k;
      if (i < nv) {
        const float a = buf[k].x - mu, bb = buf[k].y - mu, c = buf[k].z - mu, e = buf[k].w - mu;
        q += (a * a + bb * bb) + (c * c + e * e);
      }
    }
  }
  q = warp_sum(q);
  if (lane == 0) red[1][warp] = q;
  __syncthreads();
  if (!live) return;
  float u = 0.f;
#pragma unroll
  for (int p = 0; p < kSplit; ++p) u += red[1][first + p];
  const float rs = rsqrtf(u / d + 1e-5f);
  Y* yr = y + static_cast<long>(row) * d;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int i = part * 32 + lane + 32 * kSplit * k;
    if (i < nv) {
      const float4 gg = g4[i], bb = b4[i];
      st4(yr + 4 * i, make_float4((buf[k].x - mu) * rs * gg.x + bb.x, (buf[k].y - mu) * rs * gg.y + bb.y,
                                  (buf[k].z - mu) * rs * gg.z + bb.z, (buf[k].w - mu) * rs * gg.w + bb.w));
    }
  }
  if (part == 0 && lane == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
}

// LayerNorm backward as two HBM-streaming passes (d <= 4096):
//  ln_bwd_dx_kernel  — warp per row: the row sums in a first sweep, dx in a second sweep that
//                      re-reads x, dy from L1 (no per-row state kept in registers);
//  ln_bwd_dgb_kernel — column strips (32 lanes x float4) over row ranges: dγ = Σ dy·x̂,
//                      dβ = Σ dy, per-block partials folded by the strip's last block (atomic
//                      ticket, fixed block order: deterministic), added into dg, db.
// Each pass keeps many warps in flight per SM; the single-pass kernel below carried dγ/dβ
// for a whole row per lane and ran at ~1.4 TB/s at d = 1600.
// The row in registers, split over kDxSplit warps (each lane holds <= kVec float4 of x, dy and
// the dx being accumulated into: ~70 registers at kVec 4, three 8-warp blocks per SM), so every
// load of the row is in flight before its first use and the SM keeps 24 warps' worth of them;
// the parts' row sums meet in shared memory. At d = 1600 this took the dx pass from 8 warps
// per SM (a whole row per warp, 225 registers) to 24, and LayerNorm backward 91 -> 64 us.
template <int kVec, int kDxSplit>
__global__ void __launch_bounds__(256) ln_bwd_dx_kernel(int rows, int d, const float* __restrict__ x,
                                                        const float* __restrict__ g, const float* __restrict__ mean,
                                                        const float* __restrict__ rstd, const float* __restrict__ dy,
                                                        float* __restrict__ dx, int accumulate) {
  constexpr int kDxRows = kWarpsPerBlock / kDxSplit;  // rows per 256-thread block
  __shared__ float2 red[kWarpsPerBlock];
  pdl_wait_and_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * kDxRows + warp / kDxSplit;
  const int part = warp % kDxSplit;
  const int nv = d >> 2;
  const bool live = row < rows;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long>(row) * d);
  const float4* dyr = reinterpret_cast<const float4*>(dy + static_cast<long>(row) * d);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* dxr = reinterpret_cast<float4*>(dx + static_cast<long>(row) * d);
  float4 xv[kVec], gv[kVec], pv[kVec];
  float mu = 0.f, rs = 0.f, s1 = 0.f, s2 = 0.f;
  if (live) {
    mu = mean[row];
    rs = rstd[row];
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      const int i = part * 32 + lane + 32 * kDxSplit * k;
      if (i < nv) {
        xv[k] = xr[i];
        gv[k] = dyr[i];
        if (accumulate) pv[k] = dxr[i];
      }
    }
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      const int i = part * 32 + lane + 32 * kDxSplit * k;
      if (i < nv) {
        const float4 w = g4[i];
        gv[k] = make_float4(gv[k].x * w.x, gv[k].y * w.y, gv[k].z * w.z, gv[k].w * w.w);  // dy * g
        xv[k] = make_float4((xv[k].x - mu) * rs, (xv[k].y - mu) * rs, (xv[k].z - mu) * rs, (xv[k].w - mu) * rs);
        s1 += (gv[k].x + gv[k].y) + (gv[k].z + gv[k].w);
        s2 += (gv[k].x * xv[k].x + gv[k].y * xv[k].y) + (gv[k].z * xv[k].z + gv[k].w * xv[k].w);
      }
    }
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) red[warp] = make_float2(s1, s2);
  __syncthreads();
  if (!live) return;
  float t1 = 0.f, t2 = 0.f;
#pragma unroll
  for (int p = 0; p < kDxSplit; ++p) {  // fixed order: deterministic
    const float2 r = red[(warp / kDxSplit) * kDxSplit + p];
    t1 += r.x;
    t2 += r.y;
  }
  const float m1 = t1 / d, m2 = t2 / d;
#pragma unroll
  for (int k = 0; k < kVec; ++k) {
    const int i = part * 32 + lane + 32 * kDxSplit * k;
    if (i < nv) {
      float4 o = make_float4(rs * (gv[k].x - m1 - xv[k].x * m2), rs * (gv[k].y - m1 - xv[k].y * m2),
                             rs * (gv[k].z - m1 - xv[k].z * m2), rs * (gv[k].w - m1 - xv[k].w * m2));
      if (accumulate) {
        o.x += pv[k].x;
        o.y += pv[k].y;
        o.z += pv[k].z;
        o.w += pv[k].w;
      }
      dxr[i] = o;
    }
  }
}

__global__ void __launch_bounds__(256) ln_bwd_dgb_kernel(int rows, int d, const float* __restrict__ x,
                                                         const float* __restrict__ mean,
                                                         const float* __restrict__ rstd,
                                                         const float* __restrict__ dy, float* __restrict__ part,
                                                         float* __restrict__ dg, float* __restrict__ db,
                                                         int rows_per_block, unsigned* __restrict__ ticket) {
  pdl_wait_and_trigger();
  __shared__ float4 red[2][8][33];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = (blockIdx.x * 32 + lane) * 4;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float4 ag = make_float4(0.f, 0.f, 0.f, 0.f), ab = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < d) {
#pragma unroll 4
    for (int r = r0 + ty; r < r1; r += 8) {
      const float mu = mean[r], rs = rstd[r];
      const float4 xv = *reinterpret_cast<const float4*>(x + static_cast<long>(r) * d + c);
      const float4 dv = *reinterpret_cast<const float4*>(dy + static_cast<long>(r) * d + c);
      ag.x += dv.x * (xv.x - mu) * rs;
      ag.y += dv.y * (xv.y - mu) * rs;
      ag.z += dv.z * (xv.z - mu) * rs;
      ag.w += dv.w * (xv.w - mu) * rs;
      ab.x += dv.x;
      ab.y += dv.y;
      ab.z += dv.z;
      ab.w += dv.w;
    }
  }
  red[0][ty][lane] = ag;
  red[1][ty][lane] = ab;
  __syncthreads();
  float* pg = part;                                     // [nb][d] dγ partials
  float* pb = part + static_cast<long>(gridDim.y) * d;  // [nb][d] dβ partials
  if (ty < 2) {
    float4 t = red[ty][0][lane];
#pragma unroll
    for (int y = 1; y < 8; ++y) {
      const float4 u = red[ty][y][lane];
      t.x += u.x;
      t.y += u.y;
      t.z += u.z;
      t.w += u.w;
    }
    if (c < d) *reinterpret_cast<float4*>((ty ? pb : pg) + static_cast<long>(blockIdx.y) * d + c) = t;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ticket[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // fold: 4 row groups per output (dγ: ty 0-3, dβ: ty 4-7), fixed block order
  const int which = ty >> 2, grp = ty & 3;
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < d) {
    const float* src = which ? pb : pg;
    for (int b = grp; b < static_cast<int>(gridDim.y); b += 4) {
      const float4 u = __ldcg(reinterpret_cast<const float4*>(src + static_cast<long>(b) * d + c));
      t.x += u.x;
      t.y += u.y;
      t.z += u.z;
      t.w += u.w;
    }
  }
  red[which][grp][lane] = t;
  __syncthreads();
  if (ty < 2) {
    float4 f = red[ty][0][lane];
#pragma unroll
    for (int y = 1; y < 4; ++y) {
      const float4 u = red[ty][y][lane];
      f.x += u.x;
      f.y += u.y;
      f.z += u.z;
      f.w += u.w;
    }
    if (c < d) {
      float4* o = reinterpret_cast<float4*>((ty ? db : dg) + c);
      const float4 p = *o;
      *o = make_float4(p.x + f.x, p.y + f.y, p.z + f.z, p.w + f.w);
    }
  }
  if (threadIdx.x == 0) ticket[blockIdx.x] = 0;
}

// Register-accumulating form (d <= 2048): two sweeps over each row — the first only forms the
// row sums (and adds dy * xhat, dy into per-lane dγ / dβ accumulators held in registers for the
// whole block), the second re-reads x, dy from L1 to write dx — so neither the row nor the
// column partials need per-element shared-memory traffic.
template <int kMaxVec>
__global__ void __launch_bounds__(256) ln_bwd_rr_kernel(int rows, int d, const float* __restrict__ x,
                                                        const float* __restrict__ g, const float* __restrict__ mean,
                                                        const float* __restrict__ rstd, const float* __restrict__ dy,
                                                        float* __restrict__ dx, int accumulate,
                                                        float* __restrict__ ws_dg, float* __restrict__ ws_db,
                                                        int rows_per_block) {
  pdl_wait_and_trigger();
  extern __shared__ float sh[];  // [warps][2][d], only for the final block reduction
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_warps = blockDim.x >> 5;
  const int nv = d >> 2;
  float4 ag[kMaxVec], ab[kMaxVec];
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    ag[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    ab[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int row = r0 + warp; row < r1; row += n_warps) {
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long>(row) * d);
    const float4* dyr = reinterpret_cast<const float4*>(dy + static_cast<long>(row) * d);
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int i = lane + 32 * k;
      if (i < nv) {
        const float4 xv = xr[i], dv = dyr[i], gv = g4[i];
        const float4 xh = make_float4((xv.x - mu) * rs, (xv.y - mu) * rs, (xv.z - mu) * rs, (xv.w - mu) * rs);
        s1 += (dv.x * gv.x + dv.y * gv.y) + (dv.z * gv.z + dv.w * gv.w);
        s2 += (dv.x * gv.x * xh.x + dv.y * gv.y * xh.y) + (dv.z * gv.z * xh.z + dv.w * gv.w * xh.w);
        ag[k].x += dv.x * xh.x;
        ag[k].y += dv.y * xh.y;
        ag[k].z += dv.z * xh.z;
        ag[k].w += dv.w * xh.w;
        ab[k].x += dv.x;
        ab[k].y += dv.y;
        ab[k].z += dv.z;
        ab[k].w += dv.w;
      }
    }
    const float m1 = warp_sum(s1) / d, m2 = warp_sum(s2) / d;
    float4* dxr = reinterpret_cast<float4*>(dx + static_cast<long>(row) * d);
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int i = lane + 32 * k;
      if (i < nv) {
        const float4 xv = xr[i], dv = dyr[i], gv = g4[i];
        const float hx = (xv.x - mu) * rs, hy = (xv.y - mu) * rs, hz = (xv.z - mu) * rs, hw = (xv.w - mu) * rs;
        float4 o = make_float4(rs * (dv.x * gv.x - m1 - hx * m2), rs * (dv.y * gv.y - m1 - hy * m2),
                               rs * (dv.z * gv.z - m1 - hz * m2), rs * (dv.w * gv.w - m1 - hw * m2));
        if (accumulate) {
          const float4 p = dxr[i];
          o.x += p.x;
          o.y += p.y;
          o.z += p.z;
          o.w += p.w;
        }
        dxr[i] = o;
      }
    }
  }
  float4* my_dg = reinterpret_cast<float4*>(sh + warp * 2 * d);
  float4* my_db = reinterpret_cast<float4*>(sh + warp * 2 * d + d);
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int i = lane + 32 * k;
    if (i < nv) {
      my_dg[i] = ag[k];
      my_db[i] = ab[k];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float a = 0.f, c = 0.f;
    for (int w = 0; w < n_warps; ++w) {
      a += sh[w * 2 * d + i];
      c += sh[w * 2 * d + d + i];
    }
    ws_dg[static_cast<long>(blockIdx.x) * d + i] = a;
    ws_db[static_cast<long>(blockIdx.x) * d + i] = c;
  }
}

// dx = rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat)); per-block partial dg/db.
template <int kMaxVec>
__global__ void ln_bwd_kernel(int rows, int d, const float* __restrict__ x, const float* __restrict__ g,
                              const float* __restrict__ mean, const float* __restrict__ rstd,
                              const float* __restrict__ dy, float* __restrict__ dx, int accumulate,
                              float* __restrict__ ws_dg, float* __restrict__ ws_db, int rows_per_block) {
  pdl_wait_and_trigger();
  extern __shared__ float sh[];  // [warps][2][d]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_warps = blockDim.x >> 5;
  const int nv = d >> 2;
  float* my_dg = sh + warp * 2 * d;
  float* my_db = my_dg + d;
  for (int i = lane; i < d; i += 32) {
    my_dg[i] = 0.f;
    my_db[i] = 0.f;
  }
  __syncwarp();
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int row = r0 + warp; row < r1; row += n_warps) {
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long>(row) * d);
    const float4* dyr = reinterpret_cast<const float4*>(dy + static_cast<long>(row) * d);
    const float mu = mean[row], rs = rstd[row];
    float4 xh[kMaxVec], gy[kMaxVec];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int i = lane + 32 * k;
      if (i < nv) {
        const float4 xv = xr[i], dv = dyr[i], gv = g4[i];
        xh[k] = make_float4((xv.x - mu) * rs, (xv.y - mu) * rs, (xv.z - mu) * rs, (xv.w - mu) * rs);
        gy[k] = make_float4(dv.x * gv.x, dv.y * gv.y, dv.z * gv.z, dv.w * gv.w);
        s1 += (gy[k].x + gy[k].y) + (gy[k].z + gy[k].w);
        s2 += (gy[k].x * xh[k].x + gy[k].y * xh[k].y) + (gy[k].z * xh[k].z + gy[k].w * xh[k].w);
        float* dgp = my_dg + 4 * i;
        float* dbp = my_db + 4 * i;
        dgp[0] += dv.x * xh[k].x;
        dgp[1] += dv.y * xh[k].y;
        dgp[2] += dv.z * xh[k].z;
        dgp[3] += dv.w * xh[k].w;
        dbp[0] += dv.x;
        dbp[1] += dv.y;
        dbp[2] += dv.z;
        dbp[3] += dv.w;
      }
    }
    const float m1 = warp_sum(s1) / d, m2 = warp_sum(s2) / d;
    float4* dxr = reinterpret_cast<float4*>(dx + static_cast<long>(row) * d);
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int i = lane + 32 * k;
      if (i < nv) {
        float4 o = make_float4(rs * (gy[k].x - m1 - xh[k].x * m2), rs * (gy[k].y - m1 - xh[k].y * m2),
                               rs * (gy[k].z - m1 - xh[k].z * m2), rs * (gy[k].w - m1 - xh[k].w * m2));
        if (accumulate) {
          const float4 p = dxr[i];
          o.x += p.x;
          o.y += p.y;
          o.z += p.z;
          o.w += p.w;
        }
        dxr[i] = o;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float a = 0.f, c = 0.f;
    for (int w = 0; w < n_warps; ++w) {
      a += sh[w * 2 * d + i];
      c += sh[w * 2 * d + d + i];
    }
    ws_dg[static_cast<long>(blockIdx.x) * d + i] = a;
    ws_db[static_cast<long>(blockIdx.x) * d + i] = c;
  }
}

// out[n] (+)= sum_b part[b][n], fixed order => deterministic.
// Block (32 columns x 8 part-lanes): lane y sums parts y, y+8, ... then lane 0 adds the 8
// partials in fixed order => deterministic, and 8x the memory parallelism of one thread/column.
__global__ void reduce_parts_kernel(int parts, int N, const float* __restrict__ part, float* __restrict__ out,
                                    int accumulate) {
  pdl_wait_and_trigger();
  __shared__ float acc[8][33];
  const int n = blockIdx.x * 32 + threadIdx.x;
  float s = 0.f;
  if (n < N) {
    for (int b = threadIdx.y; b < parts; b += 8) s += part[static_cast<long>(b) * N + n];
  }
  acc[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
    float t = 0.f;
#pragma unroll
    for (int y = 0; y < 8; ++y) t += acc[y][threadIdx.x];
    out[n] = accumulate ? out[n] + t : t;
  }
}

// Column sums in one launch, deterministic: block (x, y) sums rows [y*rpb, (y+1)*rpb) of the
// 128-column strip x (32 lanes x float4, 8 row groups, fixed-order smem reduction) into
// part[y]; the last block of a strip to finish (atomic ticket) adds the strip's partials in
// row-block order and resets the ticket, so the result does not depend on block timing.
template <typename XT = float>
__global__ void __launch_bounds__(256) colsum_fused_kernel(int M, int N, const XT* __restrict__ X, long ldx,
                                                           float* __restrict__ part, float* __restrict__ out,
                                                           int accumulate, int rows_per_block,
                                                           unsigned* __restrict__ ticket) {
  pdl_wait_and_trigger();
  __shared__ float4 red[8][33];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = (blockIdx.x * 32 + lane) * 4;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(M, r0 + rows_per_block);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < N) {
#pragma unroll 8
    for (int r = r0 + ty; r < r1; r += 8) {
      const float4 v = ld4(X + static_cast<long>(r) * ldx + c);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
  }
  red[ty][lane] = acc;
  __syncthreads();
  if (ty == 0) {
    float4 t = red[0][lane];
#pragma unroll
    for (int y = 1; y < 8; ++y) {
      const float4 u = red[y][lane];
      t.x += u.x;
      t.y += u.y;
      t.z += u.z;
      t.w += u.w;
    }
    if (c < N) *reinterpret_cast<float4*>(part + static_cast<long>(blockIdx.y) * N + c) = t;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ticket[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // this strip's 128 columns over gridDim.y partials: 8 row groups, fixed order
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < N) {
    for (int b = ty; b < static_cast<int>(gridDim.y); b += 8) {
      const float4 u = __ldcg(reinterpret_cast<const float4*>(part + static_cast<long>(b) * N + c));
      t.x += u.x;
      t.y += u.y;
      t.z += u.z;
      t.w += u.w;
    }
  }
  red[ty][lane] = t;
  __syncthreads();
  if (ty == 0) {
    float4 f = red[0][lane];
#pragma unroll
    for (int y = 1; y < 8; ++y) {
      const float4 u = red[y][lane];
      f.x += u.x;
      f.y += u.y;
      f.z += u.z;
      f.w += u.w;
    }
    if (c < N) {
      float4* o = reinterpret_cast<float4*>(out + c);
      if (accumulate) {
        const float4 p = *o;
        f.x += p.x;
        f.y += p.y;
        f.z += p.z;
        f.w += p.w;
      }
      *o = f;
    }
    if (lane == 0) ticket[blockIdx.x] = 0;
  }
}

// Partial column sums over a row range per block; 256 threads stride the columns.
__global__ void colsum_part_kernel(int M, int N, const float* __restrict__ X, long ldx, float* __restrict__ part,
                                   int rows_per_block) {
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(M, r0 + rows_per_block);
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int r = r0; r < r1; ++r) s += X[static_cast<long>(r) * ldx + n];
    part[static_cast<long>(blockIdx.y) * N + n] = s;
  }
}

// ---- embedding -----------------------------------------------------------------
__global__ void embed_fwd_kernel(int rows, int T, int d, const int32_t* __restrict__ tok,
                                 const float* __restrict__ wte, const float* __restrict__ wpe, float* __restrict__ h) {
  const int nv = d >> 2;
  const long total = static_cast<long>(rows) * nv;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / nv), c = static_cast<int>(i % nv);
    const float4 a = reinterpret_cast<const float4*>(wte + static_cast<long>(tok[r]) * d)[c];
    const float4 p = reinterpret_cast<const float4*>(wpe + static_cast<long>(r % T) * d)[c];
    reinterpret_cast<float4*>(h)[i] = make_float4(a.x + p.x, a.y + p.y, a.z + p.z, a.w + p.w);
  }
}

__global__ void embed_scatter_kernel(int rows, int d, const int32_t* __restrict__ tok, const float* __restrict__ dh,
                                     float* __restrict__ dwte) {
  const long total = static_cast<long>(rows) * d;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / d), c = static_cast<int>(i % d);
    atomicAdd(dwte + static_cast<long>(tok[r]) * d + c, dh[i]);
  }
}

// dwpe[t][c] = sum_b dh[b*T + t][c]
__global__ void embed_pos_kernel(int B, int T, int d, const float* __restrict__ dh, float* __restrict__ dwpe) {
  const long total = static_cast<long>(T) * d;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int b = 0; b < B; ++b) s += dh[static_cast<long>(b) * T * d + i];
    dwpe[i] = s;
  }
}

// ---- softmax cross-entropy ------------------------------------------------------
__global__ void xent_kernel(int V, float* __restrict__ logits, long ldl, const int32_t* __restrict__ targets,
                            float grad_scale, float* __restrict__ row_loss) {
  pdl_wait_and_trigger();
  __shared__ float red_m[32], red_s[32];
  const int row = blockIdx.x;
  float* lr = logits + static_cast<long>(row) * ldl;
  const int tid = threadIdx.x, nw = blockDim.x >> 5, warp = tid >> 5, lane = tid & 31;
  float m = -FLT_MAX, s = 0.f;
  for (int i = tid; i < V; i += blockDim.x) {
    const float z = lr[i];
    if (z > m) {
      s = s * __expf(m - z) + 1.f;
      m = z;
    } else {
      s += __expf(z - m);
    }
  }
  // combine (m, s) across the block
  float wm = warp_max(m);
  float ws = s * __expf(m - wm);
  ws = warp_sum(ws);
  if (lane == 0) {
    red_m[warp] = wm;
    red_s[warp] = ws;
  }
  __syncthreads();
  if (warp == 0) {
    float mm = lane < nw ? red_m[lane] : -FLT_MAX;
    float ss = lane < nw ? red_s[lane] : 0.f;
    const float gm = warp_max(mm);
    ss = warp_sum(lane < nw ? ss * __expf(mm - gm) : 0.f);
    if (lane == 0) {
      red_m[0] = gm;
      red_s[0] = ss;
    }
  }
  __syncthreads();
  const float gm = red_m[0], gs = red_s[0];
  const float inv = 1.f / gs;
  const int tgt = targets[row];
  const float zt = lr[tgt];
  __syncthreads();
  for (int i = tid; i < V; i += blockDim.x) {
    const float p = __expf(lr[i] - gm) * inv;
    lr[i] = (p - (i == tgt ? 1.f : 0.f)) * grad_scale;
  }
  if (tid == 0) row_loss[row] = logf(gs) + gm - zt;
}

// Register-resident variant (V <= 512 * 4 * kV4): the row is read from HBM once into
// registers as float4 (rows are 16-byte aligned: ldl = HY_VOCAB_PAD), reduced for max and
// sum, and written once — 2 x V x 4 bytes of traffic instead of 3 passes.
template <int kV4>
__global__ void __launch_bounds__(512) xent_reg_kernel(int V, float* __restrict__ logits, long ldl,
                                                       const int32_t* __restrict__ targets, float grad_scale,
                                                       float* __restrict__ row_loss) {
  pdl_wait_and_trigger();
  __shared__ float red[32];
  __shared__ float bcast;
  const int row = blockIdx.x;
  float* lr = logits + static_cast<long>(row) * ldl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n4 = V >> 2;  // full float4s; V & 3 tail elements handled by thread 0
  float4 z[kV4];
  float m = -FLT_MAX;
#pragma unroll
  for (int k = 0; k < kV4; ++k) {
    const int i4 = tid + k * 512;
    if (i4 < n4) {
      z[k] = reinterpret_cast<const float4*>(lr)[i4];
      m = fmaxf(m, fmaxf(fmaxf(z[k].x, z[k].y), fmaxf(z[k].z, z[k].w)));
    }
  }
  float tail[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
  if (tid == 0) {
    for (int t = 0; t < (V & 3); ++t) {
      tail[t] = lr[4 * n4 + t];
      m = fmaxf(m, tail[t]);
    }
  }
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (warp == 0) {
    float x = lane < 16 ? red[lane] : -FLT_MAX;
    x = warp_max(x);
    if (lane == 0) bcast = x;
  }
  __syncthreads();
  const float gm = bcast;
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kV4; ++k) {
    const int i4 = tid + k * 512;
    if (i4 < n4) {
      z[k].x = __expf(z[k].x - gm);
      z[k].y = __expf(z[k].y - gm);
      z[k].z = __expf(z[k].z - gm);
      z[k].w = __expf(z[k].w - gm);
      s += (z[k].x + z[k].y) + (z[k].z + z[k].w);
    }
  }
  if (tid == 0) {
    for (int t = 0; t < (V & 3); ++t) {
      tail[t] = __expf(tail[t] - gm);
      s += tail[t];
    }
  }
  s = warp_sum(s);
  __syncthreads();
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (warp == 0) {
    float x = lane < 16 ? red[lane] : 0.f;
    x = warp_sum(x);
    if (lane == 0) bcast = x;
  }
  __syncthreads();
  const float gs = bcast;
  const int tgt = targets[row];
  const float zt = lr[tgt];  // read before this thread block overwrites the row
  __syncthreads();
  const float sc = grad_scale / gs;
#pragma unroll
  for (int k = 0; k < kV4; ++k) {
    const int i4 = tid + k * 512;
    if (i4 < n4) {
      float4 o = make_float4(z[k].x * sc, z[k].y * sc, z[k].z * sc, z[k].w * sc);
      if ((tgt >> 2) == i4) (&o.x)[tgt & 3] -= grad_scale;
      reinterpret_cast<float4*>(lr)[i4] = o;
    }
  }
  if (tid == 0) {
    for (int t = 0; t < (V & 3); ++t) {
      const int i = 4 * n4 + t;
      lr[i] = tail[t] * sc - (i == tgt ? grad_scale : 0.f);
    }
    row_loss[row] = logf(gs) + gm - zt;
  }
}

__global__ void sum_double_kernel(int n, const float* __restrict__ x, double* __restrict__ out, int accumulate) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = accumulate ? out[0] + sh[0] : sh[0];
}

// ---- Adam ------------------------------------------------------------------------
__global__ void adam_kernel(long n4, float4* __restrict__ p, const float4* __restrict__ g, float4* __restrict__ m,
                            float4* __restrict__ v, AdamHyper h) {
  const float c1 = 1.f - h.beta1, c2 = 1.f - h.beta2;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    float4 pp = p[i], gg = g[i], mm = m[i], vv = v[i];
    float* pe = &pp.x;
    const float* ge = &gg.x;
    float* me = &mm.x;
    float* ve = &vv.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      me[k] = h.beta1 * me[k] + c1 * ge[k];
      ve[k] = h.beta2 * ve[k] + c2 * ge[k] * ge[k];
      const float upd = (me[k] / h.bc1) / (sqrtf(ve[k] / h.bc2) + h.eps);
      pe[k] = pe[k] - h.lr * (upd + h.weight_decay * pe[k]);
    }
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
  }
}

// Same update with the moments stored in bf16 (round-to-nearest-even after each update):
// halves the optimizer state a spilled shard streams over the host link.
__global__ void adam_bf16_kernel(long n4, float4* __restrict__ p, const float4* __restrict__ g,
                                 uint2* __restrict__ m, uint2* __restrict__ v, AdamHyper h) {
  const float c1 = 1.f - h.beta1, c2 = 1.f - h.beta2;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    float4 pp = p[i], gg = g[i];
    const uint2 mm = m[i], vv = v[i];
    __nv_bfloat16 mb[4], vb[4];
    *reinterpret_cast<uint2*>(mb) = mm;
    *reinterpret_cast<uint2*>(vb) = vv;
    float* pe = &pp.x;
    const float* ge = &gg.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float mk = h.beta1 * __bfloat162float(mb[k]) + c1 * ge[k];
      const float vk = h.beta2 * __bfloat162float(vb[k]) + c2 * ge[k] * ge[k];
      mb[k] = __float2bfloat16_rn(mk);
      vb[k] = __float2bfloat16_rn(vk);
      const float upd = (mk / h.bc1) / (sqrtf(vk / h.bc2) + h.eps);
      pe[k] = pe[k] - h.lr * (upd + h.weight_decay * pe[k]);
    }
    p[i] = pp;
    m[i] = *reinterpret_cast<uint2*>(mb);
    v[i] = *reinterpret_cast<uint2*>(vb);
  }
}

// Zero-copy AdamW: the moments and the master-param mirror live in pinned host memory and
// are read / written by the kernel itself over the host link (mapped pinned memory, UVA), so
// the optimizer needs no HBM staging and no copy-engine round trip; p is updated in place in
// the HBM slot. Each thread keeps kU independent host loads in flight to cover the PCIe
// round-trip latency. Row filter: element e belongs to row e / row4 (float4 units) and is
// processed iff flags[row] == want (flags == nullptr: every element).
// 128 threads x <= 64 registers per CTA: small enough to co-reside with a persistent GEMM
// CTA (256 threads x 191 registers) instead of evicting it from its SM for the whole transfer.
template <bool kBf16>
__global__ void __launch_bounds__(128, 8) adam_zc_kernel(long n4, long row4, const uint8_t* __restrict__ flags,
                                                      int want, float4* __restrict__ p, const float4* __restrict__ g,
                                                      void* __restrict__ mh, void* __restrict__ vh,
                                                      float4* __restrict__ ph, AdamHyper h) {
  constexpr int kU = 4;
  const float c1 = 1.f - h.beta1, c2 = 1.f - h.beta2;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long base = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; base < n4; base += stride * kU) {
    float mk[kU][4], vk[kU][4];
    bool on[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long i = base + u * stride;
      on[u] = i < n4 && (flags == nullptr || flags[i / row4] == want);
      if (!on[u]) continue;
      if constexpr (kBf16) {
        const uint2 mm = reinterpret_cast<const uint2*>(mh)[i], vv = reinterpret_cast<const uint2*>(vh)[i];
        const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mm);
        const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&vv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          mk[u][k] = __bfloat162float(mb[k]);
          vk[u][k] = __bfloat162float(vb[k]);
        }
      } else {
        const float4 mm = reinterpret_cast<const float4*>(mh)[i], vv = reinterpret_cast<const float4*>(vh)[i];
        mk[u][0] = mm.x, mk[u][1] = mm.y, mk[u][2] = mm.z, mk[u][3] = mm.w;
        vk[u][0] = vv.x, vk[u][1] = vv.y, vk[u][2] = vv.z, vk[u][3] = vv.w;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!on[u]) continue;
      const long i = base + u * stride;
      float4 pp = p[i];
      const float4 gg = g[i];
      float* pe = &pp.x;
      const float* ge = &gg.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mk[u][k] = h.beta1 * mk[u][k] + c1 * ge[k];
        vk[u][k] = h.beta2 * vk[u][k] + c2 * ge[k] * ge[k];
        const float upd = (mk[u][k] / h.bc1) / (sqrtf(vk[u][k] / h.bc2) + h.eps);
        pe[k] = pe[k] - h.lr * (upd + h.weight_decay * pe[k]);
      }
      p[i] = pp;
      if (ph) ph[i] = pp;
      if constexpr (kBf16) {
        __nv_bfloat16 mb[4], vb[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          mb[k] = __float2bfloat16_rn(mk[u][k]);
          vb[k] = __float2bfloat16_rn(vk[u][k]);
        }
        reinterpret_cast<uint2*>(mh)[i] = *reinterpret_cast<uint2*>(mb);
        reinterpret_cast<uint2*>(vh)[i] = *reinterpret_cast<uint2*>(vb);
      } else {
        reinterpret_cast<float4*>(mh)[i] = make_float4(mk[u][0], mk[u][1], mk[u][2], mk[u][3]);
        reinterpret_cast<float4*>(vh)[i] = make_float4(vk[u][0], vk[u][1], vk[u][2], vk[u][3]);
      }
    }
  }
}

// ---- embedding optimizer split (token rows vs the rest) ------------------------------
// idx[r] for the rows of layer 0 (wte rows 0..V-1, wpe rows V..V+T-1): the compact index of
// the row if this minibatch's embedding scatter touches it (token rows, every wpe row), -1
// otherwise; rows[c] = r inverts it; count[0] = number of such rows. Compact order is row order.
__global__ void row_mark_kernel(int M, const int32_t* __restrict__ tok, int V, int T, int* __restrict__ idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) idx[tok[i]] = 0;
  if (i < T) idx[V + i] = 0;
}

__global__ void __launch_bounds__(1024) row_compact_kernel(int n, int* __restrict__ idx, int* __restrict__ rows,
                                                           int* __restrict__ count) {
  __shared__ int warp_tot[32];
  const int t = threadIdx.x, per = (n + 1023) / 1024;
  const int lo = min(n, t * per), hi = min(n, lo + per);
  int c = 0;
  for (int r = lo; r < hi; ++r) c += idx[r] >= 0;
  // block exclusive scan of c
  int x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((t & 31) >= o) x += y;
  }
  if ((t & 31) == 31) warp_tot[t >> 5] = x;
  __syncthreads();
  if (t < 32) {
    int w = warp_tot[t];
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (t >= o) w += y;
    }
    warp_tot[t] = w;  // inclusive over warps
  }
  __syncthreads();
  int base = x - c + ((t >> 5) ? warp_tot[(t >> 5) - 1] : 0);
  for (int r = lo; r < hi; ++r) {
    if (idx[r] >= 0) {
      idx[r] = base;
      rows[base] = r;
      ++base;
    }
  }
  if (t == 1023) *count = base;
}

// Pass A over one staged chunk of layer 0 (elements [off, off + n) of the layer): AdamW on
// every row not in the compact set; rows in the set are only copied (m, v) into the compact
// buffers (cm, cv: [count][d]) for pass B. The chunk's p, m, v go back to the host afterwards
// unchanged for those rows.
template <bool kBf16>
__global__ void adam_masked_kernel(long n4, long off, int d, const int* __restrict__ idx, float4* __restrict__ p,
                                   const float4* __restrict__ g, void* __restrict__ m, void* __restrict__ v,
                                   void* __restrict__ cm, void* __restrict__ cv, AdamHyper h) {
  const float c1 = 1.f - h.beta1, c2 = 1.f - h.beta2;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long e = off + 4 * i;
    const int c = idx[e / d];
    const long col = e % d;
    if (c >= 0) {  // token / wpe row: stash its state for pass B
      if constexpr (kBf16) {
        reinterpret_cast<uint2*>(cm)[(static_cast<long>(c) * d + col) / 4] = reinterpret_cast<const uint2*>(m)[i];
        reinterpret_cast<uint2*>(cv)[(static_cast<long>(c) * d + col) / 4] = reinterpret_cast<const uint2*>(v)[i];
      } else {
        reinterpret_cast<float4*>(cm)[(static_cast<long>(c) * d + col) / 4] = reinterpret_cast<const float4*>(m)[i];
        reinterpret_cast<float4*>(cv)[(static_cast<long>(c) * d + col) / 4] = reinterpret_cast<const float4*>(v)[i];
      }
      continue;
    }
    float4 pp = p[i];
    const float4 gg = g[i];
    float* pe = &pp.x;
    const float* ge = &gg.x;
    float mk[4], vk[4];
    if constexpr (kBf16) {
      const uint2 mm = reinterpret_cast<const uint2*>(m)[i], vv = reinterpret_cast<const uint2*>(v)[i];
      const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mm);
      const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&vv);
#pragma unroll
      for (int k = 0; k < 4; ++k) mk[k] = __bfloat162float(mb[k]), vk[k] = __bfloat162float(vb[k]);
    } else {
      const float4 mm = reinterpret_cast<const float4*>(m)[i], vv = reinterpret_cast<const float4*>(v)[i];
      mk[0] = mm.x, mk[1] = mm.y, mk[2] = mm.z, mk[3] = mm.w;
      vk[0] = vv.x, vk[1] = vv.y, vk[2] = vv.z, vk[3] = vv.w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mk[k] = h.beta1 * mk[k] + c1 * ge[k];
      vk[k] = h.beta2 * vk[k] + c2 * ge[k] * ge[k];
      const float upd = (mk[k] / h.bc1) / (sqrtf(vk[k] / h.bc2) + h.eps);
      pe[k] = pe[k] - h.lr * (upd + h.weight_decay * pe[k]);
    }
    p[i] = pp;
    if constexpr (kBf16) {
      __nv_bfloat16 mb[4], vb[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) mb[k] = __float2bfloat16_rn(mk[k]), vb[k] = __float2bfloat16_rn(vk[k]);
      reinterpret_cast<uint2*>(m)[i] = *reinterpret_cast<uint2*>(mb);
      reinterpret_cast<uint2*>(v)[i] = *reinterpret_cast<uint2*>(vb);
    } else {
      reinterpret_cast<float4*>(m)[i] = make_float4(mk[0], mk[1], mk[2], mk[3]);
      reinterpret_cast<float4*>(v)[i] = make_float4(vk[0], vk[1], vk[2], vk[3]);
    }
  }
}

// Pass B1: AdamW on the compact rows (state from pass A's stash), p updated in the slot
// (layer 0 base `p`) and copied into cp for the write-back.
template <bool kBf16>
__global__ void adam_rows_kernel(const int* __restrict__ count, const int* __restrict__ rows, int d, float* __restrict__ p,
                                 const float* __restrict__ g, void* __restrict__ cm, void* __restrict__ cv,
                                 float* __restrict__ cp, AdamHyper h) {
  const float c1 = 1.f - h.beta1, c2 = 1.f - h.beta2;
  const long n = static_cast<long>(*count) * d;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long c = i / d, col = i % d;
    const long e = static_cast<long>(rows[c]) * d + col;
    const float gi = g[e];
    float mi, vi;
    if constexpr (kBf16) {
      mi = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(cm)[i]);
      vi = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(cv)[i]);
    } else {
      mi = reinterpret_cast<const float*>(cm)[i];
      vi = reinterpret_cast<const float*>(cv)[i];
    }
    mi = h.beta1 * mi + c1 * gi;
    vi = h.beta2 * vi + c2 * gi * gi;
    const float upd = (mi / h.bc1) / (sqrtf(vi / h.bc2) + h.eps);
    const float pi = p[e] - h.lr * (upd + h.weight_decay * p[e]);
    p[e] = pi;
    if (cp) cp[i] = pi;
    if constexpr (kBf16) {
      reinterpret_cast<__nv_bfloat16*>(cm)[i] = __float2bfloat16_rn(mi);
      reinterpret_cast<__nv_bfloat16*>(cv)[i] = __float2bfloat16_rn(vi);
    } else {
      reinterpret_cast<float*>(cm)[i] = mi;
      reinterpret_cast<float*>(cv)[i] = vi;
    }
  }
}

// Pass B2: the compact rows' p, m, v written straight into the host arrays (mapped pinned
// memory, zero-copy stores; a few MB per minibatch).
template <int kEs>
__global__ void rows_to_host_kernel(const int* __restrict__ count, const int* __restrict__ rows, int d,
                                    const float* __restrict__ cp, const void* __restrict__ cm,
                                    const void* __restrict__ cv, float* __restrict__ hp, void* __restrict__ hm,
                                    void* __restrict__ hv) {
  const long n = static_cast<long>(*count) * d;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long e = static_cast<long>(rows[i / d]) * d + i % d;
    if (hp) hp[e] = cp[i];
    if constexpr (kEs == 2) {
      reinterpret_cast<uint16_t*>(hm)[e] = reinterpret_cast<const uint16_t*>(cm)[i];
      reinterpret_cast<uint16_t*>(hv)[e] = reinterpret_cast<const uint16_t*>(cv)[i];
    } else {
      reinterpret_cast<float*>(hm)[e] = reinterpret_cast<const float*>(cm)[i];
      reinterpret_cast<float*>(hv)[e] = reinterpret_cast<const float*>(cv)[i];
    }
  }
}

int grid_for(long n, int block) {
  long g = (n + block - 1) / block;
  const long cap = static_cast<long>(sms()) * 8;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

// Column-sum blocks per SM: enough 256-thread blocks that each SM keeps ~40 KB of loads in
// flight (Little's law at ~6.5 TB/s); HY_COLSUM_WAVES overrides (diagnostics).
int colsum_waves() {
  static const int w = [] {
    const char* e = std::getenv("HY_COLSUM_WAVES");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : 4;
  }();
  return w;
}

int colsum_blocks(int rows) {
  const int target = sms() * 2;
  return rows < target ? (rows > 0 ? rows : 1) : target;
}

template <typename Y>
cudaError_t layernorm_fwd_t(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* b, Y* y,
                            float* mean, float* rstd) {
  if (d % 4 || d > 4 * 32 * kMaxVecAll) return cudaErrorInvalidValue;
  if (rows <= 0) return cudaSuccess;
  // d <= 1024: a warp per row (8 rows per block) measured faster at C2's 4096 x 768 (10.2 vs
  // 12.3 us); wider rows: 4 warps per row, 2 rows per block
  const dim3 grid((rows + 1) / 2), block(32 * kWarpsPerBlock);
  count_launch();
  if (d <= 1024) {
    check_launch(launch_pdl(ln_fwd_kernel<8, 1, Y>, dim3((rows + kWarpsPerBlock - 1) / kWarpsPerBlock), block, 0, s,
                            rows, d, x, g, b, y, mean, rstd));
  } else if (d <= 2048) {
    check_launch(launch_pdl(ln_fwd_kernel<4, 4, Y>, grid, block, 0, s, rows, d, x, g, b, y, mean, rstd));
  } else {
    check_launch(launch_pdl(ln_fwd_kernel<8, 4, Y>, grid, block, 0, s, rows, d, x, g, b, y, mean, rstd));
  }
  return cudaGetLastError();
}
cudaError_t layernorm_fwd(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* b, float* y,
                          float* mean, float* rstd) {
  return layernorm_fwd_t(s, rows, d, x, g, b, y, mean, rstd);
}
cudaError_t layernorm_fwd(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* b,
                          __nv_bfloat16* y, float* mean, float* rstd) {
  return layernorm_fwd_t(s, rows, d, x, g, b, y, mean, rstd);
}

// fp32 -> bf16 (RNE), 8 elements per thread (n % 8 == 0, 16-byte aligned), grid-stride.
__global__ void __launch_bounds__(256) cvt_bf16_kernel(long n8, const float4* __restrict__ x, uint4* __restrict__ y) {
  pdl_wait_and_trigger();
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n8; i += static_cast<long>(gridDim.x) * blockDim.x) {
    const float4 a = x[2 * i], b = x[2 * i + 1];
    __nv_bfloat162 h[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                           __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
    y[i] = *reinterpret_cast<uint4*>(h);
  }
}
cudaError_t to_bf16(cudaStream_t s, long n, const float* x, __nv_bfloat16* y) {
  if (n % 8 || (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(y) & 15)) {
    return cudaErrorInvalidValue;
  }
  if (n == 0) return cudaSuccess;
  const long n8 = n / 8;
  const int grid = static_cast<int>(std::min<long>((n8 + 255) / 256, 8L * sms()));
  count_launch();
  check_launch(launch_pdl(cvt_bf16_kernel, dim3(grid), dim3(256), 0, s, n8, reinterpret_cast<const float4*>(x),
                          reinterpret_cast<uint4*>(y)));
  return cudaGetLastError();
}

unsigned* colsum_tickets(cudaStream_t s);

cudaError_t layernorm_bwd(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* mean,
                          const float* rstd, const float* dy, float* dx, bool accumulate_dx, float* dg, float* db,
                          float* ws) {
  if (d % 4 || d > 4 * 32 * kMaxVecAll) return cudaErrorInvalidValue;
  if (rows <= 0) return cudaSuccess;
  if (unsigned* tickets = colsum_tickets(s)) {
    const int acc = accumulate_dx ? 1 : 0;
    const dim3 block(32 * kWarpsPerBlock);
    count_launch();
    const dim3 grid((rows + 1) / 2);  // kWarpsPerBlock / 4 rows per block
    if (d <= 1024) {
      check_launch(launch_pdl(ln_bwd_dx_kernel<2, 4>, grid, block, 0, s, rows, d, x, g, mean, rstd, dy, dx, acc));
    } else if (d <= 2048) {
      check_launch(launch_pdl(ln_bwd_dx_kernel<4, 4>, grid, block, 0, s, rows, d, x, g, mean, rstd, dy, dx, acc));
    } else {
      check_launch(launch_pdl(ln_bwd_dx_kernel<8, 4>, grid, block, 0, s, rows, d, x, g, mean, rstd, dy, dx, acc));
    }
    const int strips = (d + 127) / 128;
    int nb = std::max(1, std::min(colsum_blocks(rows), (colsum_waves() * sms() + strips - 1) / strips));
    nb = std::min(nb, std::max(1, rows / 32));
    const int rpb = (rows + nb - 1) / nb;
    nb = (rows + rpb - 1) / rpb;
    count_launch();
    check_launch(launch_pdl(ln_bwd_dgb_kernel, dim3(strips, nb), dim3(256), 0, s, rows, d, x, mean, rstd, dy, ws, dg,
                            db, rpb, tickets));
    return cudaGetLastError();
  }
  const int nb = colsum_blocks(rows);
  const int rpb = (rows + nb - 1) / nb;
  const int n_warps = d <= 3072 ? kWarpsPerBlock : 4;
  const size_t smem = static_cast<size_t>(n_warps) * 2 * d * sizeof(float);
  {
    cudaError_t e = ensure_smem_limit(ln_bwd_rr_kernel<8>, 200 * 1024);
    if (e == cudaSuccess) e = ensure_smem_limit(ln_bwd_rr_kernel<16>, 200 * 1024);
    if (e == cudaSuccess) e = ensure_smem_limit(ln_bwd_kernel<32>, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  float* ws_dg = ws;
  float* ws_db = ws + static_cast<long>(nb) * d;
  const int acc = accumulate_dx ? 1 : 0;
  if (d <= 1024) {
    count_launch();
    check_launch(launch_pdl(ln_bwd_rr_kernel<8>, dim3(nb), dim3(32 * n_warps), smem, s, rows, d, x, g, mean, rstd, dy, dx, acc, ws_dg, ws_db, rpb));
  } else if (d <= 2048) {
    count_launch();
    check_launch(launch_pdl(ln_bwd_rr_kernel<16>, dim3(nb), dim3(32 * n_warps), smem, s, rows, d, x, g, mean, rstd, dy, dx, acc, ws_dg, ws_db, rpb));
  } else {
    count_launch();
    check_launch(launch_pdl(ln_bwd_kernel<32>, dim3(nb), dim3(32 * n_warps), smem, s, rows, d, x, g, mean, rstd, dy, dx, acc, ws_dg, ws_db, rpb));
  }
  count_launch();
  check_launch(launch_pdl(reduce_parts_kernel, dim3((d + 31) / 32), dim3(32, 8), 0, s, nb, d, static_cast<const float*>(ws_dg), dg, 1));
  count_launch();
  check_launch(launch_pdl(reduce_parts_kernel, dim3((d + 31) / 32), dim3(32, 8), 0, s, nb, d, static_cast<const float*>(ws_db), db, 1));
  return cudaGetLastError();
}

// The colsum tickets of a stream (allocated on first use, zeroed, self-resetting). Executor
// workers sharing a GPU run colsums concurrently on their own compute streams, so the tickets
// cannot live in a module global; per stream they are serialised by stream order.
unsigned* colsum_tickets(cudaStream_t s) {
  static std::mutex mu;
  static std::map<cudaStream_t, unsigned*> per_stream;
  std::lock_guard<std::mutex> lk(mu);
  unsigned*& p = per_stream[s];
  if (!p) {
    if (cudaMalloc(&p, 4096 * sizeof(unsigned)) != cudaSuccess ||
        cudaMemsetAsync(p, 0, 4096 * sizeof(unsigned), s) != cudaSuccess) {
      p = nullptr;
    }
  }
  return p;
}

cudaError_t colsum(cudaStream_t s, int M, int N, const __nv_bfloat16* X, long ldx, float* out, bool accumulate,
                   float* ws) {
  const int strips = (N + 127) / 128;
  unsigned* tickets = colsum_tickets(s);
  if (!tickets || N % 4 || ldx % 4 || (reinterpret_cast<uintptr_t>(X) & 7) || (reinterpret_cast<uintptr_t>(out) & 15) ||
      strips > 4096) {
    return cudaErrorInvalidValue;
  }
  if (M <= 0) return cudaSuccess;
  int nb = std::max(1, std::min(colsum_blocks(M), (colsum_waves() * sms() + strips - 1) / strips));
  nb = std::min(nb, std::max(1, M / 32));
  const int rpb = (M + nb - 1) / nb;
  nb = (M + rpb - 1) / rpb;
  count_launch();
  check_launch(launch_pdl(colsum_fused_kernel<__nv_bfloat16>, dim3(strips, nb), dim3(256), 0, s, M, N, X, ldx, ws, out,
                          accumulate ? 1 : 0, rpb, tickets));
  return cudaGetLastError();
}
cudaError_t colsum(cudaStream_t s, int M, int N, const float* X, long ldx, float* out, bool accumulate, float* ws) {
  const int strips = (N + 127) / 128;
  unsigned* tickets = colsum_tickets(s);
  if (tickets && N % 4 == 0 && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(out) & 15) == 0 && strips <= 4096 && M > 0) {
    // colsum_waves() blocks per SM, >= 32 rows per block, <= colsum_blocks(M) partials (the ws size)
    int nb = std::max(1, std::min(colsum_blocks(M), (colsum_waves() * sms() + strips - 1) / strips));
    nb = std::min(nb, std::max(1, M / 32));
    const int rpb = (M + nb - 1) / nb;
    nb = (M + rpb - 1) / rpb;
    count_launch();
    check_launch(launch_pdl(colsum_fused_kernel<float>, dim3(strips, nb), dim3(256), 0, s, M, N, X, ldx, ws, out, accumulate ? 1 : 0, rpb, tickets));
    return cudaGetLastError();
  }
  const int nb = colsum_blocks(M);
  const int rpb = (M + nb - 1) / nb;
  dim3 grid((N + 255) / 256, nb);
  count_launch();
  colsum_part_kernel<<<grid, 256, 0, s>>>(M, N, X, ldx, ws, rpb);
  count_launch();
  reduce_parts_kernel<<<(N + 31) / 32, dim3(32, 8), 0, s>>>(nb, N, ws, out, accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t embed_fwd(cudaStream_t s, int rows, int T, int d, const int32_t* tok, const float* wte, const float* wpe,
                      float* h) {
  if (d % 4) return cudaErrorInvalidValue;
  const long n = static_cast<long>(rows) * (d / 4);
  count_launch();
  embed_fwd_kernel<<<grid_for(n, 256), 256, 0, s>>>(rows, T, d, tok, wte, wpe, h);
  return cudaGetLastError();
}

cudaError_t embed_bwd(cudaStream_t s, int rows, int T, int d, const int32_t* tok, const float* dh, float* dwte,
                      float* dwpe, float* /*ws*/) {
  const long n = static_cast<long>(rows) * d;
  count_launch();
  embed_scatter_kernel<<<grid_for(n, 256), 256, 0, s>>>(rows, d, tok, dh, dwte);
  count_launch();
  embed_pos_kernel<<<grid_for(static_cast<long>(T) * d, 256), 256, 0, s>>>(rows / T, T, d, dh, dwpe);
  return cudaGetLastError();
}

cudaError_t softmax_xent(cudaStream_t s, int rows, int V, float* logits, long ldl, const int32_t* targets,
                         float grad_scale, float* row_loss) {
  if (rows <= 0) return cudaSuccess;
  count_launch();
  if (V <= 512 * 4 * 25 && (ldl & 3) == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0) {
    check_launch(launch_pdl(xent_reg_kernel<25>, dim3(rows), dim3(512), 0, s, V, logits, ldl, targets, grad_scale, row_loss));
  } else {
    check_launch(launch_pdl(xent_kernel, dim3(rows), dim3(512), 0, s, V, logits, ldl, targets, grad_scale, row_loss));
  }
  return cudaGetLastError();
}

cudaError_t sum_to_double(cudaStream_t s, int n, const float* x, double* out, bool accumulate) {
  count_launch();
  sum_double_kernel<<<1, 256, 0, s>>>(n, x, out, accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t adam_update_bf16(cudaStream_t s, long n, float* p, const float* g, uint16_t* m, uint16_t* v,
                             const AdamHyper& h) {
  if (n % 4) return cudaErrorInvalidValue;
  const long n4 = n / 4;
  count_launch();
  adam_bf16_kernel<<<grid_for(n4, 256), 256, 0, s>>>(n4, reinterpret_cast<float4*>(p),
                                                     reinterpret_cast<const float4*>(g), reinterpret_cast<uint2*>(m),
                                                     reinterpret_cast<uint2*>(v), h);
  return cudaGetLastError();
}

cudaError_t adam_update(cudaStream_t s, long n, float* p, const float* g, float* m, float* v, const AdamHyper& h) {
  if (n % 4) return cudaErrorInvalidValue;
  const long n4 = n / 4;
  count_launch();
  adam_kernel<<<grid_for(n4, 256), 256, 0, s>>>(n4, reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g),
                                                reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), h);
  return cudaGetLastError();
}

cudaError_t adam_zc(cudaStream_t s, long n, float* p, const float* g, void* m_host, void* v_host, float* p_host,
                    bool bf16, const AdamHyper& h, const uint8_t* flags, int row_len, int want, int grid) {
  if (n % 4 || (flags && (row_len <= 0 || row_len % 4))) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  const long n4 = n / 4;
  const long row4 = flags ? row_len / 4 : 1;
  const long need = (n4 + 128 * 4 - 1) / (128 * 4);
  const int blocks = static_cast<int>(std::min<long>(need, grid > 0 ? grid : 96));
  count_launch();
  if (bf16) {
    adam_zc_kernel<true><<<blocks, 128, 0, s>>>(n4, row4, flags, want, reinterpret_cast<float4*>(p),
                                                reinterpret_cast<const float4*>(g), m_host, v_host,
                                                reinterpret_cast<float4*>(p_host), h);
  } else {
    adam_zc_kernel<false><<<blocks, 128, 0, s>>>(n4, row4, flags, want, reinterpret_cast<float4*>(p),
                                                 reinterpret_cast<const float4*>(g), m_host, v_host,
                                                 reinterpret_cast<float4*>(p_host), h);
  }
  return cudaGetLastError();
}

cudaError_t embed_row_index(cudaStream_t s, int M, const int32_t* tokens, int V, int T, int* idx, int* rows,
                            int* count) {
  cudaError_t e = cudaMemsetAsync(idx, 0xff, sizeof(int) * (static_cast<size_t>(V) + T), s);
  if (e != cudaSuccess) return e;
  count_launch();
  row_mark_kernel<<<(std::max(M, T) + 255) / 256, 256, 0, s>>>(M, tokens, V, T, idx);
  count_launch();
  row_compact_kernel<<<1, 1024, 0, s>>>(V + T, idx, rows, count);
  return cudaGetLastError();
}

cudaError_t adam_embed_dense(cudaStream_t s, long n, long off, int d, const int* idx, float* p, const float* g,
                             void* m, void* v, void* cm, void* cv, bool bf16, const AdamHyper& h) {
  if (n % 4 || off % 4 || d % 4) return cudaErrorInvalidValue;
  const long n4 = n / 4;
  count_launch();
  if (bf16) {
    adam_masked_kernel<true><<<grid_for(n4, 256), 256, 0, s>>>(n4, off, d, idx, reinterpret_cast<float4*>(p),
                                                               reinterpret_cast<const float4*>(g), m, v, cm, cv, h);
  } else {
    adam_masked_kernel<false><<<grid_for(n4, 256), 256, 0, s>>>(n4, off, d, idx, reinterpret_cast<float4*>(p),
                                                                reinterpret_cast<const float4*>(g), m, v, cm, cv, h);
  }
  return cudaGetLastError();
}

cudaError_t adam_embed_rows(cudaStream_t s, long max_rows, const int* count, const int* rows, int d, float* p,
                            const float* g, void* cm, void* cv, float* cp, bool bf16, const AdamHyper& h) {
  const long n = max_rows * d;
  count_launch();
  if (bf16) {
    adam_rows_kernel<true><<<grid_for(n, 256), 256, 0, s>>>(count, rows, d, p, g, cm, cv, cp, h);
  } else {
    adam_rows_kernel<false><<<grid_for(n, 256), 256, 0, s>>>(count, rows, d, p, g, cm, cv, cp, h);
  }
  return cudaGetLastError();
}

cudaError_t embed_rows_to_host(cudaStream_t s, long max_rows, const int* count, const int* rows, int d,
                               const float* cp, const void* cm, const void* cv, float* hp, void* hm, void* hv,
                               bool bf16) {
  count_launch();
  // few CTAs: host-link bound, and small enough not to crowd the compute kernels (every SM a CTA
  // of this kernel sits on cannot host a CTA of the persistent GEMMs until it finishes)
  static const int max_ctas = [] {
    const char* e = std::getenv("HY_ROWS_TO_HOST_CTAS");  // diagnostics
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : 32;
  }();
  const int grid = static_cast<int>(std::min<long>(max_ctas, (max_rows * d + 255) / 256));
  if (bf16) {
    rows_to_host_kernel<2><<<grid, 256, 0, s>>>(count, rows, d, cp, cm, cv, hp, hm, hv);
  } else {
    rows_to_host_kernel<4><<<grid, 256, 0, s>>>(count, rows, d, cp, cm, cv, hp, hm, hv);
  }
  return cudaGetLastError();
}

}  // namespace hy
