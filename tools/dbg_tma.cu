// Debug-only: TMA-load one MN-major 32x32 fp32 box (SW128) and dump smem; run a single
// 128x128x8 MN-major-A tcgen05.mma and dump the accumulator.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "../paper_2110_08633_b200/csrc/kernels/ptx.cuh"
using namespace hy;

__global__ void dump_kernel(const __grid_constant__ CUtensorMap map, float* out, int x, int y) {
  __shared__ __align__(1024) float tile[32 * 32];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(&bar, 4096); tma_load_2d(tile, &map, &bar, x, y); }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = tile[i];
}

extern "C" int dbg_tma(const float* src, long inner, long outer, long ld, float* out, int x, int y) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) { cudaDriverEntryPointQueryResult q; void* p; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q); fn = (PFN_cuTensorMapEncodeTiled_v12000)p; }
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, 32}; cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -100 - (int)r;
  dump_kernel<<<1, 128>>>(map, out, x, y);
  return (int)cudaDeviceSynchronize();
}

// One 128x128x8 MMA: A MN-major (from src A stored [K=8.. rows][M=128] via 4 boxes of 32x32
// placed at a_atom_stride apart), B K-major [N=128][K=32] via one box 32x128.
__global__ void mma_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, float* out,
                           int a_atom_stride, uint32_t lbo, uint32_t sbo, uint32_t idesc, int swap, int ltype) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = base;            // up to 64 KB
  uint8_t* sb = base + 65536;    // 16 KB
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&mbar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc<128>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, 4 * 4096 + 16384);
    for (int j = 0; j < 4; ++j) tma_load_2d(sa + j * a_atom_stride, &ma, &bar, 32 * j, 0);
    tma_load_2d(sb, &mb, &bar, 0, 0);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint64_t da = smem_desc_sw128(smem_u32(sa), lbo, sbo);
    da = (da & ~(7ull << 61)) | ((uint64_t)ltype << 61);
    uint64_t db = smem_desc_sw128(smem_u32(sb), 16, 1024);
    if (swap) mma_tf32(tm, db, da, idesc, 0); else mma_tf32(tm, da, db, idesc, 0);
    mma_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_fence_after();
  {
    int w = threadIdx.x / 32;
    for (int c = 0; c < 4; ++c) {
      float v[32];
      tmem_ld_32x32b_x32(tm + ((w * 32) << 16) + c * 32, v);
      int row = w * 32 + (threadIdx.x & 31);
      for (int i = 0; i < 32; ++i) out[row * 128 + c * 32 + i] = v[i];
    }
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<128>(tm);
}

extern "C" int dbg_mma(const float* A_mn /*[32][128]*/, const float* B /*[128][32]*/, float* out, int a_atom_stride,
                       unsigned lbo, unsigned sbo, unsigned idesc, int swap, int ltype, int tma_swz) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) { cudaDriverEntryPointQueryResult q; void* p; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q); fn = (PFN_cuTensorMapEncodeTiled_v12000)p; }
  CUtensorMap ma, mb;
  cuuint32_t es[2] = {1, 1};
  { cuuint64_t dims[2] = {128, 32}; cuuint64_t st[1] = {128 * 4}; cuuint32_t box[2] = {32, 32};
    fn(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)A_mn, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)tma_swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  { cuuint64_t dims[2] = {32, 128}; cuuint64_t st[1] = {32 * 4}; cuuint32_t box[2] = {32, 128};
    fn(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)B, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  mma_kernel<<<1, 128, 100 * 1024>>>(ma, mb, out, a_atom_stride, lbo, sbo, idesc, swap, ltype);
  return (int)cudaDeviceSynchronize();
}
