// Host entry of the tcgen05 TF32 GEMM: split-K planning and the per-mode dispatch. The
// kernels live in gemm_kernels.cuh, instantiated per epilogue mode in gemm_m{0,1,2}.cu.
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "gemm.cuh"
#include "launch_count.cuh"
#include "pdl.cuh"

namespace hy {
cudaError_t gemm_dispatch_m0(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                           long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3);
cudaError_t gemm_dispatch_m1(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                           long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3);
cudaError_t gemm_dispatch_m2(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                           long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3);
cudaError_t gemm_dispatch_m3(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                           long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3);
cudaError_t gemm_dispatch_b3(cudaStream_t st, int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_mn,
                             const __nv_bfloat16* B, long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat);
cudaError_t gemm_dispatch_b0(cudaStream_t st, int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_mn,
                             const __nv_bfloat16* B, long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat);
cudaError_t gemm_dispatch_b1(cudaStream_t st, int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_mn,
                             const __nv_bfloat16* B, long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat);
cudaError_t gemm_dispatch_b2(cudaStream_t st, int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_mn,
                             const __nv_bfloat16* B, long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat);

namespace {

constexpr int BM = 128;  // must match gemm_kernels.cuh

thread_local float* t_splitk_ws = nullptr;
thread_local bool t_prec3 = false;
thread_local bool t_bf16 = false;
thread_local long t_splitk_floats = 0;

// C = alpha * sum_s part[s] + beta * C   (fixed summation order: deterministic). Rows over
// grid.y (grid-stride), columns over grid.x, float4 when N and ldc allow; PDL-chained behind the
// split GEMM (griddepcontrol.wait before the partials are read).
template <bool VEC>
__global__ void splitk_reduce_kernel(int M, int N, int S, const float* __restrict__ part, float* __restrict__ C,
                                     long ldc, float alpha, float beta) {
  pdl_wait_and_trigger();
  const long total = static_cast<long>(M) * N;
  const int n = (blockIdx.x * blockDim.x + threadIdx.x) * (VEC ? 4 : 1);
  if (n >= N) return;
  for (int m = blockIdx.y; m < M; m += gridDim.y) {
    const long i = static_cast<long>(m) * N + n;
    float* c = C + static_cast<long>(m) * ldc + n;
    if constexpr (VEC) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < S; ++s) {
        const float4 v = *reinterpret_cast<const float4*>(part + s * total + i);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
      float4 o = make_float4(alpha * acc.x, alpha * acc.y, alpha * acc.z, alpha * acc.w);
      if (beta != 0.f) {
        const float4 p = *reinterpret_cast<const float4*>(c);
        o.x += beta * p.x;
        o.y += beta * p.y;
        o.z += beta * p.z;
        o.w += beta * p.w;
      }
      *reinterpret_cast<float4*>(c) = o;
    } else {
      float acc = 0.f;
      for (int s = 0; s < S; ++s) acc += part[s * total + i];
      *c = alpha * acc + (beta != 0.f ? beta * *c : 0.f);
    }
  }
}

int sm_count_host() {
  // every GPU of a node is the same part; initialised once, thread-safe (magic static)
  static const int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// The epilogue mode is a kernel template parameter: each instantiation carries only its own
// epilogue code (the 3-mode kernel's instruction footprint stalled the epilogue warps on
// instruction fetch).
cudaError_t dispatch(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                     long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat) {
  if (e.mode == kEpiGelu && e.Hout) return gemm_dispatch_m3(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, t_prec3);
  if (e.mode == kEpiGelu) return gemm_dispatch_m1(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, t_prec3);
  if (e.mode == kEpiGeluBwd) return gemm_dispatch_m2(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, t_prec3);
  return gemm_dispatch_m0(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, t_prec3);
}
cudaError_t dispatch(cudaStream_t st, int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_mn,
                     const __nv_bfloat16* B, long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat) {
  if (e.mode == kEpiGelu && e.Hout) return gemm_dispatch_b3(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
  if (e.mode == kEpiGelu) return gemm_dispatch_b1(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
  if (e.mode == kEpiGeluBwd) return gemm_dispatch_b2(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
  return gemm_dispatch_b0(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
}

// Split-K planning shared by both operand types (BK = K per 128-byte stage row: 32 fp32, 64 bf16).
template <typename T>
cudaError_t gemm_run(cudaStream_t stream, int M, int N, int K, const T* A, long lda, bool a_mn, const T* B, long ldb,
                     bool b_mn, const GemmEpilogue& epi, const GemmBatch* batch) {
  constexpr int BK = 128 / static_cast<int>(sizeof(T));
  constexpr long kAlign = 16 / static_cast<long>(sizeof(T));
  const bool prec3 = sizeof(T) == 4 && t_prec3;
  if (M <= 0 || N <= 0 || K <= 0) return cudaSuccess;
  if ((lda % kAlign) || (ldb % kAlign) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) {
    return cudaErrorInvalidValue;
  }
  // bf16 C: stored 4 values (8 bytes) per lane, so 8-byte aligned rows
  if (epi.c16 && (epi.beta != 0.f || batch || (epi.ldc & 3) || (reinterpret_cast<uintptr_t>(epi.C) & 7))) {
    return cudaErrorInvalidValue;
  }
  GemmBatch bat = batch ? *batch : GemmBatch{};
  GemmEpilogue e = epi;
  // Split K when the output has too few tiles to fill the GPU (e.g. the LM-head dz GEMM:
  // 24 tiles, K = 50257; dW of the attention projection: 36 tiles, K = B*T).
  int split = 1;
  const long tiles = static_cast<long>((M + BM - 1) / BM) * ((N + 127) / 128);
  const int kb_all = (K + BK - 1) / BK;
  const bool plain = !batch && e.mode == kEpiStore && !e.bias && !e.R && !e.c16;
  static const int forced_split = [] {  // diagnostics: HY_GEMM_SPLIT=S forces S-way split-K
    const char* v = std::getenv("HY_GEMM_SPLIT");
    return v ? std::atoi(v) : 0;
  }();
  if (plain && t_splitk_ws && tiles * 2 <= sm_count_host() && kb_all >= 32 * 32 / BK) {
    split = static_cast<int>(std::min<long>(sm_count_host() / tiles, kb_all / (16 * 32 / BK)));
    split = static_cast<int>(std::min<long>(split, t_splitk_floats / (static_cast<long>(M) * N)));
  }
  // Long-K GEMMs whose 256-wide CTA-pair tiles cover under half the pairs (the weight gradients,
  // K = tokens): split K so 256-wide tiles fill the GPU (BN 256 halves the operand traffic per
  // flop of the 128-wide single wave; profiles/r01_ncu_gemm_dw_mn_major.txt).
  static const bool split256 = [] {
    const char* v = std::getenv("HY_GEMM_SPLIT256");
    return !(v && v[0] == '0');
  }();
  const long tiles256 = static_cast<long>((M + 2 * BM - 1) / (2 * BM)) * ((N + 255) / 256);
  const long pairs = sm_count_host() / 2;
  if (split256 && split == 1 && plain && t_splitk_ws && !prec3 && M > BM && N > 128 && kb_all >= 64 * 32 / BK &&
      tiles256 * 2 <= pairs) {
    split = static_cast<int>(std::min<long>(pairs / tiles256, kb_all / (32 * 32 / BK)));
    split = static_cast<int>(std::min<long>(split, t_splitk_floats / (static_cast<long>(M) * N)));
  }
  if (forced_split >= 2 && plain && t_splitk_ws) {
    split = static_cast<int>(std::min<long>(forced_split, t_splitk_floats / (static_cast<long>(M) * N)));
  }
  if (split >= 2) {
    bat.nb1 = split;
    bat.causal = kSplitK;
    bat.c_s1 = static_cast<long>(M) * N;
    GemmEpilogue pe;
    pe.C = t_splitk_ws;
    pe.ldc = N;
    const cudaError_t r = dispatch(stream, M, N, K, A, lda, a_mn, B, ldb, b_mn, pe, bat);
    if (r != cudaSuccess) return r;
    const bool vec = (N % 4 == 0) && (e.ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(e.C) % 16 == 0);
    const int cols = vec ? N / 4 : N;
    const int gx = (cols + 255) / 256;
    const int gy = static_cast<int>(std::min<long>(M, std::max<long>(1, sm_count_host() * 8L / gx)));
    count_launch();
    return vec ? launch_pdl(splitk_reduce_kernel<true>, dim3(gx, gy), dim3(256), 0, stream, M, N, split,
                            static_cast<const float*>(t_splitk_ws), e.C, e.ldc, e.alpha, e.beta)
               : launch_pdl(splitk_reduce_kernel<false>, dim3(gx, gy), dim3(256), 0, stream, M, N, split,
                            static_cast<const float*>(t_splitk_ws), e.C, e.ldc, e.alpha, e.beta);
  }
  return dispatch(stream, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
}

}  // namespace

void gemm_set_precision_fp32(bool three_pass) { t_prec3 = three_pass; }
bool gemm_precision_fp32() { return t_prec3; }

cudaError_t gemm_tf32(cudaStream_t stream, int M, int N, int K, const float* A, long lda, bool a_mn,
                      const float* B, long ldb, bool b_mn, const GemmEpilogue& epi, const GemmBatch* batch) {
  return gemm_run<float>(stream, M, N, K, A, lda, a_mn, B, ldb, b_mn, epi, batch);
}

cudaError_t gemm_bf16(cudaStream_t stream, int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_mn,
                      const __nv_bfloat16* B, long ldb, bool b_mn, const GemmEpilogue& epi) {
  return gemm_run<__nv_bfloat16>(stream, M, N, K, A, lda, a_mn, B, ldb, b_mn, epi, nullptr);
}

void gemm_set_compute_bf16(bool on) { t_bf16 = on; }
bool gemm_compute_bf16() { return t_bf16; }

void gemm_set_splitk_workspace(float* ws, long floats) {
  t_splitk_ws = ws;
  t_splitk_floats = floats;
}

}  // namespace hy
