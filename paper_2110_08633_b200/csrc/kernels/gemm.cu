// Host entry of the tcgen05 TF32 GEMM: split-K planning and the per-mode dispatch. The
// kernels live in gemm_kernels.cuh, instantiated per epilogue mode in gemm_m{0,1,2}.cu.
#include <cstdlib>
#include <cuda.h>

#include <algorithm>

#include "gemm.cuh"
#include "launch_count.cuh"

namespace hy {
cudaError_t gemm_dispatch_m0(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                           long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3);
cudaError_t gemm_dispatch_m1(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                           long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3);
cudaError_t gemm_dispatch_m2(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                           long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3);

namespace {

constexpr int BM = 128;  // must match gemm_kernels.cuh
constexpr int BK = 32;

thread_local float* t_splitk_ws = nullptr;
thread_local bool t_prec3 = false;
thread_local long t_splitk_floats = 0;

// C = alpha * sum_s part[s] + beta * C   (fixed summation order: deterministic)
__global__ void splitk_reduce_kernel(int M, int N, int S, const float* __restrict__ part, float* __restrict__ C,
                                     long ldc, float alpha, float beta) {
  const long total = static_cast<long>(M) * N;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < S; ++s) acc += part[s * total + i];
    const long m = i / N, n = i % N;
    float* c = C + m * ldc + n;
    *c = alpha * acc + (beta != 0.f ? beta * *c : 0.f);
  }
}

int sm_count_host() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// The epilogue mode is a kernel template parameter: each instantiation carries only its own
// epilogue code (the 3-mode kernel's instruction footprint stalled the epilogue warps on
// instruction fetch).
cudaError_t dispatch(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                     long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat) {
  if (e.mode == kEpiGelu) return gemm_dispatch_m1(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, t_prec3);
  if (e.mode == kEpiGeluBwd) return gemm_dispatch_m2(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, t_prec3);
  return gemm_dispatch_m0(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, t_prec3);
}

}  // namespace

void gemm_set_precision_fp32(bool three_pass) { t_prec3 = three_pass; }
bool gemm_precision_fp32() { return t_prec3; }

cudaError_t gemm_tf32(cudaStream_t stream, int M, int N, int K, const float* A, long lda, bool a_mn,
                      const float* B, long ldb, bool b_mn, const GemmEpilogue& epi, const GemmBatch* batch) {
  if (M <= 0 || N <= 0 || K <= 0) return cudaSuccess;
  if ((lda & 3) || (ldb & 3) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) {
    return cudaErrorInvalidValue;
  }
  GemmBatch bat = batch ? *batch : GemmBatch{};
  GemmEpilogue e = epi;
  // Split K when the output has too few tiles to fill the GPU (e.g. the LM-head dz GEMM:
  // 24 tiles, K = 50257; dW of the attention projection: 36 tiles, K = B*T).
  int split = 1;
  const long tiles = static_cast<long>((M + BM - 1) / BM) * ((N + 127) / 128);
  const int kb_all = (K + BK - 1) / BK;
  const bool plain = !batch && e.mode == kEpiStore && !e.bias && !e.R;
  static const int forced_split = [] {  // diagnostics: HY_GEMM_SPLIT=S forces S-way split-K
    const char* v = std::getenv("HY_GEMM_SPLIT");
    return v ? std::atoi(v) : 0;
  }();
  if (plain && t_splitk_ws && tiles * 2 <= sm_count_host() && kb_all >= 32) {
    split = static_cast<int>(std::min<long>(sm_count_host() / tiles, kb_all / 16));
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
    const long total = static_cast<long>(M) * N;
    const int grid = static_cast<int>(std::min<long>((total + 255) / 256, sm_count_host() * 8L));
    count_launch();
    splitk_reduce_kernel<<<grid, 256, 0, stream>>>(M, N, split, t_splitk_ws, e.C, e.ldc, e.alpha, e.beta);
    return cudaGetLastError();
  }
  return dispatch(stream, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat);
}

void gemm_set_splitk_workspace(float* ws, long floats) {
  t_splitk_ws = ws;
  t_splitk_floats = floats;
}

}  // namespace hy
