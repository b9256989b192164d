// tcgen05/TMEM/TMA GEMM (kind::tf32, fp32 accumulate) with fused epilogues.
#pragma once

#include <cuda_runtime.h>

namespace hy {

enum EpiMode : int {
  kEpiStore = 0,    // C = beta*C + acc (+bias) (+R)
  kEpiGelu = 1,     // Hout = acc + bias ; C = gelu(Hout)
  kEpiGeluBwd = 2,  // C = (acc) * gelu'(Hin)
};

struct GemmEpilogue {
  float* C = nullptr;
  long ldc = 0;
  const float* bias = nullptr;  // [N]
  const float* R = nullptr;     // residual [M, N]
  long ldr = 0;
  float* Hout = nullptr;  // GELU pre-activation out
  long ldho = 0;
  const float* Hin = nullptr;  // GELU pre-activation in (backward)
  long ldhi = 0;
  float beta = 0.f;
  int mode = kEpiStore;
};

// C[M,N] = op(A)[M,K] * op(B)[N,K]^T.
//  a_mn == false: A stored row-major [M][lda] (K contiguous).   true: stored [K][lda] (M contiguous).
//  b_mn == false: B stored row-major [N][ldb] (K contiguous).   true: stored [K][ldb] (N contiguous).
// All leading dims in elements, multiples of 4 (16-byte TMA strides); pointers 16-byte aligned.
cudaError_t gemm_tf32(cudaStream_t stream, int M, int N, int K, const float* A, long lda, bool a_mn,
                      const float* B, long ldb, bool b_mn, const GemmEpilogue& epi);

}  // namespace hy
