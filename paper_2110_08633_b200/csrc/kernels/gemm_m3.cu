// GEMM instantiations for epilogue mode kEpiGeluSave (GELU + gelu' store) (see gemm_kernels.cuh).
#include "gemm_kernels.cuh"

namespace hy {
cudaError_t gemm_dispatch_m3(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool a_mn, const float* B,
                           long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat, bool prec3) {
  return dispatch_mode<float, kEpiGeluSave>(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, prec3);
}
}  // namespace hy
