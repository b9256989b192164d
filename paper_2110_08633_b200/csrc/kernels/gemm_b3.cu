// bf16-operand GEMM instantiations (kind::f16) for epilogue mode kEpiGeluSave (GELU + gelu' store) (see gemm_kernels.cuh).
#include "gemm_kernels.cuh"

namespace hy {
cudaError_t gemm_dispatch_b3(cudaStream_t st, int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_mn,
                             const __nv_bfloat16* B, long ldb, bool b_mn, const GemmEpilogue& e, const GemmBatch& bat) {
  return dispatch_mode<__nv_bfloat16, kEpiGeluSave>(st, M, N, K, A, lda, a_mn, B, ldb, b_mn, e, bat, false);
}
}  // namespace hy
