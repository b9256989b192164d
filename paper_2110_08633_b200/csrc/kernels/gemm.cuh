// tcgen05/TMEM/TMA GEMM (kind::tf32, fp32 accumulate) with fused epilogues.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace hy {

enum EpiMode : int {
  kEpiStore = 0,    // C = beta*C + acc (+bias) (+R)
  kEpiGelu = 1,     // C = gelu(acc + bias); Hout = gelu'(acc + bias) (skipped when Hout is null)
  kEpiGeluBwd = 2,  // C = acc * Hin  (Hin = the gelu' the forward stored)
  kEpiGeluSave = 3,  // internal: kEpiGelu with Hout set (its own instantiation: each kernel carries
                     // only its epilogue's code, instruction fetch stalled the 2-in-1 form)
};

struct GemmEpilogue {
  float alpha = 1.f;  // C = alpha * acc + ...
  float* C = nullptr;
  long ldc = 0;
  const float* bias = nullptr;  // [N]
  const float* R = nullptr;     // residual [M, N]
  long ldr = 0;
  float* Hout = nullptr;  // gelu' of the pre-activation out (for the backward)
  long ldho = 0;
  const float* Hin = nullptr;  // gelu' of the pre-activation in (backward)
  long ldhi = 0;
  float beta = 0.f;
  int mode = kEpiStore;
  int c16 = 0;  // C is bf16 (ldc in bf16 elements; beta must be 0, unbatched): bf16 GEMM operands out
};

// Batched / causal extensions (used by tensor-core attention). A batch index z in
// [0, nb1*nb2) splits as z1 = z / nb2, z2 = z % nb2; operand X of batch z starts at
// X + z1*x_s1 + z2*x_s2 (elements). Causal modes assume square [T x T] score tiles:
//   kCausalSkipUpper : output tiles strictly above the diagonal are not computed
//   kCausalKLower    : K range limited to [0, m0 + BM)   (O = P V, dQ = dS K)
//   kCausalKUpper    : K range limited to [m0, K)        (dK = dS^T Q, dV = P^T dO)
enum CausalMode : int { kCausalNone = 0, kCausalSkipUpper = 1, kCausalKLower = 2, kCausalKUpper = 3, kSplitK = 4 };

struct GemmBatch {
  int nb1 = 1, nb2 = 1;
  long a_s1 = 0, a_s2 = 0, b_s1 = 0, b_s2 = 0, c_s1 = 0, c_s2 = 0;
  int causal = kCausalNone;
  // set by the launcher: TMA dimension order {inner, b2, outer, b1} when b2's stride is
  // smaller than the row stride (e.g. heads interleaved inside a row)
  int a_perm = 0, b_perm = 0;
  int c_tma = 0;  // set by the launcher: the CTA-pair epilogue stores C (and Hout) with TMA
};

// C[M,N] = op(A)[M,K] * op(B)[N,K]^T.
//  a_mn == false: A stored row-major [M][lda] (K contiguous).   true: stored [K][lda] (M contiguous).
//  b_mn == false: B stored row-major [N][ldb] (K contiguous).   true: stored [K][ldb] (N contiguous).
// All leading dims in elements, multiples of 4 (16-byte TMA strides); pointers 16-byte aligned.
cudaError_t gemm_tf32(cudaStream_t stream, int M, int N, int K, const float* A, long lda, bool a_mn,
                      const float* B, long ldb, bool b_mn, const GemmEpilogue& epi, const GemmBatch* batch = nullptr);

// Split-K scratch for low-occupancy GEMMs (few output tiles, long K). Per host thread
// (each executor worker drives one GPU); without one, GEMMs never split.
void gemm_set_splitk_workspace(float* ws, long floats);
// Per host thread: true = "fp32" precision (3xTF32 split on the tensor cores, ~fp32
// accuracy at 3x the MMA work), false = plain TF32 (default).
void gemm_set_precision_fp32(bool three_pass);
bool gemm_precision_fp32();

// Same contract with bf16 operands (tcgen05.mma kind::f16, fp32 accumulate; leading dims
// multiples of 8). The epilogue (bias / residual / GELU / GELU', split-K) runs in fp32 and
// stores fp32 C, or bf16 C when epi.c16 is set.
cudaError_t gemm_bf16(cudaStream_t stream, int M, int N, int K, const __nv_bfloat16* A, long lda, bool a_mn,
                      const __nv_bfloat16* B, long ldb, bool b_mn, const GemmEpilogue& epi);
// Per host thread: the shard runner's "bf16" precision (block GEMMs on bf16 operands).
void gemm_set_compute_bf16(bool on);
bool gemm_compute_bf16();

}  // namespace hy
