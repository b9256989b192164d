// HBM-bound kernels of the GPT-2 shard: LayerNorm, embedding, softmax cross-entropy,
// column reductions (bias / LN-param grads), fused Adam, flash attention.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace hy {

cudaError_t layernorm_fwd(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* b, float* y,
                          float* mean, float* rstd);
// dx (+)= LN backward; dg/db (+)= column sums. ws: >= 2 * d * colsum_blocks(rows) floats.
cudaError_t layernorm_bwd(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* mean,
                          const float* rstd, const float* dy, float* dx, bool accumulate_dx, float* dg, float* db,
                          float* ws);
int colsum_blocks(int rows);
// out[n] (+)= sum_m X[m, n]; ws >= N * colsum_blocks(M) floats.
cudaError_t colsum(cudaStream_t s, int M, int N, const float* X, long ldx, float* out, bool accumulate, float* ws);

cudaError_t embed_fwd(cudaStream_t s, int rows, int T, int d, const int32_t* tok, const float* wte, const float* wpe,
                      float* h);
// dwte[tok[r]] += dh[r] (atomic); dwpe[t] (+)= sum_b dh[b*T+t] (overwrites unless accumulate).
cudaError_t embed_bwd(cudaStream_t s, int rows, int T, int d, const int32_t* tok, const float* dh, float* dwte,
                      float* dwpe, float* ws);

// In-place softmax-CE over a [rows, V] chunk with row stride ldl. logits -> dlogits * grad_scale.
// row_loss[r] = logsumexp - logit[target].
cudaError_t softmax_xent(cudaStream_t s, int rows, int V, float* logits, long ldl, const int32_t* targets,
                         float grad_scale, float* row_loss);
// out[0] (+)= sum(x[0..n)) in double, deterministic.
cudaError_t sum_to_double(cudaStream_t s, int n, const float* x, double* out, bool accumulate);

struct AdamHyper {
  float lr, beta1, beta2, eps, weight_decay, bc1, bc2;  // bc = 1 - beta^step
};
cudaError_t adam_update(cudaStream_t s, long n, float* p, const float* g, float* m, float* v, const AdamHyper& h);
// Moments stored as bf16 bit patterns (RNE after each update); params/grads fp32.
cudaError_t adam_update_bf16(cudaStream_t s, long n, float* p, const float* g, uint16_t* m, uint16_t* v,
                             const AdamHyper& h);

// Tensor-core attention (attention_tc.cu). `work` holds score matrices: forward needs
// T*T floats per (batch, head) processed at once, backward 2*T*T; chunks are sized to fit.
cudaError_t attention_fwd_tc(cudaStream_t s, int B, int T, int H, const float* qkv, float* out, float* work,
                             long work_floats);
// dqkv overwritten ([B*T, 3*H*64]).
cudaError_t attention_bwd_tc(cudaStream_t s, int B, int T, int H, const float* qkv, const float* dout, float* dqkv,
                             float* work, long work_floats);

}  // namespace hy
