// HBM-bound kernels of the GPT-2 shard: LayerNorm, embedding, softmax cross-entropy,
// column reductions (bias / LN-param grads), fused Adam, flash attention.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace hy {

cudaError_t layernorm_fwd(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* b, float* y,
                          float* mean, float* rstd);
// bf16 output (the "bf16" precision's GEMM operand); mean / rstd fp32.
cudaError_t layernorm_fwd(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* b,
                          __nv_bfloat16* y, float* mean, float* rstd);
// y = bf16(x), round to nearest even; n % 8 == 0, 16-byte aligned.
cudaError_t to_bf16(cudaStream_t s, long n, const float* x, __nv_bfloat16* y);
// dx (+)= LN backward; dg/db (+)= column sums. ws: >= 2 * d * colsum_blocks(rows) floats.
cudaError_t layernorm_bwd(cudaStream_t s, int rows, int d, const float* x, const float* g, const float* mean,
                          const float* rstd, const float* dy, float* dx, bool accumulate_dx, float* dg, float* db,
                          float* ws);
int colsum_blocks(int rows);
// out[n] (+)= sum_m X[m, n]; ws >= N * colsum_blocks(M) floats.
cudaError_t colsum(cudaStream_t s, int M, int N, const float* X, long ldx, float* out, bool accumulate, float* ws);
// Same over a bf16 matrix (N % 4 == 0, ldx % 4 == 0).
cudaError_t colsum(cudaStream_t s, int M, int N, const __nv_bfloat16* X, long ldx, float* out, bool accumulate,
                   float* ws);

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

// Zero-copy AdamW (p in HBM; m, v and the p mirror p_host in mapped pinned host memory;
// p_host may be null: the caller writes the params back itself).
// flags != nullptr: only elements of rows r (row_len floats each) with flags[r] == want.
// grid: CTAs (0 = default); the kernel is host-link bound, a few dozen CTAs saturate it.
cudaError_t adam_zc(cudaStream_t s, long n, float* p, const float* g, void* m_host, void* v_host, float* p_host,
                    bool bf16, const AdamHyper& h, const uint8_t* flags = nullptr, int row_len = 0, int want = 0,
                    int grid = 0);
// Embedding optimizer split. Rows of layer 0 (wte 0..V-1, wpe V..V+T-1) touched by this
// minibatch's embedding scatter (token rows, all wpe rows) get compact indices:
// idx[V+T] (-1 = untouched), rows[<= M+T] (inverse), count[1].
cudaError_t embed_row_index(cudaStream_t s, int M, const int32_t* tokens, int V, int T, int* idx, int* rows,
                            int* count);
// Pass A on a staged chunk (layer-0 elements [off, off+n)): AdamW for untouched rows; touched
// rows' m, v copied to the compact buffers cm, cv ([rows][d]).
cudaError_t adam_embed_dense(cudaStream_t s, long n, long off, int d, const int* idx, float* p, const float* g,
                             void* m, void* v, void* cm, void* cv, bool bf16, const AdamHyper& h);
// Pass B1: AdamW on the compact rows; p (layer-0 base in HBM) updated in place, cp = new p.
cudaError_t adam_embed_rows(cudaStream_t s, long max_rows, const int* count, const int* rows, int d, float* p,
                            const float* g, void* cm, void* cv, float* cp, bool bf16, const AdamHyper& h);
// Pass B2: compact rows' p, m, v -> host arrays (layer-0 base pointers), zero-copy stores.
cudaError_t embed_rows_to_host(cudaStream_t s, long max_rows, const int* count, const int* rows, int d,
                               const float* cp, const void* cm, const void* cv, float* hp, void* hm, void* hv,
                               bool bf16);

// Fused causal attention (attention_fa.cu), kind::tf32, head dim 64. qkv [B*T, 3*H*64];
// out [B*T, H*64]; lse2 [B*H*T] = per-row log2-domain logsumexp of S/8 (for the backward).
cudaError_t attention_fwd_fa(cudaStream_t s, int B, int T, int H, const float* qkv, float* out, float* lse2);
// dqkv overwritten; Di: [B*H*T] scratch.
cudaError_t attention_bwd_fa(cudaStream_t s, int B, int T, int H, const float* qkv, const float* out,
                             const float* dout, const float* lse2, float* dqkv, float* Di);

// Tensor-core attention (attention_tc.cu). `work` holds score matrices: forward needs
// T*T floats per (batch, head) processed at once, backward 2*T*T; chunks are sized to fit.
cudaError_t attention_fwd_tc(cudaStream_t s, int B, int T, int H, const float* qkv, float* out, float* work,
                             long work_floats);
// dqkv overwritten ([B*T, 3*H*64]).
cudaError_t attention_bwd_tc(cudaStream_t s, int B, int T, int H, const float* qkv, const float* dout, float* dqkv,
                             float* work, long work_floats);

}  // namespace hy
