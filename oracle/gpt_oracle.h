/* ORACLE / TEST INFRASTRUCTURE ONLY — CPU restatement of the shard-execution numerics.
 *
 * The reference (spillsim) never executes tensors, so loss/parameter parity is
 * NOT pinned by reference code: this oracle restates the standard GPT-2 definition the
 * reference's cost model describes (proj/core/src/model.cpp:165-216: embed, n blocks with
 * QKV / attn-proj / 4d MLP, tied head with the loss folded in) together with the
 * reference's shard semantics (proj/core/src/strategies.cpp:743-782: F(s) consumes the
 * boundary activation of s-1 and demotes its own; B(s) promotes the checkpoint + grad_in,
 * recomputes the shard forward, back-propagates, and offloads the shard's parameter
 * gradients; optimizer kept off the device footprint).
 * Layout/init/tokens: include/hydra_gpt.h. fp32 storage, fp64 accumulation, OpenMP.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg call this.
 */
#ifndef GPT_ORACLE_H_
#define GPT_ORACLE_H_

#include <stdint.h>

#include "../include/hydra_gpt.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Forward of layers [l0, l1). act_in: [B*T, d] (ignored when l0 == 0: tokens used).
 * act_out: [B*T, d] written unless the shard contains the head; *loss set if it does. */
int oracle_shard_fwd(const hy_dims* m, const float* params, int l0, int l1, const int32_t* tokens,
                     const int32_t* targets, const float* act_in, float* act_out, double* loss);

/* Backward of layers [l0, l1) with in-shard recompute from act_in (the checkpoint).
 * grad_out: dL/d(act_out) (ignored when the shard contains the head). grads: full-size
 * gradient vector, accumulated into (+=). grad_in: dL/d(act_in), written when l0 > 0. */
int oracle_shard_bwd(const hy_dims* m, const float* params, float* grads, int l0, int l1, const int32_t* tokens,
                     const int32_t* targets, const float* act_in, const float* grad_out, float* grad_in);

/* AdamW over n elements; bias corrections computed in double from `step` (>= 1). */
void oracle_adam(long n, float* p, const float* g, float* m, float* v, float lr, float beta1, float beta2, float eps,
                 float weight_decay, int step);

/* Same with the moments rounded to bfloat16 (RNE) after each update when bf16_state != 0
 * (the update itself uses the unrounded fp32 moments), as the bf16-state GPU kernel does. */
void oracle_adam_state(long n, float* p, const float* g, float* m, float* v, float lr, float beta1, float beta2,
                       float eps, float weight_decay, int step, int bf16_state);

/* Whole-model train step (single shard) — the unsharded reference. Returns the loss. */
double oracle_train_step(const hy_dims* m, float* params, float* mom, float* var, int step, float lr,
                         const int32_t* tokens, const int32_t* targets);

/* "bf16" precision: block GEMM operands rounded to bf16 (see gpt_oracle.c); 0 restores fp32. */
void oracle_set_bf16(int on);

void oracle_init_params(const hy_dims* m, uint64_t model_key, float* params);
void oracle_make_tokens(const hy_dims* m, uint64_t seed, int job, int mb, int32_t* tokens, int32_t* targets);
int oracle_threads(void);

#ifdef __cplusplus
}
#endif
#endif
