// Device compute of one ShardTask of the GPT-2 model in include/hydra_gpt.h, as a
// sequence of sm_100a kernel launches on one stream. Transfers are the executor's job.
#pragma once

#include <algorithm>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>

#include "hydra_gpt.h"

namespace hy {

struct ShardGeom {
  int l0 = 0, l1 = 0;       // layer range [l0, l1)
  long param_floats = 0;    // contiguous layers l0..l1-1
  long wte_offset = -1;     // offset of a tied-wte copy inside the slot (head shard w/o embed), else -1
  long slot_floats = 0;     // param_floats (+ pad + V*d when wte_offset >= 0)
  bool has_embed = false, has_head = false;
  int n_blocks = 0;         // transformer blocks in the shard
};

ShardGeom shard_geom(const hy_dims& m, int l0, int l1);

// Device scratch for one worker (carved from the capped arena).
struct Scratch {
  int M = 0, d = 0;
  float* stash = nullptr;  // [max_blocks + 1][M*d] block inputs for recompute
  int stash_slots = 0;
  float *ln1, *mean1, *rstd1, *qkv, *att, *lse, *hmid, *ln2, *mean2, *rstd2, *fc, *act;
  float* tmp_h;                  // [M*d]
  float* ws;                     // colsum / LN partials
  float *z, *zmean, *zrstd, *dz;  // head
  float* row_loss;               // [M]
  double* loss;                  // [1]
  float* logits;                 // aliases fc..act, logits_rows x HY_VOCAB_PAD
  int logits_rows = 0;
  float* attn_ws;                // [B*H*T]
  // "bf16" precision (carved only then): one block's parameters as bf16, same offsets as the
  // fp32 block (hy_block_tensor_offset), converted before the block's GEMMs use them. Block
  // GEMM operands are bf16 views inside the fp32 buffers: ln1 = [ln1 | attention out],
  // ln2 = [ln2 | dh], act = [act] / [dact] / [datt (fp32) | dqkv]; see block_forward_bf16.
  __nv_bfloat16* w16 = nullptr;
};

// Stash layout for a job's shards: a backward keeps the input of each of its blocks (plus, for
// the head shard, its last block's output: the head's input). The head shard's stash sits after
// the deepest other shard's (when it has blocks and no embedding), so the forward stash of the
// shard whose backward follows the head's survives it (StashPlan::head_offset; TaskIO::head_stash).
struct StashPlan {
  int head_offset = 0;  // slot where the head shard's stash starts (0: shared with the others)
  int slots = 1;
};
inline StashPlan stash_plan(const std::vector<ShardGeom>& geom) {
  StashPlan p;
  int nohead = 0, head = 0;
  bool separate = false;
  for (const ShardGeom& sg : geom) {
    if (sg.has_head) {
      head = sg.n_blocks + 1;
      separate = sg.n_blocks > 0 && !sg.has_embed;
    } else {
      nohead = std::max(nohead, sg.n_blocks);
    }
  }
  p.head_offset = separate ? nohead : 0;
  p.slots = std::max(1, separate ? nohead + head : std::max(nohead, head));
  return p;
}
// Passed to scratch_floats / carve_scratch as `max_blocks` (they reserve max_blocks + 1 slots).
inline int stash_blocks(const std::vector<ShardGeom>& geom) { return stash_plan(geom).slots - 1; }
// Stash slots of shard s in the optional extension region (shards 1.., not the head) when
// every shard keeps its own stash; ext_stash_slots(geom) is the region's size.
inline int ext_stash_offset(const std::vector<ShardGeom>& geom, int s) {
  int off = 0;
  for (int t = 1; t < s; ++t) off += geom[static_cast<size_t>(t)].has_head ? 0 : geom[static_cast<size_t>(t)].n_blocks;
  return off;
}
inline int ext_stash_slots(const std::vector<ShardGeom>& geom) {
  return ext_stash_offset(geom, static_cast<int>(geom.size()));
}
// Bytes of scratch a worker needs for these dims with `max_blocks` blocks per shard.
// bf16: also carve Scratch::w16 (the runner then takes the bf16 block path).
long scratch_floats(const hy_dims& m, int max_blocks, bool bf16 = false);
void carve_scratch(const hy_dims& m, int max_blocks, float* base, Scratch* s, bool bf16 = false);

struct TaskIO {
  const int32_t* tokens = nullptr;   // [M] device
  const int32_t* targets = nullptr;  // [M] device
  const float* act_in = nullptr;     // boundary activation in (l0 > 0)
  float* act_out = nullptr;          // boundary activation out (forward, no head)
  const float* grad_in = nullptr;    // dL/d act_out (backward, no head)
  float* grad_out = nullptr;         // dL/d act_in (backward, l0 > 0)
  const float* z_in = nullptr;       // saved ln_f output for the deferred tied-wte grad (B of shard 0)
  float* z_out = nullptr;            // B of a head shard without the embedding: save its ln_f output here
  bool keep_stash = false;           // forward (no head): leave each block's input in the stash
  float* stash = nullptr;            // this shard's stash region (default: the scratch's shared stash)
  bool stash_ready = false;          // backward: the stash holds this shard's block inputs (its forward's)
  const float* wte = nullptr;        // tied wte for a head shard without the embedding
};

// Forward task: leaves the loss (when the shard has the head) in s.loss[0].
void run_forward(cudaStream_t st, const hy_dims& m, const ShardGeom& g, const float* slot, const TaskIO& io,
                 Scratch& s);
// Backward task (recompute + backward): grads (shard layout, pre-zeroed by the caller) +=.
// When the shard has the head but not the embed, the ln_f output z is left in s.z for the
// caller to demote; when it has the embed but not the head, io.z_in drives the deferred
// tied-wte gradient.
// Where a backward task's parameter gradients go. acquire(layer) returns zeroed device
// storage for that layer's gradient (layout of hy_layer_floats; the caller may insert stream
// waits), release(layer) is called once the layer's gradient is final so the optimizer can
// consume it immediately. Layers are acquired last-to-first; the embedding (layer 0) is
// acquired before the head when both are in the shard and released last.
struct GradSink {
  virtual ~GradSink() = default;
  virtual float* acquire(int layer) = 0;
  virtual void release(int layer) = 0;
  // Embedding only, before release(0): every wte row not indexed by this task's tokens is
  // final (the tied head's dense dwte is in; the embedding scatter only touches token rows
  // and wpe), so their optimizer update may start while the blocks back-propagate.
  virtual void release_dense(int layer) {}
};

void run_backward(cudaStream_t st, const hy_dims& m, const ShardGeom& g, const float* slot, GradSink& sink,
                  const TaskIO& io, Scratch& s);

void check_cuda(cudaError_t e, const char* what);

}  // namespace hy
