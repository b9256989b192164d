// GPT-2 shard compute on sm_100a kernels. Forward: embed -> blocks -> (head loss).
// Backward: recompute the shard forward from its checkpoint keeping block inputs, then
// per block recompute intermediates and back-propagate (reference semantics: backward
// compute = fwd recompute + bwd, strategies.cpp:775). Backward temporaries alias dead
// forward intermediates, so a block needs ~12 M*d floats of scratch in total.
#include "gpt_runner.hpp"
#include "prof.hpp"

#include <algorithm>
#include <string>

#include "../kernels/gemm.cuh"
#include "../kernels/ops.cuh"
#include "spillsim/errors.hpp"

namespace hy {

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw spillsim::DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

ShardGeom shard_geom(const hy_dims& m, int l0, int l1) {
  ShardGeom g;
  g.l0 = l0;
  g.l1 = l1;
  g.has_embed = l0 == 0;
  g.has_head = l1 == m.L + 2;
  g.n_blocks = std::min(l1, m.L + 1) - std::max(l0, 1);
  if (g.n_blocks < 0) g.n_blocks = 0;
  g.param_floats = hy_layer_offset(&m, l1) - hy_layer_offset(&m, l0);
  g.slot_floats = g.param_floats;
  if (g.has_head && !g.has_embed) {
    g.wte_offset = hy_pad32(g.param_floats);
    g.slot_floats = g.wte_offset + static_cast<long>(m.V) * m.d;
  }
  return g;
}

namespace {

using bf16 = __nv_bfloat16;

// floats of scratch holding one transformer block's parameters as bf16
long w16_floats(const hy_dims& m) { return hy_pad32((hy_layer_floats(&m, 1) + 1) / 2); }

inline long lo(const hy_dims& m, int layer, int l0) { return hy_layer_offset(&m, layer) - hy_layer_offset(&m, l0); }
inline const float* bt(const float* w, int d, int t) { return w + hy_block_tensor_offset(d, t); }
inline float* btw(float* w, int d, int t) { return w + hy_block_tensor_offset(d, t); }

void gemm(cudaStream_t st, int M, int N, int K, const float* A, long lda, bool amn, const float* B, long ldb,
          bool bmn, float* C, long ldc, const float* bias = nullptr, const float* R = nullptr, long ldr = 0,
          float beta = 0.f, int mode = kEpiStore, float* hout = nullptr, const float* hin = nullptr, long ldh = 0) {
  GemmEpilogue e;
  e.C = C;
  e.ldc = ldc;
  e.bias = bias;
  e.R = R;
  e.ldr = ldr;
  e.beta = beta;
  e.mode = mode;
  e.Hout = hout;
  e.ldho = ldh;
  e.Hin = hin;
  e.ldhi = ldh;
  check_cuda(gemm_tf32(st, M, N, K, A, lda, amn, B, ldb, bmn, e), "gemm");
}

void gemm16(cudaStream_t st, int M, int N, int K, const bf16* A, long lda, bool amn, const bf16* B, long ldb, bool bmn,
            void* C, long ldc, bool c16, const float* bias = nullptr, const float* R = nullptr, long ldr = 0,
            float beta = 0.f, int mode = kEpiStore, float* hout = nullptr, const float* hin = nullptr, long ldh = 0) {
  GemmEpilogue e;
  e.C = static_cast<float*>(C);
  e.ldc = ldc;
  e.c16 = c16 ? 1 : 0;
  e.bias = bias;
  e.R = R;
  e.ldr = ldr;
  e.beta = beta;
  e.mode = mode;
  e.Hout = hout;
  e.ldho = ldh;
  e.Hin = hin;
  e.ldhi = ldh;
  check_cuda(gemm_bf16(st, M, N, K, A, lda, amn, B, ldb, bmn, e), "gemm bf16");
}

// The block's parameters as bf16 into s.w16 (same offsets as the fp32 block).
const bf16* block_w16(cudaStream_t st, const hy_dims& m, const float* w, Scratch& s) {
  HY_PROF(st, "w16");
  check_cuda(to_bf16(st, hy_layer_floats(&m, 1), w, s.w16), "w16");
  return s.w16;
}
inline const bf16* bt16(const bf16* w, int d, int t) { return w + hy_block_tensor_offset(d, t); }

// bf16 views of the block scratch (Scratch::w16 comment).
struct Views16 {
  bf16 *ln1, *att, *ln2, *dh, *act, *dqkv;
  float* datt;
};
inline Views16 views16(Scratch& s) {
  const long n = static_cast<long>(s.M) * s.d;
  Views16 v;
  v.ln1 = reinterpret_cast<bf16*>(s.ln1);
  v.att = v.ln1 + n;
  v.ln2 = reinterpret_cast<bf16*>(s.ln2);
  v.dh = v.ln2 + n;
  v.act = reinterpret_cast<bf16*>(s.act);
  v.datt = s.act;
  v.dqkv = reinterpret_cast<bf16*>(s.act + n);
  return v;
}

// "bf16" precision, the autocast split: every block GEMM reads bf16 operands (weights, LN
// outputs, attention output, GELU output, and the gradients feeding dX / dW GEMMs) with fp32
// accumulation and fp32 epilogues; the residual stream, LayerNorm statistics, attention
// (TF32 flash kernels on fp32 Q/K/V), softmax-CE, the head and every parameter gradient stay
// fp32. The CPU oracle's bf16 mode rounds exactly these operands (oracle/gpt_oracle.c).
void block_forward_bf16(cudaStream_t st, const hy_dims& m, const float* w, const float* h_in, float* h_out,
                        Scratch& s, bool keep_h) {
  const int M = s.M, d = m.d;
  const bf16* w16 = block_w16(st, m, w, s);
  const Views16 v = views16(s);
  { HY_PROF(st, "ln1");
  check_cuda(layernorm_fwd(st, M, d, h_in, bt(w, d, HY_LN1_G), bt(w, d, HY_LN1_B), v.ln1, s.mean1, s.rstd1), "ln1");
  }
  { HY_PROF(st, "qkv");
  gemm16(st, M, 3 * d, d, v.ln1, d, false, bt16(w16, d, HY_WQKV), d, false, s.qkv, 3 * d, false, bt(w, d, HY_BQKV));
  }
  { HY_PROF(st, "attn_fwd");
  check_cuda(attention_fwd_fa(st, m.B, m.T, m.H, s.qkv, s.att, s.lse), "attn_fwd");
  check_cuda(to_bf16(st, static_cast<long>(M) * d, s.att, v.att), "att16");
  }
  { HY_PROF(st, "o_proj");
  gemm16(st, M, d, d, v.att, d, false, bt16(w16, d, HY_WO), d, false, s.hmid, d, false, bt(w, d, HY_BO), h_in, d);
  }
  { HY_PROF(st, "ln2");
  check_cuda(layernorm_fwd(st, M, d, s.hmid, bt(w, d, HY_LN2_G), bt(w, d, HY_LN2_B), v.ln2, s.mean2, s.rstd2), "ln2");
  }
  { HY_PROF(st, "fc");
  gemm16(st, M, 4 * d, d, v.ln2, d, false, bt16(w16, d, HY_WFC), d, false, v.act, 4 * d, true, bt(w, d, HY_BFC),
         nullptr, 0, 0.f, kEpiGelu, keep_h ? s.fc : nullptr, nullptr, 4 * d);
  }
  if (h_out) {
    HY_PROF(st, "mlp_proj");
    gemm16(st, M, d, 4 * d, v.act, 4 * d, false, bt16(w16, d, HY_WPR), 4 * d, false, h_out, d, false, bt(w, d, HY_BPR),
           s.hmid, d);
  }
}

// Backward of block_forward_bf16 (its intermediates and s.w16 must be this block's).
void block_backward_bf16(cudaStream_t st, const hy_dims& m, const float* w, float* gw, const float* h_in, float* dh,
                         Scratch& s) {
  const int M = s.M, d = m.d;
  const long n = static_cast<long>(M) * d;
  const bf16* w16 = s.w16;
  const Views16 v = views16(s);
  check_cuda(to_bf16(st, n, dh, v.dh), "dh16");
  { HY_PROF(st, "bwd_dW_proj");
  gemm16(st, d, 4 * d, M, v.dh, d, true, v.act, 4 * d, true, btw(gw, d, HY_WPR), 4 * d, false, nullptr, nullptr, 0, 1.f);
  }
  { HY_PROF(st, "bwd_bias");
  check_cuda(colsum(st, M, d, dh, d, btw(gw, d, HY_BPR), true, s.ws), "colsum bpr");
  }
  bf16* dact = v.act;  // act is dead after dWpr
  { HY_PROF(st, "bwd_dact");
  gemm16(st, M, 4 * d, d, v.dh, d, false, bt16(w16, d, HY_WPR), 4 * d, true, dact, 4 * d, true, nullptr, nullptr, 0,
         0.f, kEpiGeluBwd, nullptr, s.fc, 4 * d);
  }
  { HY_PROF(st, "bwd_dW_fc");
  gemm16(st, 4 * d, d, M, dact, 4 * d, true, v.ln2, d, true, btw(gw, d, HY_WFC), d, false, nullptr, nullptr, 0, 1.f);
  }
  { HY_PROF(st, "bwd_bias");
  check_cuda(colsum(st, M, 4 * d, dact, 4 * d, btw(gw, d, HY_BFC), true, s.ws), "colsum bfc");
  }
  float* dln2 = s.fc;  // fc dead after dact
  { HY_PROF(st, "bwd_dln2");
  gemm16(st, M, d, 4 * d, dact, 4 * d, false, bt16(w16, d, HY_WFC), d, true, dln2, d, false);
  }
  { HY_PROF(st, "bwd_ln");
  check_cuda(layernorm_bwd(st, M, d, s.hmid, bt(w, d, HY_LN2_G), s.mean2, s.rstd2, dln2, dh, true,
                           btw(gw, d, HY_LN2_G), btw(gw, d, HY_LN2_B), s.ws),
             "ln2 bwd");
  }
  check_cuda(to_bf16(st, n, dh, v.dh), "dh16");
  { HY_PROF(st, "bwd_dW_o");
  gemm16(st, d, d, M, v.dh, d, true, v.att, d, true, btw(gw, d, HY_WO), d, false, nullptr, nullptr, 0, 1.f);
  }
  { HY_PROF(st, "bwd_bias");
  check_cuda(colsum(st, M, d, dh, d, btw(gw, d, HY_BO), true, s.ws), "colsum bo");
  }
  { HY_PROF(st, "bwd_datt");
  gemm16(st, M, d, d, v.dh, d, false, bt16(w16, d, HY_WO), d, true, v.datt, d, false);
  }
  float* dqkv = s.fc;
  { HY_PROF(st, "attn_bwd");
  check_cuda(attention_bwd_fa(st, m.B, m.T, m.H, s.qkv, s.att, v.datt, s.lse, dqkv, s.attn_ws), "attn bwd");
  check_cuda(to_bf16(st, 3 * n, dqkv, v.dqkv), "dqkv16");
  }
  { HY_PROF(st, "bwd_dW_qkv");
  gemm16(st, 3 * d, d, M, v.dqkv, 3 * d, true, v.ln1, d, true, btw(gw, d, HY_WQKV), d, false, nullptr, nullptr, 0, 1.f);
  }
  { HY_PROF(st, "bwd_bias");
  check_cuda(colsum(st, M, 3 * d, dqkv, 3 * d, btw(gw, d, HY_BQKV), true, s.ws), "colsum bqkv");
  }
  float* dln1 = s.hmid;
  { HY_PROF(st, "bwd_dln1");
  gemm16(st, M, d, 3 * d, v.dqkv, 3 * d, false, bt16(w16, d, HY_WQKV), d, true, dln1, d, false);
  }
  { HY_PROF(st, "bwd_ln");
  check_cuda(layernorm_bwd(st, M, d, h_in, bt(w, d, HY_LN1_G), s.mean1, s.rstd1, dln1, dh, true,
                           btw(gw, d, HY_LN1_G), btw(gw, d, HY_LN1_B), s.ws),
             "ln1 bwd");
  }
}

// keep_h: also store gelu' of the MLP pre-activation (s.fc), which only the backward's GELU' needs; the
// forward tasks and the backward's stash recompute skip that M x 4d write. h_out == nullptr:
// the block's output is not needed (the backward's per-block recompute, or the last block of a
// shard without the head in the stash pass) — the MLP projection GEMM is skipped.
void block_forward(cudaStream_t st, const hy_dims& m, const float* w, const float* h_in, float* h_out, Scratch& s,
                   bool keep_h) {
  if (s.w16) return block_forward_bf16(st, m, w, h_in, h_out, s, keep_h);
  const int M = s.M, d = m.d;
  { HY_PROF(st, "ln1");
  check_cuda(layernorm_fwd(st, M, d, h_in, bt(w, d, HY_LN1_G), bt(w, d, HY_LN1_B), s.ln1, s.mean1, s.rstd1), "ln1");
  }
  { HY_PROF(st, "qkv");
  gemm(st, M, 3 * d, d, s.ln1, d, false, bt(w, d, HY_WQKV), d, false, s.qkv, 3 * d, bt(w, d, HY_BQKV));
  }
  // scores live in the (not yet written) MLP buffers fc+act: 8*M*d floats, contiguous
  { HY_PROF(st, "attn_fwd");
  // TF32: fused flash-style kernel (lse kept for the backward); 3xTF32 "fp32" precision:
  // score matrices in the MLP buffers fc+act (8*M*d floats) through the batched GEMMs
  if (gemm_precision_fp32()) {
    check_cuda(attention_fwd_tc(st, m.B, m.T, m.H, s.qkv, s.att, s.fc, s.act + 4L * M * d - s.fc), "attn_fwd");
  } else {
    check_cuda(attention_fwd_fa(st, m.B, m.T, m.H, s.qkv, s.att, s.lse), "attn_fwd");
  }
  }
  { HY_PROF(st, "o_proj");
  gemm(st, M, d, d, s.att, d, false, bt(w, d, HY_WO), d, false, s.hmid, d, bt(w, d, HY_BO), h_in, d);
  }
  { HY_PROF(st, "ln2");
  check_cuda(layernorm_fwd(st, M, d, s.hmid, bt(w, d, HY_LN2_G), bt(w, d, HY_LN2_B), s.ln2, s.mean2, s.rstd2), "ln2");
  }
  { HY_PROF(st, "fc");
  gemm(st, M, 4 * d, d, s.ln2, d, false, bt(w, d, HY_WFC), d, false, s.act, 4 * d, bt(w, d, HY_BFC), nullptr, 0, 0.f,
       kEpiGelu, keep_h ? s.fc : nullptr, nullptr, 4 * d);
  }
  if (h_out) {
    HY_PROF(st, "mlp_proj");
    gemm(st, M, d, 4 * d, s.act, 4 * d, false, bt(w, d, HY_WPR), 4 * d, false, h_out, d, bt(w, d, HY_BPR), s.hmid, d);
  }
}

// dh: in dL/dh_out, out dL/dh_in. Requires the intermediates of block_forward(h_in).
void block_backward(cudaStream_t st, const hy_dims& m, const float* w, float* gw, const float* h_in, float* dh,
                    Scratch& s) {
  if (s.w16) return block_backward_bf16(st, m, w, gw, h_in, dh, s);
  const int M = s.M, d = m.d;
  // MLP out: h_out = hmid + act Wpr^T + bpr
  { HY_PROF(st, "bwd_dW_proj");
  gemm(st, d, 4 * d, M, dh, d, true, s.act, 4 * d, true, btw(gw, d, HY_WPR), 4 * d, nullptr, nullptr, 0, 1.f);
  }
  { HY_PROF(st, "bwd_bias");
  check_cuda(colsum(st, M, d, dh, d, btw(gw, d, HY_BPR), true, s.ws), "colsum bpr");
  }
  float* dact = s.act;  // act is dead after dWpr
  { HY_PROF(st, "bwd_dact");
  gemm(st, M, 4 * d, d, dh, d, false, bt(w, d, HY_WPR), 4 * d, true, dact, 4 * d, nullptr, nullptr, 0, 0.f, kEpiGeluBwd,
       nullptr, s.fc, 4 * d);
  }
  { HY_PROF(st, "bwd_dW_fc");
  gemm(st, 4 * d, d, M, dact, 4 * d, true, s.ln2, d, true, btw(gw, d, HY_WFC), d, nullptr, nullptr, 0, 1.f);
  }
  { HY_PROF(st, "bwd_bias");
  check_cuda(colsum(st, M, 4 * d, dact, 4 * d, btw(gw, d, HY_BFC), true, s.ws), "colsum bfc");
  }
  float* dln2 = s.fc;  // fc dead after dact
  { HY_PROF(st, "bwd_dln2");
  gemm(st, M, d, 4 * d, dact, 4 * d, false, bt(w, d, HY_WFC), d, true, dln2, d);
  }
  { HY_PROF(st, "bwd_ln");
  check_cuda(layernorm_bwd(st, M, d, s.hmid, bt(w, d, HY_LN2_G), s.mean2, s.rstd2, dln2, dh, true,
                           btw(gw, d, HY_LN2_G), btw(gw, d, HY_LN2_B), s.ws),
             "ln2 bwd");
  }
  // attention out: hmid = h_in + att Wo^T + bo   (dh now holds dL/dhmid)
  { HY_PROF(st, "bwd_dW_o");
  gemm(st, d, d, M, dh, d, true, s.att, d, true, btw(gw, d, HY_WO), d, nullptr, nullptr, 0, 1.f);
  }
  { HY_PROF(st, "bwd_bias");
  check_cuda(colsum(st, M, d, dh, d, btw(gw, d, HY_BO), true, s.ws), "colsum bo");
  }
  float* datt = s.ln2;  // ln2 dead after dWfc
  { HY_PROF(st, "bwd_datt");
  gemm(st, M, d, d, dh, d, false, bt(w, d, HY_WO), d, true, datt, d);
  }
  // fc (dln2) and act (dact) are dead here: dqkv takes fc[0, 3Md), scores the rest of fc+act
  float* dqkv = s.fc;
  float* work = s.fc + 3L * M * d;
  { HY_PROF(st, "attn_bwd");
  if (gemm_precision_fp32()) {
    check_cuda(attention_bwd_tc(st, m.B, m.T, m.H, s.qkv, datt, dqkv, work, s.act + 4L * M * d - work), "attn bwd");
  } else {
    check_cuda(attention_bwd_fa(st, m.B, m.T, m.H, s.qkv, s.att, datt, s.lse, dqkv, s.attn_ws), "attn bwd");
  }
  }
  { HY_PROF(st, "bwd_dW_qkv");
  gemm(st, 3 * d, d, M, dqkv, 3 * d, true, s.ln1, d, true, btw(gw, d, HY_WQKV), d, nullptr, nullptr, 0, 1.f);
  }
  { HY_PROF(st, "bwd_bias");
  check_cuda(colsum(st, M, 3 * d, dqkv, 3 * d, btw(gw, d, HY_BQKV), true, s.ws), "colsum bqkv");
  }
  float* dln1 = s.hmid;  // hmid dead after ln2 bwd
  { HY_PROF(st, "bwd_dln1");
  gemm(st, M, d, 3 * d, dqkv, 3 * d, false, bt(w, d, HY_WQKV), d, true, dln1, d);
  }
  { HY_PROF(st, "bwd_ln");
  check_cuda(layernorm_bwd(st, M, d, h_in, bt(w, d, HY_LN1_G), s.mean1, s.rstd1, dln1, dh, true,
                           btw(gw, d, HY_LN1_G), btw(gw, d, HY_LN1_B), s.ws),
             "ln1 bwd");
  }
}

// z = ln_f(h); logits chunks -> xent. want_grad: dlogits scaled by 1/M; dz, dwte (if given).
void head_pass(cudaStream_t st, const hy_dims& m, const float* lnf, const float* wte, const float* h,
               const int32_t* targets, Scratch& s, bool want_grad, float* dwte, bool z_ready = false) {
  const int M = s.M, d = m.d, V = m.V;
  if (!z_ready) {
    { HY_PROF(st, "head_lnf");
    check_cuda(layernorm_fwd(st, M, d, h, lnf, lnf + hy_pad32(d), s.z, s.zmean, s.zrstd), "ln_f");
    }
  }
  check_cuda(cudaMemsetAsync(s.loss, 0, sizeof(double), st), "memset loss");
  for (int r0 = 0; r0 < M; r0 += s.logits_rows) {
    const int rows = std::min(s.logits_rows, M - r0);
    { HY_PROF(st, "head_logits");
    gemm(st, rows, V, d, s.z + static_cast<long>(r0) * d, d, false, wte, d, false, s.logits, HY_VOCAB_PAD);
    }
    { HY_PROF(st, "head_xent");
    check_cuda(softmax_xent(st, rows, V, s.logits, HY_VOCAB_PAD, targets + r0, 1.f / M, s.row_loss + r0), "xent");
    }
    if (want_grad && s.dz) {
      { HY_PROF(st, "head_dz");
      gemm(st, rows, d, V, s.logits, HY_VOCAB_PAD, false, wte, d, true, s.dz + static_cast<long>(r0) * d, d);
      }
    }
    if (want_grad && dwte) {
      { HY_PROF(st, "head_dwte");
      gemm(st, V, d, rows, s.logits, HY_VOCAB_PAD, true, s.z + static_cast<long>(r0) * d, d, true, dwte, d, nullptr,
           nullptr, 0, 1.f);
      }
    }
  }
  check_cuda(sum_to_double(st, M, s.row_loss, s.loss, false), "loss sum");
}

}  // namespace

long scratch_floats(const hy_dims& m, int max_blocks, bool bf16) {
  Scratch s;
  carve_scratch(m, max_blocks, nullptr, &s, bf16);
  const long end = bf16 ? reinterpret_cast<long>(s.w16) / static_cast<long>(sizeof(float)) + w16_floats(m)
                        : reinterpret_cast<long>(s.attn_ws) / static_cast<long>(sizeof(float)) +
                              hy_pad32(static_cast<long>(m.B) * m.H * m.T);
  return end;
}

void carve_scratch(const hy_dims& m, int max_blocks, float* base, Scratch* s, bool bf16) {
  const long M = static_cast<long>(m.B) * m.T, d = m.d;
  float* p = base;
  auto take = [&](long n) {
    float* r = p;
    p += hy_pad32(n);
    return r;
  };
  s->M = static_cast<int>(M);
  s->d = m.d;
  s->stash_slots = max_blocks + 1;
  s->stash = take(M * d * s->stash_slots);
  s->ln1 = take(M * d);
  s->mean1 = take(M);
  s->rstd1 = take(M);
  s->qkv = take(3 * M * d);
  s->att = take(M * d);
  s->lse = take(static_cast<long>(m.B) * m.H * m.T);
  s->hmid = take(M * d);
  s->ln2 = take(M * d);
  s->mean2 = take(M);
  s->rstd2 = take(M);
  // fc, act and tmp_h are adjacent: the head's logits chunk aliases them. tmp_h is free during
  // the head's chunk loop (a block output held there is read by ln_f before it; the backward's
  // dh is written after it). Chunks are balanced and rounded up to 256 rows (a CTA-pair tile row)
  // when that still fits: C2's 4096 tokens go in 8 chunks of 512 rows instead of 8 x 500 + 96.
  s->fc = take(4 * M * d);
  s->act = take(4 * M * d);
  s->tmp_h = take(M * d);
  const long span = (s->tmp_h + M * d) - s->fc;
  const long cap = std::min<long>(M, span / HY_VOCAB_PAD);
  const bool alias_logits = cap >= std::min<long>(M, 16);
  if (alias_logits) {
    const long chunks = (M + cap - 1) / cap;
    long rows = (M + chunks - 1) / chunks;
    const long r256 = (rows + 255) / 256 * 256;
    if (r256 <= cap) rows = r256;
    s->logits = s->fc;
    s->logits_rows = static_cast<int>(rows);
  } else {
    s->logits_rows = static_cast<int>(std::min<long>(M, 16));
    s->logits = take(static_cast<long>(s->logits_rows) * HY_VOCAB_PAD);
  }
  s->ws = take(512L * 4 * d);  // >= colsum_blocks(M) * max(4d, 2d)
  // the head's ln_f output and its gradient alias the QKV buffer (3 M d): the head pass runs
  // when no block intermediates are live (before the blocks' recompute in a backward, after
  // the last block in a forward); B(0)'s deferred tied-wte pass restores z there first
  s->z = s->qkv;
  s->zmean = take(M);
  s->zrstd = take(M);
  s->dz = s->qkv + M * d;
  s->row_loss = take(M);
  s->loss = reinterpret_cast<double*>(take(2));
  s->attn_ws = take(static_cast<long>(m.B) * m.H * m.T);
  s->w16 = bf16 ? reinterpret_cast<__nv_bfloat16*>(take(w16_floats(m))) : nullptr;
}

void run_forward(cudaStream_t st, const hy_dims& m, const ShardGeom& g, const float* slot, const TaskIO& io,
                 Scratch& s) {
  const long n = static_cast<long>(s.M) * m.d;
  const int b0 = std::max(g.l0, 1);
  const int b1 = std::min(g.l1, m.L + 1);
  const bool write_out = !g.has_head && io.act_out != nullptr;
  if (io.keep_stash && write_out && g.n_blocks > 0) {
    // the backward's stash pass, done here: stash[i] = input of block b0+i, so this shard's
    // backward can skip recomputing the forward if the stash survives until then
    float* const stash = io.stash ? io.stash : s.stash;
    if (g.has_embed) {
      check_cuda(embed_fwd(st, s.M, m.T, m.d, io.tokens, slot, slot + hy_pad32(static_cast<long>(m.V) * m.d),
                           stash),
                 "embed");
    } else {
      check_cuda(cudaMemcpyAsync(stash, io.act_in, n * sizeof(float), cudaMemcpyDeviceToDevice, st), "stash in");
    }
    for (int i = 0; i < g.n_blocks; ++i) {
      float* out = i == g.n_blocks - 1 ? io.act_out : stash + (i + 1) * n;
      block_forward(st, m, slot + lo(m, b0 + i, g.l0), stash + i * n, out, s, false);
    }
    return;
  }
  const float* cur = io.act_in;
  if (g.has_embed) {
    float* dst = (write_out && g.n_blocks == 0) ? io.act_out : s.tmp_h;
    check_cuda(embed_fwd(st, s.M, m.T, m.d, io.tokens, slot, slot + hy_pad32(static_cast<long>(m.V) * m.d), dst),
               "embed");
    cur = dst;
  }
  for (int l = b0; l < b1; ++l) {
    float* dst = (cur == s.tmp_h) ? s.stash : s.tmp_h;
    if (write_out && l == b1 - 1) dst = io.act_out;
    block_forward(st, m, slot + lo(m, l, g.l0), cur, dst, s, false);
    cur = dst;
  }
  if (g.has_head) {
    const float* wte = g.has_embed ? slot : (io.wte ? io.wte : slot + g.wte_offset);
    head_pass(st, m, slot + lo(m, m.L + 1, g.l0), wte, cur, io.targets, s, false, nullptr);
  } else if (write_out && cur != io.act_out) {
    check_cuda(cudaMemcpyAsync(io.act_out, cur, n * sizeof(float), cudaMemcpyDeviceToDevice, st), "act copy");
  }
}

void run_backward(cudaStream_t st, const hy_dims& m, const ShardGeom& g, const float* slot, GradSink& sink,
                  const TaskIO& io, Scratch& s) {
  const long n = static_cast<long>(s.M) * m.d;
  const int b0 = std::max(g.l0, 1);
  const int nb = g.n_blocks;
  // 0) embedding shard without the head: the deferred tied-wte gradient first (logits
  //    recomputed from the head's saved z), so the dense part of dwte is final before the
  //    blocks and its rows can go to the optimizer while they back-propagate.
  float* gembed = nullptr;
  if (g.has_embed) gembed = sink.acquire(0);  // wte/wpe grads: head (k == 1) + embedding
  if (g.has_embed && !g.has_head && io.z_in) {
    if (io.z_in != s.z) {
      check_cuda(cudaMemcpyAsync(s.z, io.z_in, n * sizeof(float), cudaMemcpyDeviceToDevice, st), "z in");
    }
    float* saved_dz = s.dz;
    s.dz = nullptr;  // only dwte is wanted
    head_pass(st, m, nullptr, slot, nullptr, io.targets, s, true, gembed, /*z_ready=*/true);
    s.dz = saved_dz;
    sink.release_dense(0);
  }
  // 1) recompute: stash[i] = input of block b0+i; stash[nb] = shard output (head shards) —
  //    unless this shard's forward left its block inputs there (io.stash_ready).
  // The last block's intermediates survive in scratch unless the head pass (whose logits
  // alias the MLP buffers) runs in between: then its recompute can be skipped.
  bool last_block_live = nb > 0 && !g.has_head && !io.stash_ready;
  // a head-only shard reads its input in place (the stash keeps another shard's block inputs)
  const bool head_only = nb == 0 && !g.has_embed;
  float* const stash = io.stash ? io.stash : s.stash;
  if (!io.stash_ready && !head_only) {
    if (g.has_embed) {
      check_cuda(embed_fwd(st, s.M, m.T, m.d, io.tokens, slot, slot + hy_pad32(static_cast<long>(m.V) * m.d), stash),
                 "embed");
    } else {
      check_cuda(cudaMemcpyAsync(stash, io.act_in, n * sizeof(float), cudaMemcpyDeviceToDevice, st), "stash in");
    }
    for (int i = 0; i < nb; ++i) {
      // the last block's output is only needed as the head's input
      float* out = (i == nb - 1 && !g.has_head) ? nullptr : stash + (i + 1) * n;
      block_forward(st, m, slot + lo(m, b0 + i, g.l0), stash + i * n, out, s, last_block_live && i == nb - 1);
    }
  }
  // 2) gradient wrt the shard output
  float* dh = s.tmp_h;
  if (g.has_head) {
    const float* lnf = slot + lo(m, m.L + 1, g.l0);
    float* glnf = sink.acquire(m.L + 1);
    const float* wte = g.has_embed ? slot : (io.wte ? io.wte : slot + g.wte_offset);
    float* dwte = g.has_embed ? gembed : nullptr;  // otherwise deferred to shard 0 via z
    const float* hfin = head_only ? io.act_in : stash + nb * n;
    head_pass(st, m, lnf, wte, hfin, io.targets, s, true, dwte);
    if (dwte) sink.release_dense(0);
    if (io.z_out) {  // z aliases the block scratch: saved before the blocks recompute
      check_cuda(cudaMemcpyAsync(io.z_out, s.z, n * sizeof(float), cudaMemcpyDeviceToDevice, st), "z save");
    }
    check_cuda(layernorm_bwd(st, s.M, m.d, hfin, lnf, s.zmean, s.zrstd, s.dz, dh, false, glnf, glnf + hy_pad32(m.d),
                             s.ws),
               "ln_f bwd");
    sink.release(m.L + 1);
  } else {
    check_cuda(cudaMemcpyAsync(dh, io.grad_in, n * sizeof(float), cudaMemcpyDeviceToDevice, st), "grad in");
  }
  // 3) blocks, last to first: recompute intermediates, back-propagate; each block's
  //    gradients are handed to the optimizer as soon as they are final.
  for (int i = nb - 1; i >= 0; --i) {
    const int layer = b0 + i;
    const float* w = slot + lo(m, layer, g.l0);
    if (!(last_block_live && i == nb - 1)) {
      block_forward(st, m, w, stash + i * n, nullptr, s, true);  // intermediates only: no MLP projection
    } else if (s.w16) {
      block_w16(st, m, w, s);
    }
    float* gw = sink.acquire(layer);
    block_backward(st, m, w, gw, stash + i * n, dh, s);
    sink.release(layer);
  }
  // 4) embedding: token rows of wte and wpe
  if (g.has_embed) {
    check_cuda(embed_bwd(st, s.M, m.T, m.d, io.tokens, dh, gembed, gembed + hy_pad32(static_cast<long>(m.V) * m.d),
                         nullptr),
               "embed bwd");
    sink.release(0);
  } else if (io.grad_out) {
    check_cuda(cudaMemcpyAsync(io.grad_out, dh, n * sizeof(float), cudaMemcpyDeviceToDevice, st), "grad out");
  }
}

}  // namespace hy
