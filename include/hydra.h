/* hydra.h — C-ABI of the B200 shard-execution library (paper_2110_08633_b200/libhydra.so).
 *
 * The reference (spillsim, /root/reference/proj) is a C++ library with no FFI; its drop-in
 * boundary is the C++ API re-declared under include/spillsim/ (*.hpp). This header is the
 * flat C boundary beneath it, for bindings (ctypes / cgo / JNI) and for kernel-level parity
 * tests. Plain pointers and sizes only; no torch / C++ types cross it.
 *
 * Conventions
 *  - Every function returns int status: HY_OK (0) or a negative HY_E* code; the message
 *    for the calling thread is available from hy_last_error(). Codes map 1:1 onto the
 *    reference exception classes (proj/core/include/spillsim/errors.hpp:23-114).
 *  - Device pointers are raw CUDA device addresses; `stream` is a cudaStream_t (NULL =
 *    legacy default stream). The caller owns every buffer; the library never frees caller
 *    memory. JSON results are written into caller buffers (hy_*_json take out/out_len and
 *    return HY_E_BUFFER_SMALL with *needed set when the buffer is too small).
 *  - Thread-compatible: distinct executors / streams may be driven from distinct threads.
 */
#ifndef HYDRA_H_
#define HYDRA_H_

#include <stddef.h>
#include <stdint.h>

#include "hydra_gpt.h"

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HY_OK = 0,
  HY_E_INVALID = -1,        /* spillsim::InvalidArgument */
  HY_E_CONFIG = -2,         /* spillsim::ConfigError */
  HY_E_CAPACITY = -3,       /* spillsim::CapacityExhausted */
  HY_E_BUFFER_OVERFLOW = -4,/* spillsim::BufferOverflow */
  HY_E_INFEASIBLE = -5,     /* InfeasibleOOM / SingleLayerTooLarge / HostOOM */
  HY_E_DEADLOCK = -6,       /* spillsim::DeadlockError */
  HY_E_BYTE_OVERFLOW = -7,  /* spillsim::ByteOverflow */
  HY_E_CUDA = -8,           /* CUDA runtime / driver failure (spillsim::DeviceError) */
  HY_E_BUFFER_SMALL = -9,   /* output buffer too small; *needed holds the size */
  HY_E_INTERNAL = -10
};

const char* hy_last_error(void);
const char* hy_version(void);

/* ---------------------------------------------------------------------------------
 * Planning (host only). Replaces the reference entry points
 *   parse_workload_config   config.hpp:70      materialize_jobs  config.hpp:79
 *   build_strategy          strategies.hpp:90  run_simulation    sim.hpp:131
 *   summarize               metrics.hpp:53     to_chrome_trace_json trace_export.hpp:28
 * request_json: {"config": {...workload v1...}, "strategy": "sharp", "gpus": G,
 *                "double_buffering": bool?, "trace": bool?}
 * result: {"partitions":[...], "tasks":[...], "dispatch":[[task,device,prefetch],...],
 *          "dispatch_hash":"...", "makespan_s":x, "report":{...}, "chrome_trace":"..."?}
 * --------------------------------------------------------------------------------- */
int hy_plan_json(const char* request_json, char* out, size_t out_len, size_t* needed);

/* ---------------------------------------------------------------------------------
 * Execution (real B200 run of a workload; replaces the simulated Engine, sim.cpp:146-587).
 * request_json: {"config": {...}, "strategy": "sharp", "gpus": G, "device_ids": [..]?,
 *                "passes": P?, "warmup_passes": W?, "mode": "plan"}
 * result: measured trace summary, per-step losses, timings.
 * --------------------------------------------------------------------------------- */
int hy_execute_json(const char* request_json, char* out, size_t out_len, size_t* needed);

/* Stateful form (what bench.py and long runs use): setup once — pinned host state,
 * capped HBM arenas, streams, GPT-2 init — then replay the plan pass by pass.
 * request_json as for hy_execute_json ("passes" + "warmup_passes" bound the total). */
int hy_executor_create(const char* request_json, void** handle);
/* Replays the plan `passes` times; timed passes are measured with CUDA events and
 * accumulate into the result JSON (pass_seconds, losses, byte counters, report).
 * timed: 0 untimed, 1 timed, 2 timed + interval log (result "links": copy-only link time
 * per direction, compute-op time and the transfer-overlap fraction per GPU; adds two event
 * records per op / copy, so throughput is measured on passes run with timed = 1). */
int hy_executor_run(void* handle, int passes, int timed, int with_trace, char* out, size_t out_len,
                    size_t* needed);
int hy_executor_dump_params(void* handle, const char* dir);
/* Job `job`'s host parameter vector (layout include/hydra_gpt.h; final after a pass) into
 * dst (n_floats >= its length) or, with dst == NULL, just its length in *total_floats. */
int hy_executor_read_params(void* handle, int job, float* dst, size_t n_floats, size_t* total_floats);
void hy_executor_destroy(void* handle);
/* Diagnostics: host microseconds per back-to-back launch (kind 0 GEMM, 1 LayerNorm). */
double hy_host_launch_us(void* stream, int kind, int n, float* a, float* b, float* c);
/* Kernel launches issued by this library since load (for the bench's gpu_launches). */
long hy_kernel_launches(void);

/* ---------------------------------------------------------------------------------
 * Kernel entry points (fp32 tensors in HBM, row-major). Used by the executor and by the
 * GPU parity tests; each maps to one hand-written sm_100a kernel (csrc/kernels/).
 * --------------------------------------------------------------------------------- */

/* GEMM configuration of the calling host thread: precision_fp32 = 1 selects the 3xTF32
 * split ("fp32", ~fp32 accuracy), 0 plain TF32; splitk_ws (device, may be NULL) lets
 * low-occupancy GEMMs split K. */
int hy_gemm_config(int precision_fp32, float* splitk_ws, long splitk_floats);

/* C[M,N] = beta*C + op(A) op(B)^T (+bias[N]) (+R[M,N]) with tcgen05 kind::tf32.
 * a_mn=0: A is [M][lda] (K contiguous); a_mn=1: A is [K][lda] (M contiguous). Same for B
 * with N. mode 0 store, 1 GELU (C = gelu(acc + bias), Hout = gelu'(acc + bias)), 2 GELU-backward
 * (C = acc * Hin, Hin = the gelu' mode 1 stored). */
int hy_gemm(void* stream, int M, int N, int K, const float* A, long lda, int a_mn, const float* B, long ldb,
            int b_mn, float* C, long ldc, const float* bias, const float* R, long ldr, float beta, int mode,
            float* Hout, const float* Hin, long ldh);

/* Same with bf16 operands (bit patterns, uint16) on tcgen05 kind::f16, fp32 accumulate; leading
 * dims multiples of 8. c_bf16 = 1 stores C as bf16 (beta must be 0). The "bf16" precision's
 * block GEMMs. */
int hy_gemm_bf16(void* stream, int M, int N, int K, const uint16_t* A, long lda, int a_mn, const uint16_t* B,
                 long ldb, int b_mn, void* C, long ldc, int c_bf16, const float* bias, const float* R, long ldr,
                 float beta, int mode, float* Hout, const float* Hin, long ldh);
/* y = bf16(x) (round to nearest even), n % 8 == 0. */
int hy_to_bf16(void* stream, long n, const float* x, uint16_t* y);

int hy_layernorm_fwd(void* stream, int rows, int d, const float* x, const float* g, const float* b, float* y,
                     float* mean, float* rstd);
int hy_layernorm_bwd(void* stream, int rows, int d, const float* x, const float* g, const float* mean,
                     const float* rstd, const float* dy, float* dx, int accumulate_dx, float* dg, float* db,
                     float* ws);
/* Causal attention on tcgen05 (head dim 64). qkv [B*T, 3*H*64]; out [B*T, H*64]. `work`
 * holds score matrices: >= T*T floats (fwd) / 2*T*T (bwd); (batch, head) chunks sized to it. */
int hy_attention_fwd(void* stream, int B, int T, int H, int hd, const float* qkv, float* out, float* work,
                     long work_floats);
int hy_attention_bwd(void* stream, int B, int T, int H, int hd, const float* qkv, const float* dout, float* dqkv,
                     float* work, long work_floats);
/* Fused (flash-style) causal attention on tcgen05, kind::tf32, head dim 64 — the TF32 path of
 * the shard runner. lse2 [B*H*T]: per-query log2-domain logsumexp of S/8 written by the
 * forward, read by the backward; Di [B*H*T] backward scratch. dqkv overwritten. */
int hy_flash_attention_fwd(void* stream, int B, int T, int H, const float* qkv, float* out, float* lse2);
int hy_flash_attention_bwd(void* stream, int B, int T, int H, const float* qkv, const float* out, const float* dout,
                           const float* lse2, float* dqkv, float* Di);
int hy_embed_fwd(void* stream, int rows, int T, int d, const int32_t* tokens, const float* wte, const float* wpe,
                 float* h);
int hy_embed_bwd(void* stream, int rows, int T, int d, int V, const int32_t* tokens, const float* dh, float* dwte,
                 float* dwpe);
/* Softmax cross-entropy over a [rows, V] logits chunk (row stride ldl); overwrites the
 * chunk with dlogits * grad_scale and writes row_loss[r] = logsumexp - logit[target]. */
int hy_softmax_xent(void* stream, int rows, int V, float* logits, long ldl, const int32_t* targets,
                    float grad_scale, float* row_loss);
int hy_bias_grad(void* stream, int M, int N, const float* dy, long ldy, float* db, int accumulate, float* ws);
int hy_adam(void* stream, long n, float* p, const float* g, float* m, float* v, float lr, float beta1, float beta2,
            float eps, float weight_decay, int step);
/* AdamW with the optimizer state in pinned host memory (zero-copy, the executor's GPU-side
 * optimizer): p (HBM) updated in place and mirrored to p_host; m, v (fp32, or bf16 bit
 * patterns when bf16_state) read and written over the host link. grid = CTAs (0: default). */
int hy_adam_host_state(void* stream, long n, float* p, const float* g, void* m_host, void* v_host, float* p_host,
                       float lr, float beta1, float beta2, float eps, float weight_decay, int step, int bf16_state,
                       int grid);
/* Host-side AdamW on host memory (the reference's optimizer placement; the
 * executor's host_opt_fraction path): same update as hy_adam, on `threads` host threads
 * (0: all cores). bf16_state != 0: m, v are bf16 bit patterns (uint16), rounded RNE. */
int hy_host_adam(long n, float* p, const float* g, void* m, void* v, float lr, float beta1, float beta2, float eps,
                 float weight_decay, int step, int bf16_state, int threads);

/* ---------------------------------------------------------------------------------
 * Device level (SURVEY §8b minimum exports): what a host that runs its own engine loop needs
 * — the reference's Engine::dispatch / try_compute / on_compute_done (sim.cpp:347-474) with
 * real copies and kernels. The executor above is the packaged engine over the same pieces.
 *   hy_open: a device context with an HBM arena capped at hbm_budget (DeviceSpec::mem_bytes,
 *   model.hpp:62) — hy_arena_alloc fails with HY_E_CAPACITY beyond it — and three lanes:
 *   DOWN (H2D: ParamLoad / ActPromote), UP (D2H: ActDemote / GradOffload), COMPUTE.
 * --------------------------------------------------------------------------------- */
typedef struct hy_dev hy_dev;
enum { HY_LANE_DOWN = 0, HY_LANE_UP = 1, HY_LANE_COMPUTE = 2 };

int hy_open(int device, size_t hbm_budget, hy_dev** dev);
void hy_close(hy_dev* dev);
int hy_lane_stream(hy_dev* dev, int lane, void** stream); /* cudaStream_t for the kernel entry points */
int hy_arena_alloc(hy_dev* dev, size_t bytes, void** ptr); /* 1 KB aligned bump allocation */
int hy_arena_reset(hy_dev* dev);
int hy_arena_peak(hy_dev* dev, size_t* bytes);
int hy_pinned_alloc(size_t bytes, void** ptr);             /* portable + mapped pinned host memory */
int hy_pinned_free(void* ptr);
int hy_copy_h2d(hy_dev* dev, void* dst, const void* src, size_t bytes);            /* DOWN lane */
int hy_copy_d2h(hy_dev* dev, void* dst, const void* src, size_t bytes);            /* UP lane */
int hy_copy_p2p(hy_dev* dev, void* dst, int src_device, const void* src, size_t bytes); /* DOWN, NVLink */
int hy_event_record(hy_dev* dev, int lane, void** event);   /* creates and records a timing event */
int hy_lane_wait(hy_dev* dev, int lane, void* event);
int hy_event_query(void* event, int* done);
int hy_event_elapsed(void* start, void* end, float* ms);
int hy_event_destroy(void* event);
int hy_lane_sync(hy_dev* dev, int lane);

/* One ShardTask's compute (model.cpp:165-216 layers l0..l1-1 of the GPT in hydra_gpt.h) on the
 * COMPUTE lane. params: the shard's layers, contiguous in the hydra_gpt.h layout. wte: the tied
 * embedding when the shard has the head but not layer 0. Forward: act_in (l0 > 0) -> act_out
 * (no head) or the loss. Backward (recompute + backward, strategies.cpp:743-782): grads (same
 * layout as params, zeroed by the caller) +=, grad_in (no head) -> grad_out (l0 > 0); a head
 * shard without the embedding leaves ln_f's output in z_out for the embedding shard's deferred
 * tied-wte gradient, which that shard's backward takes as z_in. loss (host, nullable): mean
 * token cross-entropy when the shard has the head. scratch: >= hy_shard_scratch_bytes. */
typedef struct {
  hy_dims dims;
  int l0, l1;
} hy_shard_desc;

typedef struct {
  const float* params;
  const float* wte;
  const int32_t* tokens;
  const int32_t* targets;
  const float* act_in;
  float* act_out;
  const float* grad_in;
  float* grad_out;
  const float* z_in;
  float* z_out;
  float* grads;
  void* scratch;
  size_t scratch_bytes;
} hy_shard_bufs;

int hy_shard_scratch_bytes(const hy_dims* dims, int max_blocks, size_t* bytes);
int hy_shard_forward(hy_dev* dev, const hy_shard_desc* shard, const hy_shard_bufs* bufs, double* loss);
int hy_shard_backward(hy_dev* dev, const hy_shard_desc* shard, const hy_shard_bufs* bufs, double* loss);

#ifdef __cplusplus
}
#endif
#endif /* HYDRA_H_ */
