// C-ABI (include/hydra.h): status codes + thread-local error text, JSON planning entry,
// and the per-kernel entry points. Exceptions never cross this boundary.
#include "hydra.h"

#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>

#include "../kernels/gemm.cuh"
#include "../kernels/launch_count.cuh"
#include "../kernels/ops.cuh"
#include "../exec/host_opt.hpp"
#include "capi_internal.hpp"
#include "spillsim/errors.hpp"

namespace hy {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int status_from_current_exception() {
  try {
    throw;
  } catch (const spillsim::ConfigError& e) {
    return set_error(HY_E_CONFIG, e.what());
  } catch (const spillsim::CapacityExhausted& e) {
    return set_error(HY_E_CAPACITY, e.what());
  } catch (const spillsim::BufferOverflow& e) {
    return set_error(HY_E_BUFFER_OVERFLOW, e.what());
  } catch (const spillsim::InfeasibleOOM& e) {
    return set_error(HY_E_INFEASIBLE, e.what());
  } catch (const spillsim::SingleLayerTooLarge& e) {
    return set_error(HY_E_INFEASIBLE, e.what());
  } catch (const spillsim::HostOOM& e) {
    return set_error(HY_E_INFEASIBLE, e.what());
  } catch (const spillsim::DeadlockError& e) {
    return set_error(HY_E_DEADLOCK, e.what());
  } catch (const spillsim::ByteOverflow& e) {
    return set_error(HY_E_BYTE_OVERFLOW, e.what());
  } catch (const spillsim::DeviceError& e) {
    return set_error(HY_E_CUDA, e.what());
  } catch (const spillsim::InvalidArgument& e) {
    return set_error(HY_E_INVALID, e.what());
  } catch (const std::exception& e) {
    return set_error(HY_E_INTERNAL, e.what());
  } catch (...) {
    return set_error(HY_E_INTERNAL, "unknown exception");
  }
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return HY_OK;
  return set_error(HY_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int write_out(const std::string& s, char* out, size_t out_len, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (!out || out_len < s.size() + 1) return set_error(HY_E_BUFFER_SMALL, "output buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
  return HY_OK;
}

}  // namespace hy

using hy::cuda_status;

extern "C" {

const char* hy_last_error(void) { return hy::g_last_error.c_str(); }
const char* hy_version(void) { return "hydra-b200 0.1 (sm_100a)"; }

int hy_plan_json(const char* request_json, char* out, size_t out_len, size_t* needed) {
  try {
    return hy::write_out(hy::plan_json(request_json), out, out_len, needed);
  } catch (...) {
    return hy::status_from_current_exception();
  }
}

int hy_execute_json(const char* request_json, char* out, size_t out_len, size_t* needed) {
  try {
    return hy::write_out(hy::execute_json(request_json), out, out_len, needed);
  } catch (...) {
    return hy::status_from_current_exception();
  }
}

int hy_executor_create(const char* request_json, void** handle) {
  try {
    *handle = hy::session_create(request_json);
    return HY_OK;
  } catch (...) {
    *handle = nullptr;
    return hy::status_from_current_exception();
  }
}

int hy_executor_run(void* handle, int passes, int timed, int with_trace, char* out, size_t out_len,
                    size_t* needed) {
  try {
    if (!handle) return hy::set_error(HY_E_INVALID, "null executor handle");
    return hy::write_out(hy::session_run(handle, passes, timed, with_trace != 0), out, out_len, needed);
  } catch (...) {
    return hy::status_from_current_exception();
  }
}

int hy_executor_dump_params(void* handle, const char* dir) {
  try {
    hy::session_dump_params(handle, dir);
    return HY_OK;
  } catch (...) {
    return hy::status_from_current_exception();
  }
}

int hy_executor_read_params(void* handle, int job, float* dst, size_t n_floats, size_t* total_floats) {
  try {
    if (!handle) return hy::set_error(HY_E_INVALID, "null executor handle");
    const size_t n = hy::session_read_params(handle, job, dst, n_floats);
    if (total_floats) *total_floats = n;
    return HY_OK;
  } catch (...) {
    return hy::status_from_current_exception();
  }
}

void hy_executor_destroy(void* handle) {
  try {
    hy::session_destroy(handle);
  } catch (...) {
  }
}

long hy_kernel_launches(void) { return hy::g_kernel_launches.load(); }

// Diagnostics: host microseconds per launch of `kind` (0 = GEMM 128x128x64, 1 = LayerNorm
// 64x64) issued back to back from C++ on `stream`, n times. Buffers are caller-provided.
double hy_host_launch_us(void* stream, int kind, int n, float* a, float* b, float* c) {
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) {
    if (kind == 0) {
      hy::GemmEpilogue e;
      e.C = c;
      e.ldc = 128;
      hy::gemm_tf32(static_cast<cudaStream_t>(stream), 128, 128, 64, a, 64, false, b, 64, false, e);
    } else {
      hy::layernorm_fwd(static_cast<cudaStream_t>(stream), 64, 64, a, b, b + 64, c, c + 4096, c + 8192);
    }
  }
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int hy_gemm_config(int precision_fp32, float* splitk_ws, long splitk_floats) {
  hy::gemm_set_precision_fp32(precision_fp32 != 0);
  hy::gemm_set_splitk_workspace(splitk_ws, splitk_floats);
  return HY_OK;
}

int hy_gemm(void* stream, int M, int N, int K, const float* A, long lda, int a_mn, const float* B, long ldb, int b_mn,
            float* C, long ldc, const float* bias, const float* R, long ldr, float beta, int mode, float* Hout,
            const float* Hin, long ldh) {
  hy::GemmEpilogue e;
  e.C = C;
  e.ldc = ldc;
  e.bias = bias;
  e.R = R;
  e.ldr = ldr;
  e.beta = beta;
  e.mode = mode;
  e.Hout = Hout;
  e.ldho = ldh;
  e.Hin = Hin;
  e.ldhi = ldh;
  return cuda_status(hy::gemm_tf32(static_cast<cudaStream_t>(stream), M, N, K, A, lda, a_mn != 0, B, ldb, b_mn != 0, e),
                     "hy_gemm");
}

int hy_gemm_bf16(void* stream, int M, int N, int K, const uint16_t* A, long lda, int a_mn, const uint16_t* B,
                 long ldb, int b_mn, void* C, long ldc, int c_bf16, const float* bias, const float* R, long ldr,
                 float beta, int mode, float* Hout, const float* Hin, long ldh) {
  hy::GemmEpilogue e;
  e.C = static_cast<float*>(C);
  e.ldc = ldc;
  e.c16 = c_bf16 != 0;
  e.bias = bias;
  e.R = R;
  e.ldr = ldr;
  e.beta = beta;
  e.mode = mode;
  e.Hout = Hout;
  e.ldho = ldh;
  e.Hin = Hin;
  e.ldhi = ldh;
  return cuda_status(hy::gemm_bf16(static_cast<cudaStream_t>(stream), M, N, K,
                                   reinterpret_cast<const __nv_bfloat16*>(A), lda, a_mn != 0,
                                   reinterpret_cast<const __nv_bfloat16*>(B), ldb, b_mn != 0, e),
                     "hy_gemm_bf16");
}

int hy_to_bf16(void* stream, long n, const float* x, uint16_t* y) {
  return cuda_status(hy::to_bf16(static_cast<cudaStream_t>(stream), n, x, reinterpret_cast<__nv_bfloat16*>(y)),
                     "hy_to_bf16");
}

int hy_layernorm_fwd(void* stream, int rows, int d, const float* x, const float* g, const float* b, float* y,
                     float* mean, float* rstd) {
  return cuda_status(hy::layernorm_fwd(static_cast<cudaStream_t>(stream), rows, d, x, g, b, y, mean, rstd),
                     "hy_layernorm_fwd");
}

int hy_layernorm_bwd(void* stream, int rows, int d, const float* x, const float* g, const float* mean,
                     const float* rstd, const float* dy, float* dx, int accumulate_dx, float* dg, float* db,
                     float* ws) {
  return cuda_status(hy::layernorm_bwd(static_cast<cudaStream_t>(stream), rows, d, x, g, mean, rstd, dy, dx,
                                       accumulate_dx != 0, dg, db, ws),
                     "hy_layernorm_bwd");
}

int hy_attention_fwd(void* stream, int B, int T, int H, int hd, const float* qkv, float* out, float* work,
                     long work_floats) {
  if (hd != 64) return hy::set_error(HY_E_INVALID, "attention: head dim must be 64");
  return cuda_status(hy::attention_fwd_tc(static_cast<cudaStream_t>(stream), B, T, H, qkv, out, work, work_floats),
                     "hy_attention_fwd");
}

int hy_attention_bwd(void* stream, int B, int T, int H, int hd, const float* qkv, const float* dout, float* dqkv,
                     float* work, long work_floats) {
  if (hd != 64) return hy::set_error(HY_E_INVALID, "attention: head dim must be 64");
  return cuda_status(
      hy::attention_bwd_tc(static_cast<cudaStream_t>(stream), B, T, H, qkv, dout, dqkv, work, work_floats),
      "hy_attention_bwd");
}

int hy_flash_attention_fwd(void* stream, int B, int T, int H, const float* qkv, float* out, float* lse2) {
  return cuda_status(hy::attention_fwd_fa(static_cast<cudaStream_t>(stream), B, T, H, qkv, out, lse2),
                     "hy_flash_attention_fwd");
}

int hy_flash_attention_bwd(void* stream, int B, int T, int H, const float* qkv, const float* out, const float* dout,
                           const float* lse2, float* dqkv, float* Di) {
  return cuda_status(hy::attention_bwd_fa(static_cast<cudaStream_t>(stream), B, T, H, qkv, out, dout, lse2, dqkv, Di),
                     "hy_flash_attention_bwd");
}

int hy_embed_fwd(void* stream, int rows, int T, int d, const int32_t* tokens, const float* wte, const float* wpe,
                 float* h) {
  return cuda_status(hy::embed_fwd(static_cast<cudaStream_t>(stream), rows, T, d, tokens, wte, wpe, h), "hy_embed_fwd");
}

int hy_embed_bwd(void* stream, int rows, int T, int d, int /*V*/, const int32_t* tokens, const float* dh, float* dwte,
                 float* dwpe) {
  return cuda_status(hy::embed_bwd(static_cast<cudaStream_t>(stream), rows, T, d, tokens, dh, dwte, dwpe, nullptr),
                     "hy_embed_bwd");
}

int hy_softmax_xent(void* stream, int rows, int V, float* logits, long ldl, const int32_t* targets,
                    float inv_total_rows, float* row_loss) {
  return cuda_status(
      hy::softmax_xent(static_cast<cudaStream_t>(stream), rows, V, logits, ldl, targets, inv_total_rows, row_loss),
      "hy_softmax_xent");
}

int hy_bias_grad(void* stream, int M, int N, const float* dy, long ldy, float* db, int accumulate, float* ws) {
  return cuda_status(hy::colsum(static_cast<cudaStream_t>(stream), M, N, dy, ldy, db, accumulate != 0, ws),
                     "hy_bias_grad");
}

int hy_adam(void* stream, long n, float* p, const float* g, float* m, float* v, float lr, float beta1, float beta2,
            float eps, float weight_decay, int step) {
  hy::AdamHyper h{lr, beta1, beta2, eps, weight_decay, 0.f, 0.f};
  h.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta1), step));
  h.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta2), step));
  return cuda_status(hy::adam_update(static_cast<cudaStream_t>(stream), n, p, g, m, v, h), "hy_adam");
}

int hy_adam_host_state(void* stream, long n, float* p, const float* g, void* m_host, void* v_host, float* p_host,
                       float lr, float beta1, float beta2, float eps, float weight_decay, int step, int bf16_state,
                       int grid) {
  hy::AdamHyper h{lr, beta1, beta2, eps, weight_decay, 0.f, 0.f};
  h.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta1), step));
  h.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta2), step));
  return cuda_status(hy::adam_zc(static_cast<cudaStream_t>(stream), n, p, g, m_host, v_host, p_host, bf16_state != 0,
                                 h, nullptr, 0, 0, grid),
                     "hy_adam_host_state");
}

int hy_host_adam(long n, float* p, const float* g, void* m, void* v, float lr, float beta1, float beta2, float eps,
                 float weight_decay, int step, int bf16_state, int threads) {
  if (n < 0 || (n > 0 && (!p || !g || !m || !v)) || step < 1) {
    return hy::set_error(HY_E_INVALID, "hy_host_adam: bad arguments");
  }
  hy::HostAdamWork w;
  w.p = p;
  w.g = g;
  w.m = m;
  w.v = v;
  w.n = n;
  w.lr = lr;
  w.beta1 = beta1;
  w.beta2 = beta2;
  w.eps = eps;
  w.weight_decay = weight_decay;
  w.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta1), step));
  w.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(beta2), step));
  w.bf16 = bf16_state;
  w.threads = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  hy::host_adam(w);
  return HY_OK;
}

}  // extern "C"
