// Host-side AdamW — the reference's optimizer placement: "optimizer state is excluded from
// the GPU pilot footprint and charged to host DRAM" and "optimizer-update time is folded into
// the Backward task's grad_offload (host-side updates are off the critical path)"
// (SPEC.md:88). A layer placed host-side costs the link only its gradient
// (GradOffload, D2H) and its next ParamLoad; the GPU-side placement streams the moments both
// ways instead. The executor mixes the two per layer (ExecOptions::host_opt_fraction).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace hy {

struct HostAdamWork {
  float* p = nullptr;        // pinned fp32 master params of the layer
  const float* g = nullptr;  // pinned gradient (GradOffload destination)
  void* m = nullptr;         // moments: fp32, or bf16 bit patterns when bf16 != 0
  void* v = nullptr;
  long n = 0;
  float lr = 0, beta1 = 0, beta2 = 0, eps = 0, weight_decay = 0, bc1 = 1, bc2 = 1;
  int bf16 = 0;
  int threads = 1;
};

// Same arithmetic, in the same order, as adam_kernel / adam_bf16_kernel (kernels/ops.cu)
// and the CPU oracle (oracle/gpt_oracle.c oracle_adam_state). Runs on the calling thread's
// OpenMP team of `w.threads`.
void host_adam(const HostAdamWork& w);

// Enqueue host_adam on `stream` (cudaLaunchHostFunc): it runs once all prior work of the
// stream (the gradient's D2H) is done, and later work of the stream waits for it.
cudaError_t host_adam_async(cudaStream_t stream, const HostAdamWork& w);

}  // namespace hy
