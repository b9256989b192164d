// Programmatic dependent launch for the kernels of the executor's compute stream: launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, a kernel may be scheduled while the
// previous one in the stream drains; it touches nothing the previous kernel writes before
// griddepcontrol.wait (the first statement of every PDL kernel, or right after a prologue that
// only initialises its own shared memory / TMEM), and lets its own successor launch at once.
#pragma once

#include <cuda_runtime.h>

namespace hy {

__device__ __forceinline__ void pdl_wait_and_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename Kern, typename... Args>
cudaError_t launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace hy
