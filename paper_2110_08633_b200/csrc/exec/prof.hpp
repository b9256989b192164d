// Opt-in per-op device timing on the compute stream (HY_PROFILE=1): CUDA events around
// each op of the shard runner, aggregated per label after a pass. Diagnostics only.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

namespace hy {

struct OpProfiler {
  static OpProfiler& get();
  bool enabled = false;
  struct Rec {
    const char* label;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t take();
  // Sum of milliseconds per label since the last drain (synchronises).
  std::map<std::string, double> drain();
};

struct ScopedOp {
  cudaStream_t st;
  OpProfiler::Rec* rec = nullptr;
  size_t idx = 0;
  ScopedOp(cudaStream_t s, const char* label);
  ~ScopedOp();
};

#define HY_PROF(st, label) ::hy::ScopedOp hy_prof_scope_##__LINE__(st, label)

}  // namespace hy
