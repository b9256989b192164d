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
  size_t ilog_idx = static_cast<size_t>(-1);
  ScopedOp(cudaStream_t s, const char* label);
  ~ScopedOp();
};

// Interval log of one worker's pass (ExecOptions::link_log): CUDA events around every
// compute-stream op of the shard runner (HY_PROF scopes other than "wait_*") and every
// host<->device copy, giving copy-only link intervals and the transfer-overlap fraction
// (1 - link time not under compute / link time). Two event records per op / copy, so it is
// enabled for a separate measurement pass only.
struct IntervalLog {
  enum Lane { kCompute = 0, kH2D = 1, kD2H = 2 };
  struct Rec {
    int lane;
    double bytes;
    cudaEvent_t a, b;
    cudaStream_t st;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t take();
  size_t begin(int lane, double bytes, cudaStream_t st);
  void end(size_t idx, cudaStream_t st);
  void reset() {
    recs.clear();
    used = 0;
  }
  ~IntervalLog();
};
// The log of the worker running on this thread (null: not logging).
extern thread_local IntervalLog* t_ilog;

#define HY_PROF(st, label) ::hy::ScopedOp hy_prof_scope_##__LINE__(st, label)

}  // namespace hy
