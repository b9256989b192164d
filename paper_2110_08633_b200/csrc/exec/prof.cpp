#include "prof.hpp"

#include <cstdlib>
#include <cstring>

namespace hy {

OpProfiler& OpProfiler::get() {
  static OpProfiler p = [] {
    OpProfiler q;
    const char* e = std::getenv("HY_PROFILE");
    q.enabled = e && e[0] == '1';
    return q;
  }();
  return p;
}

cudaEvent_t OpProfiler::take() {
  if (used == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  return pool[used++];
}

std::map<std::string, double> OpProfiler::drain() {
  std::map<std::string, double> out;
  for (const Rec& r : recs) {
    cudaEventSynchronize(r.b);
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    out[r.label] += ms;
  }
  recs.clear();
  used = 0;
  return out;
}

thread_local IntervalLog* t_ilog = nullptr;

cudaEvent_t IntervalLog::take() {
  if (used == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  return pool[used++];
}

size_t IntervalLog::begin(int lane, double bytes, cudaStream_t st) {
  Rec r{lane, bytes, take(), take(), st};
  cudaEventRecord(r.a, st);
  recs.push_back(r);
  return recs.size() - 1;
}

void IntervalLog::end(size_t idx, cudaStream_t st) { cudaEventRecord(recs[idx].b, st); }

IntervalLog::~IntervalLog() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

ScopedOp::ScopedOp(cudaStream_t s, const char* label) : st(s) {
  if (t_ilog && std::strncmp(label, "wait", 4) != 0) ilog_idx = t_ilog->begin(IntervalLog::kCompute, 0, st);
  OpProfiler& p = OpProfiler::get();
  if (!p.enabled) return;
  OpProfiler::Rec r{label, p.take(), p.take()};
  cudaEventRecord(r.a, st);
  p.recs.push_back(r);
  idx = p.recs.size() - 1;
  rec = &p.recs.back();
}

ScopedOp::~ScopedOp() {
  if (t_ilog && ilog_idx != static_cast<size_t>(-1)) t_ilog->end(ilog_idx, st);
  if (!rec) return;
  OpProfiler& p = OpProfiler::get();
  cudaEventRecord(p.recs[idx].b, st);
}

}  // namespace hy
