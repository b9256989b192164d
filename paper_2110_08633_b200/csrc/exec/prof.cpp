#include "prof.hpp"

#include <cstdlib>

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

ScopedOp::ScopedOp(cudaStream_t s, const char* label) : st(s) {
  OpProfiler& p = OpProfiler::get();
  if (!p.enabled) return;
  OpProfiler::Rec r{label, p.take(), p.take()};
  cudaEventRecord(r.a, st);
  p.recs.push_back(r);
  idx = p.recs.size() - 1;
  rec = &p.recs.back();
}

ScopedOp::~ScopedOp() {
  if (!rec) return;
  OpProfiler& p = OpProfiler::get();
  cudaEventRecord(p.recs[idx].b, st);
}

}  // namespace hy
