// GradSink of one backward task (used by enqueue_task): embedding gradients in their own
// buffer, the other layers in the worker's FIFO ring, each released layer handed to the optimizer.
#pragma once

#include "executor_impl.hpp"

namespace spillsim {
namespace exec_detail {

// GradSink of one backward task: embedding grads in their own buffer, the other layers in
// the worker's FIFO ring; release() hands each layer to adam_layer immediately.
struct StreamingSink : hy::GradSink {
  ExecutorImpl& ex;
  Worker& w;
  HostJob& hj;
  int s;
  float* base;
  int step;
  const int32_t* tokens;  // device tokens of the task (embedding row flags)
  std::map<int, float*> live;
  bool dense_done = false;       // embedding: non-token wte rows already handed to the optimizer
  std::vector<int> host_layers;  // released to the host optimizer (slot copy now stale)

  StreamingSink(ExecutorImpl& e, Worker& wk, HostJob& h, int shard, float* b, int st, const int32_t* tok)
      : ex(e), w(wk), hj(h), s(shard), base(b), step(st), tokens(tok) {}

  float* acquire(int layer) override {
    const long len = hy_pad32(hy_layer_floats(&hj.m, layer));
    float* p;
    if (layer == 0) {
      w.gembed_tr.before_write(w.comp);
      w.gembed_tag = Tag{};  // no longer a wte cache
      p = w.gembed;
    } else {
      if (w.ring_head + len > w.ring_floats) w.ring_head = 0;
      const long lo = w.ring_head, hi = w.ring_head + len;
      // retire (wait for) every in-flight layer overlapping [lo, hi)
      HY_PROF(w.comp, "wait_ring");
      std::deque<Worker::RingEntry> keep;
      for (const Worker::RingEntry& e : w.ring_live) {
        if (e.off < hi && lo < e.off + e.len) {
          if (!e.done) throw InvalidArgument("gradient ring too small for an unreleased layer");
          check_cuda(cudaStreamWaitEvent(w.comp, e.done, 0), "ring wait");
        } else {
          keep.push_back(e);
        }
      }
      w.ring_live.swap(keep);
      p = w.ring + lo;
      w.ring_head = hi;
      w.ring_live.push_back(Worker::RingEntry{lo, len, nullptr});
    }
    check_cuda(cudaMemsetAsync(p, 0, sizeof(float) * static_cast<size_t>(len), w.comp), "zero grads");
    if (layer == 0) w.gembed_tr.after_write(w.comp);
    if (layer == 0 && split_embed()) {
      w.rowidx_tr.before_write(w.comp);
      check_cuda(hy::embed_row_index(w.comp, static_cast<int>(hj.M), tokens, hj.m.V, hj.m.T, w.rowidx, w.rowlist,
                                     w.rowcount),
                 "row index");
      w.rowidx_tr.after_write(w.comp);
    }
    live[layer] = p;
    return p;
  }

  // GPU-placed embedding with its optimizer split around the scatter (not with the staging
  // aliased onto the scratch, where every update waits for the end of the backward)
  // (not when the embedding's moments are HBM-resident: one in-place update after the
  // scatter is then cheaper than the split's staged passes)
  bool split_embed() const {
    if (hj.host_layer[0] || !w.rowidx || !tokens || w.stg_alias || g_debug_skip == 2) return false;
    return !(ex.claim_moments(w, hj) && w.mv_live.count(0));
  }

  // With the Adam staging aliased onto the backward's scratch (tiny HBM caps), layers are
  // queued and handed to the optimizer only after the backward (flush()).
  bool deferred = false;
  std::vector<int> queued;

  void release(int layer) override {
    if (deferred) {
      queued.push_back(layer);
      return;
    }
    emit(layer);
  }

  void flush() {
    for (int l : queued) emit(l);
    queued.clear();
  }

  void release_dense(int layer) override {
    if (layer != 0 || !split_embed()) return;
    Tracked& mvt = *hj.mv_tr[static_cast<size_t>(s)];
    mvt.before_read(w.opt2);
    w.gembed_tr.before_read(w.opt2);
    ex.adam_layer(w, hj, s, base, 0, live.at(0), step, nullptr, /*part=*/1);
    w.gembed_tr.after_read(w.opt2);
    mvt.after_read(w.opt2);
    dense_done = true;
  }

  void emit(int layer) {
    float* p = live.at(layer);
    cudaEvent_t done = w.ev_pool[w.ev_next++ % w.ev_pool.size()];
    if (layer != 0) {
      for (auto& e : w.ring_live) {
        if (w.ring + e.off == p) e.done = done;
      }
    }
    if (hj.host_layer[static_cast<size_t>(layer)]) {
      if (layer == 0) w.gembed_tr.before_read(w.up);
      ex.host_adam_layer(w, hj, s, layer, p, step, done);
      if (layer == 0) w.gembed_tr.after_read(w.up);
      host_layers.push_back(layer);
      return;
    }
    if (layer == 0) w.gembed_tr.before_read(w.opt);
    ex.adam_layer(w, hj, s, base, layer, p, step, done, layer == 0 && dense_done ? 2 : 0);
    if (layer == 0) w.gembed_tr.after_read(w.opt);
  }
};

}  // namespace exec_detail
}  // namespace spillsim
