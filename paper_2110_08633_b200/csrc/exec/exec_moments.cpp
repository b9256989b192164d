// Optimizer-state (Adam m, v) cache of a worker: ownership, per-layer entries, hand-over to
// the next job and write-back.
#include "executor_impl.hpp"

namespace spillsim {

// Moment-cache entry of `layer` for the job `hj` (nullptr: stream it through the staging ring).
// The pool belongs to one job at a time; ownership passes to the next job only once the owner
// has no task left on this GPU in this pass (SHARP runs a GPU's jobs one after another), so
// entries are never thrashed between interleaved jobs.
bool ExecutorImpl::claim_moments(Worker& w, HostJob& hj) {
  if (!w.mvpool || !hj.write_back) return false;
  if (w.mv_owner == hj.job) {
    w.mv_owner_pass = w.cur_pass;
    return true;
  }
  if (w.mv_owner >= 0) {
    // the owner still has tasks ahead of it on this GPU in this pass: stream instead
    auto it = w.last_local_of_job.find(w.mv_owner);
    if (!exec.dynamic && w.mv_owner_pass == w.cur_pass && it != w.last_local_of_job.end() &&
        it->second > w.cur_local) {
      return false;
    }
    if (same_moment_layout(jobs.at(w.mv_owner), hj)) {
      // Same model shape: keep the entries, write the old owner's moments back in the order the
      // new owner's backward will reload them (head side first), each entry tracked on its own —
      // the new owner's first load of a layer waits only for that layer's write-back.
      flush_moments(w, hj.job);
      w.mv_owner = hj.job;
      w.mv_owner_pass = w.cur_pass;
      return true;
    }
    release_moments(w, false);
  }
  w.mv_owner = hj.job;
  w.mv_owner_pass = w.cur_pass;
  // Layout in forward order: the layers the next forward needs first (embedding, then the
  // first blocks) get resident moments, the head-side layers the backward releases first —
  // so their streamed update has the whole backward to finish — take what does not fit.
  const size_t es = exec.opt_state_bf16 ? 2 : 4;
  for (int l = 0; l < hj.m.L + 2; ++l) {
    if (hj.host_layer[static_cast<size_t>(l)]) continue;
    const long half = (static_cast<long>(es) * hy_layer_floats(&hj.m, l) + 511) / 512 * 512;
    if (w.mvpool_used + 2 * half > w.mvpool_bytes) continue;  // a smaller later layer may fit
    auto e = std::make_unique<Worker::MvEntry>();
    e->layer = l;
    e->off = w.mvpool_used;
    e->bytes = 2 * half;
    w.mvpool_used += 2 * half;
    w.mv_live[l] = std::move(e);
  }
  return true;
}

Worker::MvEntry* ExecutorImpl::acquire_moments(Worker& w, HostJob& hj, int layer, long bytes) {
  if (!claim_moments(w, hj)) return nullptr;
  auto it = w.mv_live.find(layer);
  if (it == w.mv_live.end() || it->second->bytes < bytes) return nullptr;
  if (it->second->job != hj.job) it->second->valid = false;  // holds another job's moments
  return it->second.get();
}

// Proactive handover: the owner's last update of `layer` in this pass is done, so its moments go
// back to the host right away (up) and, when the job that follows on this GPU has the same
// shape, that job's moments for the layer come in behind them (optin) — spread over the owner's
// last backward instead of piling up when the next job first needs them. The last job of a pass
// hands over to the first job of the next pass.
void ExecutorImpl::hand_over_moments(Worker& w, HostJob& hj, int layer, Worker::MvEntry& e) {
  auto nx = w.next_job.find(hj.job);
  if (nx == w.next_job.end() || nx->second == hj.job) return;
  HostJob& nj = jobs.at(nx->second);
  if (!nj.write_back || !same_moment_layout(hj, nj)) return;
  const size_t es = exec.opt_state_bf16 ? 2 : 4;
  const long nfl = hy_layer_floats(&hj.m, layer);
  const size_t sbytes = es * static_cast<size_t>(nfl);
  const size_t hoff = es * static_cast<size_t>(hy_layer_offset(&hj.m, layer));
  const long half = e.bytes / 2;
  auto shard_of = [&](const HostJob& x) {
    int s = 0;
    while (s + 1 < static_cast<int>(x.geom.size()) && x.geom[static_cast<size_t>(s) + 1].l0 <= layer) ++s;
    return s;
  };
  // write the owner's final moments back
  Tracked& mo = *hj.mv_tr[static_cast<size_t>(shard_of(hj))];
  e.tr.before_read(w.up);
  mo.before_write(w.up);
  check_cuda(xfer(reinterpret_cast<char*>(hj.mom) + hoff, w.mvpool + e.off, sbytes, cudaMemcpyDeviceToHost, w.up),
             "m hand-over write-back");
  check_cuda(xfer(reinterpret_cast<char*>(hj.var) + hoff, w.mvpool + e.off + half, sbytes, cudaMemcpyDeviceToHost,
                  w.up),
             "v hand-over write-back");
  mo.after_write(w.up);
  e.tr.after_read(w.up);
  w.st.opt_d2h_bytes += 2.0 * sbytes;
  w.st.d2h_bytes += 2.0 * sbytes;
  w.st.mv_writeback_d2h_bytes += 2.0 * sbytes;
  // ... and the next job's in behind them
  Tracked& mn = *nj.mv_tr[static_cast<size_t>(shard_of(nj))];
  e.tr.before_write(w.optin);
  mn.before_read(w.optin);
  check_cuda(xfer(w.mvpool + e.off, reinterpret_cast<char*>(nj.mom) + hoff, sbytes, cudaMemcpyHostToDevice, w.optin),
             "m hand-over load");
  check_cuda(xfer(w.mvpool + e.off + half, reinterpret_cast<char*>(nj.var) + hoff, sbytes, cudaMemcpyHostToDevice,
                  w.optin),
             "v hand-over load");
  mn.after_read(w.optin);
  e.tr.after_write(w.optin);
  w.st.opt_h2d_bytes += 2.0 * sbytes;
  w.st.h2d_bytes += 2.0 * sbytes;
  w.st.mv_load_h2d_bytes += 2.0 * sbytes;
  e.valid = true;
  e.dirty = false;
  e.job = nj.job;
}

// Old owner's dirty moments -> host (up stream), head-side layers first; every entry stays in
// place, invalid, for the next owner (same layout), ordered per entry by its tracker.
void ExecutorImpl::flush_moments(Worker& w, int new_owner) {
  HostJob& hj = jobs.at(w.mv_owner);
  const size_t es = exec.opt_state_bf16 ? 2 : 4;
  char* hm = reinterpret_cast<char*>(hj.mom);
  char* hv = reinterpret_cast<char*>(hj.var);
  for (auto it = w.mv_live.rbegin(); it != w.mv_live.rend(); ++it) {
    Worker::MvEntry& e = *it->second;
    if (e.valid && e.job == new_owner) continue;  // already handed over (proactive handover)
    e.tr.before_read(w.up);
    if (e.valid && e.dirty && e.job == w.mv_owner) {
      int s = 0;
      while (s + 1 < static_cast<int>(hj.geom.size()) && hj.geom[static_cast<size_t>(s) + 1].l0 <= e.layer) ++s;
      Tracked& mvt = *hj.mv_tr[static_cast<size_t>(s)];
      const long nfl = hy_layer_floats(&hj.m, e.layer);
      const size_t sbytes = es * static_cast<size_t>(nfl);
      const size_t hoff = es * static_cast<size_t>(hy_layer_offset(&hj.m, e.layer));
      mvt.before_write(w.up);
      check_cuda(xfer(hm + hoff, w.mvpool + e.off, sbytes, cudaMemcpyDeviceToHost, w.up), "m write-back");
      check_cuda(xfer(hv + hoff, w.mvpool + e.off + e.bytes / 2, sbytes, cudaMemcpyDeviceToHost, w.up),
                 "v write-back");
      mvt.after_write(w.up);
      w.st.opt_d2h_bytes += 2.0 * sbytes;
      w.st.d2h_bytes += 2.0 * sbytes;
      w.st.mv_writeback_d2h_bytes += 2.0 * sbytes;
    }
    e.tr.after_read(w.up);
    e.valid = false;
    e.dirty = false;
  }
}

// Write the owner's updated moments back to its host state (up stream). keep = true (end of
// a pass): entries stay resident and valid for the owner's next pass; false: the pool is
// handed over — `mv_free` (up) marks when the next owner may overwrite it.
void ExecutorImpl::release_moments(Worker& w, bool keep) {
  if (w.mv_owner < 0) return;
  HostJob& hj = jobs.at(w.mv_owner);
  const size_t es = exec.opt_state_bf16 ? 2 : 4;
  char* hm = reinterpret_cast<char*>(hj.mom);
  char* hv = reinterpret_cast<char*>(hj.var);
  for (auto& kv : w.mv_live) {
    Worker::MvEntry& e = *kv.second;
    e.tr.before_read(w.up);
    if (e.dirty && e.job == w.mv_owner) {
      int s = 0;
      while (s + 1 < static_cast<int>(hj.geom.size()) && hj.geom[static_cast<size_t>(s) + 1].l0 <= e.layer) ++s;
      Tracked& mvt = *hj.mv_tr[static_cast<size_t>(s)];
      const long nfl = hy_layer_floats(&hj.m, e.layer);
      const size_t sbytes = es * static_cast<size_t>(nfl);
      const size_t hoff = es * static_cast<size_t>(hy_layer_offset(&hj.m, e.layer));
      const long half = e.bytes / 2;
      mvt.before_write(w.up);
      check_cuda(xfer(hm + hoff, w.mvpool + e.off, sbytes, cudaMemcpyDeviceToHost, w.up), "m write-back");
      check_cuda(xfer(hv + hoff, w.mvpool + e.off + half, sbytes, cudaMemcpyDeviceToHost, w.up), "v write-back");
      mvt.after_write(w.up);
      w.st.opt_d2h_bytes += 2.0 * sbytes;
      w.st.d2h_bytes += 2.0 * sbytes;
      w.st.mv_writeback_d2h_bytes += 2.0 * sbytes;
      e.dirty = false;
    }
    e.tr.after_read(w.up);
  }
  if (keep) return;
  check_cuda(cudaEventRecord(w.mv_free, w.up), "mv free");
  w.mv_free_pending = true;
  for (auto& kv : w.mv_live) w.mv_retired.push_back(std::move(kv.second));
  w.mv_live.clear();
  w.mvpool_used = 0;
  w.mv_owner = -1;
}

}  // namespace spillsim
