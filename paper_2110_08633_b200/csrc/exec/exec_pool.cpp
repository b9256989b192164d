// Parameter cache of a worker: host-master read ordering, first-fit / LRU shard entries,
// write-back of GPU-updated layers.
#include "executor_impl.hpp"

namespace spillsim {

// Reads of a shard's host master params (ParamLoad, refresh, tied-wte reload) wait for both
// writers: the GPU optimizer's write-back (up) and the host optimizer (hopt).
void ExecutorImpl::param_read_begin(HostJob& hj, int s, cudaStream_t st) {
  hj.params_tr[static_cast<size_t>(s)]->before_read(st);
  hj.hparams_tr[static_cast<size_t>(s)]->before_read(st);
}
void ExecutorImpl::param_read_end(HostJob& hj, int s, cudaStream_t st) {
  hj.params_tr[static_cast<size_t>(s)]->after_read(st);
  hj.hparams_tr[static_cast<size_t>(s)]->after_read(st);
}


// Resident entry for (job, shard, current version), loading it (first-fit into the pool,
// evicting least-recently-used shards other than the previous task's) when absent.
Worker::PoolEntry* ExecutorImpl::acquire_params(Worker& w, HostJob& hj, int j, int s, bool* loaded) {
  const ShardGeom& g = hj.geom[static_cast<size_t>(s)];
  const Tag want{j, -1, s, hj.version[static_cast<size_t>(s)]};
  for (auto& e : w.live) {
    if (e->tag == want) {
      e->last_use = w.seq;
      *loaded = false;
      return e.get();
    }
  }
  const long len = hy_pad32(g.param_floats);
  auto find_gap = [&]() -> long {
    std::vector<std::pair<long, long>> used;
    for (auto& e : w.live) used.emplace_back(e->off, e->off + e->len);
    std::sort(used.begin(), used.end());
    long cur = 0;
    for (auto& u : used) {
      if (u.first - cur >= len) return cur;
      cur = std::max(cur, u.second);
    }
    return w.pool_floats - cur >= len ? cur : -1;
  };
  long off = find_gap();
  while (off < 0) {
    auto victim = w.live.end();
    for (auto it = w.live.begin(); it != w.live.end(); ++it) {
      if (it->get() == w.prev_entry) continue;
      if (victim == w.live.end() || (*it)->last_use < (*victim)->last_use) victim = it;
    }
    if (victim == w.live.end()) {  // only the previous task's shard is left: evict it too
      for (auto it = w.live.begin(); it != w.live.end(); ++it) victim = it;
    }
    if (victim == w.live.end()) throw InvalidArgument("parameter pool smaller than a shard");
    write_back(w, **victim);
    w.retired.splice(w.retired.end(), w.live, victim);
    off = find_gap();
  }
  auto ent = std::make_unique<Worker::PoolEntry>();
  ent->tag = want;
  ent->off = off;
  ent->len = len;
  ent->last_use = w.seq;
  // the new region may still be read/written by evicted shards' pending work
  for (auto it = w.retired.begin(); it != w.retired.end();) {
    Worker::PoolEntry& r = **it;
    if (r.off < off + len && off < r.off + r.len) {
      r.tr.before_write(w.down);
      if (r.off >= off && r.off + r.len <= off + len) {
        r.tr.destroy();
        it = w.retired.erase(it);
        continue;
      }
    }
    ++it;
  }
  *loaded = true;
  w.live.push_back(std::move(ent));
  return w.live.back().get();
}

// Write-back cache: the slot's GPU-updated layers -> host master params (up stream), before
// the slot is reused or the host copy is read.
void ExecutorImpl::write_back(Worker& w, Worker::PoolEntry& e) {
  if (e.gpu_dirty.empty()) return;
  HostJob& hj = jobs.at(e.tag.job);
  const int s = e.tag.idx;
  const long base = hy_layer_offset(&hj.m, hj.geom[static_cast<size_t>(s)].l0);
  Tracked& ptr = *hj.params_tr[static_cast<size_t>(s)];
  e.tr.before_read(w.up);
  ptr.before_write(w.up);
  for (int l : e.gpu_dirty) {
    const long off = hy_layer_offset(&hj.m, l);
    const long n = hy_layer_floats(&hj.m, l);
    check_cuda(xfer(hj.params + off, w.pool + e.off + (off - base), sizeof(float) * static_cast<size_t>(n),
                    cudaMemcpyDeviceToHost, w.up),
               "param write-back");
    w.st.d2h_bytes += 4.0 * n;
    w.st.writeback_d2h_bytes += 4.0 * n;
  }
  ptr.after_write(w.up);
  e.tr.after_read(w.up);
  e.gpu_dirty.clear();
}

}  // namespace spillsim
