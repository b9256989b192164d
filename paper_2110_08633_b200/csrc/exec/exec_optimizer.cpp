// GPU-placed AdamW streaming (staging ring / moment cache / embedding split) and the
// host-placed AdamW of the executor (ExecOptions::host_opt_fraction).
#include "executor_impl.hpp"

namespace spillsim {

// GPU-placed AdamW for one layer of shard s, as soon as its gradient is final: m, v chunks
// H2D into the staging ring -> fused Adam (params updated in place in the slot) -> params,
// m, v D2H on the up stream (the reference's GradOffload with the optimizer folded in,
// SPEC.md:225). `part`: 0 = the whole layer (opt stream). Embedding split: 1 = pass A on
// opt2, released early (release_dense) — every chunk of layer 0 is staged, untouched wte rows
// are updated and the rows this minibatch's scatter touches are stashed compactly; 2 = pass
// B after the scatter — the stashed rows are updated (opt) and written to the host with
// zero-copy stores (up, behind pass A's D2H so they land last). `done` is recorded once
// Adam no longer reads `grads`.
void ExecutorImpl::adam_layer(Worker& w, HostJob& hj, int s, float* base, int layer, const float* grads, int step,
                              cudaEvent_t done, int part) {
  const ShardGeom& g = hj.geom[static_cast<size_t>(s)];
  const long host_off = hy_layer_offset(&hj.m, layer);
  const long slot_off = host_off - hy_layer_offset(&hj.m, g.l0);
  const long nfl = hy_layer_floats(&hj.m, layer);
  const ExecJob& spec = *hj.spec;
  hy::AdamHyper h{spec.lr, spec.beta1, spec.beta2, spec.eps, spec.weight_decay, 0.f, 0.f};
  h.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(spec.beta1), step));
  h.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(spec.beta2), step));
  cudaStream_t os = part == 1 ? w.opt2 : w.opt;
  // m, v of a whole-layer update are prefetched on their own stream (optin) as soon as a
  // staging chunk frees up — ahead of the gradient; only the Adam kernels wait for it
  cudaStream_t is = part == 0 ? w.optin : os;
  // the layer's gradient is final and its params are no longer read by the compute stream
  cudaEvent_t ready = w.ev_pool[w.ev_next++ % w.ev_pool.size()];
  check_cuda(cudaEventRecord(ready, w.comp), "layer ready");
  check_cuda(cudaStreamWaitEvent(os, ready, 0), "layer ready wait");
  const bool bf16 = exec.opt_state_bf16;
  const size_t es = bf16 ? 2 : 4;  // bytes per moment element
  char* hm = reinterpret_cast<char*>(hj.mom);
  char* hv = reinterpret_cast<char*>(hj.var);
  const int d = hj.m.d;
  char* cm = reinterpret_cast<char*>(w.cbuf);
  char* cv = cm + 4 * static_cast<size_t>(w.crow_max);
  float* cp = w.cbuf + 2 * w.crow_max;
  if (part == 2) {
    check_cuda(cudaStreamWaitEvent(w.opt, w.dense_done, 0), "dense wait");
    w.cbuf_tr.before_write(w.opt);
    w.rowidx_tr.before_read(w.opt);
    check_cuda(hy::adam_embed_rows(w.opt, hj.M + hj.m.T, w.rowcount, w.rowlist, d, base + slot_off, grads, cm, cv,
                                   hj.write_back ? nullptr : cp,
                                   bf16, h),
               "adam rows");
    ++w.st.kernel_launches;
    w.rowidx_tr.after_read(w.opt);
    w.cbuf_tr.after_write(w.opt);
    if (done) check_cuda(cudaEventRecord(done, w.opt), "adam done");
    w.cbuf_tr.before_read(w.up);
    w.rowidx_tr.before_read(w.up);
    check_cuda(hy::embed_rows_to_host(w.up, hj.M + hj.m.T, w.rowcount, w.rowlist, d, cp, cm, cv,
                                      hj.write_back ? nullptr : hj.params + host_off,
                                      hm + es * host_off, hv + es * host_off, bf16),
               "rows to host");
    ++w.st.kernel_launches;
    w.rowidx_tr.after_read(w.up);
    w.cbuf_tr.after_read(w.up);
    return;
  }
  if (part == 0) {
    const long half = (static_cast<long>(es) * nfl + 511) / 512 * 512;
    if (Worker::MvEntry* e = acquire_moments(w, hj, layer, 2 * half)) {
      char* dm = w.mvpool + e->off;
      char* dv = dm + half;
      const size_t sbytes = es * static_cast<size_t>(nfl);
      const size_t hoff = es * static_cast<size_t>(host_off);
      if (!e->valid) {  // first update of this layer since the job took the cache: load once
        if (w.mv_free_pending) {
          check_cuda(cudaStreamWaitEvent(w.optin, w.mv_free, 0), "mv free wait");
          w.mv_free_pending = false;
        }
        e->tr.before_write(w.optin);
        check_cuda(xfer(dm, hm + hoff, sbytes, cudaMemcpyHostToDevice, w.optin), "m load");
        check_cuda(xfer(dv, hv + hoff, sbytes, cudaMemcpyHostToDevice, w.optin), "v load");
        e->tr.after_write(w.optin);
        e->valid = true;
        e->job = hj.job;
        w.st.opt_h2d_bytes += 2.0 * sbytes;
        w.st.h2d_bytes += 2.0 * sbytes;
        w.st.mv_load_h2d_bytes += 2.0 * sbytes;
      }
      e->tr.before_write(os);
      if (bf16) {
        check_cuda(hy::adam_update_bf16(os, nfl, base + slot_off, grads, reinterpret_cast<uint16_t*>(dm),
                                        reinterpret_cast<uint16_t*>(dv), h),
                   "adam bf16 (resident moments)");
      } else {
        check_cuda(hy::adam_update(os, nfl, base + slot_off, grads, reinterpret_cast<float*>(dm),
                                   reinterpret_cast<float*>(dv), h),
                   "adam (resident moments)");
      }
      ++w.st.kernel_launches;
      e->tr.after_write(os);
      e->dirty = true;
      w.st.mv_resident_updates += static_cast<double>(nfl);
      if (done) check_cuda(cudaEventRecord(done, os), "adam done");
      auto lb = w.last_b_local.find({hj.job, s});
      if (!exec.dynamic && lb != w.last_b_local.end() && lb->second == w.cur_local) hand_over_moments(w, hj, layer, *e);
      return;
    }
  }
  if (part == 1) {
    w.cbuf_tr.before_write(w.opt2);
    w.rowidx_tr.before_read(w.opt2);
  }
  const long chunk = w.stg_chunk;
  for (long off = 0; off < nfl; off += chunk) {
    const long n = std::min(chunk, nfl - off);
    const size_t bytes = sizeof(float) * static_cast<size_t>(n);
    const size_t sbytes = es * static_cast<size_t>(n);
    const int si = w.stg_round++ % kStaging;
    char* sm = reinterpret_cast<char*>(w.stg[si]);
    char* sv = sm + es * static_cast<size_t>(chunk);
    Tracked& stg = w.stg_tr[si];
    const size_t hoff = es * static_cast<size_t>(host_off + off);
    stg.before_write(is);
    check_cuda(xfer(sm, hm + hoff, sbytes, cudaMemcpyHostToDevice, is), "m h2d");
    check_cuda(xfer(sv, hv + hoff, sbytes, cudaMemcpyHostToDevice, is), "v h2d");
    if (is != os) {
      cudaEvent_t in = w.ev_pool[w.ev_next++ % w.ev_pool.size()];
      check_cuda(cudaEventRecord(in, is), "mv in");
      check_cuda(cudaStreamWaitEvent(os, in, 0), "mv in wait");
    }
    w.st.opt_h2d_bytes += 2.0 * sbytes;
    w.st.h2d_bytes += 2.0 * sbytes;
    if (part == 1) {
      check_cuda(hy::adam_embed_dense(os, n, off, d, w.rowidx, base + slot_off + off, grads + off, sm, sv, cm, cv,
                                      bf16, h),
                 "adam dense");
    } else if (bf16) {
      check_cuda(hy::adam_update_bf16(os, n, base + slot_off + off, grads + off, reinterpret_cast<uint16_t*>(sm),
                                      reinterpret_cast<uint16_t*>(sv), h),
                 "adam bf16");
    } else {
      check_cuda(hy::adam_update(os, n, base + slot_off + off, grads + off, reinterpret_cast<float*>(sm),
                                 reinterpret_cast<float*>(sv), h),
                 "adam");
    }
    ++w.st.kernel_launches;
    stg.after_write(os);
    stg.before_read(w.up);
    if (!hj.write_back) {  // write-through (jobs spread over GPUs); else the cache writes back
      check_cuda(xfer(hj.params + host_off + off, base + slot_off + off, bytes, cudaMemcpyDeviceToHost, w.up),
                 "p d2h");
      w.st.d2h_bytes += static_cast<double>(bytes);
    }
    check_cuda(xfer(hm + hoff, sm, sbytes, cudaMemcpyDeviceToHost, w.up), "m d2h");
    check_cuda(xfer(hv + hoff, sv, sbytes, cudaMemcpyDeviceToHost, w.up), "v d2h");
    stg.after_read(w.up);
    w.st.opt_d2h_bytes += 2.0 * sbytes;
    w.st.d2h_bytes += 2.0 * sbytes;
  }
  if (part == 1) {
    w.rowidx_tr.after_read(w.opt2);
    w.cbuf_tr.after_write(w.opt2);
    check_cuda(cudaEventRecord(w.dense_done, w.opt2), "dense done");
    return;
  }
  if (done) check_cuda(cudaEventRecord(done, w.opt), "adam done");
}

// Host-placed layer: GradOffload of the layer's gradient (up), then AdamW on the host
// (hopt stream, cudaLaunchHostFunc) over the pinned master params and moments. The HBM slot
// keeps the pre-update copy; the layer is marked dirty in the slot and refreshed from the
// host before the slot is read again (acquire hit) — a full reload refreshes it anyway.
void ExecutorImpl::host_adam_layer(Worker& w, HostJob& hj, int s, int layer, const float* grads, int step,
                                   cudaEvent_t done) {
  const long off = hy_layer_offset(&hj.m, layer);
  const long n = hy_layer_floats(&hj.m, layer);
  const ExecJob& spec = *hj.spec;
  cudaEvent_t ready = w.ev_pool[w.ev_next++ % w.ev_pool.size()];
  check_cuda(cudaEventRecord(ready, w.comp), "layer ready");
  check_cuda(cudaStreamWaitEvent(w.up, ready, 0), "layer ready wait");
  Tracked& gt = *hj.hgrad_tr[static_cast<size_t>(layer)];
  gt.before_write(w.up);
  check_cuda(xfer(hj.hgrad + off, grads, sizeof(float) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, w.up),
             "grad d2h");
  gt.after_write(w.up);
  check_cuda(cudaEventRecord(done, w.up), "grad offloaded");
  w.st.host_grad_d2h_bytes += 4.0 * n;
  w.st.d2h_bytes += 4.0 * n;
  w.st.host_opt_params += static_cast<double>(n);
  Tracked& pt = *hj.hparams_tr[static_cast<size_t>(s)];
  gt.before_read(w.hopt);
  pt.before_write(w.hopt);
  hy::HostAdamWork a;
  a.p = hj.params + off;
  a.g = hj.hgrad + off;
  const size_t es = exec.opt_state_bf16 ? 2 : 4;
  a.m = reinterpret_cast<char*>(hj.mom) + es * static_cast<size_t>(off);
  a.v = reinterpret_cast<char*>(hj.var) + es * static_cast<size_t>(off);
  a.n = n;
  a.lr = spec.lr;
  a.beta1 = spec.beta1;
  a.beta2 = spec.beta2;
  a.eps = spec.eps;
  a.weight_decay = spec.weight_decay;
  a.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(spec.beta1), step));
  a.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(spec.beta2), step));
  a.bf16 = exec.opt_state_bf16 ? 1 : 0;
  a.threads = host_threads;
  check_cuda(hy::host_adam_async(w.hopt, a), "host adam");
  pt.after_write(w.hopt);
  gt.after_read(w.hopt);
}

}  // namespace spillsim
