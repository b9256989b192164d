// Task enqueue (ParamLoad / ActPromote on down, compute on comp, ActDemote / GradOffload on
// up), NVLink peer hand-off and the dynamic-time dispatch loop.
#include "executor_impl.hpp"
#include "grad_sink.hpp"

namespace spillsim {

void ExecutorImpl::enqueue_task(Worker& w, int t, int pass) {
  const SimTask& task = tasks[static_cast<size_t>(t)];
  const int j = task.t.job;
  const int s = task.t.shard;
  HostJob& hj = jobs.at(j);
  const ShardGeom& g = hj.geom[static_cast<size_t>(s)];
  const int k = static_cast<int>(hj.geom.size());
  const int gmb = pass * job_mb[static_cast<size_t>(j)] + task.t.minibatch;
  const bool fwd = task.t.direction == Direction::kForward;
  const int local = task_local[static_cast<size_t>(t)];
  w.cur_local = local;
  w.cur_pass = pass;
  TaskTiming& tm = w.timing[static_cast<size_t>(local)];
  const size_t act_bytes = sizeof(float) * static_cast<size_t>(hj.n_act);

  // Cross-device predecessors (only with jobs migrating, e.g. double_buffering=false):
  // wait until their producer has been enqueued so its events exist.
  for (int p : task.preds) {
    if (task_device[static_cast<size_t>(p)] != w.plan_dev) {
      std::unique_lock<std::mutex> lk(flag_mu);
      flag_cv.wait(lk, [&] { return enqueued_pass[static_cast<size_t>(p)] >= pass; });
    }
  }

  w.st.model_h2d_bytes += task.t.param_load_bytes + task.t.activation_in_bytes;
  w.st.model_d2h_bytes += task.t.activation_out_bytes + task.t.grad_offload_bytes;

  // ---- ParamLoad (down) -----------------------------------------------------------
  ++w.seq;
  // Interval starts are recorded after the hazard waits, right before the first copy of the
  // section (zero-length when nothing moves), so the trace's link intervals are copy time.
  bool pl0_done = false, pr0_done = false, d0_done = !fwd;
  auto mark = [](cudaEvent_t e, cudaStream_t st, bool& done) {
    if (!done) check_cuda(cudaEventRecord(e, st), "interval start");
    done = true;
  };
  bool loaded = false;
  Worker::PoolEntry* pe = acquire_params(w, hj, j, s, &loaded);
  float* pbase = w.pool + pe->off;
  if (loaded) {
    const long base = hy_layer_offset(&hj.m, g.l0);
    pe->tr.before_write(w.down);
    param_read_begin(hj, s, w.down);
    mark(tm.pl0, w.down, pl0_done);
    check_cuda(xfer(pbase, hj.params + base, sizeof(float) * static_cast<size_t>(g.param_floats),
                    cudaMemcpyHostToDevice, w.down),
               "param h2d");
    param_read_end(hj, s, w.down);
    pe->tr.after_write(w.down);
    w.st.param_h2d_bytes += 4.0 * g.param_floats;
    w.st.h2d_bytes += 4.0 * g.param_floats;
  } else if (!pe->dirty.empty()) {
    // resident, but some layers were updated host-side: refresh just those
    pe->tr.before_write(w.down);
    param_read_begin(hj, s, w.down);
    mark(tm.pl0, w.down, pl0_done);
    double bytes = 0;
    for (int l : pe->dirty) {
      const long off = hy_layer_offset(&hj.m, l);
      const long n = hy_layer_floats(&hj.m, l);
      check_cuda(xfer(pbase + (off - hy_layer_offset(&hj.m, g.l0)), hj.params + off, sizeof(float) * static_cast<size_t>(n),
                      cudaMemcpyHostToDevice, w.down),
                 "param refresh h2d");
      bytes += 4.0 * n;
    }
    param_read_end(hj, s, w.down);
    pe->tr.after_write(w.down);
    pe->dirty.clear();
    w.st.refresh_h2d_bytes += bytes;
    w.st.param_h2d_bytes += bytes;
    w.st.h2d_bytes += bytes;
    w.st.elided_param_bytes += std::max(0.0, task.t.param_load_bytes - bytes);
  } else {
    w.st.elided_param_bytes += task.t.param_load_bytes;
  }
  // Head shard without the embedding: the tied wte comes from the gembed cache (filled by a
  // D2D copy at F(0)); reload it over the link only if the cache is stale or missing.
  const float* wte_ext = nullptr;
  if (g.wte_offset >= 0) {
    const Tag wt{j, -1, -2, hj.version[0]};
    if (!(w.gembed_tag == wt)) {
      for (auto& e : w.live) {
        if (e->tag.job == j && e->tag.idx == 0) write_back(w, *e);
      }
      w.gembed_tr.before_write(w.down);
      param_read_begin(hj, 0, w.down);
      mark(tm.pl0, w.down, pl0_done);
      const size_t wb = sizeof(float) * static_cast<size_t>(hj.m.V) * static_cast<size_t>(hj.m.d);
      check_cuda(xfer(w.gembed, hj.params, wb, cudaMemcpyHostToDevice, w.down), "wte h2d");
      param_read_end(hj, 0, w.down);
      w.gembed_tr.after_write(w.down);
      w.gembed_tag = wt;
      w.st.param_h2d_bytes += static_cast<double>(wb);
      w.st.h2d_bytes += static_cast<double>(wb);
    }
    wte_ext = w.gembed;
  }
  mark(tm.pl0, w.down, pl0_done);
  check_cuda(cudaEventRecord(tm.pl1, w.down), "pl1");

  // ---- ActPromote (down): tokens, boundary activation / checkpoint, grad_in, z --------
  hy::TaskIO io;
  const bool need_tokens = g.has_embed || g.has_head;
  int tok_i = -1;
  if (need_tokens) {
    const Tag tt{j, gmb, 0, 0};
    for (int i = 0; i < 2; ++i) {
      if (w.tok_tag[i] == tt) tok_i = i;
    }
    if (tok_i < 0) {
      tok_i = 1 - w.last_tok;  // alternate: the other buffer may still feed a resident task
      w.last_tok = tok_i;
      w.tok_tr[tok_i].before_write(w.down);
      mark(tm.pr0, w.down, pr0_done);
      const size_t tb = sizeof(int32_t) * static_cast<size_t>(hj.M);
      check_cuda(xfer(w.tok[tok_i], hj.tokens + static_cast<long>(gmb) * hj.M, tb, cudaMemcpyHostToDevice,
                                 w.down),
                 "tok h2d");
      check_cuda(xfer(w.tok[tok_i] + hj.M, hj.targets + static_cast<long>(gmb) * hj.M, tb,
                                 cudaMemcpyHostToDevice, w.down),
                 "tgt h2d");
      w.tok_tr[tok_i].after_write(w.down);
      w.tok_tag[tok_i] = tt;
      w.st.h2d_bytes += 2.0 * static_cast<double>(tb);
    }
  }
  // act buffers: find resident or load
  auto find_tag = [](const Tag* tags, int n, const Tag& want_tag) {
    for (int i = 0; i < n; ++i) {
      if (tags[i] == want_tag) return i;
    }
    return -1;
  };
  int ain = -1;  // abuf holding the shard's input activation (boundary s-1)
  if (s > 0) {
    const Tag at{j, gmb, s - 1, 0};
    ain = find_tag(w.abuf_tag, 2, at);
    if (ain < 0) {
      ain = 0;
      // don't clobber a resident buffer that the forward output will need: pick the older
      if (w.abuf_tag[0].job >= 0 && w.abuf_tag[1].job < 0) ain = 1;
      if (w.abuf_dirty[ain] && !w.abuf_dirty[1 - ain]) ain = 1 - ain;  // keep live content resident
      spill_boundary(w, ain, false);
      std::lock_guard<std::mutex> lk(peer_mu);
      w.abuf_tag[ain] = Tag{};
      w.abuf_tr[ain].before_write(w.down);
      if (!peer_fetch(w, w.abuf[ain], at, false, act_bytes)) {
        hj.ckpt_tr[static_cast<size_t>(s - 1)]->before_read(w.down);
        mark(tm.pr0, w.down, pr0_done);
        check_cuda(xfer(w.abuf[ain], hj.ckpt[static_cast<size_t>(s - 1)], act_bytes, cudaMemcpyHostToDevice,
                                   w.down),
                   "act h2d");
        hj.ckpt_tr[static_cast<size_t>(s - 1)]->after_read(w.down);
        w.st.act_h2d_bytes += static_cast<double>(act_bytes);
        w.st.h2d_bytes += static_cast<double>(act_bytes);
      }
      w.abuf_tr[ain].after_write(w.down);
      w.abuf_tag[ain] = at;
    } else {
      w.st.elided_act_bytes += static_cast<double>(act_bytes);
    }
  }
  int gin = -1;  // gbd holding dL/d(boundary s) for a backward task
  if (!fwd && s < k - 1) {
    const Tag gt{j, gmb, s, 1};
    gin = find_tag(w.gbd_tag, 2, gt);
    if (gin < 0) {
      gin = w.gbd_dirty[0] && !w.gbd_dirty[1] ? 1 : 0;
      spill_boundary(w, gin, true);
      std::lock_guard<std::mutex> lk(peer_mu);
      w.gbd_tag[gin] = Tag{};
      w.gbd_tr[gin].before_write(w.down);
      if (!peer_fetch(w, w.gbd[gin], gt, true, act_bytes)) {
        hj.grad_tr[static_cast<size_t>(s)]->before_read(w.down);
        mark(tm.pr0, w.down, pr0_done);
        check_cuda(xfer(w.gbd[gin], hj.grad[static_cast<size_t>(s)], act_bytes, cudaMemcpyHostToDevice,
                                   w.down),
                   "grad h2d");
        hj.grad_tr[static_cast<size_t>(s)]->after_read(w.down);
        w.st.act_h2d_bytes += static_cast<double>(act_bytes);
        w.st.h2d_bytes += static_cast<double>(act_bytes);
      }
      w.gbd_tr[gin].after_write(w.down);
      w.gbd_tag[gin] = gt;
    } else {
      w.st.elided_act_bytes += static_cast<double>(act_bytes);
    }
  }
  const bool needs_z = !fwd && g.has_embed && !g.has_head;
  if (needs_z) {
    const Tag zt{j, gmb, 0, 2};
    if (!(w.z_tag == zt)) {
      w.z_tr.before_write(w.down);
      hj.z_tr->before_read(w.down);
      mark(tm.pr0, w.down, pr0_done);
      check_cuda(xfer(w.zbuf, hj.z, act_bytes, cudaMemcpyHostToDevice, w.down), "z h2d");
      hj.z_tr->after_read(w.down);
      w.z_tr.after_write(w.down);
      w.z_tag = zt;
      w.st.h2d_bytes += static_cast<double>(act_bytes);
    }
  }
  mark(tm.pr0, w.down, pr0_done);
  check_cuda(cudaEventRecord(tm.pr1, w.down), "pr1");

  // ---- Compute (comp) ---------------------------------------------------------------
  std::vector<int> host_dirty;  // layers of this backward updated host-side
  hy::Scratch sc;
  hy::carve_scratch(hj.m, hy::stash_blocks(hj.geom), w.scratch, &sc, exec.precision_bf16);
  if (w.stg_alias) {
    for (int i = 0; i < kStaging; ++i) w.stg_tr[i].before_write(w.comp);  // scratch reused as staging
  }
  {
  HY_PROF(w.comp, fwd ? "wait_task_F" : "wait_task_B");
  pe->tr.before_read(w.comp);
  if (wte_ext) w.gembed_tr.before_read(w.comp);
  if (need_tokens) w.tok_tr[tok_i].before_read(w.comp);
  if (ain >= 0) w.abuf_tr[ain].before_read(w.comp);
  if (gin >= 0) w.gbd_tr[gin].before_read(w.comp);
  if (needs_z) w.z_tr.before_read(w.comp);
  }
  check_cuda(cudaEventRecord(tm.c0, w.comp), "c0");
  int aout = -1, gout = -1;
  if (fwd) {
    io.tokens = need_tokens ? w.tok[tok_i] : nullptr;
    io.act_in = ain >= 0 ? w.abuf[ain] : nullptr;
    if (!g.has_head) {
      aout = ain >= 0 ? 1 - ain : (w.abuf_tag[0].job < 0 ? 0 : (w.abuf_tag[1].job < 0 ? 1 : 0));
      if (ain < 0 && w.abuf_dirty[aout] && !w.abuf_dirty[1 - aout]) aout = 1 - aout;
      spill_boundary(w, aout, false);
      std::lock_guard<std::mutex> lk(peer_mu);
      w.abuf_tag[aout] = Tag{};  // being overwritten: no peer may copy the old content now
      w.abuf_tr[aout].before_write(w.comp);
      io.act_out = w.abuf[aout];
    }
  } else {
    io.tokens = need_tokens ? w.tok[tok_i] : nullptr;
    io.act_in = ain >= 0 ? w.abuf[ain] : nullptr;
    io.grad_in = gin >= 0 ? w.gbd[gin] : nullptr;
    if (s > 0) {
      gout = gin >= 0 ? 1 - gin : (w.gbd_dirty[0] && !w.gbd_dirty[1] ? 1 : 0);
      spill_boundary(w, gout, true);
      std::lock_guard<std::mutex> lk(peer_mu);
      w.gbd_tag[gout] = Tag{};
      w.gbd_tr[gout].before_write(w.comp);
      io.grad_out = w.gbd[gout];
    }
    if (needs_z) io.z_in = w.zbuf;
  }
  io.wte = wte_ext;
  // targets live in the second half of the token buffer ([tokens | targets], 2*M ints)
  io.targets = need_tokens ? w.tok[tok_i] + hj.M : nullptr;
  // F of the head shard has no boundary output: when its B follows on this GPU (always
  // with double buffering) the B task's forward recompute is the forward, and reports the
  // loss. The plan and the transfers are unchanged; only the duplicate compute is elided.
  bool skip_fwd = false;
  if (fwd && g.has_head && local + 1 < static_cast<int>(w.tasks.size())) {
    const ShardTask& nx = tasks[static_cast<size_t>(w.tasks[static_cast<size_t>(local) + 1])].t;
    skip_fwd = nx.job == j && nx.minibatch == task.t.minibatch && nx.shard == s &&
               nx.direction == Direction::kBackward;
  }
  if (g_debug_skip == 2) skip_fwd = true;
  const Tag my_stash{j, gmb, s, 4};
  // this shard's stash region: its own slice of stash_ext when the arena has room for one per
  // shard (shards 1.., not the head), the head shard's after the others' (StashPlan), else the
  // scratch's shared stash (region 0)
  int stash_region = 0;
  float* stash_base = sc.stash;
  {
    const hy::StashPlan sp = hy::stash_plan(hj.geom);
    if (g.has_head && sp.head_offset > 0) {
      stash_region = 1;
      stash_base = sc.stash + static_cast<long>(sp.head_offset) * hj.n_act;
    } else if (!g.has_head && s > 0 && w.stash_ext &&
               static_cast<long>(hy::ext_stash_offset(hj.geom, s) + g.n_blocks) * hj.n_act <= w.stash_ext_floats) {
      stash_region = 2 + s;
      stash_base = w.stash_ext + static_cast<long>(hy::ext_stash_offset(hj.geom, s)) * hj.n_act;
    }
  }
  io.stash = stash_base;
  if (fwd && !skip_fwd) {
    io.keep_stash = !g.has_head && g.n_blocks > 0 && g_debug_skip == 0;
    hy::run_forward(w.comp, hj.m, g, pbase, io, sc);
    // a forward without the kept stash ping-pongs through the shared stash's first slot
    if (g.n_blocks > 0 || g.has_embed) w.stash_tags[io.keep_stash ? stash_region : 0] = io.keep_stash ? my_stash : Tag{};
    if (g.has_head) {
      check_cuda(cudaMemcpyAsync(w.loss_dev + local, sc.loss, sizeof(double), cudaMemcpyDeviceToDevice, w.comp),
                 "loss copy");
    }
  } else if (fwd) {
    w.st.elided_compute_tasks += 1;
  } else {
    // Gradients stream into the optimizer layer by layer (StreamingSink -> adam_layer on
    // the opt stream, zero-copy: host params / m / v of the shard are rewritten by the
    // optimizer kernels themselves; host-placed layers go through host_adam_layer).
    Tracked& ptr = *hj.params_tr[static_cast<size_t>(s)];
    Tracked& mvt = *hj.mv_tr[static_cast<size_t>(s)];
    mvt.before_read(w.opt);
    mvt.before_read(w.optin);
    ptr.before_write(w.up);
    mvt.before_write(w.up);
    check_cuda(cudaEventRecord(tm.d0, w.up), "d0");
    StreamingSink sink(*this, w, hj, s, pbase, gmb + 1, need_tokens ? w.tok[tok_i] : nullptr);
    sink.deferred = w.stg_alias;
    if (g_debug_skip == 2) {  // gradients "computed": only the optimizer/transfer pipeline runs
      if (g.has_embed) sink.acquire(0);
      if (g.has_head) {
        sink.acquire(hj.m.L + 1);
        sink.release(hj.m.L + 1);
      }
      for (int l = std::min(g.l1, hj.m.L + 1) - 1; l >= std::max(g.l0, 1); --l) {
        sink.acquire(l);
        sink.release(l);
      }
      if (g.has_embed) sink.release(0);
    } else {
      if (g.has_head && !g.has_embed) {
        w.z_tr.before_write(w.comp);
        io.z_out = w.zbuf;
      }
      io.stash_ready = g.n_blocks > 0 && w.stash_tags[stash_region] == my_stash;
      if (io.stash_ready) w.st.stash_reuses += 1;
      hy::run_backward(w.comp, hj.m, g, pbase, sink, io, sc);
      if (g.n_blocks > 0 || g.has_embed) w.stash_tags[stash_region] = Tag{};  // consumed / rewritten
    }
    if (w.stg_alias) {
      for (int i = 0; i < kStaging; ++i) w.stg_tr[i].after_write(w.comp);  // staging = scratch: after the backward
    }
    sink.flush();
    host_dirty = sink.host_layers;
    if (hj.write_back) {
      for (int l = g.l0; l < g.l1; ++l) {
        if (!hj.host_layer[static_cast<size_t>(l)] &&
            std::find(pe->gpu_dirty.begin(), pe->gpu_dirty.end(), l) == pe->gpu_dirty.end()) {
          pe->gpu_dirty.push_back(l);
        }
      }
    }
    mvt.after_read(w.opt);
    mvt.after_read(w.optin);
    ptr.after_write(w.up);
    mvt.after_write(w.up);
    pe->tr.after_write(w.opt);  // Adam rewrote the params in place (opt waited for opt2)
    pe->tr.after_read(w.up);    // ... and the up stream writes them back
    if (g.has_head && !g.has_embed) {  // run_backward saved the ln_f output (io.z_out)
      w.z_tr.after_write(w.comp);
      w.z_tag = Tag{j, gmb, 0, 2};
    }
    if (g.has_head) {  // the backward's recompute produced this minibatch's loss
      check_cuda(cudaMemcpyAsync(w.loss_dev + local, sc.loss, sizeof(double), cudaMemcpyDeviceToDevice, w.comp),
                 "loss copy");
    }
  }
  check_cuda(cudaEventRecord(tm.c1, w.comp), "c1");
  pe->tr.after_read(w.comp);
  if (wte_ext) w.gembed_tr.after_read(w.comp);
  // F(0) of a job whose head shard lacks the embedding: cache the (current) wte in gembed
  if (fwd && g.has_embed && !g.has_head && hj.geom.back().wte_offset >= 0 && w.gembed) {
    const Tag wt{j, -1, -2, hj.version[0]};
    if (!(w.gembed_tag == wt)) {
      w.gembed_tr.before_write(w.comp);
      check_cuda(cudaMemcpyAsync(w.gembed, pbase, sizeof(float) * static_cast<size_t>(hj.m.V) * hj.m.d,
                                 cudaMemcpyDeviceToDevice, w.comp),
                 "wte cache");
      w.gembed_tr.after_write(w.comp);
      w.gembed_tag = wt;
    }
  }
  if (need_tokens) w.tok_tr[tok_i].after_read(w.comp);
  if (ain >= 0) w.abuf_tr[ain].after_read(w.comp);
  if (gin >= 0) w.gbd_tr[gin].after_read(w.comp);
  if (needs_z) w.z_tr.after_read(w.comp);
  if (aout >= 0) {
    std::lock_guard<std::mutex> lk(peer_mu);
    w.abuf_tr[aout].after_write(w.comp);
    w.abuf_tag[aout] = Tag{j, gmb, s, 0};
  }
  if (gout >= 0) {
    std::lock_guard<std::mutex> lk(peer_mu);
    w.gbd_tr[gout].after_write(w.comp);
    w.gbd_tag[gout] = Tag{j, gmb, s - 1, 1};
  }

  // ---- ActDemote + GradOffload (up) ---------------------------------------------------
  // Write-back jobs (every task on this GPU) keep boundary activations / gradients resident
  // and demote them only if their buffer is reused before the last consumer (spill_boundary):
  // B(s+1) reads activation s from here, B(s-1) gradient s-1. With two buffers per kind, the
  // activations of all but the last two boundaries are reused by the forward before their
  // backward, so those still go out eagerly right behind their producer (no stall later).
  // The reference's transfers (the plan) are unchanged; only physical copies are elided.
  if (!fwd) {  // B(s) was the last consumer of activation s-1 and of gradient s: dead now
    for (int i = 0; i < 2; ++i) {
      if (w.abuf_tag[i] == Tag{j, gmb, s - 1, 0}) w.abuf_dirty[i] = false;
      if (w.gbd_tag[i] == Tag{j, gmb, s, 1}) w.gbd_dirty[i] = false;
    }
  }
  if (aout >= 0 && hj.write_back && s >= k - 3) {
    w.abuf_dirty[aout] = true;
    w.st.elided_act_bytes += static_cast<double>(act_bytes);
    aout = -1;
  }
  if (gout >= 0 && hj.write_back) {
    w.gbd_dirty[gout] = true;
    w.st.elided_act_bytes += static_cast<double>(act_bytes);
    gout = -1;
  }
  if (aout >= 0) {  // forward boundary activation -> checkpoint store
    Tracked& host = *hj.ckpt_tr[static_cast<size_t>(s)];
    w.abuf_tr[aout].before_read(w.up);
    host.before_write(w.up);
    mark(tm.d0, w.up, d0_done);
    check_cuda(xfer(hj.ckpt[static_cast<size_t>(s)], w.abuf[aout], act_bytes, cudaMemcpyDeviceToHost, w.up),
               "act d2h");
    host.after_write(w.up);
    w.abuf_tr[aout].after_read(w.up);
    w.st.act_d2h_bytes += static_cast<double>(act_bytes);
    w.st.d2h_bytes += static_cast<double>(act_bytes);
  }
  if (gout >= 0) {  // dL/d(input boundary) -> host
    Tracked& host = *hj.grad_tr[static_cast<size_t>(s - 1)];
    w.gbd_tr[gout].before_read(w.up);
    host.before_write(w.up);
    mark(tm.d0, w.up, d0_done);
    check_cuda(xfer(hj.grad[static_cast<size_t>(s - 1)], w.gbd[gout], act_bytes, cudaMemcpyDeviceToHost,
                               w.up),
               "grad d2h");
    host.after_write(w.up);
    w.gbd_tr[gout].after_read(w.up);
    w.st.act_d2h_bytes += static_cast<double>(act_bytes);
    w.st.d2h_bytes += static_cast<double>(act_bytes);
  }
  if (!fwd && g.has_head && !g.has_embed) {  // saved ln_f output for shard 0's tied-wte grad
    w.z_tr.before_read(w.up);
    hj.z_tr->before_write(w.up);
    mark(tm.d0, w.up, d0_done);
    check_cuda(xfer(hj.z, w.zbuf, act_bytes, cudaMemcpyDeviceToHost, w.up), "z d2h");
    hj.z_tr->after_write(w.up);
    w.z_tr.after_read(w.up);
    w.st.d2h_bytes += static_cast<double>(act_bytes);
  }
  mark(tm.d0, w.up, d0_done);
  check_cuda(cudaEventRecord(tm.d1, w.up), "d1");
  if (!fwd) {
    hj.version[static_cast<size_t>(s)] += 1;
    pe->tag = Tag{j, -1, s, hj.version[static_cast<size_t>(s)]};
    pe->dirty.insert(pe->dirty.end(), host_dirty.begin(), host_dirty.end());
  }
  w.prev_entry = pe;
  {
    std::lock_guard<std::mutex> lk(flag_mu);
    enqueued_pass[static_cast<size_t>(t)] = pass;
  }
  flag_cv.notify_all();
}

// P2P hand-off (BoundaryOut::kPeer's role for SHARP chains that change GPU): when a
// task's boundary input is still resident on another GPU of this process (the producer ran
// there), copy it over NVLink on this GPU's down stream instead of promoting it from the host
// checkpoint (the producer's ActDemote still writes the checkpoint, as the reference does). The
// copy waits for the producer's write on the other GPU and registers a read, so the producer's
// next reuse of that buffer waits for it. Caller holds peer_mu.
bool ExecutorImpl::peer_fetch(Worker& w, float* dst, const Tag& want, bool grad, size_t bytes) {
  if (!exec.p2p || workers.size() < 2) return false;
  for (auto& op : workers) {
    Worker& o = *op;
    if (&o == &w) continue;
    for (int i = 0; i < 2; ++i) {
      if (!((grad ? o.gbd_tag[i] : o.abuf_tag[i]) == want)) continue;
      Tracked& src = grad ? o.gbd_tr[i] : o.abuf_tr[i];
      src.before_read(w.down);
      check_cuda(cudaMemcpyPeerAsync(dst, w.cuda_dev, grad ? o.gbd[i] : o.abuf[i], o.cuda_dev, bytes, w.down),
                 "p2p hand-off");
      src.after_read(w.down);
      w.st.p2p_bytes += static_cast<double>(bytes);
      return true;
    }
  }
  return false;
}

// Dynamic-time scheduling (ExecOptions::dynamic): instead of replaying the virtual engine's
// dispatch log, every GPU's worker asks the strategy's own TaskScheduler (a fresh instance per
// pass, shared under one mutex, so its single-threaded semantics hold) with the engine's
// protocol (sim.cpp enqueue / start_compute / compute_finished / finish): an idle GPU asks
// next_task(dev, false, -1); when a task starts computing with nothing queued behind it the
// GPU asks for a prefetch next_task(dev, true, task) whose loads overlap that compute; a task
// completes (on_complete) when its compute ends on the device (CUDA event), and idle GPUs
// re-ask. Durations are therefore the
// real ones: which GPU frees up first, and so which job goes where, follows the hardware
// rather than the cost model.
void ExecutorImpl::dynamic_dispatch(Worker& w, int pass) {
  w.tasks.clear();
  std::deque<int> queue;  // dispatched, compute not yet finished
  auto dispatch = [&](int t, bool prefetch) {
    task_device[static_cast<size_t>(t)] = w.plan_dev;
    task_local[static_cast<size_t>(t)] = static_cast<int>(w.tasks.size());
    w.tasks.push_back(t);
    dyn.sched->on_dispatch(t, w.plan_dev);
    dyn.log.push_back(Dispatch{t, w.plan_dev, prefetch, 0.0});
  };
  const int total = static_cast<int>(tasks.size());
  for (;;) {
    if (queue.empty()) {  // idle GPU: ask for new work
      int t = -1;
      {
        std::unique_lock<std::mutex> lk(dyn.mu);
        if (dyn.done >= total) break;
        const std::optional<int> pick = dyn.sched->next_task(w.plan_dev, false, -1);
        if (pick) {
          t = *pick;
          dispatch(t, false);
        } else {
          dyn.cv.wait_for(lk, std::chrono::milliseconds(1));  // until another GPU completes a task
          continue;
        }
      }
      enqueue_task(w, t, pass);
      queue.push_back(t);
    }
    const int front = queue.front();
    if (queue.size() == 1 && options.double_buffering) {  // front starts computing: prefetch ask
      int t2 = -1;
      {
        std::lock_guard<std::mutex> lk(dyn.mu);
        const std::optional<int> pick = dyn.sched->next_task(w.plan_dev, true, front);
        if (pick) {
          t2 = *pick;
          dispatch(t2, true);
        }
      }
      if (t2 >= 0) {
        enqueue_task(w, t2, pass);
        queue.push_back(t2);
      }
    }
    const TaskTiming& tm = w.timing[static_cast<size_t>(task_local[static_cast<size_t>(front)])];
    check_cuda(cudaEventSynchronize(tm.c1), "compute done");
    queue.pop_front();
    {
      // The engine completes a task before its chain successor may start computing (the
      // successor's predecessors include it); here its drains may still be in flight, but
      // every data hazard is ordered on the device, so the scheduler is told now.
      std::lock_guard<std::mutex> lk(dyn.mu);
      dyn.sched->on_complete(front);
      ++dyn.done;
    }
    dyn.cv.notify_all();
  }
}

void ExecutorImpl::spill_boundary(Worker& w, int i, bool grad) {
  bool& dirty = grad ? w.gbd_dirty[i] : w.abuf_dirty[i];
  if (!dirty) return;
  dirty = false;
  const Tag t = grad ? w.gbd_tag[i] : w.abuf_tag[i];
  if (t.job < 0) return;
  HostJob& oj = jobs.at(t.job);
  const size_t bytes = sizeof(float) * static_cast<size_t>(oj.n_act);
  Tracked& dev = grad ? w.gbd_tr[i] : w.abuf_tr[i];
  Tracked& host = grad ? *oj.grad_tr[static_cast<size_t>(t.idx)] : *oj.ckpt_tr[static_cast<size_t>(t.idx)];
  float* dst = grad ? oj.grad[static_cast<size_t>(t.idx)] : oj.ckpt[static_cast<size_t>(t.idx)];
  dev.before_read(w.up);
  host.before_write(w.up);
  check_cuda(xfer(dst, grad ? w.gbd[i] : w.abuf[i], bytes, cudaMemcpyDeviceToHost, w.up),
             grad ? "grad spill d2h" : "act spill d2h");
  host.after_write(w.up);
  dev.after_read(w.up);
  w.st.act_d2h_bytes += static_cast<double>(bytes);
  w.st.d2h_bytes += static_cast<double>(bytes);
  w.st.elided_act_bytes -= static_cast<double>(bytes);
}

}  // namespace spillsim
