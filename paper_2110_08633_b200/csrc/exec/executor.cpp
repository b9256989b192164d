// Plan-mode B200 executor: replays the virtual engine's dispatch plan on real GPUs.
//
// One host worker thread per GPU enqueues its task list asynchronously on five streams:
//   down    ParamLoad + ActPromote  (H2D, pinned host -> HBM; the reference's down channel)
//   comp    shard forward / recompute+backward (sm_100a kernels)
//   up      ActDemote (D2H) + the gradients of host-placed layers (GradOffload)
//   opt     GPU-placed AdamW: zero-copy kernels that read m, v from pinned host memory and
//           write params, m, v back over the link, layer by layer as the backward releases
//           them (the reference folds the optimizer into GradOffload)
//   hopt    host-placed AdamW (cudaLaunchHostFunc, OpenMP) after the gradient's D2H
// Double buffering falls out of the stream structure: task t+1's ParamLoad is enqueued right
// after task t's compute and runs on the copy engine while t computes (slot t+1 only waits
// for slot t-1's last reader). Every buffer shared between streams carries a hazard tracker
// (last-writer / last-reader-per-stream CUDA events), so no host-side synchronisation is
// needed inside a pass. Physical optimisations that keep the plan unchanged: a ParamLoad is
// skipped when the slot already holds that shard at the current version (B(k-1) after
// F(k-1) — the reference's elision, sim.cpp:356-365 — and F(0) of the next minibatch after
// B(0)); an ActPromote is skipped when the producer's output is still resident on this GPU.
#include <limits>
#include <set>

#include "executor_impl.hpp"

namespace spillsim {

namespace exec_detail {
int g_debug_skip = 0;
}  // namespace exec_detail

ExecutorImpl::~ExecutorImpl() {
  for (auto& wp : workers) {
    Worker& w = *wp;
    cudaSetDevice(w.cuda_dev);
    cudaDeviceSynchronize();
    for (auto& tm : w.timing) {
      for (cudaEvent_t e : {tm.pl0, tm.pl1, tm.pr0, tm.pr1, tm.c0, tm.c1, tm.d0, tm.d1}) {
        if (e) cudaEventDestroy(e);
      }
    }
    for (int i = 0; i < 2; ++i) {
      (void)i;
      w.abuf_tr[i].destroy();
      w.gbd_tr[i].destroy();
      w.tok_tr[i].destroy();
    }
    for (int i = 0; i < kStaging; ++i) w.stg_tr[i].destroy();
    w.rowidx_tr.destroy();
    w.cbuf_tr.destroy();
    for (cudaEvent_t e : w.ev_pool) cudaEventDestroy(e);
    if (w.gembed_free) cudaEventDestroy(w.gembed_free);
    for (auto& e : w.live) e->tr.destroy();
    for (auto& e : w.retired) e->tr.destroy();
    for (auto& kv : w.mv_live) kv.second->tr.destroy();
    for (auto& e : w.mv_retired) e->tr.destroy();
    if (w.mv_free) cudaEventDestroy(w.mv_free);
    w.gembed_tr.destroy();
    w.z_tr.destroy();
    for (cudaEvent_t e : {w.t0, w.t_end, w.join[0], w.join[1], w.join[2], w.join[3], w.join[4], w.join[5],
                          w.dense_done}) {
      if (e) cudaEventDestroy(e);
    }
    if (w.arena) cudaFree(w.arena);
    for (cudaStream_t s : {w.comp, w.down, w.up, w.opt, w.opt2, w.hopt, w.optin}) {
      if (s) cudaStreamDestroy(s);
    }
  }
  for (auto& kv : jobs) {
    HostJob& hj = kv.second;
    for (auto& t : hj.params_tr) t->destroy();
    for (auto& t : hj.mv_tr) t->destroy();
    for (auto& t : hj.ckpt_tr) t->destroy();
    for (auto& t : hj.grad_tr) t->destroy();
    for (auto& t : hj.hgrad_tr) t->destroy();
    for (auto& t : hj.hparams_tr) t->destroy();
    if (hj.z_tr) hj.z_tr->destroy();
    for (void* p : {static_cast<void*>(hj.params), static_cast<void*>(hj.mom), static_cast<void*>(hj.var),
                    static_cast<void*>(hj.z), static_cast<void*>(hj.tokens), static_cast<void*>(hj.targets)}) {
      if (p) cudaFreeHost(p);
    }
    for (float* p : hj.ckpt) cudaFreeHost(p);
    for (float* p : hj.grad) cudaFreeHost(p);
    if (hj.hgrad) cudaFreeHost(hj.hgrad);
  }
  if (host_loss) cudaFreeHost(host_loss);
}


void* exec_detail::pinned(size_t bytes) {
  void* p = nullptr;
  // mapped: the zero-copy optimizer kernels read / write moments and params in place (UVA:
  // the device pointer is the host pointer)
  check_cuda(cudaHostAlloc(&p, bytes ? bytes : 4, cudaHostAllocPortable | cudaHostAllocMapped), "cudaHostAlloc");
  return p;
}


double exec_detail::host_available_bytes() {
  // MemAvailable of /proc/meminfo minus a 4 GB margin for the process itself; +inf if unknown
  FILE* f = std::fopen("/proc/meminfo", "r");
  if (!f) return std::numeric_limits<double>::infinity();
  char line[256];
  double kb = -1;
  while (std::fgets(line, sizeof line, f)) {
    if (std::sscanf(line, "MemAvailable: %lf kB", &kb) == 1) break;
  }
  std::fclose(f);
  if (kb < 0) return std::numeric_limits<double>::infinity();
  return std::max(0.0, kb * 1024.0 - 4e9);
}

double ExecutorImpl::host_job_pinned_bytes(int j) const {
  // mirrors setup_host_job's pinned allocations
  const ExecJob& spec = exec.jobs.at(static_cast<size_t>(j));
  const hy_dims m = spec.dims;
  const double total = static_cast<double>(hy_total_floats(&m));
  const double n_act = static_cast<double>(m.B) * m.T * m.d;
  const double k = static_cast<double>(spec.shard_starts.size());
  const double n_gmb = static_cast<double>(job_mb[static_cast<size_t>(j)]) * (exec.passes + exec.warmup_passes);
  double b = 4.0 * total + 2.0 * (exec.opt_state_bf16 ? 2.0 : 4.0) * total;  // params, m, v
  b += 4.0 * n_act * (2.0 * (k - 1) + 1.0);                                  // checkpoints, grads, z
  b += 8.0 * static_cast<double>(m.B) * m.T * n_gmb;                         // tokens, targets
  if (exec.host_opt_fraction > 0) b += 4.0 * total;                          // host-optimizer grads
  return b;
}

void ExecutorImpl::setup_host_job(int j) {
  HostJob& hj = jobs[j];
  const ExecJob& spec = exec.jobs.at(static_cast<size_t>(j));
  hj.spec = &spec;
  hj.job = j;
  hj.m = spec.dims;
  hj.M = static_cast<long>(hj.m.B) * hj.m.T;
  hj.n_act = hj.M * hj.m.d;
  hj.total = hy_total_floats(&hj.m);
  const int n_layers = hj.m.L + 2;
  const std::vector<int>& starts = spec.shard_starts;
  const int k = static_cast<int>(starts.size());
  for (int s = 0; s < k; ++s) {
    hj.geom.push_back(hy::shard_geom(hj.m, starts[static_cast<size_t>(s)],
                                     s + 1 < k ? starts[static_cast<size_t>(s) + 1] : n_layers));
  }
  hj.params = static_cast<float*>(pinned(sizeof(float) * static_cast<size_t>(hj.total)));
  const size_t state_bytes = (exec.opt_state_bf16 ? 2 : 4) * static_cast<size_t>(hj.total);
  hj.mom = static_cast<float*>(pinned(state_bytes));
  hj.var = static_cast<float*>(pinned(state_bytes));
  // GPT-2 init, layers in parallel (each layer's stream is independent of the others).
#pragma omp parallel for schedule(dynamic)
  for (int l = 0; l < n_layers; ++l) hy_init_layer(&hj.m, spec.model_key, l, hj.params + hy_layer_offset(&hj.m, l));
  std::memset(hj.mom, 0, state_bytes);
  std::memset(hj.var, 0, state_bytes);
  for (int b = 0; b + 1 < k; ++b) {
    hj.ckpt.push_back(static_cast<float*>(pinned(sizeof(float) * static_cast<size_t>(hj.n_act))));
    hj.grad.push_back(static_cast<float*>(pinned(sizeof(float) * static_cast<size_t>(hj.n_act))));
    hj.ckpt_tr.emplace_back(new Tracked);
    hj.grad_tr.emplace_back(new Tracked);
  }
  hj.z = static_cast<float*>(pinned(sizeof(float) * static_cast<size_t>(hj.n_act)));
  hj.z_tr.reset(new Tracked);
  for (int s = 0; s < k; ++s) {
    hj.params_tr.emplace_back(new Tracked);
    hj.mv_tr.emplace_back(new Tracked);
    hj.hparams_tr.emplace_back(new Tracked);
  }
  // Host-placed optimizer layers: from the head-side shards down (in a SHARP chain the shards
  // a backward task leaves behind are the ones reloaded before their next use anyway, so the
  // host update costs the link nothing extra; shards 0 and 1 stay resident into the next
  // minibatch's first forwards and would need a refresh), each shard's layers in the order
  // the backward releases them (head, last block .. first block, embedding).
  hj.host_layer.assign(static_cast<size_t>(n_layers), 0);
  if (exec.host_opt_fraction > 0) {
    const double target = exec.host_opt_fraction * static_cast<double>(hj.total);
    double acc = 0;
    for (int s = k - 1; s >= 0 && acc < target; --s) {
      const int l0 = starts[static_cast<size_t>(s)];
      const int l1 = s + 1 < k ? starts[static_cast<size_t>(s) + 1] : n_layers;
      for (int l = l1 - 1; l >= l0 && acc < target; --l) {
        const double n = static_cast<double>(hy_layer_floats(&hj.m, l));
        if (acc + 0.5 * n > target) continue;
        hj.host_layer[static_cast<size_t>(l)] = 1;
        acc += n;
      }
    }
    if (acc > 0) hj.hgrad = static_cast<float*>(pinned(sizeof(float) * static_cast<size_t>(hj.total)));
  }
  for (int l = 0; l < n_layers; ++l) hj.hgrad_tr.emplace_back(new Tracked);
  hj.version.assign(static_cast<size_t>(k), 0);
  hj.n_gmb = job_mb[static_cast<size_t>(j)] * (exec.passes + exec.warmup_passes);
  hj.tokens = static_cast<int32_t*>(pinned(sizeof(int32_t) * static_cast<size_t>(hj.M * hj.n_gmb)));
  hj.targets = static_cast<int32_t*>(pinned(sizeof(int32_t) * static_cast<size_t>(hj.M * hj.n_gmb)));
#pragma omp parallel for schedule(static)
  for (int g = 0; g < hj.n_gmb; ++g) {
    for (int r = 0; r < hj.m.B; ++r) {
      for (int t = 0; t < hj.m.T; ++t) {
        const long i = static_cast<long>(g) * hj.M + static_cast<long>(r) * hj.m.T + t;
        hj.tokens[i] = hy_token(exec.seed, j, g, r, t);
        hj.targets[i] = hy_token(exec.seed, j, g, r, t + 1);
      }
    }
  }
}

void ExecutorImpl::setup_worker(Worker& w) {
  check_cuda(cudaSetDevice(w.cuda_dev), "set device");
  {
    static const int comp_prio = [] {  // diagnostics: HY_COMP_PRIORITY=1 runs the compute stream at high priority
      const char* v = std::getenv("HY_COMP_PRIORITY");
      return v ? std::atoi(v) : 0;
    }();
    int lo = 0, hi = 0;
    check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    check_cuda(cudaStreamCreateWithPriority(&w.comp, cudaStreamNonBlocking, comp_prio ? hi : 0), "stream");
  }
  check_cuda(cudaStreamCreateWithFlags(&w.down, cudaStreamNonBlocking), "stream");
  check_cuda(cudaStreamCreateWithFlags(&w.up, cudaStreamNonBlocking), "stream");
  // the Adam kernels sit between an H2D and a D2H copy of each moment chunk: at high priority the
  // block scheduler runs them ahead of queued compute blocks so the link pipeline does not drain
  int prio_lo = 0, prio_hi = 0;
  if (exec.opt_priority) check_cuda(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "priority range");
  check_cuda(cudaStreamCreateWithPriority(&w.opt, cudaStreamNonBlocking, prio_hi), "stream");
  check_cuda(cudaStreamCreateWithFlags(&w.hopt, cudaStreamNonBlocking), "stream");
  check_cuda(cudaStreamCreateWithPriority(&w.opt2, cudaStreamNonBlocking, prio_hi), "stream");
  check_cuda(cudaStreamCreateWithFlags(&w.optin, cudaStreamNonBlocking), "stream");
  // Size the arena from the tasks this GPU will run.
  bool all_write_back = true;
  long model_f = 0;  // the largest job's parameters (all shards): what the cache can usefully hold
  for (int t : w.tasks) {
    const HostJob& hj = jobs.at(tasks[static_cast<size_t>(t)].t.job);
    all_write_back = all_write_back && hj.write_back;
    long sum = 0;
    for (const ShardGeom& sg : hj.geom) sum += hy_pad32(sg.param_floats);
    model_f = std::max(model_f, sum + 256L * static_cast<long>(hj.geom.size()));
  }
  long slot_f = 0, embed_f = 0, layer_f = 0, act_f = 0, scratch_f = 0, tok_n = 0, idx_n = 0, list_n = 0, crow = 0;
  for (int t : w.tasks) {
    const HostJob& hj = jobs.at(tasks[static_cast<size_t>(t)].t.job);
    const ShardGeom& g = hj.geom[static_cast<size_t>(tasks[static_cast<size_t>(t)].t.shard)];
    slot_f = std::max(slot_f, g.param_floats);
    if (g.has_embed || g.wte_offset >= 0) embed_f = std::max(embed_f, hy_layer_floats(&hj.m, 0));
    if (g.has_embed) {
      idx_n = std::max(idx_n, static_cast<long>(hj.m.V) + hj.m.T);
      list_n = std::max(list_n, hj.M + hj.m.T);
      crow = std::max(crow, (hj.M + hj.m.T) * static_cast<long>(hj.m.d));
    }
    for (int l = std::max(g.l0, 1); l < g.l1; ++l) layer_f = std::max(layer_f, hy_layer_floats(&hj.m, l));
    act_f = std::max(act_f, hj.n_act);
    tok_n = std::max(tok_n, hj.M);
    scratch_f = std::max(scratch_f, hy::scratch_floats(hj.m, hy::stash_blocks(hj.geom), exec.precision_bf16));
  }
  const long base_floats = 2 * hy_pad32(slot_f) + hy_pad32(embed_f) + 5 * hy_pad32(act_f) +
                           2 * hy_pad32(2 * tok_n) + hy_pad32(scratch_f) +
                           hy_pad32(2 * static_cast<long>(w.tasks.size()) + 2) + hy_pad32(idx_n > 0 ? 32 + idx_n + list_n : 0) +
                           hy_pad32((all_write_back ? 2 : 3) * crow);
  const DeviceSpec& dev = cluster.devices[static_cast<size_t>(w.plan_dev)];
  const double cap = dev.mem_bytes + exec.hbm_slack_bytes;
  long budget_floats = static_cast<long>(cap / 4) - base_floats - 2048;
  // gradient ring: at least two of the largest non-embedding layers
  long ring_f = 2 * hy_pad32(layer_f) + 64;
  budget_floats -= ring_f;
  // split-K partials (<= splitk_max_floats) from what the cap leaves, the Adam staging ring, then the
  // parameter cache beyond its two slots
  long splitk_f = std::min(exec.splitk_max_floats, std::max(0L, budget_floats / 4)) / 1024 * 1024;
  if (splitk_f < (256L << 10)) splitk_f = 0;
  budget_floats -= splitk_f;
  // staging: first its base chunk (<= 2M elements), then — after the parameter cache has grown
  // toward the whole job — up to opt_chunk_floats from what is left: deeper m, v prefetch keeps
  // the host link busier (C2: 2M -> 4M-element chunks took a pass 1.97 -> 1.82 s with 120 MB
  // of extra HBM, tools/skip_sweep.py)
  const long base_chunk = std::min(exec.opt_chunk_floats, 2L << 20);
  long chunk = std::min(base_chunk, budget_floats / (2 * kStaging));
  chunk = chunk / 1024 * 1024;
  // alias the staging ring onto the scratch only when the cap leaves no room for the
  // requested chunks (or for 1M-element chunks, whichever is smaller)
  w.stg_alias = chunk < std::min(base_chunk / 1024 * 1024, 1L << 20);
  if (w.stg_alias) chunk = 0;
  budget_floats -= kStaging * 2 * hy_pad32(chunk);
  if (w.stg_alias) {
    // deferred optimizer: the ring must hold every non-embedding layer of a shard
    long shard_f = 0;
    for (int t : w.tasks) {
      const HostJob& hj = jobs.at(tasks[static_cast<size_t>(t)].t.job);
      const ShardGeom& g = hj.geom[static_cast<size_t>(tasks[static_cast<size_t>(t)].t.shard)];
      long sum = 0;
      for (int l = std::max(g.l0, 1); l < g.l1; ++l) sum += hy_pad32(hy_layer_floats(&hj.m, l));
      shard_f = std::max(shard_f, sum + 64);
    }
    budget_floats -= std::max(0L, shard_f - ring_f);
    ring_f = std::max(ring_f, shard_f);
  }
  // The parameter cache (LRU over shard entries) grows toward the whole of the largest job:
  // shards that stay resident skip their ParamLoad (and, with write-back, their write-back)
  // — physical traffic only, the plan is unchanged.
  long pool_f = 2 * hy_pad32(slot_f);
  if (budget_floats > 0 && model_f > pool_f) {
    long ext = std::min(budget_floats, model_f - pool_f);
    if (exec.pool_extra_max_bytes >= 0) ext = std::min(ext, static_cast<long>(exec.pool_extra_max_bytes / 4));
    ext = ext / 32 * 32;
    pool_f += ext;
    budget_floats -= ext;
  }
  if (!w.stg_alias && chunk > 0 && exec.opt_chunk_floats > chunk && budget_floats > 0) {
    const long grow = std::min(exec.opt_chunk_floats - chunk, budget_floats / (2 * kStaging)) / 1024 * 1024;
    if (grow > 0) {
      budget_floats -= kStaging * 2 * (hy_pad32(chunk + grow) - hy_pad32(chunk));
      chunk += grow;
    }
  }
  // Per-shard stash regions (a forward's block inputs then survive until its shard's backward,
  // which skips its recompute pass): next in line, ahead of the deeper ring and the moment cache —
  // a shard's recompute costs a block forward per block, its moments only link time.
  long stash_ext_f = 0;
  for (int t : w.tasks) {
    const HostJob& hj = jobs.at(tasks[static_cast<size_t>(t)].t.job);
    stash_ext_f = std::max(stash_ext_f, static_cast<long>(hy::ext_stash_slots(hj.geom)) * hj.n_act);
  }
  stash_ext_f = hy_pad32(stash_ext_f);
  if (stash_ext_f <= 0 || stash_ext_f > budget_floats || g_debug_skip != 0) stash_ext_f = 0;
  budget_floats -= stash_ext_f;
  // Spare budget: a deeper gradient ring (up to 4 layers) and optimizer moments kept resident
  // (write-back jobs only). Resident moments save their link bytes every minibatch, so they
  // come first when the budget is tight (exec.ring_first = false); the ring takes the rest.
  auto deepen_ring = [&]() {
    if (budget_floats > 0) {
      const long deep = std::min(budget_floats, 2 * hy_pad32(layer_f)) / 32 * 32;
      ring_f += deep;
      budget_floats -= deep;
    }
  };
  if (exec.ring_first) deepen_ring();
  long mv_f = 0;
  if (exec.mv_cache && all_write_back && !w.stg_alias && budget_floats > (2L << 20)) {
    long job_mv_f = 0;  // the largest job's moments: what the cache can usefully hold
    const long es = exec.opt_state_bf16 ? 2 : 4;
    for (int t : w.tasks) {
      const HostJob& hj = jobs.at(tasks[static_cast<size_t>(t)].t.job);
      job_mv_f = std::max(job_mv_f, (2 * es * hj.total) / 4 + 64L * (hj.m.L + 2));
    }
    mv_f = std::min(budget_floats - (1L << 20), job_mv_f);
    if (exec.mv_cache_max_bytes >= 0) mv_f = std::min(mv_f, static_cast<long>(exec.mv_cache_max_bytes / 4));
    mv_f = mv_f / 256 * 256;
    budget_floats -= mv_f;
  }
  if (!exec.ring_first) deepen_ring();
  if (std::getenv("HY_DEBUG_ARENA")) {  // diagnostics: where the capped HBM goes (MB)
    std::fprintf(stderr,
                 "arena dev %d: slots %.1f embed %.1f act %.1f scratch %.1f crow %.1f | ring %.1f splitk %.1f "
                 "staging %.1f pool+ %.1f stash+ %.1f mv %.1f | left %.1f\n",
                 w.plan_dev, 8.0 * hy_pad32(slot_f) / 1e6, 4.0 * hy_pad32(embed_f) / 1e6, 20.0 * hy_pad32(act_f) / 1e6,
                 4.0 * hy_pad32(scratch_f) / 1e6, 4.0 * (all_write_back ? 2 : 3) * crow / 1e6, 4.0 * ring_f / 1e6,
                 4.0 * splitk_f / 1e6, 4.0 * kStaging * 2 * hy_pad32(chunk) / 1e6,
                 4.0 * (pool_f - 2 * hy_pad32(slot_f)) / 1e6, 4.0 * stash_ext_f / 1e6, 4.0 * mv_f / 1e6,
                 4.0 * budget_floats / 1e6);
  }
  const long floats = base_floats + ring_f + splitk_f + kStaging * 2 * hy_pad32(chunk) + (pool_f - 2 * hy_pad32(slot_f)) +
                      stash_ext_f + mv_f;
  w.arena_bytes = floats * 4 + 4096;
  if (static_cast<double>(w.arena_bytes) > cap) {
    throw InfeasibleOOM("sharp-executor", "(all jobs on this device)", dev.device_id,
                        static_cast<double>(w.arena_bytes), cap);
  }
  check_cuda(cudaMalloc(&w.arena, static_cast<size_t>(w.arena_bytes)), "arena cudaMalloc");
  float* p = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(w.arena) + 1023) & ~uintptr_t(1023));
  auto take = [&](long n) {
    float* r = p;
    p += hy_pad32(n);
    return r;
  };
  w.pool = take(pool_f);
  w.pool_floats = pool_f;
  w.gembed = embed_f > 0 ? take(embed_f) : nullptr;
  w.ring = take(ring_f);
  w.ring_floats = ring_f;
  w.abuf[0] = take(act_f);
  w.abuf[1] = take(act_f);
  w.gbd[0] = take(act_f);
  w.gbd[1] = take(act_f);
  w.zbuf = take(act_f);
  w.tok[0] = reinterpret_cast<int32_t*>(take(2 * tok_n));
  w.tok[1] = reinterpret_cast<int32_t*>(take(2 * tok_n));
  if (!w.stg_alias) {
    for (int i = 0; i < kStaging; ++i) w.stg[i] = take(2 * chunk);
  }
  w.scratch = take(scratch_f);
  w.splitk = splitk_f > 0 ? take(splitk_f) : nullptr;
  w.splitk_floats = splitk_f;
  w.stash_ext = stash_ext_f > 0 ? take(stash_ext_f) : nullptr;
  w.stash_ext_floats = stash_ext_f;
  if (w.stg_alias) {
    // staging inside the scratch fc/act block of the largest job on this GPU
    long best = 0;
    for (int t : w.tasks) {
      const HostJob& hj = jobs.at(tasks[static_cast<size_t>(t)].t.job);
      hy::Scratch sc;
      hy::carve_scratch(hj.m, hy::stash_blocks(hj.geom), w.scratch, &sc, exec.precision_bf16);
      const long avail = 8L * hj.M * hj.m.d;  // fc + act
      if (avail > best) {
        best = avail;
        chunk = avail / (2 * kStaging) / 1024 * 1024;
        for (int i = 0; i < kStaging; ++i) w.stg[i] = sc.fc + static_cast<long>(i) * 2 * chunk;
      }
    }
  }
  w.stg_chunk = chunk;
  if (idx_n > 0) {
    int* ip = reinterpret_cast<int*>(take(32 + idx_n + list_n));
    w.rowcount = ip;
    w.rowidx = ip + 32;
    w.rowlist = w.rowidx + idx_n;
    w.crow_max = crow;
    w.cbuf = take((all_write_back ? 2 : 3) * crow);
  }
  w.loss_dev = reinterpret_cast<double*>(take(2 * static_cast<long>(w.tasks.size()) + 2));
  if (mv_f > 0) {
    w.mvpool = reinterpret_cast<char*>(take(mv_f));
    w.mvpool_bytes = 4 * mv_f;
  }
  for (size_t i = 0; i < w.tasks.size(); ++i) {
    const ShardTask& st = tasks[static_cast<size_t>(w.tasks[i])].t;
    w.last_local_of_job[st.job] = static_cast<int>(i);
    if (st.direction == Direction::kBackward) w.last_b_local[{st.job, st.shard}] = static_cast<int>(i);
  }
  if (!exec.dynamic && !w.tasks.empty()) {
    // the job that follows each job on this GPU; the last one is followed by the first of the
    // next pass (the plan repeats)
    std::vector<int> order;
    for (int t : w.tasks) {
      const int j = tasks[static_cast<size_t>(t)].t.job;
      if (order.empty() || order.back() != j) order.push_back(j);
    }
    for (size_t i = 0; i < order.size(); ++i) w.next_job[order[i]] = order[(i + 1) % order.size()];
  }
  w.mv_free = new_event(false);
  check_cuda(cudaMemset(w.arena, 0, static_cast<size_t>(w.arena_bytes)), "arena memset");
  w.timing.resize(w.tasks.size());
  for (TaskTiming& tm : w.timing) {
    for (cudaEvent_t* e : {&tm.pl0, &tm.pl1, &tm.pr0, &tm.pr1, &tm.c0, &tm.c1, &tm.d0, &tm.d1}) *e = new_event(true);
  }
  for (int i = 0; i < 256; ++i) w.ev_pool.push_back(new_event(false));
  w.gembed_free = new_event(false);
  w.dense_done = new_event(false);
  w.t0 = new_event(true);
  w.t_end = new_event(true);
  for (auto& e : w.join) e = new_event(false);
  w.st.arena_bytes.push_back(static_cast<double>(w.arena_bytes));
}

void ExecutorImpl::setup(ExecResult& res) {
  const auto t_start = std::chrono::steady_clock::now();
  const int G = static_cast<int>(cluster.devices.size());
  std::vector<int> run = exec.run_devices;
  if (run.empty()) {
    for (int d = 0; d < G; ++d) run.push_back(d);
  }
  const auto per_dev = plan.per_device(G);
  task_local.assign(tasks.size(), -1);
  task_device.assign(tasks.size(), -1);
  for (int d = 0; d < G; ++d) {
    for (size_t i = 0; i < per_dev[static_cast<size_t>(d)].size(); ++i) {
      task_device[static_cast<size_t>(per_dev[static_cast<size_t>(d)][i])] = d;
      task_local[static_cast<size_t>(per_dev[static_cast<size_t>(d)][i])] = static_cast<int>(i);
    }
  }
  // minibatches per job per pass
  job_mb.assign(exec.jobs.size(), 0);
  for (const SimTask& t : tasks) {
    job_mb[static_cast<size_t>(t.t.job)] = std::max(job_mb[static_cast<size_t>(t.t.job)], t.t.minibatch + 1);
  }
  {
    // Real-bytes host check (the reference's HostOOM, strategies.cpp:613-626, charges the cost
    // model's 2P + boundary activations; this counts what setup_host_job pins): every job this
    // process executes, against the config's host_dram_bytes and this host's available memory.
    std::set<int> mine;
    for (int d : run) {
      if (exec.dynamic) {
        for (const SimTask& t : tasks) mine.insert(t.t.job);
      } else {
        for (int t : per_dev[static_cast<size_t>(d)]) mine.insert(tasks[static_cast<size_t>(t)].t.job);
      }
    }
    double need = 0;
    for (int j : mine) need += host_job_pinned_bytes(j);
    const double avail = std::min(cluster.host_dram_bytes, exec_detail::host_available_bytes());
    if (need > avail) throw HostOOM(need, avail);
  }
  for (int d : run) {
    auto w = std::make_unique<Worker>();
    w->ex = this;
    w->plan_dev = d;
    w->cuda_dev = exec.device_ids.empty() ? d : exec.device_ids.at(static_cast<size_t>(d));
    w->tasks = per_dev[static_cast<size_t>(d)];
    if (exec.dynamic) {  // any job may land on any executed GPU: size for all of them
      w->tasks.clear();
      for (size_t t = 0; t < tasks.size(); ++t) w->tasks.push_back(static_cast<int>(t));
    }
    for (int t : w->tasks) {
      const int j = tasks[static_cast<size_t>(t)].t.job;
      if (!jobs.count(j)) {
        check_cuda(cudaSetDevice(w->cuda_dev), "set device");
        setup_host_job(j);
      }
    }
    workers.push_back(std::move(w));
  }
  for (auto& kv : jobs) {
    int dev = -1;
    bool one = true;
    for (size_t t = 0; t < tasks.size(); ++t) {
      if (tasks[t].t.job != kv.first) continue;
      if (dev < 0) dev = task_device[t];
      one = one && task_device[t] == dev;
    }
    // dynamic mode: with double buffering the scheduler keeps a job on one GPU within a pass
    // (its prefetch is always the running job's successor), and every cache is written back and
    // released at the end of each pass; without it jobs migrate, so they are write-through
    kv.second.write_back = (one || (exec.dynamic && options.double_buffering)) && !exec.write_through;
  }
  for (auto& w : workers) setup_worker(*w);
  // NVLink peer access between the GPUs of this process (P2P hand-off)
  for (auto& a : workers) {
    for (auto& b : workers) {
      if (a->cuda_dev == b->cuda_dev) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a->cuda_dev, b->cuda_dev);
      if (!can) continue;
      check_cuda(cudaSetDevice(a->cuda_dev), "set device");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b->cuda_dev, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) check_cuda(e, "enable peer access");
      cudaGetLastError();
    }
  }
  host_loss = static_cast<double*>(pinned(sizeof(double) * tasks.size()));
  host_threads = exec.host_opt_threads > 0 ? exec.host_opt_threads
                                           : std::max(1, static_cast<int>(std::thread::hardware_concurrency()) - 4);
  enqueued_pass.assign(tasks.size(), -1);
  res.losses.assign(exec.jobs.size(), {});
  double pinned_total = 0;
  for (auto& kv : jobs) {
    const HostJob& hj = kv.second;
    pinned_total += 3.0 * 4 * hj.total + 4.0 * hj.n_act * (2 * hj.ckpt.size() + 1) + 8.0 * hj.M * hj.n_gmb +
                    (hj.hgrad ? 4.0 * hj.total : 0.0);
  }
  res.stats.pinned_bytes.push_back(pinned_total);
  res.stats.setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

void ExecutorImpl::run_pass(int pass, bool timed, ExecResult& res, bool interval_log) {
  if (exec.dynamic) {
    dyn.sched = exec.scheduler_factory();
    dyn.done = 0;
    dyn.log.clear();
  }
  std::vector<std::thread> threads;
  std::vector<std::exception_ptr> errs(workers.size());
  for (size_t i = 0; i < workers.size(); ++i) {
    threads.emplace_back([&, i] {
      Worker& w = *workers[i];
      try {
        check_cuda(cudaSetDevice(w.cuda_dev), "set device");
        hy::gemm_set_splitk_workspace(w.splitk, w.splitk_floats);
        hy::gemm_set_precision_fp32(exec.precision_fp32);
        hy::gemm_set_compute_bf16(exec.precision_bf16);
        g_debug_skip = exec.debug_skip;
        check_cuda(cudaDeviceSynchronize(), "pre-pass sync");
        w.ilog.reset();
        hy::t_ilog = interval_log ? &w.ilog : nullptr;
        check_cuda(cudaEventRecord(w.t0, w.comp), "t0");
        for (cudaStream_t s : {w.down, w.up, w.opt, w.opt2, w.hopt, w.optin}) {
          check_cuda(cudaStreamWaitEvent(s, w.t0, 0), "t0 wait");
        }
        const auto h0 = std::chrono::steady_clock::now();
        if (exec.dynamic) {
          dynamic_dispatch(w, pass);
        } else {
          for (int t : w.tasks) enqueue_task(w, t, pass);
        }
        // end of pass: the cache's updated params reach the host (they stay cached)
        for (auto& e : w.live) write_back(w, *e);
        // (dynamic: a job may run on another GPU next pass, so moments are released too)
        release_moments(w, !exec.dynamic);
        w.enqueue_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
        // join all streams into comp, then record the end
        cudaStream_t others[6] = {w.down, w.up, w.opt, w.hopt, w.opt2, w.optin};
        for (int k = 0; k < 6; ++k) {
          check_cuda(cudaEventRecord(w.join[k], others[k]), "join");
          check_cuda(cudaStreamWaitEvent(w.comp, w.join[k], 0), "join wait");
        }
        check_cuda(cudaEventRecord(w.t_end, w.comp), "t_end");
        check_cuda(cudaEventSynchronize(w.t_end), "pass sync");
        check_cuda(cudaGetLastError(), "pass");
        hy::t_ilog = nullptr;
      } catch (...) {
        hy::t_ilog = nullptr;
        errs[i] = std::current_exception();
        std::lock_guard<std::mutex> lk(flag_mu);
        for (auto& e : enqueued_pass) e = std::max(e, pass);  // unblock peers
        flag_cv.notify_all();
      }
    });
  }
  for (auto& th : threads) th.join();
  for (auto& e : errs) {
    if (e) std::rethrow_exception(e);
  }
  if (exec.dynamic) res.dispatch_log = dyn.log;
  if (timed) collect(pass, res, interval_log);
}

namespace {

using Spans = std::vector<std::pair<double, double>>;

// sorted, disjoint union of [a, b) intervals
Spans merge_spans(Spans v) {
  std::sort(v.begin(), v.end());
  Spans out;
  for (const auto& iv : v) {
    if (iv.second <= iv.first) continue;
    if (!out.empty() && iv.first <= out.back().second) {
      out.back().second = std::max(out.back().second, iv.second);
    } else {
      out.push_back(iv);
    }
  }
  return out;
}

double span_len(const Spans& v) {
  double t = 0;
  for (const auto& iv : v) t += iv.second - iv.first;
  return t;
}

// total length of the intersection of two merged span lists
double span_overlap(const Spans& a, const Spans& b) {
  double t = 0;
  size_t i = 0, j = 0;
  while (i < a.size() && j < b.size()) {
    const double lo = std::max(a[i].first, b[j].first), hi = std::min(a[i].second, b[j].second);
    if (hi > lo) t += hi - lo;
    (a[i].second < b[j].second) ? ++i : ++j;
  }
  return t;
}

}  // namespace

void ExecutorImpl::collect(int pass, ExecResult& res, bool interval_log) {
  // losses
  double pass_max = 0;
  SimTrace tr;
  const int G = static_cast<int>(cluster.devices.size());
  tr.device_resource.assign(static_cast<size_t>(G), -1);
  std::vector<int> down_res(static_cast<size_t>(G), -1), up_res(static_cast<size_t>(G), -1);
  for (int d = 0; d < G; ++d) {
    const std::string& id = cluster.devices[static_cast<size_t>(d)].device_id;
    tr.device_resource[static_cast<size_t>(d)] = static_cast<int>(tr.resource_names.size());
    tr.resource_names.push_back(id);
    tr.resource_device.push_back(d);
    down_res[static_cast<size_t>(d)] = static_cast<int>(tr.resource_names.size());
    tr.resource_names.push_back("h2d." + id + ".down");
    tr.resource_device.push_back(d);
    up_res[static_cast<size_t>(d)] = static_cast<int>(tr.resource_names.size());
    tr.resource_names.push_back("h2d." + id + ".up");
    tr.resource_device.push_back(d);
  }
  for (size_t i = 0; i < tasks.size(); ++i) {
    const SimTask& t = tasks[i];
    tr.task_labels.push_back("j" + std::to_string(t.t.job) + ".mb" + std::to_string(t.t.minibatch) + ".s" +
                             std::to_string(t.t.shard) + (t.t.direction == Direction::kForward ? ".F" : ".B"));
  }
  for (auto& wp : workers) {
    Worker& w = *wp;
    check_cuda(cudaSetDevice(w.cuda_dev), "set device");
    float ms = 0;
    check_cuda(cudaEventElapsedTime(&ms, w.t0, w.t_end), "elapsed");
    pass_max = std::max(pass_max, ms * 1e-3);
    auto rel = [&](cudaEvent_t e) {
      float v = 0;
      check_cuda(cudaEventElapsedTime(&v, w.t0, e), "elapsed");
      return static_cast<double>(v) * 1e-3;
    };
    // losses of forward head tasks
    std::vector<double> lbuf(w.tasks.size() + 1, 0.0);
    check_cuda(cudaMemcpy(lbuf.data(), w.loss_dev, sizeof(double) * w.tasks.size(), cudaMemcpyDeviceToHost),
               "loss d2h");
    double busy = 0;
    for (size_t li = 0; li < w.tasks.size(); ++li) {
      const int t = w.tasks[li];
      const SimTask& task = tasks[static_cast<size_t>(t)];
      const HostJob& hj = jobs.at(task.t.job);
      const ShardGeom& g = hj.geom[static_cast<size_t>(task.t.shard)];
      TaskTiming& tm = w.timing[li];
      const double pl0 = rel(tm.pl0), pl1 = rel(tm.pl1), pr0 = rel(tm.pr0), pr1 = rel(tm.pr1);
      const double c0 = rel(tm.c0), c1 = rel(tm.c1), d0 = rel(tm.d0), d1 = rel(tm.d1);
      if (pl1 > pl0) tr.events.push_back(SimEvent{down_res[static_cast<size_t>(w.plan_dev)], EventKind::kParamLoad, t, pl0, pl1});
      if (pr1 > pr0) tr.events.push_back(SimEvent{down_res[static_cast<size_t>(w.plan_dev)], EventKind::kActPromote, t, pr0, pr1});
      tr.events.push_back(SimEvent{tr.device_resource[static_cast<size_t>(w.plan_dev)], EventKind::kCompute, t, c0, c1});
      busy += c1 - c0;
      if (d1 > d0) {
        const EventKind k = task.t.direction == Direction::kForward ? EventKind::kActDemote : EventKind::kGradOffload;
        tr.events.push_back(SimEvent{up_res[static_cast<size_t>(w.plan_dev)], k, t, d0, d1});
      }
      tr.makespan_s = std::max(tr.makespan_s, std::max(c1, d1));
      if (task.t.direction == Direction::kBackward && g.has_head) {
        const int gmb = pass * job_mb[static_cast<size_t>(task.t.job)] + task.t.minibatch;
        auto& L = res.losses[static_cast<size_t>(task.t.job)];
        if (static_cast<int>(L.size()) <= gmb) L.resize(static_cast<size_t>(gmb) + 1, 0.0);
        L[static_cast<size_t>(gmb)] = lbuf[li] / static_cast<double>(hj.M);
      }
    }
    res.stats.device_busy_s.push_back(busy);
    res.stats.enqueue_s.push_back(w.enqueue_s);
    if (interval_log) {
      LinkStats ls;
      ls.plan_device = w.plan_dev;
      ls.pass_s = ms * 1e-3;
      Spans lane[3];
      static const bool dump = std::getenv("HY_LINK_DUMP") != nullptr;
      for (const hy::IntervalLog::Rec& r : w.ilog.recs) {
        lane[r.lane].emplace_back(rel(r.a), rel(r.b));
        if (dump) {
          const cudaStream_t ss[6] = {w.comp, w.down, w.up, w.opt, w.opt2, w.optin};
          int code = 6;
          for (int i = 0; i < 6; ++i) code = (r.st == ss[i] && code == 6) ? i : code;
          ls.raw.push_back({static_cast<double>(r.lane), static_cast<double>(code), rel(r.a), rel(r.b), r.bytes});
        }
        if (r.lane == hy::IntervalLog::kH2D) ls.h2d_bytes += r.bytes, ++ls.copies;
        if (r.lane == hy::IntervalLog::kD2H) ls.d2h_bytes += r.bytes, ++ls.copies;
        if (r.lane == hy::IntervalLog::kCompute) ++ls.ops;
      }
      Spans comp = merge_spans(lane[0]);
      Spans h2d = merge_spans(lane[1]), d2h = merge_spans(lane[2]);
      Spans both = lane[1];
      both.insert(both.end(), lane[2].begin(), lane[2].end());
      both = merge_spans(both);
      ls.h2d_busy_s = span_len(h2d);
      ls.d2h_busy_s = span_len(d2h);
      ls.link_busy_s = span_len(both);
      ls.compute_busy_s = span_len(comp);
      ls.exposed_s = ls.link_busy_s - span_overlap(both, comp);
      if (res.links.size() < workers.size()) res.links.resize(workers.size());
      res.links[static_cast<size_t>(&wp - &workers[0])] = ls;
    }
  }
  if (hy::OpProfiler::get().enabled) res.op_profile_ms = hy::OpProfiler::get().drain();
  std::sort(tr.events.begin(), tr.events.end(), [](const SimEvent& a, const SimEvent& b) {
    return std::tie(a.resource, a.start_s, a.end_s) < std::tie(b.resource, b.start_s, b.end_s);
  });
  res.trace = std::move(tr);
  res.pass_seconds.push_back(pass_max);
}

Executor::Executor(const ClusterSpec& cluster, const std::vector<SimTask>& tasks, const DispatchPlan& plan,
                   const SimOptions& options, const ExecOptions& exec)
    : impl_(new ExecutorImpl(cluster, tasks, plan, options, exec)) {
  impl_->setup(res_);
}

Executor::~Executor() = default;

void Executor::run(int passes, bool timed, bool interval_log) {
  const int limit = impl_->exec.warmup_passes + impl_->exec.passes;
  for (int i = 0; i < passes; ++i) {
    if (next_pass_ >= limit) throw InvalidArgument("executor: more passes than ExecOptions allowed");
    for (auto& w : impl_->workers) w->st = ExecStats{};
    impl_->run_pass(next_pass_++, timed, res_, interval_log && timed);
    if (!timed) continue;
    ExecStats& a = res_.stats;
    for (auto& w : impl_->workers) {
      const ExecStats& b = w->st;
      a.h2d_bytes += b.h2d_bytes;
      a.d2h_bytes += b.d2h_bytes;
      a.model_h2d_bytes += b.model_h2d_bytes;
      a.model_d2h_bytes += b.model_d2h_bytes;
      a.param_h2d_bytes += b.param_h2d_bytes;
      a.opt_h2d_bytes += b.opt_h2d_bytes;
      a.opt_d2h_bytes += b.opt_d2h_bytes;
      a.act_h2d_bytes += b.act_h2d_bytes;
      a.act_d2h_bytes += b.act_d2h_bytes;
      a.elided_param_bytes += b.elided_param_bytes;
      a.host_opt_params += b.host_opt_params;
      a.host_grad_d2h_bytes += b.host_grad_d2h_bytes;
      a.refresh_h2d_bytes += b.refresh_h2d_bytes;
      a.writeback_d2h_bytes += b.writeback_d2h_bytes;
      a.mv_load_h2d_bytes += b.mv_load_h2d_bytes;
      a.mv_writeback_d2h_bytes += b.mv_writeback_d2h_bytes;
      a.mv_resident_updates += b.mv_resident_updates;
      a.p2p_bytes += b.p2p_bytes;
      a.elided_act_bytes += b.elided_act_bytes;
      a.kernel_launches += b.kernel_launches;
      a.stash_reuses += b.stash_reuses;
    }
  }
  double total = 0;
  for (double x : res_.pass_seconds) total += x;
  res_.stats.makespan_s = res_.pass_seconds.empty() ? 0 : total / static_cast<double>(res_.pass_seconds.size());
  res_.stats.arena_bytes.clear();
  res_.stats.mv_cache_bytes.clear();
  for (auto& w : impl_->workers) {
    res_.stats.arena_bytes.push_back(static_cast<double>(w->arena_bytes));
    res_.stats.mv_cache_bytes.push_back(static_cast<double>(w->mvpool_bytes));
  }
}

void Executor::dump_params(const std::string& dir) const {
  for (auto& kv : impl_->jobs) {
    const std::string path = dir + "/job" + std::to_string(kv.first) + ".f32";
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw InvalidArgument("cannot write " + path);
    std::fwrite(kv.second.params, sizeof(float), static_cast<size_t>(kv.second.total), f);
    std::fclose(f);
  }
}

size_t Executor::read_params(int job, float* dst, size_t n_floats) const {
  auto it = impl_->jobs.find(job);
  if (it == impl_->jobs.end()) throw InvalidArgument("read_params: job " + std::to_string(job) + " is not executed here");
  const size_t total = static_cast<size_t>(it->second.total);
  if (dst) {
    if (n_floats < total) throw InvalidArgument("read_params: buffer holds " + std::to_string(n_floats) +
                                                " floats, job needs " + std::to_string(total));
    std::memcpy(dst, it->second.params, total * sizeof(float));
  }
  return total;
}

ExecResult run_execution(const ClusterSpec& cluster, const std::vector<SimTask>& tasks, const DispatchPlan& plan,
                         const SimOptions& options, const ExecOptions& exec) {
  Executor ex(cluster, tasks, plan, options, exec);
  ex.run(exec.warmup_passes, false);
  ex.run(exec.passes, true);
  if (!exec.params_out_dir.empty()) ex.dump_params(exec.params_out_dir);
  return std::move(ex.result());
}

}  // namespace spillsim
