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
#include "spillsim/executor.hpp"

#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <optional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "../kernels/gemm.cuh"
#include "../kernels/ops.cuh"
#include "gpt_runner.hpp"
#include "host_opt.hpp"
#include "prof.hpp"
#include "spillsim/errors.hpp"

namespace spillsim {
namespace {

using hy::check_cuda;
using hy::ShardGeom;

// Diagnostics only (ExecOptions::debug_skip): 1 = skip host<->device copies, 2 = skip the
// shard compute — to split a pass into its link-bound and compute-bound parts.
int g_debug_skip = 0;

constexpr int kStaging = 4;

cudaError_t xfer(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
  if (g_debug_skip == 1 && (kind == cudaMemcpyHostToDevice || kind == cudaMemcpyDeviceToHost)) return cudaSuccess;
  return cudaMemcpyAsync(dst, src, bytes, kind, st);
}

cudaEvent_t new_event(bool timing) {
  cudaEvent_t e;
  check_cuda(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming), "event create");
  return e;
}

int device_of_stream(cudaStream_t s) {
  int dev = 0;
  check_cuda(cudaStreamGetDevice(s, &dev), "stream device");
  return dev;
}

// Hazard tracker for one buffer accessed from several streams (possibly several GPUs).
struct Tracked {
  std::mutex mu;
  cudaStream_t writer = nullptr;
  std::map<cudaStream_t, cudaEvent_t> write_ev, read_ev;
  std::map<cudaStream_t, bool> read_live;

  cudaEvent_t ev(std::map<cudaStream_t, cudaEvent_t>& m, cudaStream_t s) {
    auto it = m.find(s);
    if (it != m.end()) return it->second;
    int cur = 0;
    cudaGetDevice(&cur);
    const int dev = device_of_stream(s);
    if (dev != cur) cudaSetDevice(dev);
    cudaEvent_t e = new_event(false);
    if (dev != cur) cudaSetDevice(cur);
    m[s] = e;
    return e;
  }
  void before_write(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    for (auto& kv : read_live) {
      if (kv.second && kv.first != s) check_cuda(cudaStreamWaitEvent(s, read_ev[kv.first], 0), "wait read");
    }
    if (writer && writer != s) check_cuda(cudaStreamWaitEvent(s, write_ev[writer], 0), "wait write");
  }
  void after_write(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    check_cuda(cudaEventRecord(ev(write_ev, s), s), "record write");
    writer = s;
    for (auto& kv : read_live) kv.second = false;
  }
  void before_read(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    if (writer && writer != s) check_cuda(cudaStreamWaitEvent(s, write_ev[writer], 0), "wait write");
  }
  void after_read(cudaStream_t s) {
    std::lock_guard<std::mutex> g(mu);
    check_cuda(cudaEventRecord(ev(read_ev, s), s), "record read");
    read_live[s] = true;
  }
  void destroy() {
    for (auto& kv : write_ev) cudaEventDestroy(kv.second);
    for (auto& kv : read_ev) cudaEventDestroy(kv.second);
    write_ev.clear();
    read_ev.clear();
  }
};

struct Tag {
  int job = -1, gmb = -1, idx = -1, ver = -1;
  bool operator==(const Tag& o) const { return job == o.job && gmb == o.gmb && idx == o.idx && ver == o.ver; }
};

struct HostJob {
  const ExecJob* spec = nullptr;
  int job = -1;
  hy_dims m{};
  long M = 0, n_act = 0, total = 0;
  std::vector<ShardGeom> geom;
  float *params = nullptr, *mom = nullptr, *var = nullptr, *z = nullptr;
  std::vector<float*> ckpt, grad;  // per boundary 0..k-2
  int32_t *tokens = nullptr, *targets = nullptr;  // [n_gmb][M]
  int n_gmb = 0;
  std::vector<std::unique_ptr<Tracked>> params_tr, mv_tr, ckpt_tr, grad_tr;
  std::unique_ptr<Tracked> z_tr;
  std::vector<int> version;  // per shard: Adam updates applied
  // host-placed optimizer (ExecOptions::host_opt_fraction)
  std::vector<char> host_layer;                      // per layer: AdamW runs host-side
  float* hgrad = nullptr;                            // pinned gradients of host layers
  std::vector<std::unique_ptr<Tracked>> hgrad_tr;    // per layer
  std::vector<std::unique_ptr<Tracked>> hparams_tr;  // per shard: host-side writes of params
  // every task of the job on one GPU (SHARP with double buffering): its updated params may
  // stay in that GPU's parameter cache and reach the host only on eviction / at pass end
  bool write_back = false;
};

struct TaskTiming {
  cudaEvent_t pl0 = nullptr, pl1 = nullptr, pr0 = nullptr, pr1 = nullptr, c0 = nullptr, c1 = nullptr,
              d0 = nullptr, d1 = nullptr;
  bool loaded = false, promoted = false, demoted = false;
};


}  // namespace

struct ExecutorImpl;

namespace {

struct Worker {
  ExecutorImpl* ex = nullptr;
  int plan_dev = 0, cuda_dev = 0;
  std::vector<int> tasks;  // plan order
  cudaStream_t comp{}, down{}, up{}, opt{}, opt2{}, hopt{}, optin{};
  cudaEvent_t dense_done = nullptr;  // opt2: the embedding's early (non-token rows) update
  char* arena = nullptr;
  long arena_bytes = 0;
  // Parameter cache: shards live anywhere in `pool` (2 x the largest shard), first-fit,
  // evicting least-recently-used shards; a ParamLoad is skipped whenever the shard is still
  // resident at its current version (generalises the reference's F(k-1)->B(k-1) elision).
  struct PoolEntry {
    Tag tag;
    long off = 0, len = 0;
    long last_use = -1;
    Tracked tr;
    std::vector<int> dirty;      // layers updated host-side since the slot was filled (refresh)
    std::vector<int> gpu_dirty;  // layers updated in the slot, host copy stale (write back)
  };
  float* pool = nullptr;
  long pool_floats = 0;
  std::list<std::unique_ptr<PoolEntry>> live, retired;
  PoolEntry* prev_entry = nullptr;
  long seq = 0;
  // the embedding-gradient buffer doubles as a cache of the tied wte between F(0) and the
  // head shard's tasks (a D2D copy instead of reloading V*d floats over the host link)
  Tag gembed_tag;
  Tracked gembed_tr;
  // Parameter gradients: the embedding's in its own buffer, every other layer in a ring
  // (FIFO, released as each layer's Adam finishes reading), so the optimizer streams a
  // layer's state while the backward is still working on earlier layers.
  float* gembed = nullptr;
  cudaEvent_t gembed_free = nullptr;  // Adam of the last embedding gradient done
  float* ring = nullptr;
  long ring_floats = 0, ring_head = 0;
  struct RingEntry {
    long off, len;
    cudaEvent_t done;
  };
  std::deque<RingEntry> ring_live;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  float* abuf[2] = {nullptr, nullptr};
  Tag abuf_tag[2];
  Tracked abuf_tr[2];
  float* gbd[2] = {nullptr, nullptr};
  Tag gbd_tag[2];
  Tracked gbd_tr[2];
  float* zbuf = nullptr;
  Tag z_tag;
  Tracked z_tr;
  int32_t* tok[2] = {nullptr, nullptr};
  Tag tok_tag[2];
  Tracked tok_tr[2];
  float* stg[kStaging] = {nullptr, nullptr, nullptr, nullptr};
  Tracked stg_tr[kStaging];
  bool stg_alias = false;
  long stg_chunk = 0;
  int stg_round = 0;
  // embedding optimizer split (B of the embedding shard): rows touched by the minibatch's
  // tokens (+ wpe) are updated after the embedding scatter from a compact stash, all other
  // wte rows early, while the blocks back-propagate
  int* rowidx = nullptr;   // [V + T]
  int* rowlist = nullptr;  // [M + T]
  int* rowcount = nullptr;
  float* cbuf = nullptr;   // compact m | v (| p for write-through jobs) of those rows
  long crow_max = 0;
  Tracked rowidx_tr, cbuf_tr;
  // Optimizer-state cache: the HBM the cap leaves after every other region keeps whole
  // layers' Adam moments resident across the minibatches of the job that owns it (write-back:
  // the host copy is refreshed when ownership passes to the next job on this GPU and at the
  // end of each pass). Layers that do not fit stream through the staging ring as before.
  struct MvEntry {
    int layer = -1;
    long off = 0, bytes = 0;  // m at off, v at off + bytes / 2
    bool valid = false, dirty = false;
    int job = -1;             // whose moments the entry holds while valid
    Tracked tr;
  };
  char* mvpool = nullptr;
  long mvpool_bytes = 0, mvpool_used = 0;
  int mv_owner = -1;                         // job whose moments the pool holds
  int mv_owner_pass = -1;                    // last pass in which the owner used the pool
  std::map<int, std::unique_ptr<MvEntry>> mv_live;  // layer -> entry (owner's)
  std::vector<std::unique_ptr<MvEntry>> mv_retired;
  cudaEvent_t mv_free = nullptr;             // up: previous owner's write-back done
  bool mv_free_pending = false;
  std::map<int, int> last_local_of_job;      // job -> its last local task index on this GPU
  std::map<std::pair<int, int>, int> last_b_local;  // (job, shard) -> local index of its last backward
  std::map<int, int> next_job;               // job -> the job this GPU runs after it (plan mode; -1 none)
  int cur_local = -1, cur_pass = -1;
  float* scratch = nullptr;
  double* loss_dev = nullptr;  // per task slot
  int last_slot = -1;
  int last_tok = 1;
  float* splitk = nullptr;
  long splitk_floats = 0;
  double enqueue_s = 0;
  std::vector<TaskTiming> timing;  // per local task index
  cudaEvent_t t0 = nullptr, t_end = nullptr;
  cudaEvent_t join[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  ExecStats st;  // per pass accumulation (bytes)
};

}  // namespace

struct ExecutorImpl {
  const ClusterSpec& cluster;
  const std::vector<SimTask>& tasks;
  const DispatchPlan& plan;
  const SimOptions& options;
  const ExecOptions& exec;
  std::map<int, HostJob> jobs;  // executed jobs
  std::vector<std::unique_ptr<Worker>> workers;
  std::vector<int> task_local;    // task -> local index on its worker
  std::vector<int> task_device;   // task -> plan device
  int mb_per_job_max = 0;
  int host_threads = 1;
  std::vector<int> job_mb;        // minibatches per job per pass
  double* host_loss = nullptr;    // [task] per pass (pinned)
  // cross-device ordering: task enqueued flags
  std::mutex flag_mu;
  std::condition_variable flag_cv;
  std::vector<int> enqueued_pass;  // per task: last pass enqueued

  ExecutorImpl(const ClusterSpec& c, const std::vector<SimTask>& t, const DispatchPlan& p, const SimOptions& o,
               const ExecOptions& e)
      : cluster(c), tasks(t), plan(p), options(o), exec(e) {}
  ~ExecutorImpl();

  void setup(ExecResult& res);
  void setup_host_job(int j);
  void setup_worker(Worker& w);
  void run_pass(int pass, bool timed, ExecResult& res);
  void dynamic_dispatch(Worker& w, int pass);
  // P2P hand-off between the GPUs of this process: boundary activations / gradients resident
  // on the producer's GPU are copied device to device (NVLink) instead of through the host.
  std::mutex peer_mu;  // guards the act/grad buffer tags of every worker
  bool peer_fetch(Worker& w, float* dst, const Tag& want, bool grad, size_t bytes);
  // dynamic-time scheduling state (one scheduler per pass, shared by the GPU workers)
  struct Dynamic {
    std::mutex mu;
    std::condition_variable cv;
    std::unique_ptr<TaskScheduler> sched;
    int done = 0;
    std::vector<Dispatch> log;
  } dyn;
  void enqueue_task(Worker& w, int t, int pass);
  void adam_layer(Worker& w, HostJob& hj, int s, float* base, int layer, const float* grads, int step,
                  cudaEvent_t done, int part = 0);
  void host_adam_layer(Worker& w, HostJob& hj, int s, int layer, const float* grads, int step, cudaEvent_t done);
  void param_read_begin(HostJob& hj, int s, cudaStream_t st);
  void param_read_end(HostJob& hj, int s, cudaStream_t st);
  Worker::PoolEntry* acquire_params(Worker& w, HostJob& hj, int j, int s, bool* loaded);
  Worker::MvEntry* acquire_moments(Worker& w, HostJob& hj, int layer, long bytes);
  bool claim_moments(Worker& w, HostJob& hj);
  bool same_moment_layout(const HostJob& a, const HostJob& b) const {
    return a.m.L == b.m.L && a.m.d == b.m.d && a.m.V == b.m.V && a.host_layer == b.host_layer;
  }
  void flush_moments(Worker& w, int new_owner);
  void hand_over_moments(Worker& w, HostJob& hj, int layer, Worker::MvEntry& e);
  void release_moments(Worker& w, bool keep);
  void write_back(Worker& w, Worker::PoolEntry& e);
  void collect(int pass, ExecResult& res);
};

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

namespace {

void* pinned(size_t bytes) {
  void* p = nullptr;
  // mapped: the zero-copy optimizer kernels read / write moments and params in place (UVA:
  // the device pointer is the host pointer)
  check_cuda(cudaHostAlloc(&p, bytes ? bytes : 4, cudaHostAllocPortable | cudaHostAllocMapped), "cudaHostAlloc");
  return p;
}

}  // namespace

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
  check_cuda(cudaStreamCreateWithFlags(&w.comp, cudaStreamNonBlocking), "stream");
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
    int max_blocks = 0;
    for (const ShardGeom& sg : hj.geom) max_blocks = std::max(max_blocks, sg.n_blocks);
    scratch_f = std::max(scratch_f, hy::scratch_floats(hj.m, max_blocks));
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
  long chunk = std::min(exec.opt_chunk_floats, budget_floats / (2 * kStaging));
  chunk = chunk / 1024 * 1024;
  // alias the staging ring onto the scratch only when the cap leaves no room for the
  // requested chunks (or for 1M-element chunks, whichever is smaller)
  w.stg_alias = chunk < std::min(exec.opt_chunk_floats / 1024 * 1024, 1L << 20);
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
                 "staging %.1f pool+ %.1f mv %.1f | left %.1f\n",
                 w.plan_dev, 8.0 * hy_pad32(slot_f) / 1e6, 4.0 * hy_pad32(embed_f) / 1e6, 20.0 * hy_pad32(act_f) / 1e6,
                 4.0 * hy_pad32(scratch_f) / 1e6, 4.0 * (all_write_back ? 2 : 3) * crow / 1e6, 4.0 * ring_f / 1e6,
                 4.0 * splitk_f / 1e6, 4.0 * kStaging * 2 * hy_pad32(chunk) / 1e6,
                 4.0 * (pool_f - 2 * hy_pad32(slot_f)) / 1e6, 4.0 * mv_f / 1e6, 4.0 * budget_floats / 1e6);
  }
  const long floats = base_floats + ring_f + splitk_f + kStaging * 2 * hy_pad32(chunk) + (pool_f - 2 * hy_pad32(slot_f)) +
                      mv_f;
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
  if (w.stg_alias) {
    // staging inside the scratch fc/act block of the largest job on this GPU
    long best = 0;
    for (int t : w.tasks) {
      const HostJob& hj = jobs.at(tasks[static_cast<size_t>(t)].t.job);
      int mb = 0;
      for (const ShardGeom& sg : hj.geom) mb = std::max(mb, sg.n_blocks);
      hy::Scratch sc;
      hy::carve_scratch(hj.m, mb, w.scratch, &sc);
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

namespace {

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

}  // namespace

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
  check_cuda(cudaEventRecord(tm.pl0, w.down), "pl0");
  bool loaded = false;
  Worker::PoolEntry* pe = acquire_params(w, hj, j, s, &loaded);
  float* pbase = w.pool + pe->off;
  if (loaded) {
    const long base = hy_layer_offset(&hj.m, g.l0);
    pe->tr.before_write(w.down);
    param_read_begin(hj, s, w.down);
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
  check_cuda(cudaEventRecord(tm.pl1, w.down), "pl1");

  // ---- ActPromote (down): tokens, boundary activation / checkpoint, grad_in, z --------
  check_cuda(cudaEventRecord(tm.pr0, w.down), "pr0");
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
      std::lock_guard<std::mutex> lk(peer_mu);
      w.abuf_tag[ain] = Tag{};
      w.abuf_tr[ain].before_write(w.down);
      if (!peer_fetch(w, w.abuf[ain], at, false, act_bytes)) {
        hj.ckpt_tr[static_cast<size_t>(s - 1)]->before_read(w.down);
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
      gin = 0;
      std::lock_guard<std::mutex> lk(peer_mu);
      w.gbd_tag[gin] = Tag{};
      w.gbd_tr[gin].before_write(w.down);
      if (!peer_fetch(w, w.gbd[gin], gt, true, act_bytes)) {
        hj.grad_tr[static_cast<size_t>(s)]->before_read(w.down);
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
      check_cuda(xfer(w.zbuf, hj.z, act_bytes, cudaMemcpyHostToDevice, w.down), "z h2d");
      hj.z_tr->after_read(w.down);
      w.z_tr.after_write(w.down);
      w.z_tag = zt;
      w.st.h2d_bytes += static_cast<double>(act_bytes);
    }
  }
  check_cuda(cudaEventRecord(tm.pr1, w.down), "pr1");

  // ---- Compute (comp) ---------------------------------------------------------------
  std::vector<int> host_dirty;  // layers of this backward updated host-side
  hy::Scratch sc;
  int max_blocks = 0;
  for (const ShardGeom& sg : hj.geom) max_blocks = std::max(max_blocks, sg.n_blocks);
  hy::carve_scratch(hj.m, max_blocks, w.scratch, &sc);
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
      gout = gin >= 0 ? 1 - gin : 0;
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
  if (fwd && !skip_fwd) {
    hy::run_forward(w.comp, hj.m, g, pbase, io, sc);
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
      hy::run_backward(w.comp, hj.m, g, pbase, sink, io, sc);
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
    if (g.has_head && !g.has_embed) {
      w.z_tr.before_write(w.comp);
      check_cuda(cudaMemcpyAsync(w.zbuf, sc.z, act_bytes, cudaMemcpyDeviceToDevice, w.comp), "z save");
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
  if (fwd) check_cuda(cudaEventRecord(tm.d0, w.up), "d0");
  if (aout >= 0) {  // forward boundary activation -> checkpoint store
    Tracked& host = *hj.ckpt_tr[static_cast<size_t>(s)];
    w.abuf_tr[aout].before_read(w.up);
    host.before_write(w.up);
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
    check_cuda(xfer(hj.z, w.zbuf, act_bytes, cudaMemcpyDeviceToHost, w.up), "z d2h");
    hj.z_tr->after_write(w.up);
    w.z_tr.after_read(w.up);
    w.st.d2h_bytes += static_cast<double>(act_bytes);
  }
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

void ExecutorImpl::run_pass(int pass, bool timed, ExecResult& res) {
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
        g_debug_skip = exec.debug_skip;
        check_cuda(cudaDeviceSynchronize(), "pre-pass sync");
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
      } catch (...) {
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
  if (timed) collect(pass, res);
}

void ExecutorImpl::collect(int pass, ExecResult& res) {
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

void Executor::run(int passes, bool timed) {
  const int limit = impl_->exec.warmup_passes + impl_->exec.passes;
  for (int i = 0; i < passes; ++i) {
    if (next_pass_ >= limit) throw InvalidArgument("executor: more passes than ExecOptions allowed");
    for (auto& w : impl_->workers) w->st = ExecStats{};
    impl_->run_pass(next_pass_++, timed, res_);
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

ExecResult run_execution(const ClusterSpec& cluster, const std::vector<SimTask>& tasks, const DispatchPlan& plan,
                         const SimOptions& options, const ExecOptions& exec) {
  Executor ex(cluster, tasks, plan, options, exec);
  ex.run(exec.warmup_passes, false);
  ex.run(exec.passes, true);
  if (!exec.params_out_dir.empty()) ex.dump_params(exec.params_out_dir);
  return std::move(ex.result());
}

}  // namespace spillsim
