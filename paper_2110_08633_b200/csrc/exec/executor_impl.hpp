// Internal types of the plan-mode executor (not installed; shared by the exec/*.cpp
// translation units): hazard trackers, host-side job state, the per-GPU worker and the
// executor implementation. See executor.cpp for the stream structure.
#pragma once

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

struct ExecutorImpl;

namespace exec_detail {


using hy::check_cuda;
using hy::ShardGeom;

// Diagnostics only (ExecOptions::debug_skip): 1 = skip host<->device copies, 2 = skip the
// shard compute — to split a pass into its link-bound and compute-bound parts.
extern int g_debug_skip;

constexpr int kStaging = 4;

inline cudaError_t xfer(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
  const bool link = kind == cudaMemcpyHostToDevice || kind == cudaMemcpyDeviceToHost;
  if (g_debug_skip == 1 && link) return cudaSuccess;
  if (link && hy::t_ilog) {  // copy-only link interval (ExecOptions::link_log)
    const size_t i = hy::t_ilog->begin(kind == cudaMemcpyHostToDevice ? hy::IntervalLog::kH2D : hy::IntervalLog::kD2H,
                                       static_cast<double>(bytes), st);
    const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, st);
    hy::t_ilog->end(i, st);
    return e;
  }
  return cudaMemcpyAsync(dst, src, bytes, kind, st);
}

inline cudaEvent_t new_event(bool timing) {
  cudaEvent_t e;
  check_cuda(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming), "event create");
  return e;
}

inline int device_of_stream(cudaStream_t s) {
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
  // per stash region (0: the scratch's shared stash, 1: the head shard's, 2 + s: shard s's own
  // in stash_ext): {job, gmb, shard, 4} when it holds that forward's block inputs (its backward
  // may skip the recompute pass); cleared by any task that rewrites the region
  std::map<int, Tag> stash_tags;
  float* stash_ext = nullptr;  // per-shard stash regions, when the cap leaves room for them
  long stash_ext_floats = 0;
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
  // write-back boundary buffers (write-back jobs): the content is live and not yet in the
  // host checkpoint store; it is demoted only if the buffer is reused before its last consumer
  bool abuf_dirty[2] = {false, false};
  bool gbd_dirty[2] = {false, false};
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
  hy::IntervalLog ilog;            // ExecOptions::link_log
  cudaEvent_t t0 = nullptr, t_end = nullptr;
  cudaEvent_t join[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  ExecStats st;  // per pass accumulation (bytes)
};


}  // namespace exec_detail

using namespace exec_detail;  // internal header: the exec/*.cpp units share these types

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
  double host_job_pinned_bytes(int j) const;
  void setup_worker(Worker& w);
  void run_pass(int pass, bool timed, ExecResult& res, bool interval_log = false);
  void dynamic_dispatch(Worker& w, int pass);
  // P2P hand-off between the GPUs of this process: boundary activations / gradients resident
  // on the producer's GPU are copied device to device (NVLink) instead of through the host.
  std::mutex peer_mu;  // guards the act/grad buffer tags of every worker
  bool peer_fetch(Worker& w, float* dst, const Tag& want, bool grad, size_t bytes);
  // demote a dirty boundary buffer (activation: grad = false, gradient: true) to the host
  // checkpoint store of the job / boundary in its tag before the buffer is overwritten
  void spill_boundary(Worker& w, int i, bool grad);
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
  void collect(int pass, ExecResult& res, bool interval_log);
};

namespace exec_detail {
// pinned + mapped host allocation (zero-copy optimizer kernels address it directly)
void* pinned(size_t bytes);
// MemAvailable of this host minus a 4 GB margin (bytes; +inf if unknown).
double host_available_bytes();
}  // namespace exec_detail

}  // namespace spillsim
