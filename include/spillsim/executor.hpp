// Real B200 execution of a compiled strategy — the B200 build's replacement for the
// reference's simulated Engine (proj/core/src/sim.cpp:146-587). Same inputs as
// run_simulation (cluster, tasks, scheduler via its dispatch plan, options) plus the real
// model of every job; returns the same SimTrace type with CUDA-event timestamps, so
// summarize() and to_chrome_trace_json() apply unchanged.
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "hydra_gpt.h"
#include "spillsim/sim.hpp"

namespace spillsim {

struct ExecJob {
  hy_dims dims{};              // the real GPT-2 (include/hydra_gpt.h)
  uint64_t model_key = 0;      // init stream (jobs of one model share it)
  float lr = 1e-4f;
  float beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f, weight_decay = 0.f;
  std::vector<int> shard_starts;  // from the partitioner (layer indices)
};

struct ExecOptions {
  std::vector<ExecJob> jobs;       // indexed like ShardTask::job
  std::vector<int> device_ids;     // plan device -> CUDA ordinal (default: identity)
  std::vector<int> run_devices;    // plan devices executed by this process (default: all)
  uint64_t seed = 0;               // synthetic tokens
  int passes = 1;                  // times the whole plan is replayed (minibatch index continues)
  int warmup_passes = 0;           // replays before the timed ones (not in the trace)
  long opt_chunk_floats = 4L << 20;  // Adam m/v streaming chunk, upper bound (elements; the arena grants <= 2M first)
  long splitk_max_floats = 4672L << 10;  // split-K partials cap (elements): two 3072x768 partials (GPT-2 dW(fc))
  bool ring_first = true;             // spare HBM: deepen the gradient ring before the moment cache
  bool opt_priority = false;          // optimizer streams at the device's highest stream priority
  double pool_extra_max_bytes = -1;   // cap on the parameter cache beyond its two slots (< 0: none)
  bool opt_state_bf16 = false;       // Adam moments stored/streamed as bf16 (halves their link bytes)
  std::string params_out_dir;      // if set: final params of every executed job as job<j>.f32
  bool precision_fp32 = false;     // GEMMs as 3xTF32 (~fp32) instead of TF32
  bool precision_bf16 = false;     // block GEMMs on bf16 operands (kind::f16), fp32 accumulate / residual / head
  double hbm_slack_bytes = 0;      // physical arena may exceed mem_bytes by this much (toy configs
                                   // whose cost model leaves no room for real activations)
  int debug_skip = 0;              // diagnostics: 1 skip host<->device copies, 2 skip shard compute
  // Optimizer placement. The reference keeps optimizer state in host DRAM and updates it
  // host-side: a host-placed layer moves only its gradient (D2H) and its next
  // ParamLoad over the link, at 28 B/param of host DRAM traffic. GPU-placed layers stream their
  // moments through HBM instead (no host compute, 16 B/param more on the link). This is the
  // fraction of every job's parameters updated host-side (layers chosen from the shards that
  // are reloaded anyway, head side first); 0 = all on the GPU.
  double host_opt_fraction = 0;
  int host_opt_threads = 0;        // OpenMP threads of the host optimizer (0: cores - 4)
  // Parameter cache policy. Default: write-back — a job whose tasks all run on one GPU
  // (SHARP with double buffering) keeps its updated params in the GPU's cache and copies them
  // to the host only on eviction and at the end of each pass. write_through: every backward
  // writes its params back immediately (always the case for jobs spread over GPUs).
  bool write_through = false;
  // Optimizer-state cache: HBM left under the cap after every other region keeps whole
  // layers' moments resident across the owning job's minibatches (write-back jobs only).
  bool mv_cache = true;
  double mv_cache_max_bytes = -1;  // < 0: no limit beyond the cap (tests use a small limit)
  // Dynamic-time scheduling: run the strategy's TaskScheduler live on measured completions
  // (one fresh scheduler per pass from the factory) instead of replaying the plan. Jobs may
  // then land on other GPUs than in the virtual plan; all of them are set up on every GPU of
  // this process.
  bool dynamic = false;
  // P2P hand-off: a boundary activation / gradient still resident on another GPU of this process
  // is copied device to device instead of promoted from the host checkpoint
  bool p2p = true;
  std::function<std::unique_ptr<TaskScheduler>()> scheduler_factory;
};

struct ExecStats {
  double makespan_s = 0;           // timed passes, max over executed devices
  double h2d_bytes = 0, d2h_bytes = 0;            // physical, timed passes
  double model_h2d_bytes = 0, model_d2h_bytes = 0;  // cost-model bytes of the executed tasks
  double param_h2d_bytes = 0, opt_h2d_bytes = 0, opt_d2h_bytes = 0, act_h2d_bytes = 0, act_d2h_bytes = 0;
  double elided_param_bytes = 0, elided_act_bytes = 0;
  double host_opt_params = 0;       // parameter updates done host-side
  double host_grad_d2h_bytes = 0, refresh_h2d_bytes = 0;  // their GradOffload / resident-slot refresh
  double writeback_d2h_bytes = 0;   // params written back by the cache (eviction / pass end)
  double mv_load_h2d_bytes = 0, mv_writeback_d2h_bytes = 0;  // moment cache fills / write-backs
  double p2p_bytes = 0;             // boundary activations / gradients handed over GPU to GPU
  double mv_resident_updates = 0;   // parameter updates whose moments were HBM-resident
  std::vector<double> mv_cache_bytes;  // per executed device: HBM given to the moment cache
  std::vector<double> arena_bytes;  // per executed device: HBM reserved (<= mem_bytes)
  std::vector<double> device_busy_s;
  std::vector<double> enqueue_s;    // host time to enqueue a pass (per executed GPU)
  std::vector<double> pinned_bytes;
  int kernel_launches = 0;
  int elided_compute_tasks = 0;  // head-shard forwards folded into their backward
  int stash_reuses = 0;          // backwards that skipped the recompute pass (their forward's stash survived)
  double setup_s = 0;
};

// Copy-only link intervals of one GPU's last logged pass (Executor::run interval_log).
// overlap = 1 - exposed / link_busy: the share of link time hidden under shard compute.
struct LinkStats {
  int plan_device = -1;
  double pass_s = 0;
  double h2d_busy_s = 0, d2h_busy_s = 0;  // union of copy intervals per direction
  double link_busy_s = 0;                 // union over both directions
  double compute_busy_s = 0;              // union of compute-stream op intervals
  double exposed_s = 0;                   // link busy while no compute op runs
  double h2d_bytes = 0, d2h_bytes = 0;    // bytes of the logged copies
  long copies = 0, ops = 0;
  // HY_LINK_DUMP=1 (diagnostics): every logged interval {lane 0 compute / 1 H2D / 2 D2H,
  // stream 0 comp 1 down 2 up 3 opt 4 opt2 5 optin 6 other, start s, end s, bytes}
  std::vector<std::vector<double>> raw;
};

struct ExecResult {
  SimTrace trace;                              // measured, last timed pass
  std::vector<std::vector<double>> losses;     // [job][global minibatch] (executed jobs)
  std::vector<double> pass_seconds;            // per timed pass (max over devices)
  std::map<std::string, double> op_profile_ms; // HY_PROFILE=1: compute-stream time per op (last pass)
  ExecStats stats;
  std::vector<Dispatch> dispatch_log;          // dynamic mode: the measured dispatch order (last pass)
  std::vector<LinkStats> links;                // interval-logged pass: per executed GPU
};

struct ExecutorImpl;

/// Stateful form: setup (pinned host state, HBM arenas, streams, init) once, then replay
/// the plan pass by pass. Inputs are borrowed and must outlive the executor. At most
/// exec.warmup_passes + exec.passes passes may be run in total (tokens are pre-drawn).
class Executor {
 public:
  Executor(const ClusterSpec& cluster, const std::vector<SimTask>& tasks, const DispatchPlan& plan,
           const SimOptions& options, const ExecOptions& exec);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  /// Replays the plan `passes` times. Timed passes append to result(): pass_seconds (CUDA
  /// events on each GPU, max over this process's GPUs), losses, byte counters, trace.
  /// interval_log: also record every compute op and host<->device copy of the (timed) passes
  /// (result().links: copy-only link time and the transfer-overlap fraction); it adds two
  /// event records per op / copy, so measure throughput on passes without it.
  void run(int passes, bool timed, bool interval_log = false);
  ExecResult& result() { return res_; }
  void dump_params(const std::string& dir) const;
  // Copies job `job`'s current host parameter vector (final after a pass) into dst when
  // dst != nullptr (n_floats must cover it); returns its length in floats.
  size_t read_params(int job, float* dst, size_t n_floats) const;

 private:
  std::unique_ptr<ExecutorImpl> impl_;
  ExecResult res_;
  int next_pass_ = 0;
};

ExecResult run_execution(const ClusterSpec& cluster, const std::vector<SimTask>& tasks, const DispatchPlan& plan,
                         const SimOptions& options, const ExecOptions& exec);

}  // namespace spillsim
