// Task/trace contract and the virtual-time engine — B200 build of
// proj/core/include/spillsim/sim.hpp:26-139. ShardTask/SimTask/TaskScheduler/SimTrace
// keep the reference layout so strategies, schedulers and reports are drop-in. The
// real executor (spillsim/executor.hpp) consumes the same tasks and scheduler and
// returns the same SimTrace type, filled with CUDA-event timestamps.
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "spillsim/model.hpp"

namespace spillsim {

enum class Direction { kForward, kBackward };

struct ShardTask {
  int job = 0;
  int minibatch = 0;
  int shard = 0;
  Direction direction = Direction::kForward;
  int microbatch = -1;

  double param_load_bytes = 0;
  double activation_in_bytes = 0;
  double activation_out_bytes = 0;
  double compute_s = 0;
  double grad_offload_bytes = 0;
};

enum class BoundaryOut { kNone, kHost, kPeer };

struct SimTask {
  ShardTask t;
  std::vector<int> preds;
  int bound_device = -1;
  bool act_in_from_host = true;
  BoundaryOut act_out = BoundaryOut::kHost;
  int act_out_peer = -1;
  bool flush_marker = false;
  std::string label;
};

/// Work source (sim.hpp:70-77). next_task(device, prefetch=false, -1) when a device
/// idles; next_task(device, true, running) at compute start for double buffering.
class TaskScheduler {
 public:
  virtual ~TaskScheduler() = default;
  virtual std::optional<int> next_task(int device, bool prefetch, int running_task) = 0;
  virtual void on_dispatch(int task, int device) { (void)task; (void)device; }
  virtual void on_complete(int task) { (void)task; }
};

enum class EventKind {
  kParamLoad,
  kActPromote,
  kActDemote,
  kGradOffload,
  kCompute,
  kIdle,
  kFlush,
};

const char* to_string(EventKind kind);

struct SimEvent {
  int resource = 0;
  EventKind kind = EventKind::kCompute;
  int task = -1;
  double start_s = 0;
  double end_s = 0;
};

struct SimTrace {
  std::vector<std::string> resource_names;
  std::vector<int> resource_device;
  std::vector<int> device_resource;
  std::vector<std::string> task_labels;
  std::vector<SimEvent> events;
  double makespan_s = 0;

  double device_busy_s(int device) const;
  double total_compute_s() const;
};

double transfer_time(double bytes, const InterconnectSpec& link);

struct SimOptions {
  bool double_buffering = true;
  std::vector<double> prefetch_buffer_bytes;
  std::vector<std::string> job_names;
};

/// Virtual-time run (sim.cpp:146-597). Deterministic; DeadlockError if work remains
/// when the event queue drains.
SimTrace run_simulation(const ClusterSpec& cluster, const std::vector<SimTask>& tasks,
                        TaskScheduler& scheduler, const SimOptions& options = {});

void check_trace_invariants(const SimTrace& trace);

// ---- B200 build extensions (not in the reference) --------------------------------

/// One scheduler decision as the engine applied it.
struct Dispatch {
  int task = -1;
  int device = -1;
  bool prefetch = false;
  double time_s = 0;  // virtual time of the dispatch
};

/// Plan = the virtual engine's dispatch log. The real executor replays it ("plan
/// mode") so shard-to-GPU assignment and per-GPU order are bit-identical to the
/// reference engine on the same cost model.
struct DispatchPlan {
  std::vector<Dispatch> order;  // global dispatch order
  SimTrace trace;               // the virtual trace the plan came from

  std::vector<std::vector<int>> per_device(int n_devices) const;
  /// FNV-1a 64 (whole-value steps) over (task * 8 + device) in dispatch order (BASELINE.md §3 hash).
  unsigned long long hash() const;
};

DispatchPlan plan_simulation(const ClusterSpec& cluster, const std::vector<SimTask>& tasks,
                             TaskScheduler& scheduler, const SimOptions& options = {});

}  // namespace spillsim
