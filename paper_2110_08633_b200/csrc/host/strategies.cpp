// SHARP task compiler, Sharded-LRTF and the task-parallel comparison leg.
// Reference: proj/core/src/strategies.cpp (SHARP :98-198, :663-807; task-parallel
// :207-304, :809-877; feasibility :558-656; reduced instances :1014-1077).
#include "spillsim/strategies.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>

#include "spillsim/errors.hpp"

namespace spillsim {

namespace {

struct KindName {
  StrategyKind kind;
  const char* name;
};
constexpr KindName kKindNames[] = {
    {StrategyKind::kSharp, "sharp"},
    {StrategyKind::kTaskParallel, "task-parallel"},
    {StrategyKind::kModelParallel, "model-parallel"},
    {StrategyKind::kPipelineParallel, "pipeline-parallel"},
    {StrategyKind::kHybridTaskOverModel, "hybrid-task-over-model"},
    {StrategyKind::kExactOptimal, "exact-optimal"},
};

// A transfer that is issued costs latency + bytes/bw; a zero-byte one is elided.
double xfer_s(double bytes, const InterconnectSpec& link) {
  return bytes > 0 ? transfer_time(bytes, link) : 0.0;
}

std::vector<std::string> job_names(size_t n) {
  std::vector<std::string> v;
  v.reserve(n);
  for (size_t i = 0; i < n; ++i) v.push_back("j" + std::to_string(i));
  return v;
}

// First device with the smallest memory (ties keep the lower index).
int tightest_device(const ClusterSpec& c) {
  int best = 0;
  for (size_t d = 1; d < c.devices.size(); ++d) {
    if (c.devices[d].mem_bytes < c.devices[static_cast<size_t>(best)].mem_bytes) {
      best = static_cast<int>(d);
    }
  }
  return best;
}

[[noreturn]] void unsupported(StrategyKind kind) {
  throw InvalidArgument("strategy '" + to_string(kind) +
                        "' is a reference baseline outside the B200 build's hot path");
}

}  // namespace

std::string to_string(StrategyKind kind) {
  for (const KindName& kn : kKindNames) {
    if (kn.kind == kind) return kn.name;
  }
  return "?";
}

StrategyKind strategy_kind_from_string(const std::string& name) {
  for (const KindName& kn : kKindNames) {
    if (name == kn.name) return kn.kind;
  }
  throw InvalidArgument("unknown strategy: '" + name + "'");
}

double resident_training_footprint(const ModelProfile& model) {
  double params = 0, acts = 0, worst = 0;
  for (const LayerProfile& l : model.layers) {
    params += l.param_bytes;
    acts += l.activation_out_bytes;
    worst = std::max(worst, l.activation_out_bytes + l.workspace_bytes);
  }
  return 2 * params + acts + worst + model.input_batch_bytes;
}

double spilled_host_bytes(const ModelProfile& model, const Partitioning& p) {
  double ckpt = 0;
  for (const Shard& sh : p.shards) ckpt += sh.boundary_activation_bytes;
  return 2 * model.total_param_bytes() + ckpt + model.input_batch_bytes;
}

// ---------------------------------------------------------------------------
// Sharded-LRTF

SharpScheduler::SharpScheduler(const std::vector<SimTask>& tasks, std::vector<double> est) {
  if (est.size() != tasks.size()) throw InvalidArgument("one estimate per task required");
  slot_.assign(tasks.size(), -1);
  std::vector<int> slot_of_job;
  for (size_t i = 0; i < tasks.size(); ++i) {
    const int job = tasks[i].t.job;
    if (job >= static_cast<int>(slot_of_job.size())) slot_of_job.resize(static_cast<size_t>(job) + 1, -1);
    int& slot = slot_of_job[static_cast<size_t>(job)];
    if (slot < 0) {
      slot = static_cast<int>(jobs_.size());
      jobs_.emplace_back();
    }
    slot_[i] = slot;
    jobs_[static_cast<size_t>(slot)].tasks.push_back(static_cast<int>(i));
  }
  for (Chain& c : jobs_) {
    c.tail.assign(c.tasks.size() + 1, 0.0);
    for (size_t i = c.tasks.size(); i > 0; --i) {
      c.tail[i - 1] = c.tail[i] + est[static_cast<size_t>(c.tasks[i - 1])];
    }
  }
}

double SharpScheduler::remaining_estimate(int job) const {
  const Chain& c = jobs_[static_cast<size_t>(job)];
  return c.tail[static_cast<size_t>(c.done)];
}

std::optional<int> SharpScheduler::next_task(int /*device*/, bool prefetch, int running_task) {
  if (prefetch) {
    // Only the running task's own successor may take the prefetch buffer.
    if (running_task < 0) return std::nullopt;
    const Chain& c = jobs_[static_cast<size_t>(slot_[static_cast<size_t>(running_task)])];
    const bool successor_free = c.running == 1 && c.last == running_task &&
                                c.cursor < static_cast<int>(c.tasks.size());
    if (!successor_free) return std::nullopt;
    return c.tasks[static_cast<size_t>(c.cursor)];
  }
  int best = -1;
  double best_left = -1;
  for (size_t j = 0; j < jobs_.size(); ++j) {
    const Chain& c = jobs_[j];
    if (c.cursor >= static_cast<int>(c.tasks.size()) || c.running != 0) continue;
    const double left = c.tail[static_cast<size_t>(c.done)];
    if (left > best_left) {  // strict: ties keep the lower slot
      best_left = left;
      best = static_cast<int>(j);
    }
  }
  if (best < 0) return std::nullopt;
  const Chain& c = jobs_[static_cast<size_t>(best)];
  return c.tasks[static_cast<size_t>(c.cursor)];
}

void SharpScheduler::on_dispatch(int task, int /*device*/) {
  Chain& c = jobs_[static_cast<size_t>(slot_[static_cast<size_t>(task)])];
  ++c.cursor;
  ++c.running;
  c.last = task;
}

void SharpScheduler::on_complete(int task) {
  Chain& c = jobs_[static_cast<size_t>(slot_[static_cast<size_t>(task)])];
  ++c.done;
  --c.running;
}

std::vector<double> sharp_task_estimates(const std::vector<SimTask>& tasks,
                                         const InterconnectSpec& h2d) {
  std::vector<double> out(tasks.size(), 0.0);
  for (size_t i = 0; i < tasks.size(); ++i) {
    const ShardTask& t = tasks[i].t;
    double e = t.compute_s;
    e += xfer_s(t.activation_in_bytes, h2d);
    e += xfer_s(t.activation_out_bytes, h2d);
    e += xfer_s(t.grad_offload_bytes, h2d);
    const double load = xfer_s(t.param_load_bytes, h2d);
    if (tasks[i].preds.empty()) {
      e += load;
    } else {
      // Double buffering hides the load behind the chain predecessor's compute.
      e += std::max(0.0, load - tasks[static_cast<size_t>(tasks[i].preds.front())].t.compute_s);
    }
    out[i] = e;
  }
  return out;
}

// ---------------------------------------------------------------------------
// Job-granular binding (task parallelism): whole jobs bind to single devices,
// longest total estimate first, ties to the lower job.

namespace {

class WholeJobScheduler : public TaskScheduler {
 public:
  WholeJobScheduler(std::vector<std::vector<int>> lists, std::vector<double> totals,
                    std::vector<int> job_of_task, int n_devices)
      : lists_(std::move(lists)), totals_(std::move(totals)), job_of_(std::move(job_of_task)) {
    next_.assign(lists_.size(), 0);
    left_.resize(lists_.size());
    for (size_t j = 0; j < lists_.size(); ++j) left_[j] = static_cast<int>(lists_[j].size());
    bound_.assign(lists_.size(), false);
    on_device_.assign(static_cast<size_t>(n_devices), -1);
    device_of_.assign(lists_.size(), -1);
  }

  std::optional<int> next_task(int device, bool prefetch, int /*running*/) override {
    int job = on_device_[static_cast<size_t>(device)];
    if (job < 0) {
      if (prefetch) return std::nullopt;  // never bind a second model early
      double best_total = -1;
      for (size_t j = 0; j < lists_.size(); ++j) {
        if (!bound_[j] && totals_[j] > best_total) {
          best_total = totals_[j];
          job = static_cast<int>(j);
        }
      }
      if (job < 0) return std::nullopt;
      on_device_[static_cast<size_t>(device)] = job;
      bound_[static_cast<size_t>(job)] = true;
      device_of_[static_cast<size_t>(job)] = device;
    }
    const auto& list = lists_[static_cast<size_t>(job)];
    const int nx = next_[static_cast<size_t>(job)];
    if (nx >= static_cast<int>(list.size())) return std::nullopt;
    return list[static_cast<size_t>(nx)];
  }

  void on_dispatch(int task, int) override { ++next_[static_cast<size_t>(job_of_[static_cast<size_t>(task)])]; }

  void on_complete(int task) override {
    const int job = job_of_[static_cast<size_t>(task)];
    if (--left_[static_cast<size_t>(job)] == 0) {
      on_device_[static_cast<size_t>(device_of_[static_cast<size_t>(job)])] = -1;
    }
  }

 private:
  std::vector<std::vector<int>> lists_;
  std::vector<double> totals_;
  std::vector<int> job_of_;
  std::vector<int> next_, left_;
  std::vector<bool> bound_;
  std::vector<int> on_device_, device_of_;
};

SimTask plain_task(int job, int mb, int shard, Direction dir, double load, double in, double out,
                   double compute, double grad) {
  SimTask task;
  task.t.job = job;
  task.t.minibatch = mb;
  task.t.shard = shard;
  task.t.direction = dir;
  task.t.microbatch = -1;
  task.t.param_load_bytes = load;
  task.t.activation_in_bytes = in;
  task.t.activation_out_bytes = out;
  task.t.compute_s = compute;
  task.t.grad_offload_bytes = grad;
  return task;
}

CompiledStrategy compile_sharp(const StrategyConfig& cfg, const std::vector<ModelJob>& jobs,
                               const ClusterSpec& cluster, const BufferPolicy& policy,
                               const PinnedBoundaries* pinned = nullptr) {
  CompiledStrategy out;
  out.config = cfg;
  const DeviceSpec& tight = cluster.devices[static_cast<size_t>(tightest_device(cluster))];
  auto pinned_for = [&](size_t j) -> const std::vector<int>* {
    if (!pinned || j >= pinned->size() || (*pinned)[j].empty()) return nullptr;
    return &(*pinned)[j];
  };

  std::vector<Partitioning> parts;
  parts.reserve(jobs.size());
  for (size_t j = 0; j < jobs.size(); ++j) {
    // A pinned job reuses its boundaries (partitioner.cpp:157-184: validated against the cap).
    const std::vector<int>* pin = pinned_for(j);
    parts.push_back(pin ? partition_with_boundaries(jobs[j].model, *pin, tight, policy)
                        : partition(jobs[j].model, tight, policy));
  }

  if (policy.kind == BufferPolicy::Kind::kAuto) {
    // One shared prefetch reserve (the largest any job wanted); re-cut the rest.
    double shared = 0;
    for (const Partitioning& p : parts) shared = std::max(shared, p.buffer_reserve_bytes);
    BufferPolicy fixed = BufferPolicy::absolute(shared);
    fixed.framework_overhead_bytes = policy.framework_overhead_bytes;
    for (size_t j = 0; j < jobs.size(); ++j) {
      if (parts[j].buffer_reserve_bytes == shared) continue;
      const std::vector<int>* pin = pinned_for(j);
      parts[j] = pin ? partition_with_boundaries(jobs[j].model, *pin, tight, fixed) : partition(jobs[j].model, tight, fixed);
    }
  }

  double host_need = 0;
  for (size_t j = 0; j < jobs.size(); ++j) host_need += spilled_host_bytes(jobs[j].model, parts[j]);
  if (host_need > cluster.host_dram_bytes) throw HostOOM(host_need, cluster.host_dram_bytes);

  for (size_t j = 0; j < jobs.size(); ++j) {
    const Partitioning& p = parts[j];
    const int job = static_cast<int>(j);
    const int k = p.shard_count();
    const int n_mb = jobs[j].total_minibatches();
    int prev = -1;
    auto emit = [&](SimTask task) {
      if (prev >= 0) task.preds.push_back(prev);
      prev = static_cast<int>(out.tasks.size());
      out.tasks.push_back(std::move(task));
    };
    if (k == 1) {
      // Whole model fits the execution region: resident training, loaded once.
      const Shard& sh = p.shards[0];
      for (int mb = 0; mb < n_mb; ++mb) {
        SimTask f = plain_task(job, mb, 0, Direction::kForward, mb == 0 ? sh.param_bytes : 0.0, 0.0,
                               0.0, sh.fwd_compute_s, 0.0);
        f.act_in_from_host = false;
        f.act_out = BoundaryOut::kNone;
        emit(std::move(f));
        SimTask b = plain_task(job, mb, 0, Direction::kBackward, 0.0, 0.0, 0.0, sh.bwd_compute_s, 0.0);
        b.act_in_from_host = false;
        b.act_out = BoundaryOut::kNone;
        emit(std::move(b));
      }
      continue;
    }
    for (int mb = 0; mb < n_mb; ++mb) {
      for (int s = 0; s < k; ++s) {  // forward sweep
        const Shard& sh = p.shards[static_cast<size_t>(s)];
        const double in = s > 0 ? p.shards[static_cast<size_t>(s - 1)].boundary_activation_bytes : 0.0;
        SimTask f = plain_task(job, mb, s, Direction::kForward, sh.param_bytes, in,
                               sh.boundary_activation_bytes, sh.fwd_compute_s, 0.0);
        f.act_in_from_host = in > 0;
        f.act_out = BoundaryOut::kHost;
        emit(std::move(f));
      }
      for (int s = k - 1; s >= 0; --s) {  // backward sweep: checkpoint (+ grad_in) in, recompute + bwd
        const Shard& sh = p.shards[static_cast<size_t>(s)];
        const double ckpt = s > 0 ? p.shards[static_cast<size_t>(s - 1)].boundary_activation_bytes : 0.0;
        const double grad_in = s < k - 1 ? sh.boundary_activation_bytes : 0.0;
        SimTask b = plain_task(job, mb, s, Direction::kBackward, sh.param_bytes, ckpt + grad_in, ckpt,
                               sh.fwd_compute_s + sh.bwd_compute_s, sh.param_bytes);
        b.act_in_from_host = b.t.activation_in_bytes > 0;
        b.act_out = BoundaryOut::kHost;
        emit(std::move(b));
      }
    }
  }

  out.options.job_names = job_names(jobs.size());
  for (const DeviceSpec& dev : cluster.devices) {
    double reserve = 0;
    if (policy.kind == BufferPolicy::Kind::kAuto) {
      reserve = parts.empty() ? 0 : parts.front().buffer_reserve_bytes;
    } else if (policy.kind == BufferPolicy::Kind::kFraction) {
      reserve = policy.value * dev.mem_bytes;
    } else {
      reserve = policy.value;
    }
    out.options.prefetch_buffer_bytes.push_back(reserve);
  }
  out.scheduler = std::make_unique<SharpScheduler>(out.tasks, sharp_task_estimates(out.tasks, cluster.h2d));
  out.partitionings = std::move(parts);
  return out;
}

CompiledStrategy compile_task_parallel(const StrategyConfig& cfg, const std::vector<ModelJob>& jobs,
                                       const ClusterSpec& cluster) {
  CompiledStrategy out;
  out.config = cfg;
  const DeviceSpec& tight = cluster.devices[static_cast<size_t>(tightest_device(cluster))];
  std::vector<std::vector<int>> lists;
  std::vector<double> totals;
  std::vector<int> job_of;
  for (size_t j = 0; j < jobs.size(); ++j) {
    const ModelProfile& m = jobs[j].model;
    const double need = resident_training_footprint(m);
    if (need > tight.mem_bytes) {
      throw InfeasibleOOM("task-parallel", "j" + std::to_string(j), tight.device_id, need, tight.mem_bytes);
    }
    std::vector<int> list;
    int prev = -1;
    for (int mb = 0; mb < jobs[j].total_minibatches(); ++mb) {
      for (int half = 0; half < 2; ++half) {
        const bool fwd = half == 0;
        SimTask task = plain_task(static_cast<int>(j), mb, 0, fwd ? Direction::kForward : Direction::kBackward,
                                  fwd && mb == 0 ? m.total_param_bytes() : 0.0, 0.0, 0.0,
                                  fwd ? m.total_fwd_compute_s() : m.total_bwd_compute_s(), 0.0);
        task.act_in_from_host = false;
        task.act_out = BoundaryOut::kNone;
        if (prev >= 0) task.preds.push_back(prev);
        prev = static_cast<int>(out.tasks.size());
        out.tasks.push_back(std::move(task));
        job_of.push_back(static_cast<int>(j));
        list.push_back(prev);
      }
    }
    double total = 0;
    for (int t : list) {
      const ShardTask& st = out.tasks[static_cast<size_t>(t)].t;
      total += st.compute_s + xfer_s(st.param_load_bytes, cluster.h2d);
    }
    lists.push_back(std::move(list));
    totals.push_back(total);
  }
  out.options.job_names = job_names(jobs.size());
  out.scheduler = std::make_unique<WholeJobScheduler>(std::move(lists), std::move(totals), std::move(job_of),
                                                      static_cast<int>(cluster.devices.size()));
  return out;
}

}  // namespace

Feasibility check_feasibility(const StrategyConfig& cfg, const std::vector<ModelJob>& jobs,
                              const ClusterSpec& cluster, const BufferPolicy& policy) {
  Feasibility f;
  f.strategy = to_string(cfg.kind);
  try {
    validate(cluster);
    for (const ModelJob& job : jobs) validate(job);
    const DeviceSpec& dev = cluster.devices[static_cast<size_t>(tightest_device(cluster))];
    switch (cfg.kind) {
      case StrategyKind::kTaskParallel:
        for (size_t j = 0; j < jobs.size(); ++j) {
          const double need = resident_training_footprint(jobs[j].model);
          if (need > dev.mem_bytes) {
            throw InfeasibleOOM(f.strategy, "j" + std::to_string(j), dev.device_id, need, dev.mem_bytes);
          }
        }
        break;
      case StrategyKind::kSharp:
      case StrategyKind::kExactOptimal: {
        double host_need = 0;
        for (const ModelJob& job : jobs) host_need += spilled_host_bytes(job.model, partition(job.model, dev, policy));
        if (host_need > cluster.host_dram_bytes) throw HostOOM(host_need, cluster.host_dram_bytes);
        break;
      }
      default:
        unsupported(cfg.kind);
    }
  } catch (const InfeasibleOOM& e) {
    f.ok = false;
    f.detail = e.what();
    f.job = e.job;
    f.device = e.device;
    f.required_bytes = e.required_bytes;
    f.available_bytes = e.available_bytes;
  } catch (const SingleLayerTooLarge& e) {
    f.ok = false;
    f.detail = e.what();
    f.required_bytes = e.footprint_bytes;
    f.available_bytes = e.capacity_bytes;
  } catch (const HostOOM& e) {
    f.ok = false;
    f.detail = e.what();
    f.required_bytes = e.required_bytes;
    f.available_bytes = e.available_bytes;
  } catch (const CapacityExhausted& e) {
    f.ok = false;
    f.detail = e.what();
    f.device = e.device;
    f.required_bytes = e.required_bytes;
    f.available_bytes = e.available_bytes;
  } catch (const Error& e) {
    f.ok = false;
    f.detail = e.what();
  }
  return f;
}

CompiledStrategy build_strategy(const StrategyConfig& cfg, const std::vector<ModelJob>& jobs,
                                const ClusterSpec& cluster, const BufferPolicy& policy) {
  return build_strategy(cfg, jobs, cluster, policy, PinnedBoundaries{});
}

CompiledStrategy build_strategy(const StrategyConfig& cfg, const std::vector<ModelJob>& jobs,
                                const ClusterSpec& cluster, const BufferPolicy& policy,
                                const PinnedBoundaries& pinned) {
  validate(cluster);
  for (const ModelJob& job : jobs) validate(job);
  if (jobs.empty()) throw InvalidArgument("no jobs to schedule");
  bool any_pinned = false;
  for (const auto& b : pinned) any_pinned = any_pinned || !b.empty();
  if (any_pinned && cfg.kind != StrategyKind::kSharp) {
    throw InvalidArgument("pinned shard boundaries apply to the sharp strategy only");
  }
  switch (cfg.kind) {
    case StrategyKind::kSharp: return compile_sharp(cfg, jobs, cluster, policy, any_pinned ? &pinned : nullptr);
    case StrategyKind::kTaskParallel: return compile_task_parallel(cfg, jobs, cluster);
    default: unsupported(cfg.kind);
  }
}

SimTrace run_strategy(const StrategyConfig& cfg, const std::vector<ModelJob>& jobs,
                      const ClusterSpec& cluster, const BufferPolicy& policy, bool double_buffering) {
  CompiledStrategy compiled = build_strategy(cfg, jobs, cluster, policy);
  compiled.options.double_buffering = double_buffering;
  return run_simulation(cluster, compiled.tasks, *compiled.scheduler, compiled.options);
}

// ---------------------------------------------------------------------------
// Reduced instances (chains of plain durations)

void validate(const TaskInstance& inst) {
  if (inst.devices < 1) throw InvalidArgument("instance needs >= 1 device");
  for (size_t i = 0; i < inst.tasks.size(); ++i) {
    const TaskInstance::Task& t = inst.tasks[i];
    if (!(t.duration_s > 0) || !std::isfinite(t.duration_s)) {
      throw InvalidArgument("task durations must be positive and finite");
    }
    if (t.pred >= static_cast<int>(i) || t.pred < -1) {
      throw InvalidArgument("chain predecessors must precede their task in the list");
    }
  }
}

std::pair<double, double> lower_bounds(const TaskInstance& inst) {
  validate(inst);
  double total = 0, longest = 0;
  std::vector<double> chain(inst.tasks.size(), 0.0);
  for (size_t i = 0; i < inst.tasks.size(); ++i) {
    const TaskInstance::Task& t = inst.tasks[i];
    total += t.duration_s;
    chain[i] = t.duration_s + (t.pred >= 0 ? chain[static_cast<size_t>(t.pred)] : 0.0);
    longest = std::max(longest, chain[i]);
  }
  return {total / inst.devices, longest};
}

}  // namespace spillsim
