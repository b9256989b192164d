// ORACLE / TEST INFRASTRUCTURE ONLY — a C shim over the REFERENCE's compiled core so
// Python tests and bench.py's reference arm can call the reference planner in-process
// (ctypes). Built into oracle/_ref/libspillsim_ref.so by oracle/Makefile.
#include <chrono>
#include <cstring>
#include <string>

#include "spillsim/config.hpp"
#include "spillsim/errors.hpp"
#include "spillsim/strategies.hpp"

using namespace spillsim;

extern "C" {

// Plans and simulates `strategy` for the config with its devices replicated to `gpus`
// entries. Returns 0 and fills makespan + wall seconds, or -1 with msg filled.
int ref_run_strategy(const char* config_json, const char* strategy, int gpus, double* makespan_s,
                     double* wall_s, char* msg, int msg_len) {
  try {
    WorkloadConfig cfg = parse_workload_config(config_json);
    if (gpus > 0) {
      DeviceSpec proto = cfg.cluster.devices.front();
      cfg.cluster.devices.clear();
      for (int d = 0; d < gpus; ++d) {
        DeviceSpec dev = proto;
        dev.device_id = "gpu" + std::to_string(d);
        cfg.cluster.devices.push_back(dev);
      }
    }
    const auto jobs = materialize_jobs(cfg);
    const auto kind = strategy_kind_from_string(strategy);
    const auto t0 = std::chrono::steady_clock::now();
    const SimTrace tr = run_strategy(strategy_for(cfg, kind), jobs, cfg.cluster, cfg.options.buffer_policy,
                                     cfg.options.double_buffering);
    const auto t1 = std::chrono::steady_clock::now();
    *makespan_s = tr.makespan_s;
    *wall_s = std::chrono::duration<double>(t1 - t0).count();
    return 0;
  } catch (const std::exception& e) {
    if (msg && msg_len > 0) {
      std::strncpy(msg, e.what(), static_cast<size_t>(msg_len) - 1);
      msg[msg_len - 1] = 0;
    }
    return -1;
  }
}

// Shard starts of job `job` under SHARP for the config (the reference partitioner).
int ref_shard_starts(const char* config_json, int job, int* out, int max_out) {
  try {
    const WorkloadConfig cfg = parse_workload_config(config_json);
    const auto jobs = materialize_jobs(cfg);
    const auto cs = build_strategy(strategy_for(cfg, StrategyKind::kSharp), jobs, cfg.cluster, cfg.options.buffer_policy);
    const auto& starts = cs.partitionings.at(static_cast<size_t>(job)).shard_starts;
    const int n = static_cast<int>(starts.size());
    for (int i = 0; i < n && i < max_out; ++i) out[i] = starts[static_cast<size_t>(i)];
    return n;
  } catch (...) {
    return -1;
  }
}

}
