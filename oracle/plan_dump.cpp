// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// plan_dump: runs the planning path of the spillsim API (partition -> build_strategy ->
// Sharded-LRTF dispatch -> virtual-time engine -> report / Chrome trace) on a case file
// and prints everything as canonical JSON. The same source is compiled twice:
//   * against the REFERENCE sources (/root/reference/proj/core, built by oracle/Makefile
//     into oracle/_ref/plan_dump_ref) -> golden files under tests/golden/plan_*.json
//   * against this repo's B200 build (build/plan_dump_b200) -> compared byte-for-byte
// Only the reference's public API (spillsim/*.hpp) is used, so parity is on the
// drop-in boundary itself.
//
// Case file: {"config": <workload config v1>, "gpus": [1,2,...], "strategies": [...],
//             "double_buffering": [true,false], "events": true|false}
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>

#include "nlohmann/json.hpp"
#include "spillsim/config.hpp"
#include "spillsim/errors.hpp"
#include "spillsim/metrics.hpp"
#include "spillsim/partitioner.hpp"
#include "spillsim/sim.hpp"
#include "spillsim/strategies.hpp"
#include "spillsim/trace_export.hpp"

using namespace spillsim;
using ojson = nlohmann::ordered_json;

namespace {

std::string g17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

// Forwards to the strategy's scheduler and records each dispatch.
class Recorder : public TaskScheduler {
 public:
  explicit Recorder(TaskScheduler& inner) : inner_(inner) {}
  std::optional<int> next_task(int device, bool prefetch, int running) override {
    last_prefetch_ = prefetch;
    return inner_.next_task(device, prefetch, running);
  }
  void on_dispatch(int task, int device) override {
    log.push_back({task, device, last_prefetch_ ? 1 : 0});
    inner_.on_dispatch(task, device);
  }
  void on_complete(int task) override { inner_.on_complete(task); }
  std::vector<std::array<int, 3>> log;

 private:
  TaskScheduler& inner_;
  bool last_prefetch_ = false;
};

unsigned long long fnv_dispatch(const std::vector<std::array<int, 3>>& log) {
  unsigned long long h = 1469598103934665603ULL;
  for (const auto& e : log) {
    const unsigned long long v = static_cast<unsigned long long>(e[0]) * 8ULL + static_cast<unsigned long long>(e[1]);
    h ^= v;  // whole-value FNV-1a step, as quoted in BASELINE.md §3
    h *= 1099511628211ULL;
  }
  return h;
}

ClusterSpec with_gpus(const ClusterSpec& base, int g) {
  ClusterSpec c = base;
  c.devices.clear();
  for (int d = 0; d < g; ++d) {
    DeviceSpec dev = base.devices[static_cast<size_t>(d) % base.devices.size()];
    dev.device_id = "gpu" + std::to_string(d);
    c.devices.push_back(dev);
  }
  return c;
}

ojson dump_partition(const Partitioning& p) {
  ojson j;
  j["model"] = p.model_name;
  j["shard_starts"] = p.shard_starts;
  j["reserve"] = g17(p.buffer_reserve_bytes);
  j["cap"] = g17(p.effective_capacity_bytes);
  ojson shards = ojson::array();
  for (const Shard& s : p.shards) {
    shards.push_back({s.layer_begin, s.layer_end, g17(s.param_bytes), g17(s.boundary_activation_bytes),
                      g17(s.fwd_compute_s), g17(s.bwd_compute_s), g17(s.peak_exec_bytes)});
  }
  j["shards"] = shards;
  return j;
}

ojson dump_tasks(const std::vector<SimTask>& tasks) {
  ojson arr = ojson::array();
  for (const SimTask& t : tasks) {
    arr.push_back({t.t.job, t.t.minibatch, t.t.shard, t.t.direction == Direction::kForward ? "F" : "B",
                   g17(t.t.param_load_bytes), g17(t.t.activation_in_bytes), g17(t.t.activation_out_bytes),
                   g17(t.t.compute_s), g17(t.t.grad_offload_bytes), t.preds, t.act_in_from_host ? 1 : 0,
                   static_cast<int>(t.act_out)});
  }
  return arr;
}

ojson run_case(const WorkloadConfig& cfg, const std::string& strategy, int g, bool db, bool with_events) {
  ojson j;
  j["strategy"] = strategy;
  j["gpus"] = g;
  j["double_buffering"] = db;
  const ClusterSpec cluster = with_gpus(cfg.cluster, g);
  const std::vector<ModelJob> jobs = materialize_jobs(cfg);
  const StrategyConfig sc = strategy_for(cfg, strategy_kind_from_string(strategy));
  const Feasibility f = check_feasibility(sc, jobs, cluster, cfg.options.buffer_policy);
  j["feasible"] = f.ok;
  j["feasibility_detail"] = f.detail;
  try {
    CompiledStrategy cs = build_strategy(sc, jobs, cluster, cfg.options.buffer_policy);
    cs.options.double_buffering = db;
    ojson parts = ojson::array();
    for (const Partitioning& p : cs.partitionings) parts.push_back(dump_partition(p));
    j["partitions"] = parts;
    j["n_tasks"] = cs.tasks.size();
    j["tasks"] = dump_tasks(cs.tasks);
    if (sc.kind == StrategyKind::kSharp) {
      ojson est = ojson::array();
      for (double e : sharp_task_estimates(cs.tasks, cluster.h2d)) est.push_back(g17(e));
      j["estimates"] = est;
    }
    ojson pbuf = ojson::array();
    for (double b : cs.options.prefetch_buffer_bytes) pbuf.push_back(g17(b));
    j["prefetch_buffer_bytes"] = pbuf;
    Recorder rec(*cs.scheduler);
    const SimTrace tr = run_simulation(cluster, cs.tasks, rec, cs.options);
    check_trace_invariants(tr);
    ojson disp = ojson::array();
    for (const auto& e : rec.log) disp.push_back({e[0], e[1], e[2]});
    j["dispatch"] = disp;
    char hbuf[32];
    std::snprintf(hbuf, sizeof hbuf, "%016llx", fnv_dispatch(rec.log));
    j["dispatch_hash"] = hbuf;
    j["makespan"] = g17(tr.makespan_s);
    j["n_events"] = tr.events.size();
    j["resource_names"] = tr.resource_names;
    j["task_labels_head"] = std::vector<std::string>(
        tr.task_labels.begin(), tr.task_labels.begin() + std::min<size_t>(tr.task_labels.size(), 16));
    if (with_events) {
      ojson ev = ojson::array();
      for (const SimEvent& e : tr.events) {
        ev.push_back({e.resource, to_string(e.kind), e.task, g17(e.start_s), g17(e.end_s)});
      }
      j["events"] = ev;
      j["chrome_trace"] = to_chrome_trace_json(tr);
    }
    const RunReport rep = summarize(tr, cluster, strategy);
    j["report_json"] = report_to_json(rep);
    j["report_csv"] = report_to_csv(rep);
    j["report_text"] = report_to_text(rep);
  } catch (const Error& e) {
    j["error"] = e.what();
  }
  return j;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: plan_dump CASE.json\n");
    return 2;
  }
  std::ifstream in(argv[1]);
  std::stringstream ss;
  ss << in.rdbuf();
  const nlohmann::json spec = nlohmann::json::parse(ss.str());
  ojson out;
  try {
    const WorkloadConfig cfg = parse_workload_config(spec["config"].dump());
    out["serialized"] = serialize_workload_config(cfg);
    const WorkloadConfig again = parse_workload_config(serialize_workload_config(cfg));
    out["roundtrip_equal"] = serialize_workload_config(again) == serialize_workload_config(cfg);
    const bool events = spec.value("events", true);
    ojson runs = ojson::array();
    for (const auto& strat : spec["strategies"]) {
      for (const auto& g : spec["gpus"]) {
        for (const auto& db : spec.value("double_buffering", std::vector<bool>{true})) {
          runs.push_back(run_case(cfg, strat.get<std::string>(), g.get<int>(), db, events));
        }
      }
    }
    out["runs"] = runs;
  } catch (const Error& e) {
    out["config_error"] = e.what();
  }
  std::cout << out.dump(1) << "\n";
  return 0;
}
