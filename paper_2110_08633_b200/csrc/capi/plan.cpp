// hy_plan_json: the planning path (config -> partitions -> SHARP tasks -> virtual-time
// dispatch plan -> report) behind one JSON call, for bindings that cannot use C++.
#include <cstdio>

#include "capi_internal.hpp"
#include "nlohmann/json.hpp"
#include "spillsim/config.hpp"
#include "spillsim/errors.hpp"
#include "spillsim/metrics.hpp"
#include "spillsim/trace_export.hpp"
#include "workload.hpp"

namespace hy {

using json = nlohmann::json;
using ojson = nlohmann::ordered_json;
using namespace spillsim;

std::string plan_json(const std::string& request) {
  const json req = json::parse(request);
  WorkloadConfig cfg = parse_workload_config(req.at("config").dump());
  const int gpus = req.value("gpus", 0);
  if (gpus > 0) replicate_devices(cfg.cluster, gpus);
  const std::string strategy = req.value("strategy", std::string("sharp"));
  const bool db = req.value("double_buffering", cfg.options.double_buffering);
  const std::vector<ModelJob> jobs = materialize_jobs(cfg);
  CompiledStrategy cs = build_strategy(strategy_for(cfg, strategy_kind_from_string(strategy)), jobs, cfg.cluster,
                                       cfg.options.buffer_policy, pinned_boundaries(req, jobs.size()));
  cs.options.double_buffering = db;
  const DispatchPlan plan = plan_simulation(cfg.cluster, cs.tasks, *cs.scheduler, cs.options);

  ojson out;
  ojson parts = ojson::array();
  for (const Partitioning& p : cs.partitionings) {
    ojson pj;
    pj["model"] = p.model_name;
    pj["shard_starts"] = p.shard_starts;
    pj["buffer_reserve_bytes"] = p.buffer_reserve_bytes;
    pj["effective_capacity_bytes"] = p.effective_capacity_bytes;
    ojson shards = ojson::array();
    for (const Shard& s : p.shards) {
      shards.push_back({{"layer_begin", s.layer_begin}, {"layer_end", s.layer_end}, {"param_bytes", s.param_bytes},
                        {"boundary_activation_bytes", s.boundary_activation_bytes},
                        {"fwd_compute_s", s.fwd_compute_s}, {"bwd_compute_s", s.bwd_compute_s},
                        {"peak_exec_bytes", s.peak_exec_bytes}});
    }
    pj["shards"] = shards;
    parts.push_back(pj);
  }
  out["partitions"] = parts;
  ojson tasks = ojson::array();
  for (const SimTask& t : cs.tasks) {
    tasks.push_back({{"job", t.t.job}, {"minibatch", t.t.minibatch}, {"shard", t.t.shard},
                     {"dir", t.t.direction == Direction::kForward ? "F" : "B"},
                     {"param_load_bytes", t.t.param_load_bytes}, {"activation_in_bytes", t.t.activation_in_bytes},
                     {"activation_out_bytes", t.t.activation_out_bytes}, {"compute_s", t.t.compute_s},
                     {"grad_offload_bytes", t.t.grad_offload_bytes}, {"preds", t.preds}});
  }
  out["tasks"] = tasks;
  ojson disp = ojson::array();
  for (const Dispatch& d : plan.order) disp.push_back({d.task, d.device, d.prefetch ? 1 : 0});
  out["dispatch"] = disp;
  char h[32];
  std::snprintf(h, sizeof h, "%016llx", plan.hash());
  out["dispatch_hash"] = h;
  out["makespan_s"] = plan.trace.makespan_s;
  out["report"] = ojson::parse(report_to_json(summarize(plan.trace, cfg.cluster, strategy)));
  if (req.value("trace", false)) out["chrome_trace"] = to_chrome_trace_json(plan.trace);
  return out.dump();
}

}  // namespace hy
