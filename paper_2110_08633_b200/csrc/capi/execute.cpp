// hy_execute_json: config -> SHARP (or task-parallel) plan -> real B200 execution.
#include <chrono>
#include <cmath>
#include <cstdio>

#include "capi_internal.hpp"
#include "nlohmann/json.hpp"
#include "spillsim/config.hpp"
#include "spillsim/errors.hpp"
#include "spillsim/executor.hpp"
#include "spillsim/metrics.hpp"
#include "spillsim/trace_export.hpp"
#include "workload.hpp"

namespace hy {

using json = nlohmann::json;
using ojson = nlohmann::ordered_json;
using namespace spillsim;

namespace {

// Real model of a job: only transformer-generator models describe a trainable network.
ExecJob exec_job_for(const WorkloadConfig& cfg, const JobConfig& jc, const std::vector<int>& starts) {
  for (size_t mi = 0; mi < cfg.models.size(); ++mi) {
    const ModelSpec& spec = cfg.models[mi];
    if (spec.name != jc.model) continue;
    if (!spec.transformer) {
      throw InvalidArgument("model '" + spec.name + "' is not a transformer generator: nothing to execute");
    }
    const TransformerParams& t = *spec.transformer;
    if (t.d_model < 64 || t.d_model % 64 != 0) {
      throw InvalidArgument("model '" + spec.name + "': d_model must be a positive multiple of 64 (head dim 64)");
    }
    ExecJob e;
    e.dims.V = kTransformerVocab;
    e.dims.d = t.d_model;
    e.dims.L = t.n_blocks;
    e.dims.T = t.seq_len;
    e.dims.B = t.batch_size;
    e.dims.H = t.d_model / 64;
    e.model_key = hy_mix64(static_cast<uint64_t>(cfg.seed) * 0x100000001B3ull + mi);
    auto it = jc.hyperparams.find("lr");
    e.lr = it == jc.hyperparams.end() ? 1e-4f : static_cast<float>(std::stod(it->second));
    e.shard_starts = starts;
    return e;
  }
  throw InvalidArgument("unknown model '" + jc.model + "'");
}

}  // namespace

std::string execute_json(const std::string& request) {
  const auto t_call = std::chrono::steady_clock::now();
  const json req = json::parse(request);
  WorkloadConfig cfg = parse_workload_config(req.at("config").dump());
  const int gpus = req.value("gpus", 0);
  if (gpus > 0) replicate_devices(cfg.cluster, gpus);
  const std::string strategy = req.value("strategy", std::string("sharp"));
  const bool db = req.value("double_buffering", cfg.options.double_buffering);
  const std::vector<ModelJob> jobs = materialize_jobs(cfg);
  CompiledStrategy cs = build_strategy(strategy_for(cfg, strategy_kind_from_string(strategy)), jobs, cfg.cluster,
                                       cfg.options.buffer_policy);
  cs.options.double_buffering = db;
  const auto t_plan0 = std::chrono::steady_clock::now();
  const DispatchPlan plan = plan_simulation(cfg.cluster, cs.tasks, *cs.scheduler, cs.options);
  const double plan_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_plan0).count();

  ExecOptions ex;
  ex.seed = req.value("seed", static_cast<uint64_t>(cfg.seed));
  ex.passes = req.value("passes", 1);
  ex.warmup_passes = req.value("warmup_passes", 0);
  ex.params_out_dir = req.value("params_out_dir", std::string());
  ex.hbm_slack_bytes = req.value("hbm_slack_bytes", 0.0);
  if (req.contains("device_ids")) ex.device_ids = req["device_ids"].get<std::vector<int>>();
  if (req.contains("run_devices")) ex.run_devices = req["run_devices"].get<std::vector<int>>();
  if (req.contains("opt_chunk_floats")) ex.opt_chunk_floats = req["opt_chunk_floats"].get<long>();
  for (size_t j = 0; j < cfg.jobs.size(); ++j) {
    std::vector<int> starts{0};
    if (j < cs.partitionings.size()) starts = cs.partitionings[j].shard_starts;
    ex.jobs.push_back(exec_job_for(cfg, cfg.jobs[j], starts));
  }
  ExecResult r = run_execution(cfg.cluster, cs.tasks, plan, cs.options, ex);

  // Work of the executed devices per pass: samples and cost-model roofline terms.
  const int G = static_cast<int>(cfg.cluster.devices.size());
  const auto per_dev = plan.per_device(G);
  std::vector<int> run = ex.run_devices;
  if (run.empty()) {
    for (int d = 0; d < G; ++d) run.push_back(d);
  }
  double samples = 0, roofline_link_s = 0, model_flops = 0;
  for (int d : run) {
    for (int t : per_dev[static_cast<size_t>(d)]) {
      const ShardTask& task = cs.tasks[static_cast<size_t>(t)].t;
      const ModelJob& job = jobs[static_cast<size_t>(task.job)];
      const auto* spec = &cfg.models[0];
      for (const auto& m : cfg.models) {
        if (m.name == cfg.jobs[static_cast<size_t>(task.job)].model) spec = &m;
      }
      const double F = spec->transformer ? spec->transformer->device_reference_flops : 1.0;
      model_flops += task.compute_s * F;
      if (task.direction == Direction::kBackward && task.shard == 0) samples += job.batch_size;
    }
  }
  (void)roofline_link_s;

  ojson out;
  char h[32];
  std::snprintf(h, sizeof h, "%016llx", plan.hash());
  out["dispatch_hash"] = h;
  out["virtual_makespan_s"] = plan.trace.makespan_s;
  out["plan_wall_s"] = plan_s;
  out["pass_seconds"] = r.pass_seconds;
  out["makespan_s"] = r.stats.makespan_s;
  out["samples_per_pass"] = samples;
  out["model_flops_per_pass"] = model_flops;
  ojson losses = ojson::array();
  for (const auto& l : r.losses) losses.push_back(l);
  out["losses"] = losses;
  ojson parts = ojson::array();
  for (const Partitioning& p : cs.partitionings) parts.push_back(p.shard_starts);
  out["shard_starts"] = parts;
  ojson st;
  const double np = std::max<size_t>(1, r.pass_seconds.size());
  st["h2d_bytes_per_pass"] = r.stats.h2d_bytes / np;
  st["d2h_bytes_per_pass"] = r.stats.d2h_bytes / np;
  st["model_h2d_bytes_per_pass"] = r.stats.model_h2d_bytes / np;
  st["model_d2h_bytes_per_pass"] = r.stats.model_d2h_bytes / np;
  st["param_h2d_bytes_per_pass"] = r.stats.param_h2d_bytes / np;
  st["opt_h2d_bytes_per_pass"] = r.stats.opt_h2d_bytes / np;
  st["opt_d2h_bytes_per_pass"] = r.stats.opt_d2h_bytes / np;
  st["act_h2d_bytes_per_pass"] = r.stats.act_h2d_bytes / np;
  st["act_d2h_bytes_per_pass"] = r.stats.act_d2h_bytes / np;
  st["elided_param_bytes_per_pass"] = r.stats.elided_param_bytes / np;
  st["elided_act_bytes_per_pass"] = r.stats.elided_act_bytes / np;
  st["arena_bytes"] = r.stats.arena_bytes;
  st["pinned_bytes"] = r.stats.pinned_bytes;
  st["device_busy_s_last_pass"] = r.stats.device_busy_s.empty() ? 0.0 : r.stats.device_busy_s.back();
  st["setup_s"] = r.stats.setup_s;
  st["adam_launches"] = r.stats.kernel_launches;
  out["stats"] = st;
  out["report"] = ojson::parse(report_to_json(summarize(r.trace, cfg.cluster, strategy)));
  if (req.value("trace", false)) out["chrome_trace"] = to_chrome_trace_json(r.trace);
  out["wall_s"] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call).count();
  return out.dump();
}

}  // namespace hy
