// hy_execute_json: config -> SHARP (or task-parallel) plan -> real B200 execution.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <memory>

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

// Everything one execution needs, owned together (the Executor borrows from it).
struct Session {
  WorkloadConfig cfg;
  std::string strategy;
  std::vector<ModelJob> jobs;
  PinnedBoundaries pinned;
  CompiledStrategy cs;
  DispatchPlan plan;
  ExecOptions ex;
  double plan_s = 0;
  std::unique_ptr<Executor> exec;
  double samples_per_pass = 0, model_flops_per_pass = 0;
};

std::unique_ptr<Session> make_session(const std::string& request) {
  auto S = std::make_unique<Session>();
  const json req = json::parse(request);
  S->cfg = parse_workload_config(req.at("config").dump());
  const int gpus = req.value("gpus", 0);
  if (gpus > 0) replicate_devices(S->cfg.cluster, gpus);
  S->strategy = req.value("strategy", std::string("sharp"));
  const bool db = req.value("double_buffering", S->cfg.options.double_buffering);
  S->jobs = materialize_jobs(S->cfg);
  S->pinned = pinned_boundaries(req, S->jobs.size());
  S->cs = build_strategy(strategy_for(S->cfg, strategy_kind_from_string(S->strategy)), S->jobs, S->cfg.cluster,
                         S->cfg.options.buffer_policy, S->pinned);
  S->cs.options.double_buffering = db;
  const auto t0 = std::chrono::steady_clock::now();
  S->plan = plan_simulation(S->cfg.cluster, S->cs.tasks, *S->cs.scheduler, S->cs.options);
  S->plan_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  ExecOptions& ex = S->ex;
  ex.seed = req.value("seed", static_cast<uint64_t>(S->cfg.seed));
  ex.passes = req.value("passes", 1);
  ex.warmup_passes = req.value("warmup_passes", 0);
  ex.params_out_dir = req.value("params_out_dir", std::string());
  ex.hbm_slack_bytes = req.value("hbm_slack_bytes", 0.0);
  ex.debug_skip = req.value("debug_skip", 0);
  ex.host_opt_fraction = req.value("host_opt_fraction", 0.0);
  if (ex.host_opt_fraction < 0 || ex.host_opt_fraction > 1) throw InvalidArgument("host_opt_fraction must be in [0, 1]");
  ex.host_opt_threads = req.value("host_opt_threads", 0);
  ex.write_through = req.value("write_through", false);
  ex.mv_cache = req.value("mv_cache", true);
  ex.mv_cache_max_bytes = req.value("mv_cache_max_bytes", -1.0);
  ex.p2p = req.value("p2p", true);
  const std::string schedule = req.value("schedule", std::string("plan"));
  if (schedule != "plan" && schedule != "dynamic") throw InvalidArgument("schedule must be 'plan' or 'dynamic'");
  if (schedule == "dynamic") {
    ex.dynamic = true;
    Session* raw = S.get();
    ex.scheduler_factory = [raw]() {
      CompiledStrategy c = build_strategy(strategy_for(raw->cfg, strategy_kind_from_string(raw->strategy)), raw->jobs,
                                          raw->cfg.cluster, raw->cfg.options.buffer_policy, raw->pinned);
      return std::move(c.scheduler);
    };
  }
  const std::string prec = req.value("precision", std::string("tf32"));
  if (prec != "tf32" && prec != "fp32" && prec != "bf16") {
    throw InvalidArgument("precision must be 'tf32', 'fp32' or 'bf16'");
  }
  ex.precision_fp32 = prec == "fp32";
  ex.precision_bf16 = prec == "bf16";
  const std::string state = req.value("opt_state", std::string("fp32"));
  if (state != "fp32" && state != "bf16") throw InvalidArgument("opt_state must be 'fp32' or 'bf16'");
  ex.opt_state_bf16 = state == "bf16";
  if (req.contains("device_ids")) ex.device_ids = req["device_ids"].get<std::vector<int>>();
  if (req.contains("run_devices")) ex.run_devices = req["run_devices"].get<std::vector<int>>();
  if (req.contains("opt_chunk_floats")) ex.opt_chunk_floats = req["opt_chunk_floats"].get<long>();
  if (req.contains("splitk_max_floats")) ex.splitk_max_floats = req["splitk_max_floats"].get<long>();
  ex.ring_first = req.value("ring_first", true);
  ex.opt_priority = req.value("opt_priority", ex.opt_priority);
  ex.pool_extra_max_bytes = req.value("pool_extra_max_bytes", -1.0);
  for (size_t j = 0; j < S->cfg.jobs.size(); ++j) {
    std::vector<int> starts{0};
    if (j < S->cs.partitionings.size()) starts = S->cs.partitionings[j].shard_starts;
    ex.jobs.push_back(exec_job_for(S->cfg, S->cfg.jobs[j], starts));
  }
  // Work of the GPUs this process executes, per pass.
  const int G = static_cast<int>(S->cfg.cluster.devices.size());
  const auto per_dev = S->plan.per_device(G);
  std::vector<int> run = ex.run_devices;
  if (run.empty()) {
    for (int d = 0; d < G; ++d) run.push_back(d);
  }
  for (int d : run) {
    for (int t : per_dev[static_cast<size_t>(d)]) {
      const ShardTask& task = S->cs.tasks[static_cast<size_t>(t)].t;
      const JobConfig& jc = S->cfg.jobs[static_cast<size_t>(task.job)];
      double F = 1.0;
      for (const ModelSpec& m : S->cfg.models) {
        if (m.name == jc.model && m.transformer) F = m.transformer->device_reference_flops;
      }
      S->model_flops_per_pass += task.compute_s * F;
      if (task.direction == Direction::kBackward && task.shard == 0) S->samples_per_pass += jc.batch_size;
    }
  }
  S->exec = std::make_unique<Executor>(S->cfg.cluster, S->cs.tasks, S->plan, S->cs.options, ex);
  return S;
}

ojson session_result(Session& S, bool with_trace) {
  const ExecResult& r = S.exec->result();
  ojson out;
  char h[32];
  std::snprintf(h, sizeof h, "%016llx", S.plan.hash());
  out["dispatch_hash"] = h;
  if (!r.dispatch_log.empty()) {  // dynamic mode: what actually ran (last pass)
    DispatchPlan measured;
    measured.order = r.dispatch_log;
    std::snprintf(h, sizeof h, "%016llx", measured.hash());
    out["dispatch_hash_measured"] = h;
    ojson dl = ojson::array();
    for (const Dispatch& d : r.dispatch_log) dl.push_back({d.task, d.device, d.prefetch ? 1 : 0});
    out["dispatch_measured"] = dl;
    out["schedule"] = "dynamic";
  }
  out["virtual_makespan_s"] = S.plan.trace.makespan_s;
  out["plan_wall_s"] = S.plan_s;
  out["pass_seconds"] = r.pass_seconds;
  out["makespan_s"] = r.stats.makespan_s;
  out["samples_per_pass"] = S.samples_per_pass;
  out["model_flops_per_pass"] = S.model_flops_per_pass;
  ojson losses = ojson::array();
  for (const auto& l : r.losses) losses.push_back(l);
  out["losses"] = losses;
  ojson parts = ojson::array();
  for (const Partitioning& p : S.cs.partitionings) parts.push_back(p.shard_starts);
  out["shard_starts"] = parts;
  ojson st;
  const double np = static_cast<double>(std::max<size_t>(1, r.pass_seconds.size()));
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
  st["host_opt_params_per_pass"] = r.stats.host_opt_params / np;
  st["host_grad_d2h_bytes_per_pass"] = r.stats.host_grad_d2h_bytes / np;
  st["refresh_h2d_bytes_per_pass"] = r.stats.refresh_h2d_bytes / np;
  st["writeback_d2h_bytes_per_pass"] = r.stats.writeback_d2h_bytes / np;
  st["mv_load_h2d_bytes_per_pass"] = r.stats.mv_load_h2d_bytes / np;
  st["mv_writeback_d2h_bytes_per_pass"] = r.stats.mv_writeback_d2h_bytes / np;
  st["mv_resident_updates_per_pass"] = r.stats.mv_resident_updates / np;
  st["mv_cache_bytes"] = r.stats.mv_cache_bytes;
  st["p2p_bytes_per_pass"] = r.stats.p2p_bytes / np;
  st["stash_reuses_per_pass"] = r.stats.stash_reuses / np;
  st["arena_bytes"] = r.stats.arena_bytes;
  st["pinned_bytes"] = r.stats.pinned_bytes;
  st["device_busy_s_last_pass"] = r.stats.device_busy_s.empty() ? 0.0 : r.stats.device_busy_s.back();
  st["setup_s"] = r.stats.setup_s;
  st["enqueue_s_last_pass"] = r.stats.enqueue_s.empty() ? 0.0 : r.stats.enqueue_s.back();
  out["stats"] = st;
  if (!r.op_profile_ms.empty()) out["op_profile_ms"] = r.op_profile_ms;
  if (!r.links.empty()) {
    ojson ls = ojson::array();
    for (const LinkStats& l : r.links) {
      ls.push_back({{"plan_device", l.plan_device}, {"pass_s", l.pass_s}, {"h2d_busy_s", l.h2d_busy_s},
                    {"d2h_busy_s", l.d2h_busy_s}, {"link_busy_s", l.link_busy_s},
                    {"compute_busy_s", l.compute_busy_s}, {"exposed_s", l.exposed_s},
                    {"overlap_frac", l.link_busy_s > 0 ? 1.0 - l.exposed_s / l.link_busy_s : 1.0},
                    {"h2d_bytes", l.h2d_bytes}, {"d2h_bytes", l.d2h_bytes}, {"copies", l.copies}, {"ops", l.ops}});
      if (!l.raw.empty()) ls.back()["raw"] = l.raw;
    }
    out["links"] = ls;
  }
  if (!r.pass_seconds.empty()) {
    out["report"] = ojson::parse(report_to_json(summarize(r.trace, S.cfg.cluster, S.strategy)));
    if (with_trace) out["chrome_trace"] = to_chrome_trace_json(r.trace);
  }
  return out;
}

std::string execute_json(const std::string& request) {
  const auto t_call = std::chrono::steady_clock::now();
  const json req = json::parse(request);
  std::unique_ptr<Session> S = make_session(request);
  S->exec->run(S->ex.warmup_passes, false);
  S->exec->run(S->ex.passes, true);
  if (!S->ex.params_out_dir.empty()) S->exec->dump_params(S->ex.params_out_dir);
  ojson out = session_result(*S, req.value("trace", false));
  out["wall_s"] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call).count();
  return out.dump();
}

void* session_create(const std::string& request) { return make_session(request).release(); }

std::string session_run(void* handle, int passes, int timed, bool with_trace) {
  Session* S = static_cast<Session*>(handle);
  const auto t0 = std::chrono::steady_clock::now();
  S->exec->run(passes, timed != 0, timed == 2);
  ojson out = session_result(*S, with_trace);
  out["wall_s"] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out.dump();
}

void session_dump_params(void* handle, const std::string& dir) { static_cast<Session*>(handle)->exec->dump_params(dir); }
size_t session_read_params(void* handle, int job, float* dst, size_t n) {
  return static_cast<Session*>(handle)->exec->read_params(job, dst, n);
}

void session_destroy(void* handle) { delete static_cast<Session*>(handle); }

}  // namespace hy
