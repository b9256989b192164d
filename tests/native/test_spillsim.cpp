// Native unit tests of the B200 build's host library (libhydra.so) against the
// reference's known-answer cases (proj/tests/test_model.cpp, test_partitioner.cpp,
// test_sim.cpp, test_strategies.cpp, test_config.cpp; cited per case). Plain C++: a
// failure prints the case and the process exits non-zero (driven by
// tests/test_native_host.py).
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "spillsim/config.hpp"
#include "spillsim/errors.hpp"
#include "spillsim/metrics.hpp"
#include "spillsim/partitioner.hpp"
#include "spillsim/sim.hpp"
#include "spillsim/strategies.hpp"
#include "spillsim/trace_export.hpp"

using namespace spillsim;

static int g_fail = 0, g_pass = 0;
#define EXPECT(cond)                                                          \
  do {                                                                        \
    if (cond) {                                                               \
      ++g_pass;                                                               \
    } else {                                                                  \
      ++g_fail;                                                               \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);             \
    }                                                                         \
  } while (0)
#define NEAR(a, b, tol) EXPECT(std::fabs((a) - (b)) <= (tol) * std::max(1.0, std::fabs(b)))

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// Platform-pinned draws (mt19937_64 with hand mapping), as the reference tests use.
struct Rng {
  std::mt19937_64 g;
  explicit Rng(unsigned long long s) : g(s) {}
  int integer(int lo, int hi) { return lo + static_cast<int>(g() % static_cast<unsigned long long>(hi - lo + 1)); }
  double real(double lo, double hi) { return lo + static_cast<double>(g() >> 11) * (1.0 / 9007199254740992.0) * (hi - lo); }
};

static LayerProfile fp_layer(double footprint) {  // pilot footprint all workspace, unit compute
  LayerProfile l;
  l.workspace_bytes = footprint;
  l.fwd_compute_s = 1;
  l.bwd_compute_s = 2;
  return l;
}
static ModelProfile fp_model(const std::vector<double>& fps) {
  ModelProfile m;
  m.name = "fp";
  for (double f : fps) m.layers.push_back(fp_layer(f));
  return m;
}
static std::vector<int> prefix_cuts(const std::vector<double>& fps, double cap) {
  std::vector<int> s{0};
  double run = 0;
  for (size_t i = 0; i < fps.size(); ++i) {
    if (run + fps[i] > cap) {
      s.push_back(static_cast<int>(i));
      run = fps[i];
    } else {
      run += fps[i];
    }
  }
  return s;
}
static DeviceSpec dev(double mem) {
  DeviceSpec d;
  d.device_id = "gpu0";
  d.mem_bytes = mem;
  return d;
}
static ClusterSpec cluster(int n, double mem, double bw, double lat = 0, bool shared = false, bool duplex = true) {
  ClusterSpec c;
  for (int i = 0; i < n; ++i) {
    DeviceSpec d = dev(mem);
    d.device_id = "gpu" + std::to_string(i);
    d.busy_power_w = 300;
    d.idle_power_w = 50;
    d.hourly_price = 3;
    c.devices.push_back(d);
  }
  c.host_dram_bytes = 1e15;
  c.h2d.bandwidth_Bps = bw;
  c.h2d.latency_s = lat;
  c.h2d.shared = shared;
  c.h2d.duplex = duplex;
  return c;
}

struct InOrder : TaskScheduler {  // feeds tasks by index to whichever device asks
  size_t n, next = 0;
  explicit InOrder(size_t total) : n(total) {}
  std::optional<int> next_task(int, bool, int) override {
    return next < n ? std::optional<int>(static_cast<int>(next)) : std::nullopt;
  }
  void on_dispatch(int, int) override { ++next; }
};

static std::vector<SimTask> fwd_chain(const std::vector<double>& loads, const std::vector<double>& comps) {
  std::vector<SimTask> v;
  for (size_t s = 0; s < loads.size(); ++s) {
    SimTask t;
    t.t.shard = static_cast<int>(s);
    t.t.param_load_bytes = loads[s];
    t.t.compute_s = comps[s];
    t.act_in_from_host = false;
    t.act_out = BoundaryOut::kNone;
    if (s) t.preds.push_back(static_cast<int>(s) - 1);
    v.push_back(t);
  }
  return v;
}
static double chain_makespan(const std::vector<SimTask>& t, bool db = true) {
  ClusterSpec c = cluster(1, 1e12, 1.0);
  InOrder sch(t.size());
  SimOptions o;
  o.double_buffering = db;
  const SimTrace tr = run_simulation(c, t, sch, o);
  check_trace_invariants(tr);
  return tr.makespan_s;
}
static int count(const SimTrace& tr, EventKind k) {
  int n = 0;
  for (const SimEvent& e : tr.events) n += e.kind == k;
  return n;
}

static void model_tests() {
  // test_model.cpp:25-32
  const LayerProfile l = make_layer(10, 3, 5, 1);
  EXPECT(pilot_footprint(l) == 2 * 10 + 2 * 3 + 5);
  EXPECT(l.bwd_compute_s == 2.0);
  // test_model.cpp:82-109: GPT-2 XL parameter count, independent formula
  TransformerParams p;
  p.n_blocks = 48;
  p.d_model = 1600;
  p.seq_len = 512;
  p.batch_size = 16;
  p.device_reference_flops = 1e15;
  const ModelProfile xl = make_transformer_model(p);
  EXPECT(xl.layers.size() == 50);
  const double params = xl.total_param_bytes() / 4;
  EXPECT(params == 50257.0 * 1600 + 48 * 12.0 * 1600 * 1600);
  EXPECT(std::fabs(params - 1.5e9) / 1.5e9 < 0.10);
  // test_model.cpp:123-137: block durations linear in batch
  TransformerParams p2 = p;
  p2.batch_size = 32;
  const ModelProfile xl2 = make_transformer_model(p2);
  EXPECT(xl2.layers[1].fwd_compute_s == 2 * xl.layers[1].fwd_compute_s);
  // test_model.cpp:139-147: byte overflow
  TransformerParams huge = p;
  huge.d_model = 1 << 30;
  EXPECT(throws<ByteOverflow>([&] { make_transformer_model(huge); }));
  EXPECT(throws<InvalidArgument>([&] { make_uniform_model(0, l, 0); }));
}

static void partitioner_tests() {
  // test_partitioner.cpp:60-88
  EXPECT(partition(fp_model({6, 6, 6, 6}), dev(16), BufferPolicy::absolute(0)).shard_starts == std::vector<int>({0, 2}));
  EXPECT(partition(fp_model({8, 8}), dev(16), BufferPolicy::absolute(0)).shard_starts == std::vector<int>({0}));
  bool caught = false;
  try {
    partition(fp_model({10, 20}), dev(16), BufferPolicy::absolute(0));
  } catch (const SingleLayerTooLarge& e) {
    caught = e.layer_index == 1;
  }
  EXPECT(caught);
  // test_partitioner.cpp:90-127: random instances vs the prefix-sum oracle
  Rng r(42);
  for (int trial = 0; trial < 300; ++trial) {
    const int n = r.integer(1, 40);
    std::vector<double> fps;
    double mx = 0;
    for (int i = 0; i < n; ++i) {
      fps.push_back(r.integer(1, 50));
      mx = std::max(mx, fps.back());
    }
    const double cap = mx + r.integer(0, 200);
    EXPECT(partition(fp_model(fps), dev(cap), BufferPolicy::absolute(0)).shard_starts == prefix_cuts(fps, cap));
  }
  // test_partitioner.cpp:129-146: auto reserve widens to the largest shard's params
  LayerProfile big;
  big.param_bytes = 40;
  big.fwd_compute_s = 1;
  big.bwd_compute_s = 2;
  const ModelProfile m8 = make_uniform_model(8, big, 0);
  const Partitioning pa = partition(m8, dev(320), BufferPolicy::auto_reserve(0.10));
  EXPECT(pa.buffer_reserve_bytes >= 40);
  double largest = 0;
  for (const Shard& s : pa.shards) largest = std::max(largest, s.param_bytes);
  EXPECT(pa.buffer_reserve_bytes >= largest);
  // test_partitioner.cpp:148-166: imbalance = max fwd / mean fwd
  ModelProfile m2;
  m2.name = "imb";
  LayerProfile a = fp_layer(10), b = fp_layer(10);
  a.fwd_compute_s = 3;
  b.fwd_compute_s = 1;
  m2.layers = {a, b};
  const Partitioning pi = partition_with_boundaries(m2, {0, 1}, dev(100), BufferPolicy::absolute(0));
  NEAR(partition_stats(pi).imbalance, 1.5, 1e-12);
  // boundary text round trip + validation
  EXPECT(boundaries_from_text(boundaries_to_text(pi)) == pi.shard_starts);
  EXPECT(throws<InvalidArgument>([&] { boundaries_from_text("0\n1x\n"); }));
  EXPECT(throws<InvalidArgument>([&] { partition_with_boundaries(m2, {1}, dev(100), BufferPolicy::absolute(0)); }));
  EXPECT(throws<CapacityExhausted>([&] { effective_capacity(dev(1), fp_model({1}), BufferPolicy::absolute(2)); }));
  // monotone: more capacity never yields more shards (acceptance.cpp criterion 1)
  Rng r2(1001);
  for (int trial = 0; trial < 200; ++trial) {
    std::vector<double> fps;
    const int n = r2.integer(1, 60);
    double mx = 0;
    for (int i = 0; i < n; ++i) {
      fps.push_back(r2.integer(1, 100));
      mx = std::max(mx, fps.back());
    }
    const double cap = mx + r2.integer(0, 400);
    const auto p1 = partition(fp_model(fps), dev(cap), BufferPolicy::absolute(0));
    EXPECT(p1.shard_starts == prefix_cuts(fps, cap));
    const auto p2 = partition(fp_model(fps), dev(cap + r2.integer(1, 400)), BufferPolicy::absolute(0));
    EXPECT(p2.shard_count() <= p1.shard_count());
  }
}

static void engine_tests() {
  InterconnectSpec link;
  link.bandwidth_Bps = 16e9;
  link.latency_s = 10e-6;
  NEAR(transfer_time(4e9, link), 0.25001, 1e-12);
  // test_sim.cpp:100-124: F then B with resident-param elision: 2 + 5 + 15
  {
    std::vector<SimTask> t(2);
    t[0].t.param_load_bytes = 2;
    t[0].t.compute_s = 5;
    t[0].act_in_from_host = false;
    t[0].act_out = BoundaryOut::kNone;
    t[1].t.direction = Direction::kBackward;
    t[1].t.param_load_bytes = 2;
    t[1].t.compute_s = 15;
    t[1].act_in_from_host = false;
    t[1].act_out = BoundaryOut::kNone;
    t[1].preds = {0};
    ClusterSpec c = cluster(1, 1e12, 1.0);
    InOrder sch(2);
    const SimTrace tr = run_simulation(c, t, sch);
    NEAR(tr.makespan_s, 22.0, 1e-12);
    EXPECT(count(tr, EventKind::kParamLoad) == 1);
  }
  // test_sim.cpp:126-138: compute-bound hiding and transfer-bound
  NEAR(chain_makespan(fwd_chain({2, 2, 2}, {5, 5, 5})), 17.0, 1e-12);
  NEAR(chain_makespan(fwd_chain({5, 5, 5}, {2, 2, 2})), 17.0, 1e-12);
  // test_sim.cpp:140-151: infinite bandwidth
  {
    ClusterSpec c = cluster(1, 1e12, std::numeric_limits<double>::infinity());
    auto t = fwd_chain({7, 9, 11}, {1.5, 2.5, 3.0});
    for (auto& x : t) {
      x.act_out = BoundaryOut::kHost;
      x.t.activation_out_bytes = 123;
    }
    InOrder sch(t.size());
    NEAR(run_simulation(c, t, sch).makespan_s, 7.0, 1e-12);
  }
  // test_sim.cpp:153-175: zero-byte elision; demote then promote serializes
  {
    auto t = fwd_chain({0, 0}, {1, 1});
    for (auto& x : t) x.act_out = BoundaryOut::kHost;
    ClusterSpec c = cluster(1, 1e12, 1.0);
    InOrder sch(t.size());
    const SimTrace tr = run_simulation(c, t, sch);
    NEAR(tr.makespan_s, 2.0, 1e-12);
    EXPECT(count(tr, EventKind::kParamLoad) == 0 && count(tr, EventKind::kActDemote) == 0);
    auto u = fwd_chain({0, 0}, {4, 6});
    u[0].act_out = BoundaryOut::kHost;
    u[0].t.activation_out_bytes = 3;
    u[1].act_in_from_host = true;
    u[1].t.activation_in_bytes = 3;
    NEAR(chain_makespan(u), 4 + 3 + 3 + 6, 1e-12);
  }
  // test_sim.cpp:177-201: dedicated vs shared down channel
  {
    std::vector<SimTask> t(2);
    for (int j = 0; j < 2; ++j) {
      t[j].t.job = j;
      t[j].t.param_load_bytes = 2;
      t[j].t.compute_s = 1;
      t[j].act_in_from_host = false;
      t[j].act_out = BoundaryOut::kNone;
    }
    ClusterSpec ded = cluster(2, 1e12, 1.0, 0, false);
    SharpScheduler s1(t, {1.0, 1.0});
    NEAR(run_simulation(ded, t, s1).makespan_s, 3.0, 1e-12);
    ClusterSpec sh = cluster(2, 1e12, 1.0, 0, true);
    SharpScheduler s2(t, {1.0, 1.0});
    NEAR(run_simulation(sh, t, s2).makespan_s, 5.0, 1e-12);
  }
  // test_sim.cpp:203-235: full vs half duplex
  {
    std::vector<SimTask> t(2);
    t[0].t.job = 0;
    t[0].t.compute_s = 2;
    t[0].t.activation_out_bytes = 4;
    t[0].act_in_from_host = false;
    t[0].act_out = BoundaryOut::kHost;
    t[1].t.job = 1;
    t[1].t.param_load_bytes = 4;
    t[1].t.compute_s = 2;
    t[1].act_in_from_host = false;
    t[1].act_out = BoundaryOut::kNone;
    InOrder a(2), b(2);
    NEAR(run_simulation(cluster(1, 1e12, 1.0, 0, false, true), t, a).makespan_s, 6.0, 1e-12);
    NEAR(run_simulation(cluster(1, 1e12, 1.0, 0, false, false), t, b).makespan_s, 8.0, 1e-12);
  }
  // test_sim.cpp:237-257: deadlock and buffer overflow are errors
  {
    struct Never : TaskScheduler {
      std::optional<int> next_task(int, bool, int) override { return std::nullopt; }
    } never;
    auto t = fwd_chain({1}, {1});
    ClusterSpec c = cluster(1, 1e12, 1.0);
    EXPECT(throws<DeadlockError>([&] { run_simulation(c, t, never); }));
    auto u = fwd_chain({1, 5}, {3, 3});
    InOrder sch(u.size());
    SimOptions o;
    o.prefetch_buffer_bytes = {2.0};
    EXPECT(throws<BufferOverflow>([&] { run_simulation(c, u, sch, o); }));
  }
  // test_sim.cpp:282-320: random spilled SHARP workloads: conservation + determinism
  Rng r(19);
  for (int trial = 0; trial < 40; ++trial) {
    const int ndev = r.integer(1, 3);
    const bool shared = r.integer(0, 1) == 1;
    ClusterSpec c = cluster(ndev, 64, 8.0, 1e-4, shared);
    c.host_dram_bytes = 1e9;
    std::vector<ModelJob> jobs;
    const int nj = r.integer(1, 4);
    for (int j = 0; j < nj; ++j) {
      LayerProfile l;
      l.param_bytes = r.real(1, 4);
      l.activation_out_bytes = r.real(0, 2);
      l.workspace_bytes = r.real(0, 4);
      l.fwd_compute_s = r.real(0.2, 2);
      l.bwd_compute_s = 2 * l.fwd_compute_s;
      ModelJob job;
      job.model = make_uniform_model(r.integer(1, 6), l, 0, "m" + std::to_string(j));
      job.minibatches_per_epoch = r.integer(1, 2);
      jobs.push_back(job);
    }
    StrategyConfig cfg;
    const BufferPolicy pol = BufferPolicy::absolute(16);
    const SimTrace tr = run_strategy(cfg, jobs, c, pol);
    check_trace_invariants(tr);
    double comp = 0;
    for (const SimTask& t : build_strategy(cfg, jobs, c, pol).tasks) comp += t.t.compute_s;
    NEAR(tr.total_compute_s(), comp, 1e-9);
    EXPECT(to_chrome_trace_json(tr) == to_chrome_trace_json(run_strategy(cfg, jobs, c, pol)));
  }
  // test_sim.cpp:322-341: devices offered work in ascending order
  {
    std::vector<SimTask> t(2);
    for (int j = 0; j < 2; ++j) {
      t[j].t.job = j;
      t[j].t.compute_s = 1;
      t[j].act_in_from_host = false;
      t[j].act_out = BoundaryOut::kNone;
    }
    SharpScheduler s(t, {1.0, 1.0});
    const SimTrace tr = run_simulation(cluster(2, 1e12, 1.0), t, s);
    for (const SimEvent& e : tr.events) {
      if (e.kind == EventKind::kCompute) EXPECT(tr.resource_names[e.resource] == (e.task == 0 ? "gpu0" : "gpu1"));
    }
  }
}

static void scheduler_tests() {
  std::vector<SimTask> t(3);
  for (int j = 0; j < 3; ++j) {
    t[j].t.job = j;
    t[j].t.compute_s = 1;
  }
  {  // test_strategies.cpp:69-135: argmax remaining, ties -> lower job id
    SharpScheduler s(t, {10, 6, 4});
    auto pick = s.next_task(0, false, -1);
    EXPECT(pick && t[*pick].t.job == 0);
    SharpScheduler tie(t, {10, 10, 4});
    pick = tie.next_task(0, false, -1);
    EXPECT(pick && t[*pick].t.job == 0);
  }
  {  // one device per job; the prefetch slot takes the chain successor
    std::vector<SimTask> chain(2);
    chain[0].t.compute_s = chain[1].t.compute_s = 1;
    chain[1].t.shard = 1;
    chain[1].preds = {0};
    SharpScheduler s(chain, {1, 1});
    auto first = s.next_task(0, false, -1);
    EXPECT(first.has_value());
    s.on_dispatch(*first, 0);
    EXPECT(!s.next_task(1, false, -1).has_value());
    auto pf = s.next_task(0, true, *first);
    EXPECT(pf && *pf == 1);
  }
  {  // suffix sums non-increasing and exactly zero at completion
    std::vector<SimTask> c(3);
    for (int i = 0; i < 3; ++i) {
      c[i].t.shard = i;
      c[i].t.compute_s = 1 + i;
      if (i) c[i].preds = {i - 1};
    }
    SharpScheduler s(c, {1, 2, 3});
    double prev = s.remaining_estimate(0);
    EXPECT(prev == 6);
    for (int i = 0; i < 3; ++i) {
      s.on_dispatch(i, 0);
      s.on_complete(i);
      EXPECT(s.remaining_estimate(0) <= prev);
      prev = s.remaining_estimate(0);
    }
    EXPECT(prev == 0.0);
  }
  // test_strategies.cpp:267-286: identical spilled jobs scale; one job cannot use 2 GPUs
  {
    LayerProfile l;
    l.param_bytes = 2;
    l.activation_out_bytes = 1;
    l.fwd_compute_s = 1;
    l.bwd_compute_s = 2;
    std::vector<ModelJob> jobs(4);
    for (auto& j : jobs) j.model = make_uniform_model(4, l, 0);
    const BufferPolicy pol = BufferPolicy::absolute(4);
    const double one = run_strategy(StrategyConfig{}, jobs, cluster(1, 20, 4.0), pol).makespan_s;
    const double two = run_strategy(StrategyConfig{}, jobs, cluster(2, 20, 4.0), pol).makespan_s;
    EXPECT(std::fabs(one / two - 2.0) < 0.02 * 2.0);
    std::vector<ModelJob> single(1, jobs[0]);
    const double s1 = run_strategy(StrategyConfig{}, single, cluster(1, 20, 4.0), pol).makespan_s;
    const double s4 = run_strategy(StrategyConfig{}, single, cluster(4, 20, 4.0), pol).makespan_s;
    NEAR(s1, s4, 1e-12);
  }
  // test_strategies.cpp:324-347: with free transfers SHARP <= task-parallel
  {
    LayerProfile l;
    l.param_bytes = 1;
    l.fwd_compute_s = 1;
    l.bwd_compute_s = 2;
    std::vector<ModelJob> jobs;
    for (int n : {3, 1, 2, 5, 4}) {
      ModelJob j;
      j.model = make_uniform_model(n, l, 0);
      jobs.push_back(j);
    }
    ClusterSpec c = cluster(2, 1e6, std::numeric_limits<double>::infinity());
    StrategyConfig tp;
    tp.kind = StrategyKind::kTaskParallel;
    const double sharp = run_strategy(StrategyConfig{}, jobs, c, BufferPolicy::absolute(10)).makespan_s;
    const double task = run_strategy(tp, jobs, c, BufferPolicy::absolute(10)).makespan_s;
    EXPECT(sharp <= task + 1e-9);
  }
  // feasibility verdicts carry the refusal (test_strategies.cpp:366-385)
  {
    LayerProfile l;
    l.param_bytes = 100;
    l.fwd_compute_s = 1;
    l.bwd_compute_s = 2;
    std::vector<ModelJob> jobs(1);
    jobs[0].model = make_uniform_model(4, l, 0);
    StrategyConfig tp;
    tp.kind = StrategyKind::kTaskParallel;
    const Feasibility f = check_feasibility(tp, jobs, cluster(1, 500, 1.0));
    EXPECT(!f.ok && f.required_bytes > f.available_bytes && f.device == "gpu0");
    ClusterSpec tiny_host = cluster(1, 500, 1.0);
    tiny_host.host_dram_bytes = 10;
    EXPECT(!check_feasibility(StrategyConfig{}, jobs, tiny_host, BufferPolicy::absolute(100)).ok);
    EXPECT(throws<HostOOM>([&] { build_strategy(StrategyConfig{}, jobs, tiny_host, BufferPolicy::absolute(100)); }));
  }
  EXPECT(strategy_kind_from_string("sharp") == StrategyKind::kSharp);
  EXPECT(throws<InvalidArgument>([] { strategy_kind_from_string("nope"); }));
}

static void config_tests() {
  const char* base = R"({"schema_version": 1,
    "cluster": {"devices": [{"id": "g", "mem_bytes": 64}], "host_dram_bytes": 1e9,
                "h2d": {"bandwidth_Bps": 8}},
    "models": [{"name": "m", "generator": {"kind": "uniform", "n_layers": 4,
               "layer": {"param_bytes": 4, "fwd_compute_s": 1}}}],
    "jobs": [{"model": "m", "minibatches_per_epoch": 2}]})";
  const WorkloadConfig cfg = parse_workload_config(base);
  EXPECT(cfg.jobs.size() == 1 && cfg.models.size() == 1);
  const std::string s1 = serialize_workload_config(cfg);
  EXPECT(serialize_workload_config(parse_workload_config(s1)) == s1);
  // unknown fields are rejected at every level (test_config.cpp:66-77)
  std::string bad = base;
  bad.replace(bad.find("\"jobs\""), 6, "\"jobz\"");
  EXPECT(throws<ConfigError>([&] { parse_workload_config(bad); }));
  std::string bad2 = base;
  bad2.replace(bad2.find("\"mem_bytes\""), 11, "\"mem_byte\"");
  EXPECT(throws<ConfigError>([&] { parse_workload_config(bad2); }));
  EXPECT(throws<ConfigError>([] { parse_workload_config("{not json"); }));
  // preset expansion (config.cpp:151-191)
  const char* preset = R"({"schema_version": 1,
    "cluster": {"devices": [{"id": "g", "mem_bytes": 16e9}], "host_dram_bytes": 1e12,
                "h2d": {"bandwidth_Bps": 16e9}},
    "models": [{"preset": "gpt2-gridsearch"}], "jobs": [{"preset": "gpt2-gridsearch"}]})";
  const WorkloadConfig pc = parse_workload_config(preset);
  EXPECT(pc.models.size() == 2 && pc.jobs.size() == 12);
  EXPECT(materialize_jobs(pc)[0].model.layers.size() == 50);
}

int main() {
  model_tests();
  partitioner_tests();
  engine_tests();
  scheduler_tests();
  config_tests();
  std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
