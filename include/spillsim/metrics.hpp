// Run report (reference: proj/core/include/spillsim/metrics.hpp:27-99). The same
// summarize() consumes virtual traces and the executor's measured traces.
#pragma once

#include <string>
#include <vector>

#include "spillsim/model.hpp"
#include "spillsim/sim.hpp"
#include "spillsim/strategies.hpp"

namespace spillsim {

struct DeviceUsage {
  std::string device_id;
  double busy_s = 0;
  double idle_s = 0;
  double utilization = 0;
  double energy_j = 0;
};

struct ChannelUsage {
  std::string name;
  double busy_s = 0;
};

struct RunReport {
  std::string strategy;
  double makespan_s = 0;
  std::vector<DeviceUsage> devices;
  std::vector<ChannelUsage> channels;
  double energy_j = 0;
  double cost = 0;
  Feasibility feasibility;
};

RunReport summarize(const SimTrace& trace, const ClusterSpec& cluster, const std::string& strategy_name);
RunReport infeasible_report(const Feasibility& f);

std::string report_to_json(const RunReport& report);
std::string report_to_csv(const RunReport& report);
std::string report_to_text(const RunReport& report);

// (The reference's compare() / ComparisonTable build its paper tables and are out of scope
// here.)

}  // namespace spillsim
