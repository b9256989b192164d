// Small helpers shared by the planning and execution entry points.
#pragma once

#include <string>
#include <vector>

#include "nlohmann/json.hpp"
#include "spillsim/errors.hpp"
#include "spillsim/model.hpp"
#include "spillsim/partitioner.hpp"
#include "spillsim/strategies.hpp"

namespace hy {

// Replace the cluster's device list with `n` copies of device 0 named gpu0..gpu{n-1}.
inline void replicate_devices(spillsim::ClusterSpec& c, int n) {
  spillsim::DeviceSpec proto = c.devices.front();
  c.devices.clear();
  for (int d = 0; d < n; ++d) {
    spillsim::DeviceSpec dev = proto;
    dev.device_id = "gpu" + std::to_string(d);
    c.devices.push_back(dev);
  }
}

// Request field "shard_boundaries": one entry per job — a list of shard starts, the
// boundary text of boundaries_to_text (partitioner.cpp:206-231), or null (greedy cut).
inline spillsim::PinnedBoundaries pinned_boundaries(const nlohmann::json& req, size_t n_jobs) {
  spillsim::PinnedBoundaries out;
  if (!req.contains("shard_boundaries") || req["shard_boundaries"].is_null()) return out;
  const nlohmann::json& b = req["shard_boundaries"];
  if (!b.is_array() || b.size() > n_jobs) throw spillsim::InvalidArgument("shard_boundaries: a list with at most one entry per job");
  for (const nlohmann::json& e : b) {
    if (e.is_null()) out.emplace_back();
    else if (e.is_string()) out.push_back(spillsim::boundaries_from_text(e.get<std::string>()));
    else if (e.is_array()) out.push_back(e.get<std::vector<int>>());
    else throw spillsim::InvalidArgument("shard_boundaries entries are lists of starts, boundary text or null");
  }
  return out;
}

}  // namespace hy
