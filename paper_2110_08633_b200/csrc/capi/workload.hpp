// Small helpers shared by the planning and execution entry points.
#pragma once

#include <string>

#include "spillsim/model.hpp"

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

}  // namespace hy
