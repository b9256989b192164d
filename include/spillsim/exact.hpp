// Reduced scheduling instance + classical makespan bounds (reference:
// proj/core/include/spillsim/exact.hpp:27-52, src/exact.cpp:27-54). The branch-and-bound
// optimum (exact_optimal) is out of scope for the B200 build; the
// bounds are kept because C5 reports makespan against the LRTF lower bound.
#pragma once

#include <string>
#include <utility>
#include <vector>

namespace spillsim {

struct TaskInstance {
  struct Task {
    std::string id;
    double duration_s = 0;
    int pred = -1;
  };
  std::vector<Task> tasks;
  int devices = 1;
};

void validate(const TaskInstance& instance);

/// (sum of durations / devices, longest chain).
std::pair<double, double> lower_bounds(const TaskInstance& instance);

}  // namespace spillsim
