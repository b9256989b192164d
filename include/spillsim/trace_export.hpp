// Chrome trace-event export (reference: proj/core/include/spillsim/trace_export.hpp:28).
#pragma once

#include <string>

#include "spillsim/sim.hpp"

namespace spillsim {

std::string to_chrome_trace_json(const SimTrace& trace);

}  // namespace spillsim
