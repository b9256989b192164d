#include "capi_internal.hpp"
#include "spillsim/errors.hpp"
namespace hy {
std::string execute_json(const std::string&) { throw spillsim::InvalidArgument("executor not built yet"); }
}  // namespace hy
