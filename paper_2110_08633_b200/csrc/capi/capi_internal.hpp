// Internal glue between the C-ABI and the C++ layers.
#pragma once

#include <cstddef>
#include <string>

namespace hy {

int set_error(int code, const std::string& msg);
int status_from_current_exception();

// JSON request -> JSON result; throw spillsim exceptions on failure.
std::string plan_json(const std::string& request);
std::string execute_json(const std::string& request);
void* session_create(const std::string& request);
std::string session_run(void* handle, int passes, int timed, bool with_trace);
void session_dump_params(void* handle, const std::string& dir);
size_t session_read_params(void* handle, int job, float* dst, size_t n);
void session_destroy(void* handle);

}  // namespace hy
