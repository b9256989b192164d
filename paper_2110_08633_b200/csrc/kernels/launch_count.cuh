// Process-wide count of kernel launches issued by this library (reported as gpu_launches).
#pragma once

#include <atomic>

namespace hy {
inline std::atomic<long> g_kernel_launches{0};
inline void count_launch() { g_kernel_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace hy
