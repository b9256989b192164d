#include "host_opt.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>

namespace hy {
namespace {

inline float bf16_to_f(uint16_t b) {
  const uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
inline uint16_t f_to_bf16_rne(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// target_clones: AVX-512 on the B200 hosts (Sapphire/Emerald Rapids), AVX2 elsewhere.
__attribute__((target_clones("avx512f", "avx2", "default"))) void adam_f32(
    long lo, long hi, float* __restrict p, const float* __restrict g, float* __restrict m, float* __restrict v,
    float lr, float b1, float b2, float eps, float wd, float bc1, float bc2) {
  const float c1 = 1.f - b1, c2 = 1.f - b2;
  for (long i = lo; i < hi; ++i) {
    const float gi = g[i];
    const float mi = b1 * m[i] + c1 * gi;
    const float vi = b2 * v[i] + c2 * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float upd = (mi / bc1) / (std::sqrt(vi / bc2) + eps);
    p[i] = p[i] - lr * (upd + wd * p[i]);
  }
}

__attribute__((target_clones("avx512f", "avx2", "default"))) void adam_bf16(
    long lo, long hi, float* __restrict p, const float* __restrict g, uint16_t* __restrict m,
    uint16_t* __restrict v, float lr, float b1, float b2, float eps, float wd, float bc1, float bc2) {
  const float c1 = 1.f - b1, c2 = 1.f - b2;
  for (long i = lo; i < hi; ++i) {
    const float gi = g[i];
    const float mi = b1 * bf16_to_f(m[i]) + c1 * gi;
    const float vi = b2 * bf16_to_f(v[i]) + c2 * gi * gi;
    m[i] = f_to_bf16_rne(mi);
    v[i] = f_to_bf16_rne(vi);
    const float upd = (mi / bc1) / (std::sqrt(vi / bc2) + eps);
    p[i] = p[i] - lr * (upd + wd * p[i]);
  }
}

void CUDART_CB host_adam_cb(void* arg) {
  HostAdamWork* w = static_cast<HostAdamWork*>(arg);
  host_adam(*w);
  delete w;
}

}  // namespace

void host_adam(const HostAdamWork& w) {
  const int nt = w.threads > 0 ? w.threads : 1;
  // contiguous 64-byte-aligned ranges per thread
#pragma omp parallel num_threads(nt)
  {
    const int t = omp_get_thread_num(), T = omp_get_num_threads();
    const long per = ((w.n + T - 1) / T + 15) / 16 * 16;
    const long lo = std::min(w.n, per * t), hi = std::min(w.n, lo + per);
    if (lo < hi) {
      if (w.bf16) {
        adam_bf16(lo, hi, w.p, w.g, static_cast<uint16_t*>(w.m), static_cast<uint16_t*>(w.v), w.lr, w.beta1,
                  w.beta2, w.eps, w.weight_decay, w.bc1, w.bc2);
      } else {
        adam_f32(lo, hi, w.p, w.g, static_cast<float*>(w.m), static_cast<float*>(w.v), w.lr, w.beta1, w.beta2,
                 w.eps, w.weight_decay, w.bc1, w.bc2);
      }
    }
  }
}

cudaError_t host_adam_async(cudaStream_t stream, const HostAdamWork& w) {
  return cudaLaunchHostFunc(stream, host_adam_cb, new HostAdamWork(w));
}

}  // namespace hy
