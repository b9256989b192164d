// Probe (diagnostics, not product): host-side fused AdamW throughput on the box's cores, alone
// and while the GPU's copy engines stream H2D + D2H over pinned memory (the DRAM they share).
// Decides how much of the optimizer the executor can place host-side (the reference's
// placement) without the host becoming the bottleneck.
//   nvcc -O3 -Xcompiler -fopenmp,-march=x86-64-v4,-fno-math-errno tools/host_adam_probe.cu -o /tmp/hap -lgomp
#include <cuda_runtime.h>
#include <omp.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>

static void adam(long n, float* __restrict p, const float* __restrict g, float* __restrict m, float* __restrict v) {
  const float b1 = 0.9f, b2 = 0.999f, lr = 1e-4f, eps = 1e-8f, bc1 = 0.1f, bc2 = 0.001f;
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * ((mi / bc1) / (sqrtf(vi / bc2) + eps));
  }
}

static double time_adam(long n, float* p, float* g, float* m, float* v, int reps) {
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    const double t0 = omp_get_wtime();
    adam(n, p, g, m, v);
    best = std::min(best, omp_get_wtime() - t0);
  }
  return best;
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : (1L << 27);
  const size_t cb = 1L << 30;
  float *p, *g;
  cudaHostAlloc(&p, n * 4, cudaHostAllocPortable);
  cudaHostAlloc(&g, n * 4, cudaHostAllocPortable);
  float* m = static_cast<float*>(aligned_alloc(2 << 20, n * 4));
  float* v = static_cast<float*>(aligned_alloc(2 << 20, n * 4));
#pragma omp parallel for
  for (long i = 0; i < n; ++i) {
    p[i] = 0.01f * (i % 97);
    g[i] = 0.001f * (i % 13);
    m[i] = 0;
    v[i] = 0;
  }
  char *hs, *hd, *ds, *dd;
  cudaHostAlloc(&hs, cb, cudaHostAllocPortable);
  cudaHostAlloc(&hd, cb, cudaHostAllocPortable);
  cudaMalloc(&ds, cb);
  cudaMalloc(&dd, cb);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  const int maxt = omp_get_max_threads();
  for (int t : {4, 8, 12, maxt - 2, maxt}) {
    if (t > maxt || t < 1) continue;
    omp_set_num_threads(t);
    adam(n, p, g, m, v);
    const double alone = time_adam(n, p, g, m, v, 3);
    // concurrent duplex DMA
    std::atomic<bool> stop{false};
    std::atomic<long> bytes{0};
    std::thread dma([&] {
      while (!stop.load()) {
        cudaMemcpyAsync(dd, hs, cb, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(hd, ds, cb, cudaMemcpyDeviceToHost, s2);
        cudaStreamSynchronize(s1);
        cudaStreamSynchronize(s2);
        bytes += 2 * cb;
      }
    });
    std::this_thread::sleep_for(std::chrono::milliseconds(200));
    const long b0 = bytes.load();
    const auto w0 = std::chrono::steady_clock::now();
    const double busy = time_adam(n, p, g, m, v, 3);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    const long b1 = bytes.load();
    stop = true;
    dma.join();
    printf("{\"threads\": %d, \"alone_Gupd_s\": %.3f, \"alone_GBps\": %.1f, \"with_dma_Gupd_s\": %.3f, "
           "\"dma_GBps_during\": %.1f}\n",
           t, n / alone / 1e9, 28.0 * n / alone / 1e9, n / busy / 1e9, (b1 - b0) / wall / 1e9);
    fflush(stdout);
  }
  // DMA alone for reference
  const auto w0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 4; ++i) {
    cudaMemcpyAsync(dd, hs, cb, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(hd, ds, cb, cudaMemcpyDeviceToHost, s2);
  }
  cudaDeviceSynchronize();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
  printf("{\"dma_alone_duplex_GBps_total\": %.1f}\n", 8.0 * cb / wall / 1e9);
  return 0;
}
