// Device-level C-ABI (SURVEY §8b "C-ABI exports (minimum)"): a device context with a capped,
// budget-enforced HBM arena and three lanes (DOWN = H2D, UP = D2H, COMPUTE), pinned host
// buffers, asynchronous copies, events, and one shard task's forward / recompute+backward on
// the sm_100a kernels — the pieces a host that drives its own engine loop (the reference's
// Engine::dispatch / try_compute / on_compute_done, sim.cpp:347-474) needs. The executor
// (hy_execute_json / hy_executor_*) is the packaged engine built from the same pieces.
#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <string>

#include "../exec/gpt_runner.hpp"
#include "capi_internal.hpp"
#include "hydra.h"

struct hy_dev {
  int device = 0;
  size_t budget = 0, used = 0, peak = 0;
  char* arena = nullptr;
  cudaStream_t lane[3] = {nullptr, nullptr, nullptr};
};

namespace {

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return HY_OK;
  return hy::set_error(HY_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool lane_ok(int lane) { return lane >= HY_LANE_DOWN && lane <= HY_LANE_COMPUTE; }

// Parameter gradients of a backward task go into the caller's shard-layout buffer.
struct BufferSink : hy::GradSink {
  float* grads;
  long base;
  const hy_dims& m;
  BufferSink(float* g, long b, const hy_dims& dims) : grads(g), base(b), m(dims) {}
  float* acquire(int layer) override { return grads + (hy_layer_offset(&m, layer) - base); }
  void release(int) override {}
};

}  // namespace

extern "C" {

int hy_open(int device, size_t hbm_budget, hy_dev** out) {
  if (!out || hbm_budget == 0) return hy::set_error(HY_E_INVALID, "hy_open: null handle or zero budget");
  auto* d = new (std::nothrow) hy_dev;
  if (!d) return hy::set_error(HY_E_INTERNAL, "hy_open: out of host memory");
  d->device = device;
  d->budget = hbm_budget;
  int rc = cuda_status(cudaSetDevice(device), "hy_open set device");
  if (rc == HY_OK) rc = cuda_status(cudaMalloc(&d->arena, hbm_budget), "hy_open arena");
  for (int i = 0; i < 3 && rc == HY_OK; ++i) {
    rc = cuda_status(cudaStreamCreateWithFlags(&d->lane[i], cudaStreamNonBlocking), "hy_open lane");
  }
  if (rc != HY_OK) {
    hy_close(d);
    return rc;
  }
  *out = d;
  return HY_OK;
}

void hy_close(hy_dev* d) {
  if (!d) return;
  cudaSetDevice(d->device);
  for (cudaStream_t s : d->lane) {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
  if (d->arena) cudaFree(d->arena);
  delete d;
}

int hy_lane_stream(hy_dev* d, int lane, void** stream) {
  if (!d || !stream || !lane_ok(lane)) return hy::set_error(HY_E_INVALID, "hy_lane_stream: bad handle or lane");
  *stream = d->lane[lane];
  return HY_OK;
}

int hy_arena_alloc(hy_dev* d, size_t bytes, void** ptr) {
  if (!d || !ptr) return hy::set_error(HY_E_INVALID, "hy_arena_alloc: null argument");
  const size_t off = (d->used + 1023) / 1024 * 1024;
  if (off + bytes > d->budget) {
    return hy::set_error(HY_E_CAPACITY, "hy_arena_alloc: " + std::to_string(bytes) + " B exceeds the HBM budget (" +
                                            std::to_string(d->budget - off) + " B left)");
  }
  *ptr = d->arena + off;
  d->used = off + bytes;
  if (d->used > d->peak) d->peak = d->used;
  return HY_OK;
}

int hy_arena_reset(hy_dev* d) {
  if (!d) return hy::set_error(HY_E_INVALID, "hy_arena_reset: null handle");
  d->used = 0;
  return HY_OK;
}

int hy_arena_peak(hy_dev* d, size_t* bytes) {
  if (!d || !bytes) return hy::set_error(HY_E_INVALID, "hy_arena_peak: null argument");
  *bytes = d->peak;
  return HY_OK;
}

int hy_pinned_alloc(size_t bytes, void** ptr) {
  if (!ptr) return hy::set_error(HY_E_INVALID, "hy_pinned_alloc: null argument");
  return cuda_status(cudaHostAlloc(ptr, bytes ? bytes : 4, cudaHostAllocPortable | cudaHostAllocMapped),
                     "hy_pinned_alloc");
}

int hy_pinned_free(void* ptr) { return ptr ? cuda_status(cudaFreeHost(ptr), "hy_pinned_free") : HY_OK; }

int hy_copy_h2d(hy_dev* d, void* dst, const void* src, size_t bytes) {
  if (!d) return hy::set_error(HY_E_INVALID, "hy_copy_h2d: null handle");
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, d->lane[HY_LANE_DOWN]), "hy_copy_h2d");
}

int hy_copy_d2h(hy_dev* d, void* dst, const void* src, size_t bytes) {
  if (!d) return hy::set_error(HY_E_INVALID, "hy_copy_d2h: null handle");
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, d->lane[HY_LANE_UP]), "hy_copy_d2h");
}

int hy_copy_p2p(hy_dev* d, void* dst, int src_device, const void* src, size_t bytes) {
  if (!d) return hy::set_error(HY_E_INVALID, "hy_copy_p2p: null handle");
  return cuda_status(cudaMemcpyPeerAsync(dst, d->device, src, src_device, bytes, d->lane[HY_LANE_DOWN]),
                     "hy_copy_p2p");
}

int hy_event_record(hy_dev* d, int lane, void** event) {
  if (!d || !event || !lane_ok(lane)) return hy::set_error(HY_E_INVALID, "hy_event_record: bad handle or lane");
  cudaEvent_t e = nullptr;
  int rc = cuda_status(cudaEventCreate(&e), "hy_event_record create");
  if (rc == HY_OK) rc = cuda_status(cudaEventRecord(e, d->lane[lane]), "hy_event_record");
  *event = e;
  return rc;
}

int hy_lane_wait(hy_dev* d, int lane, void* event) {
  if (!d || !event || !lane_ok(lane)) return hy::set_error(HY_E_INVALID, "hy_lane_wait: bad handle or lane");
  return cuda_status(cudaStreamWaitEvent(d->lane[lane], static_cast<cudaEvent_t>(event), 0), "hy_lane_wait");
}

int hy_event_query(void* event, int* done) {
  if (!event || !done) return hy::set_error(HY_E_INVALID, "hy_event_query: null argument");
  const cudaError_t e = cudaEventQuery(static_cast<cudaEvent_t>(event));
  if (e == cudaErrorNotReady) {
    *done = 0;
    return HY_OK;
  }
  *done = 1;
  return cuda_status(e, "hy_event_query");
}

int hy_event_elapsed(void* start, void* end, float* ms) {
  if (!start || !end || !ms) return hy::set_error(HY_E_INVALID, "hy_event_elapsed: null argument");
  return cuda_status(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(end)),
                     "hy_event_elapsed");
}

int hy_event_destroy(void* event) {
  return event ? cuda_status(cudaEventDestroy(static_cast<cudaEvent_t>(event)), "hy_event_destroy") : HY_OK;
}

int hy_lane_sync(hy_dev* d, int lane) {
  if (!d || !lane_ok(lane)) return hy::set_error(HY_E_INVALID, "hy_lane_sync: bad handle or lane");
  return cuda_status(cudaStreamSynchronize(d->lane[lane]), "hy_lane_sync");
}

int hy_shard_scratch_bytes(const hy_dims* m, int max_blocks, size_t* bytes) {
  if (!m || !bytes || max_blocks < 0) return hy::set_error(HY_E_INVALID, "hy_shard_scratch_bytes: bad argument");
  *bytes = sizeof(float) * static_cast<size_t>(hy::scratch_floats(*m, max_blocks)) + 4096;
  return HY_OK;
}

static int shard_task(hy_dev* d, const hy_shard_desc* desc, const hy_shard_bufs* b, double* loss, bool backward) {
  if (!d || !desc || !b || !b->params || !b->scratch) return hy::set_error(HY_E_INVALID, "hy_shard_*: null argument");
  const hy_dims& m = desc->dims;
  if (desc->l0 < 0 || desc->l1 <= desc->l0 || desc->l1 > m.L + 2) {
    return hy::set_error(HY_E_INVALID, "hy_shard_*: layer range outside the model");
  }
  try {
    const hy::ShardGeom g = hy::shard_geom(m, desc->l0, desc->l1);
    size_t need = 0;
    hy_shard_scratch_bytes(&m, g.n_blocks, &need);
    if (b->scratch_bytes < need) {
      return hy::set_error(HY_E_INVALID, "hy_shard_*: scratch smaller than hy_shard_scratch_bytes");
    }
    if (g.has_head && !g.has_embed && !b->wte) {
      return hy::set_error(HY_E_INVALID, "hy_shard_*: a head shard without the embedding needs the tied wte");
    }
    if (backward && !b->grads) return hy::set_error(HY_E_INVALID, "hy_shard_backward: null grads");
    cudaSetDevice(d->device);
    const uintptr_t a = (reinterpret_cast<uintptr_t>(b->scratch) + 1023) & ~uintptr_t(1023);
    hy::Scratch s;
    hy::carve_scratch(m, g.n_blocks, reinterpret_cast<float*>(a), &s);
    hy::TaskIO io;
    io.tokens = b->tokens;
    io.targets = b->targets;
    io.act_in = b->act_in;
    io.act_out = b->act_out;
    io.grad_in = b->grad_in;
    io.grad_out = b->grad_out;
    io.z_in = b->z_in;
    io.wte = b->wte;
    cudaStream_t st = d->lane[HY_LANE_COMPUTE];
    if (backward) {
      BufferSink sink(b->grads, hy_layer_offset(&m, desc->l0), m);
      if (g.has_head && !g.has_embed) io.z_out = b->z_out;  // saved right after the head pass
      hy::run_backward(st, m, g, b->params, sink, io, s);
    } else {
      hy::run_forward(st, m, g, b->params, io, s);
    }
    if (loss && g.has_head) {
      hy::check_cuda(cudaMemcpyAsync(loss, s.loss, sizeof(double), cudaMemcpyDeviceToHost, st), "loss d2h");
      hy::check_cuda(cudaStreamSynchronize(st), "loss sync");
      *loss /= static_cast<double>(m.B) * m.T;
    }
    return cuda_status(cudaGetLastError(), backward ? "hy_shard_backward" : "hy_shard_forward");
  } catch (...) {
    return hy::status_from_current_exception();
  }
}

int hy_shard_forward(hy_dev* d, const hy_shard_desc* desc, const hy_shard_bufs* bufs, double* loss) {
  return shard_task(d, desc, bufs, loss, false);
}

int hy_shard_backward(hy_dev* d, const hy_shard_desc* desc, const hy_shard_bufs* bufs, double* loss) {
  return shard_task(d, desc, bufs, loss, true);
}

}  // extern "C"
