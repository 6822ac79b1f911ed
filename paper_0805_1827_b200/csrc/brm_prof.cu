// brm_prof.cu -- launch accounting and CUDA-event kernel timing for bench.py.
//
// Every kernel launch of the library goes through prof_begin / prof_end.
// Launches are always counted; when profiling is enabled each launch is
// bracketed by a pair of CUDA events recorded on the stream it is launched
// on, and brm_profile_read() folds the elapsed times per kernel family.
// Walker kernels also count the path-steps they execute into a per-device
// counter (one atomic per warp), the unit of the roofline.
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "../../include/bermuda_b200.h"
#include "brm_internal.h"

namespace brm {
namespace {
struct Rec {
  int kind, device;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_pending;
double g_ms[kProfKinds] = {};
uint64_t g_launches[kProfKinds] = {};
unsigned long long *g_counter[64] = {};  // per device: [kProfKinds] executed path-steps
uint64_t g_h2d = 0, g_d2h = 0;
}  // namespace

void count_transfer(size_t h2d, size_t d2h) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_h2d += h2d;
  g_d2h += d2h;
}

unsigned long long *step_counter(int kind) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_counter[dev]) {
    if (cudaMalloc(&g_counter[dev], sizeof(unsigned long long) * kProfKinds) != cudaSuccess) {
      cudaGetLastError();
      g_counter[dev] = nullptr;
      return nullptr;
    }
    cudaMemset(g_counter[dev], 0, sizeof(unsigned long long) * kProfKinds);
  }
  return g_counter[dev] + kind;
}

int prof_begin(int kind, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches[kind] += 1;
  if (!g_on) return -1;
  Rec r{kind, 0, nullptr, nullptr};
  cudaGetDevice(&r.device);
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s);
  g_pending.push_back(r);
  return (int)g_pending.size() - 1;
}

void prof_end(int token, cudaStream_t s) {
  if (token < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (token < (int)g_pending.size()) cudaEventRecord(g_pending[token].b, s);
}

}  // namespace brm

using namespace brm;

extern "C" int brm_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on != 0;
  return BRM_OK;
}

extern "C" int brm_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto &r : g_pending) {
    cudaEventSynchronize(r.b);
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_pending.clear();
  for (int k = 0; k < kProfKinds; ++k) g_ms[k] = 0.0, g_launches[k] = 0;
  g_h2d = g_d2h = 0;
  for (int d = 0; d < 64; ++d)
    if (g_counter[d]) {
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(d);
      cudaMemset(g_counter[d], 0, sizeof(unsigned long long) * kProfKinds);
      cudaSetDevice(prev);
    }
  return BRM_OK;
}

// Totals per kernel family since the last reset: device milliseconds (events,
// profiling enabled), launches, executed path-steps (summed over devices).
extern "C" int brm_profile_read(int32_t kind, double *ms, uint64_t *launches, uint64_t *path_steps) {
  if (kind < 0 || kind >= kProfKinds) return set_error(BRM_EINVAL, "unknown kernel family %d", kind);
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto &r : g_pending) {
    float t = 0.f;
    cudaEventSynchronize(r.b);
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) g_ms[r.kind] += t;
    cudaGetLastError();
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_pending.clear();
  if (ms) *ms = g_ms[kind];
  if (launches) *launches = g_launches[kind];
  if (path_steps) {
    uint64_t total = 0;
    for (int d = 0; d < 64; ++d)
      if (g_counter[d]) {
        unsigned long long v[kProfKinds];
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(d);
        cudaMemcpy(v, g_counter[d], sizeof v, cudaMemcpyDeviceToHost);
        cudaSetDevice(prev);
        total += v[kind];
      }
    *path_steps = total;
  }
  return BRM_OK;
}

// Host<->device bytes the library staged since the last reset.
extern "C" int brm_transfer_read(uint64_t *h2d, uint64_t *d2h) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (h2d) *h2d = g_h2d;
  if (d2h) *d2h = g_d2h;
  return BRM_OK;
}
