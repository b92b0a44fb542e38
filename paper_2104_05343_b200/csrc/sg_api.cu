// Library-wide host entry points: error reporting and device queries.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <atomic>
#include <cstdint>

#include "sg.h"
#include "sg_internal.h"

namespace sg {
static thread_local char g_err[512] = {0};
int set_error(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg ? msg : "");
  return code;
}
void clear_error() { g_err[0] = 0; }
}  // namespace sg

extern "C" const char* sg_last_error(void) { return sg::g_err; }

namespace sg {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace sg

extern "C" int64_t sg_launch_count(void) { return sg::g_launches.load(std::memory_order_relaxed); }

extern "C" int sg_device_sm_count(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  // Cached per device ordinal (a process may drive several devices).
  static int cache[64] = {0};
  if (dev < 64 && cache[dev] > 0) return cache[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (dev < 64) cache[dev] = n;
  return n;
}

namespace sg {
static std::atomic<int> g_sm_reserve{0};
}  // namespace sg

// SMs left free by the persistent GEMM grid (dist meshes: room for the NCCL kernels
// that move step l+1's panels while step l's product runs, summa.py).
extern "C" int sg_set_sm_reserve(int n) {
  if (n < 0 || n > 64) return sg::set_error(SG_ERR_CONFIG, "sm reserve must lie in [0, 64]");
  sg::g_sm_reserve.store(n, std::memory_order_relaxed);
  return SG_OK;
}

extern "C" int sg_gemm_sm_budget(void) {
  const int sms = sg_device_sm_count();
  if (sms <= 0) return sms;
  const int left = sms - sg::g_sm_reserve.load(std::memory_order_relaxed);
  return left < 2 ? 2 : (left & ~1);  // CTA pairs need an even grid
}

extern "C" const char* sg_build_info(void) {
  return "libsg sm_100a (tcgen05/TMA) built with nvcc " __DATE__;
}
