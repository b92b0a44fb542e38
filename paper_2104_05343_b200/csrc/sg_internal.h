// Shared host-side helpers of libsg (error slot, device queries).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

namespace sg {
// cudaFuncSetAttribute(max dynamic smem) once per (kernel, device): a process may drive
// several devices, and the attribute is per device.
inline bool ensure_smem(const void* kern, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_pair(kern, dev);
  if (done.count(key)) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  done.insert(key);
  return true;
}

int set_error(int code, const char* msg);
void clear_error();
void count_launch();  // every kernel this library launches (bench gpu_launches)
}  // namespace sg

extern "C" int sg_device_sm_count(void);
extern "C" int sg_gemm_sm_budget(void);


namespace sg {
// Programmatic dependent launch (opt-in, SG_PDL=1): every libsg kernel triggers its
// dependents at entry and waits for its predecessor (griddepcontrol) before
// touching memory, so with the launch attribute set a kernel's launch and prologue
// overlap the tail of the previous one (also inside CUDA graphs). Measured on the
// BERT step it costs ~1.3% (679 vs 688 samples/s: early-resident CTAs of the next
// kernel only spin), so plain launches are the default; the device-side
// griddepcontrol instructions are no-ops then.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SG_PDL");
    return e && atoi(e) != 0;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace sg

// Phase-timeline stamps for the instrumented build only (tools/trace_build.py
// compiles with -DSG_TRACE into libsg_trace.so; the product library has none):
// SG_TR(cond, buffer, index, event) appends (event << 56 | clock64) to a per-TU
// device buffer read back by sg_debug_trace (tools/ftrace.py).
#ifdef SG_TRACE
namespace sg {
static __device__ unsigned long long g_sgtrace[4][8192];
__device__ __forceinline__ void sg_trace_stamp(int buf, int& i, int ev) {
  if (i < 8192) g_sgtrace[buf][i++] = ((unsigned long long)ev << 56) | (clock64() & 0xffffffffffffffull);
}
}  // namespace sg
#define SG_TR(cond, buf, idx, ev) \
  do {                            \
    if (cond) sg::sg_trace_stamp(buf, idx, ev); \
  } while (0)
#else
#define SG_TR(cond, buf, idx, ev) \
  do {                            \
  } while (0)
#endif
