// Peer memory for the SPMD ("dist") mesh: symmetric device arenas shared between the
// mesh's processes through CUDA IPC, and a device-side group barrier over them.
//
// The reference's row / column reduces of AB^T / A^T B partial products
// (mesh.py:458-482, called per SUMMA step from summa.py:128-139, 152-163) become
// remote accumulation: every position's GEMM epilogue reduce-adds (TMA
// cp.reduce.async.bulk) its partial tile straight into the destination position's
// accumulator, which lives in an arena mapped into every process of the mesh
// (NVLink peer memory across GPUs; the same HBM for processes sharing one GPU).
// A barrier kernel orders "destination zeroed" -> "partials added" -> "destination
// read"; it is stream-ordered and graph-capturable (device-side epoch counters,
// no host state baked into a captured launch).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "sg.h"
#include "sg_internal.h"
#include "sg_ptx.cuh"

extern "C" int sg_sym_alloc(int64_t bytes, void** ptr, void* handle) {
  using namespace sg;
  clear_error();
  if (bytes <= 0 || !ptr || !handle) return set_error(SG_ERR_CONFIG, "sym_alloc: bad arguments");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);
  if (e != cudaSuccess) return set_error(SG_ERR_CUDA, cudaGetErrorString(e));
  e = cudaMemset(p, 0, (size_t)bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return set_error(SG_ERR_CUDA, cudaGetErrorString(e));
  }
  *ptr = p;
  return SG_OK;
}

extern "C" int sg_sym_free(void* ptr) {
  using namespace sg;
  clear_error();
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int sg_ipc_open(const void* handle, void** ptr) {
  using namespace sg;
  clear_error();
  if (!handle || !ptr) return set_error(SG_ERR_CONFIG, "ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  // mapped into the calling device's context; across GPUs this enables peer access
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int sg_ipc_close(void* ptr) {
  using namespace sg;
  clear_error();
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}

extern "C" int sg_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

namespace sg {

__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// args = [n pad pointers (int64), n member flats (int64)]; pad_i[flat] is the slot member
// `flat` writes in member i's pad. Thread t signals member t, then waits for member t's
// signal in this position's own pad (pads[me_idx]).
__global__ void peer_barrier_kernel(const long long* __restrict__ args, int n, int me_idx, int* epoch, int* err,
                                    long long timeout_cycles) {
  pdl_begin();
  __shared__ int e_sh;
  if (threadIdx.x == 0) {
    const int e = *epoch + 1;
    *epoch = e;
    e_sh = e;
  }
  __syncthreads();
  const int e = e_sh;
  const int t = threadIdx.x;
  const int my_flat = (int)args[n + me_idx];
  if (t < n) {
    // everything this position wrote before the barrier (earlier kernels, including the
    // remote reduce-adds of its GEMM epilogues) is ordered before the signal
    __threadfence_system();
    int* pad_t = reinterpret_cast<int*>(args[t]);
    st_release_sys(pad_t + my_flat, e);
  }
  if (t < n) {
    const int* mine = reinterpret_cast<const int*>(args[me_idx]) + (int)args[n + t];
    const long long t0 = clock64();
    while (ld_acquire_sys(mine) < e) {
      if (clock64() - t0 > timeout_cycles) {
        atomicOr(err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

}  // namespace sg

extern "C" int sg_peer_barrier(const int64_t* args, int n, int me_idx, int* epoch, int* err, int64_t timeout_cycles,
                               void* stream) {
  using namespace sg;
  clear_error();
  if (n < 1 || n > 32 || me_idx < 0 || me_idx >= n || !args || !epoch || !err)
    return set_error(SG_ERR_CONFIG, "peer_barrier: 1..32 members");
  launch_k(peer_barrier_kernel, dim3(1), dim3(32), 0, static_cast<cudaStream_t>(stream),
           reinterpret_cast<const long long*>(args), n, me_idx, epoch, err, (long long)timeout_cycles);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}

// ---- data movement over peer memory --------------------------------------------------
extern "C" int sg_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  using namespace sg;
  clear_error();
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return set_error(SG_ERR_CONFIG, "copy_async: bad arguments");
  if (bytes == 0) return SG_OK;
  // unified addressing: a peer-mapped source or destination is copied by the copy
  // engines over NVLink (the same HBM for processes sharing a GPU)
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}

namespace sg {
// dst[i] (op)= fold over members m = 0..n-1, in member order, of srcs[m][i] (fp32): the
// group-ordered reduce of the reference (mesh.py:464-466), read straight from the
// members' published buffers
__global__ void peer_fold_kernel(float* __restrict__ dst, const long long* __restrict__ srcs, int n, long long count,
                                 int accumulate, int op_max) {
  pdl_begin();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    float acc = accumulate ? dst[i] : reinterpret_cast<const float*>(srcs[0])[i];
    for (int m = accumulate ? 0 : 1; m < n; ++m) {
      const float v = reinterpret_cast<const float*>(srcs[m])[i];
      acc = op_max ? fmaxf(acc, v) : acc + v;
    }
    dst[i] = acc;
  }
}
}  // namespace sg

extern "C" int sg_peer_fold(float* dst, const int64_t* srcs, int n, int64_t count, int accumulate, int op_max,
                            void* stream) {
  using namespace sg;
  clear_error();
  if (n < 1 || n > 64 || count < 0 || !dst || !srcs) return set_error(SG_ERR_CONFIG, "peer_fold: bad arguments");
  if (count == 0) return SG_OK;
  const long long blocks = std::min<long long>((count + 255) / 256, 148LL * 8);
  launch_k(peer_fold_kernel, dim3((unsigned)blocks), dim3(256), 0, static_cast<cudaStream_t>(stream), dst,
           reinterpret_cast<const long long*>(srcs), n, (long long)count, accumulate, op_max);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}
