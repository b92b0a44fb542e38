// TMEM -> register load bandwidth per SM (tcgen05.ld.32x32b.x32), 4 or 8 warps.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2104_05343_b200/csrc/sg_ptx.cuh"
using namespace sg;

template <int WARPS, int BATCH>
__global__ void __launch_bounds__(32 * WARPS, 1) k(float* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    uint32_t r[BATCH][32];
#pragma unroll
    for (int b = 0; b < BATCH; ++b) tmem_ld32(base + ((b * 32 + it * 32) & 127), r[b]);
    tmem_wait_ld();
#pragma unroll
    for (int b = 0; b < BATCH; ++b)
#pragma unroll
      for (int e = 0; e < 32; ++e) acc += __uint_as_float(r[b][e]);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

template <int W, int B>
void run(float* out, int sms, int clk) {
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<W, B><<<sms, 32 * W>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)sms * W * iters * B * 4096.0;
  printf("warps %d batch %d: %.1f TB/s total, %.1f B/clk/SM (nominal %d MHz) err=%s\n", W, B, bytes / ms / 1e9,
         bytes / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 512 * 4);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  run<4, 1>(out, sms, clk);
  run<4, 4>(out, sms, clk);
  run<8, 1>(out, sms, clk);
  run<8, 4>(out, sms, clk);
  return 0;
}
