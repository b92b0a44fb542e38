// Do MUFU.EX2 and F2FP (bf16x2 pack) share a pipe? Rate of exp2 + bf16 packing
// variants per SM, one warp per SMSP (as the flash softmax runs) and 8 warps per SMSP.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack_cvt(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_prmt(float a, float b) {  // truncation
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
  return r;
}
__device__ __forceinline__ uint32_t pack_rnd(float a, float b) {  // round half up, then truncate
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(a) + 0x8000u), "r"(__float_as_uint(b) + 0x8000u));
  return r;
}

template <int MODE>
__global__ void k(uint32_t* out, int iters, float s) {
  float a[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) a[i] = -(threadIdx.x * 1e-3f + i * 0.01f);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const float p0 = ex2(a[i]), p1 = ex2(a[i + 1]);
      if (MODE == 1) acc ^= pack_cvt(p0, p1);
      if (MODE == 2) acc ^= pack_prmt(p0, p1);
      if (MODE == 3) acc ^= pack_rnd(p0, p1);
      if (MODE == 0) acc ^= __float_as_uint(p0) ^ __float_as_uint(p1);
      a[i] = fmaf(p0, s, a[i]);
      a[i + 1] = fmaf(p1, s, a[i + 1]);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 2048;
  const char* names[4] = {"ex2 only", "ex2 + cvt.bf16x2", "ex2 + prmt trunc", "ex2 + iadd+prmt rnd"};
  for (int warps : {4, 32}) {
    for (int mode = 0; mode < 4; ++mode) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<sms, 32 * warps>>>(out, iters, 1e-9f);
        if (mode == 1) k<1><<<sms, 32 * warps>>>(out, iters, 1e-9f);
        if (mode == 2) k<2><<<sms, 32 * warps>>>(out, iters, 1e-9f);
        if (mode == 3) k<3><<<sms, 32 * warps>>>(out, iters, 1e-9f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      double ex = (double)sms * 32 * warps * iters * 32;
      printf("warps/SM %2d %-22s %6.2f ex2/clk/SM (nominal %d MHz)\n", warps, names[mode],
             ex / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
    }
  }
  return 0;
}
