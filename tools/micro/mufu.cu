// Throughput of MUFU.EX2, F2FP bf16 packing and an FMA-pipe exp2 polynomial on one B200.
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
// 2^x on the FMA pipe: split into integer and fraction, degree-3 minimax on [0,1)
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float fi = floorf(x);
  const float f = x - fi;
  float p = fmaf(f, 0.0555041086648216f, 0.2402264923172690f);
  p = fmaf(p, f, 0.6931471805599453f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (static_cast<int>(fi) << 23));
}

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i * 0.01f;
  uint32_t pk = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;
      if (MODE == 1) a[i] = ex2_poly(a[i]) - 1.0f;
      if (MODE == 2) { __nv_bfloat162 h = __floats2bfloat162_rn(a[i], a[(i + 1) & 15]); pk ^= *reinterpret_cast<uint32_t*>(&h); a[i] += 1e-7f; }
    }
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + pk;
}

int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  const char* names[3] = {"MUFU.EX2", "poly exp2 (FMA)", "F2FP bf16x2 pack"};
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<sms * 4, 256>>>(out, iters);
      if (mode == 1) k<1><<<sms * 4, 256>>>(out, iters);
      if (mode == 2) k<2><<<sms * 4, 256>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 4 * 256 * iters * 16;
    printf("%-20s %8.2f Gop/s = %6.2f /clk/SM (at %d MHz nominal)\n", names[mode], ops / ms / 1e6,
           ops / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
  }
  return 0;
}
