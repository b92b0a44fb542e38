// Issue-to-completion rate of single tcgen05.mma instructions (bf16, fp32 accumulate)
// by shape and operand source: one thread per CTA issues a chain of MMAs into TMEM,
// clocks per instruction = elapsed / count. Operand contents are irrelevant.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2104_05343_b200/csrc/sg_ptx.cuh"
using namespace sg;

template <int N, bool TS, int LDW, bool AMN = false, bool BMN = false, int STW = 0>
__global__ void __launch_bounds__(384, 1) k(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ int stop_flag;
  if (threadIdx.x == 0) stop_flag = 0;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    constexpr uint32_t IDESC = umma_idesc_bf16(128, N, AMN, BMN);
    const uint32_t a = smem_u32(smem), b = a + 32768;
    const uint64_t ad = AMN ? umma_desc_sw128(a, 16384, 1024) : umma_desc_sw128(a, 0, 1024);
    const uint64_t bd = BMN ? umma_desc_sw128(b, 16384, 1024) : umma_desc_sw128(b, 0, 1024);
    // warm
    for (int i = 0; i < 8; ++i) {
      if (TS) umma_bf16_ts(tmem, tmem + 256, bd, IDESC, 1u);
      else umma_bf16(tmem, ad, bd, IDESC, 1u);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS) umma_bf16_ts(tmem, tmem + 256, bd, IDESC, 1u);
      else umma_bf16(tmem, ad, bd, IDESC, 1u);
    }
    const unsigned long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 1);
    const unsigned long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    *reinterpret_cast<volatile uint32_t*>(&slot + 0) = tmem;  // (no-op)
    stop_flag = 1;
  } else if (STW > 0 && warp >= 4 && warp < 4 + STW) {
    // shared-memory store traffic from other warps (16-byte stores into a separate 64 KB region)
    uint8_t* reg = smem + 65536 + (warp - 4) * 8192;
    uint32_t x = threadIdx.x;
    while (!*reinterpret_cast<volatile int*>(&stop_flag)) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        *reinterpret_cast<uint4*>(reg + (threadIdx.x & 31) * 128 + ((k ^ (threadIdx.x & 7)) << 4)) = make_uint4(x, x + 1, x + 2, k);
        x += 3;
      }
    }
  } else if (warp >= 4 && warp < 4 + LDW) {
    // TMEM load traffic from other warps (columns 384.., lane quadrant warp % 4)
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 384 + ((warp >> 2) & 1) * 64;
    float acc = 0.f;
    while (!*reinterpret_cast<volatile int*>(&stop_flag)) {
      uint32_t r[32];
      tmem_ld32(base, r);
      tmem_wait_ld();
      acc += __uint_as_float(r[threadIdx.x & 31]);
    }
    if (acc == 1.2345f) out[2] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool TS, int LDW = 0, bool AMN = false, bool BMN = false, int STW = 0>
void run(unsigned long long* d, int grid) {
  const int iters = 4096;
  cudaFuncSetAttribute(k<N, TS, LDW, AMN, BMN, STW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  k<N, TS, LDW, AMN, BMN, STW><<<grid, 384, 140000>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("amn %d bmn %d stw %d ldtm warps %d %s M=128 N=%3d K=16 grid %3d: issue %.1f clk/instr, complete %.1f clk/instr (ideal %d) %s\n",
         AMN, BMN, STW, LDW, TS ? "TS" : "SS", N, grid, (double)h[0] / iters, (double)h[1] / iters, 128 * N / 256, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  for (int grid : {148}) {
    run<64, false>(d, grid);
    run<128, false>(d, grid);
    run<64, true>(d, grid);
    run<128, true>(d, grid);
    run<64, false, 8>(d, grid);
    run<128, false, 8>(d, grid);
    run<64, true, 8>(d, grid);
    run<128, true, 8>(d, grid);
    run<64, false, 0, true, true>(d, grid);
    run<64, false, 0, false, true>(d, grid);
    run<128, false, 0, true, true>(d, grid);
    run<128, false, 0, false, true>(d, grid);
    run<64, true, 0, false, true>(d, grid);
    run<64, false, 0, false, false, 8>(d, grid);
    run<128, false, 0, false, false, 8>(d, grid);
    run<64, false, 0, true, true, 8>(d, grid);
    run<64, true, 0, false, true, 8>(d, grid);
    run<128, false, 0, false, false, 4>(d, grid);
  }
  return 0;
}
