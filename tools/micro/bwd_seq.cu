// Tensor-core time of the d = 64 flash-backward MMA sequence per query block, issued
// back to back by one thread per CTA (no softmax, no TMA, no drain): S^T, dP^T
// (M=128 N=128 K=64, SS, K-major), dV / dK (M=128 N=64 K=128, TS, B MN-major), dQ
// (M=128 N=64 K=128, SS, A and B MN-major), in the kernel's order and descriptors, and
// variants that isolate one feature. Prints clocks per block (ideal ~1640).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../paper_2104_05343_b200/csrc/sg_ptx.cuh"
using namespace sg;

constexpr uint32_t kT64 = 128 * 64 * 2;

// MODE: 0 full sequence; 1 S/dP only; 2 dV/dK only (TS); 3 dQ only; 4 dV/dK as SS
// (A MN-major from smem, the [queries x keys] orientation); 5 full, fixed K-step
// addresses (no advance); 6 S/dP with the D target alternating but no dependency
template <int MODE, int LDW = 0, int STW = 0, int TMAW = 0, int MUW = 0>
__global__ void __launch_bounds__(512, 1) k(unsigned long long* out, int iters, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ uint64_t cb[8];
  __shared__ int stop_flag;
  if (threadIdx.x == 0) stop_flag = 0;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    for (int j = 0; j < 8; ++j) mbar_init(&cb[j], 1);
    fence_mbar_init();
    if (MODE == 8) mbar_arrive(&cb[7]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    constexpr uint32_t ID_ST = umma_idesc_bf16(128, 128, false, false);
    constexpr uint32_t ID_KV = umma_idesc_bf16(128, 64, false, true);
    constexpr uint32_t ID_KVSS = umma_idesc_bf16(128, 64, true, true);
    constexpr uint32_t ID_DQ = umma_idesc_bf16(128, 64, true, true);
    const uint32_t base = smem_u32(smem);
    const uint32_t k_base = base, v_base = base + kT64, q_base = base + 2 * kT64, do_base = base + 3 * kT64,
                   ds_base = base + 4 * kT64;  // dS: 2 atoms
    const uint32_t t_s = tmem, t_dp = tmem + 128, t_p = tmem + 256, t_dv = tmem + 320, t_dk = tmem + 384,
                   t_dq = tmem + 448;
    const int adv = MODE == 5 ? 0 : 1;
    unsigned long long t0 = 0;
    for (int i = 0; i < iters + 2; ++i) {
      if (i == 2) t0 = clock64();
      if (MODE == 8) {
        // full sequence with the kernel's commits and its wait pattern: before each
        // group a wait on an already completed barrier + tcgen05.fence::after_thread_sync
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(t_s, umma_desc_sw128(k_base + kk * 32, 0, 1024), umma_desc_sw128(q_base + kk * 32, 0, 1024), ID_ST,
                    kk > 0 ? 1u : 0u);
        umma_commit(&cb[0]);
        mbar_wait(&cb[7], 0);
        tc_fence_after();
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          umma_bf16_ts(t_dv, t_p + kq * 8, umma_desc_sw128(do_base + kq * 2048, kT64, 1024), ID_KV, 1u);
        mbar_wait(&cb[7], 0);
        tc_fence_after();
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          umma_bf16_ts(t_dk, t_dp + ((kq >> 2) * 64 + (kq & 3) * 8), umma_desc_sw128(q_base + kq * 2048, kT64, 1024),
                       ID_KV, 1u);
        umma_commit(&cb[2]);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(t_dp, umma_desc_sw128(v_base + kk * 32, 0, 1024), umma_desc_sw128(do_base + kk * 32, 0, 1024),
                    ID_ST, kk > 0 ? 1u : 0u);
        umma_commit(&cb[3]);
        mbar_wait(&cb[7], 0);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(t_dq, umma_desc_sw128(ds_base + kk * 2048, kT64, 1024), umma_desc_sw128(k_base + kk * 2048, kT64, 1024),
                    ID_DQ, kk > 0 ? 1u : 0u);
        umma_commit(&cb[4]);
        mbar_wait(&cb[7], 0);
        tc_fence_after();
      }
      if (MODE == 7) {
        // full sequence with the kernel's commits (barriers never waited on)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(t_s, umma_desc_sw128(k_base + kk * 32, 0, 1024), umma_desc_sw128(q_base + kk * 32, 0, 1024), ID_ST,
                    kk > 0 ? 1u : 0u);
        umma_commit(&cb[0]);
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          umma_bf16_ts(t_dv, t_p + kq * 8, umma_desc_sw128(do_base + kq * 2048, kT64, 1024), ID_KV, 1u);
        umma_commit(&cb[1]);
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          umma_bf16_ts(t_dk, t_dp + ((kq >> 2) * 64 + (kq & 3) * 8), umma_desc_sw128(q_base + kq * 2048, kT64, 1024),
                       ID_KV, 1u);
        umma_commit(&cb[2]);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(t_dp, umma_desc_sw128(v_base + kk * 32, 0, 1024), umma_desc_sw128(do_base + kk * 32, 0, 1024),
                    ID_ST, kk > 0 ? 1u : 0u);
        umma_commit(&cb[3]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(t_dq, umma_desc_sw128(ds_base + kk * 2048, kT64, 1024), umma_desc_sw128(k_base + kk * 2048, kT64, 1024),
                    ID_DQ, kk > 0 ? 1u : 0u);
        umma_commit(&cb[4]);
        umma_commit(&cb[5]);
        if (MODE == 7 && (i & 3) == 3) {
          umma_commit(&cb[6]);
          umma_commit(&cb[7]);
        }
      }
      if (MODE == 0 || MODE == 1 || MODE == 5 || MODE == 6) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(t_s, umma_desc_sw128(k_base + adv * kk * 32, 0, 1024),
                    umma_desc_sw128(q_base + adv * kk * 32, 0, 1024), ID_ST, kk > 0 ? 1u : 0u);
      }
      if (MODE == 0 || MODE == 2 || MODE == 5) {
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          umma_bf16_ts(t_dv, t_p + adv * kq * 8, umma_desc_sw128(do_base + adv * kq * 2048, kT64, 1024), ID_KV, 1u);
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          umma_bf16_ts(t_dk, t_dp + adv * ((kq >> 2) * 64 + (kq & 3) * 8),
                       umma_desc_sw128(q_base + adv * kq * 2048, kT64, 1024), ID_KV, 1u);
      }
      if (MODE == 4) {
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          umma_bf16(t_dv, umma_desc_sw128(ds_base + kq * 2048, kT64, 1024),
                    umma_desc_sw128(do_base + kq * 2048, kT64, 1024), ID_KVSS, 1u);
#pragma unroll
        for (int kq = 0; kq < 8; ++kq)
          umma_bf16(t_dk, umma_desc_sw128(ds_base + kq * 2048, kT64, 1024),
                    umma_desc_sw128(q_base + kq * 2048, kT64, 1024), ID_KVSS, 1u);
      }
      if (MODE == 0 || MODE == 1 || MODE == 5) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(t_dp, umma_desc_sw128(v_base + adv * kk * 32, 0, 1024),
                    umma_desc_sw128(do_base + adv * kk * 32, 0, 1024), ID_ST, kk > 0 ? 1u : 0u);
      }
      if (MODE == 6) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(t_dp, umma_desc_sw128(v_base + kk * 32, 0, 1024), umma_desc_sw128(do_base + kk * 32, 0, 1024),
                    ID_ST, 1u);
      }
      if (MODE == 0 || MODE == 3 || MODE == 5) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16(t_dq, umma_desc_sw128(ds_base + adv * kk * 2048, kT64, 1024),
                    umma_desc_sw128(k_base + adv * kk * 2048, kT64, 1024), ID_DQ, kk > 0 ? 1u : 0u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    *reinterpret_cast<volatile int*>(&stop_flag) = 1;
  } else if (warp >= 4 && warp < 4 + LDW) {
    // softmax-like TMEM reads: S / dP columns (0..255), lane quadrant warp % 4
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + ((warp >> 2) & 1) * 64;
    float acc = 0.f;
    int c = 0;
    while (!*reinterpret_cast<volatile int*>(&stop_flag)) {
      uint32_t r[32];
      tmem_ld32(base + (c & 3) * 32 + ((c >> 2) & 1) * 128, r);
      tmem_wait_ld();
      acc += __uint_as_float(r[threadIdx.x & 31]);
      ++c;
    }
    if (acc == 1.2345f) out[2] = 1;
  } else if (MUW > 0 && warp >= 4 && warp < 4 + MUW) {
    // softmax-like math: independent ex2 + paired FMA streams, no waits
    float a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = -(threadIdx.x * 1e-3f + i * 0.01f);
    uint32_t acc = 0;
    while (!*reinterpret_cast<volatile int*>(&stop_flag)) {
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float p0, p1;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(a[i + 1]));
        __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
        acc ^= *reinterpret_cast<uint32_t*>(&hv);
        a[i] = fmaf(p0, 1e-9f, a[i]);
        a[i + 1] = fmaf(p1, 1e-9f, a[i + 1]);
      }
    }
    if (acc == 12345u) out[3] = acc;
  } else if (TMAW && warp == 3) {
    // bulk global -> smem copies (TMA engine), 16 KB at a time, back to back
    __shared__ uint64_t tb;
    if (threadIdx.x == 96) {
      mbar_init(&tb, 1);
      fence_mbar_init();
      uint32_t ph = 0;
      const uint32_t dst = smem_u32(smem + 6 * kT64);
      size_t off = (size_t)blockIdx.x * 65536;
      while (!*reinterpret_cast<volatile int*>(&stop_flag)) {
        mbar_arrive_expect_tx(&tb, 16384);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                     ::"r"(dst), "l"(gsrc + off), "r"(smem_u32(&tb)) : "memory");
        mbar_wait(&tb, ph);
        ph ^= 1;
        off = (off + 16384) % (148 * 65536);
      }
    }
  } else if (warp >= 12 && warp < 12 + STW) {
    uint8_t* reg = smem + 6 * kT64 + (warp - 12) * 4096;
    uint32_t x = threadIdx.x;
    while (!*reinterpret_cast<volatile int*>(&stop_flag)) {
#pragma unroll
      for (int kq = 0; kq < 8; ++kq) {
        *reinterpret_cast<uint4*>(reg + (threadIdx.x & 31) * 128 + ((kq ^ (threadIdx.x & 7)) << 4)) = make_uint4(x, x + 1, x + 2, kq);
        x += 3;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

static uint8_t* g_src = nullptr;
template <int MODE, int LDW = 0, int STW = 0, int TMAW = 0, int MUW = 0>
void run(unsigned long long* d, const char* name, int ideal) {
  const int iters = 2000;
  const int smem = 6 * kT64 + 4 * 4096 + 1024;
  if (!g_src) cudaMalloc(&g_src, 148 * 65536 + 65536);
  cudaFuncSetAttribute(k<MODE, LDW, STW, TMAW, MUW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE, LDW, STW, TMAW, MUW><<<148, 512, smem>>>(d, iters, g_src);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7.0f clk per block (ideal %d) %s\n", name, (double)h / iters, ideal, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  run<0>(d, "full sequence", 1640);
  run<1>(d, "S^T + dP^T (8 x N128 SS)", 512);
  run<6>(d, "S^T + dP^T, no chain restart", 512);
  run<2>(d, "dV + dK (16 x N64 TS)", 736);
  run<4>(d, "dV + dK as SS (A MN-major)", 736);
  run<3>(d, "dQ (8 x N64 SS MN-major)", 384);
  run<5>(d, "full, fixed addresses", 1640);
  run<7>(d, "full + the kernel's commits", 1640);
  run<8>(d, "kernel commits + waits/fences", 1640);
  run<7, 8>(d, "  + 8 warps tcgen05.ld", 1640);
  run<7, 4>(d, "  + 4 warps tcgen05.ld", 1640);
  run<7, 0, 4>(d, "  + 4 warps STS", 1640);
  run<7, 8, 4>(d, "  + 8 ld warps + 4 STS warps", 1640);
  run<7, 0, 0, 1>(d, "  + TMA bulk loads (16 KB back to back)", 1640);
  run<8, 0, 0, 0, 4>(d, "waits/fences + 4 MUFU/FMA warps", 1640);
  run<8, 0, 0, 0, 8>(d, "waits/fences + 8 MUFU/FMA warps", 1640);
  run<8, 0, 0, 0, 12>(d, "waits/fences + 12 MUFU/FMA warps", 1640);
  return 0;
}
