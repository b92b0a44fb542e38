// Persistent, warp-specialised tcgen05 GEMM for sm_100a (bf16 in, fp32 TMEM
// accumulate) with a fused SUMMA epilogue. This is the local product of every
// SUMMA step of /root/reference/pkg/src/summagrid/summa.py:95-164 (there a numpy
// `a @ b` via mesh.py:349-361) and of the per-head attention products of
// layers.py:404-459.
//
// CTA layout (384 threads, 1 CTA per SM, grid = min(#tiles, #SMs)):
//   warp 0      TMA producer (one lane): A/B tiles -> SWIZZLE_128B smem ring
//   warp 1      MMA issuer (one lane): tcgen05.mma 128 x min(BN,256) x 16 into TMEM
//   warp 2      TMEM allocator
//   warps 4..11 epilogue; warp w owns TMEM lane quadrant (w % 4) = 32 tile rows and
//               every other 32-column chunk, so two warps share a quadrant
// Two TMEM accumulator buffers (one when BN = 512) let the epilogue of tile i
// overlap the MMAs of tile i+1; the smem ring has STAGES slots guarded by
// full/empty mbarriers.
//
// Epilogue modes:
//   NORMAL       tcgen05.ld (thread = row, 32 columns) -> alpha, bias, +C, GELU
//                (saves the pre-activation) or GELU', bf16/fp32 D, optional
//                bf16 copy D2 — 16-byte vector row accesses, every load of a
//                chunk issued before its stores (C may alias D); optional
//                column sums (bias gradients) via a swizzled smem transpose and
//                one atomic per column per warp.
//   SOFTMAX      D = softmax_row(alpha * acc) over the whole row (N <= 512 fits
//                TMEM): attention probabilities without an fp32 score matrix.
//   SOFTMAX_BWD  D = aux * (acc - rowsum(acc * aux)) * alpha with aux = P:
//                dS straight from the dP = dO V^T product (layers.py:447-450).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "sg.h"
#include "sg_internal.h"
#include "sg_ptx.cuh"

namespace sg {

struct GemmParams {
  int M, N, K;
  int nb2;
  int m_tiles, n_tiles, k_blocks, num_tiles;
  int a_b2_first, b_b2_first;
  int mode;
  void* D;
  long long ldd, sd1, sd2;
  int d_f32;
  const void* C;
  long long ldc, sc1, sc2;
  int c_f32;
  const float* bias;
  void* aux;
  long long ldx, sx1, sx2;
  __nv_bfloat16* D2;
  long long ld2, s21, s22;
  float* colsum;
  long long scs1, scs2;
  int act;
  float alpha;
  int vec_ok;
};

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kStg = 32 * 32;     // per-warp XOR-swizzled transpose staging for column sums (floats)
constexpr int kEpiWarps = 8;      // two epilogue warps per TMEM lane quadrant
constexpr int kThreads = 128 + 32 * kEpiWarps;

template <int BN>
struct GemmCfg {
  static constexpr int MMA_N = BN > 256 ? 256 : BN;
  static constexpr int NSPLIT = BN / MMA_N;
  static constexpr int ACC_BUFS = 2 * BN <= 512 ? 2 : 1;
  static constexpr uint32_t TMEM_COLS = ACC_BUFS * BN;
  static constexpr uint32_t A_BYTES = kBM * kBK * 2;
  static constexpr uint32_t B_BYTES = BN * kBK * 2;
  static constexpr int STAGES = BN == 512 ? 2 : (BN == 256 ? 4 : (BN == 128 ? 6 : 8));
  static constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + kEpiWarps * kStg * 4 + 1024 + 256;
};

__device__ __forceinline__ void load_box(const CUtensorMap* tm, void* dst, uint64_t* bar, int inner, int outer,
                                         int z2, int z1, int b2_first) {
  if (b2_first)
    tma_load_4d(dst, tm, bar, inner, z2, outer, z1);
  else
    tma_load_4d(dst, tm, bar, inner, outer, z2, z1);
}

__device__ __forceinline__ void decode_tile(const GemmParams& p, int t, int& mb, int& nb, int& z1, int& z2) {
  const int per = p.m_tiles * p.n_tiles;
  const int z = t / per;
  const int r = t - z * per;
  mb = r % p.m_tiles;
  nb = r / p.m_tiles;
  z1 = z / p.nb2;
  z2 = z - z1 * p.nb2;
}

__device__ __forceinline__ float gelu_fast(float x) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  return 0.5f * x * (1.f + tanh_fast(c * (x + a * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  const float t = tanh_fast(c * (x + a * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * a * x * x);
}

// 32 consecutive elements of one row: 16-byte vector accesses when aligned.
__device__ __forceinline__ void load_row32(const void* base, bool f32, bool vec, int n, float (&v)[32]) {
  if (f32) {
    const float* s = static_cast<const float*>(base);
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 x = *reinterpret_cast<const float4*>(s + j);
        v[j] = x.x; v[j + 1] = x.y; v[j + 2] = x.z; v[j + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = j < n ? s[j] : 0.f;
    }
  } else {
    const __nv_bfloat16* s = static_cast<const __nv_bfloat16*>(base);
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 x = *reinterpret_cast<const uint4*>(s + j);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(h[e]);
          v[j + 2 * e] = f.x; v[j + 2 * e + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = j < n ? __bfloat162float(s[j]) : 0.f;
    }
  }
}

__device__ __forceinline__ void store_row32(void* base, bool f32, bool vec, int n, const float (&v)[32]) {
  if (f32) {
    float* d = static_cast<float*>(base);
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(d + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < n) d[j] = v[j];
    }
  } else {
    __nv_bfloat16* d = static_cast<__nv_bfloat16*>(base);
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 x;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
        for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[j + 2 * e], v[j + 2 * e + 1]);
        *reinterpret_cast<uint4*>(d + j) = x;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < n) d[j] = __float2bfloat16_rn(v[j]);
    }
  }
}

__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Named barrier for the two epilogue warps sharing a TMEM lane quadrant.
__device__ __forceinline__ void quad_sync(int q) {
  asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ GemmParams p) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int ACC = Cfg::ACC_BUFS;
  constexpr uint32_t A_BYTES = Cfg::A_BYTES, B_BYTES = Cfg::B_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  float* stg_all = reinterpret_cast<float*>(sB + STAGES * B_BYTES);
  float* red_all = stg_all + kEpiWarps * kStg;  // [2 halves][4 quadrants][32 rows] row partials
  uint64_t* bars = reinterpret_cast<uint64_t*>(red_all + 256);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      uint32_t stage = 0, phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb, z1, z2;
        decode_tile(p, t, mb, nb, z1, z2);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], A_BYTES + B_BYTES);
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * B_BYTES;
          if (!A_MN) {
            load_box(&tmA, a_dst, &full[stage], kb * kBK, mb * kBM, z2, z1, p.a_b2_first);
          } else {
#pragma unroll
            for (int i = 0; i < kBM / 64; ++i)
              load_box(&tmA, a_dst + i * 64 * kBK * 2, &full[stage], mb * kBM + i * 64, kb * kBK, z2, z1,
                       p.a_b2_first);
          }
          if (!B_MN) {
#pragma unroll
            for (int h = 0; h < Cfg::NSPLIT; ++h)
              load_box(&tmB, b_dst + h * Cfg::MMA_N * kBK * 2, &full[stage], kb * kBK, nb * BN + h * Cfg::MMA_N, z2,
                       z1, p.b_b2_first);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              load_box(&tmB, b_dst + i * 64 * kBK * 2, &full[stage], nb * BN + i * 64, kb * kBK, z2, z1,
                       p.b_b2_first);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t IDESC = umma_idesc_bf16(kBM, Cfg::MMA_N, A_MN, B_MN);
      // byte offset of the second MMA_N-wide half of B inside a stage
      constexpr uint32_t B_HALF = Cfg::MMA_N * kBK * 2;
      uint32_t stage = 0, phase = 0, it = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
        const uint32_t as = it % ACC, aph = (it / ACC) & 1;
        mbar_wait(&tempty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * A_BYTES);
          const uint32_t b_base = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // K-major SW128: K step of 16 bf16 = 32 B inside the 128 B swizzle row,
            //   SBO = 1024 B between 8-row groups along M/N.
            // MN-major SW128: K step of 16 rows = 2048 B, LBO = 64-wide MN chunk
            //   stride (kBK rows x 128 B), SBO = 1024 B between 8-row K groups.
            const uint64_t ad = A_MN ? umma_desc_sw128(a_base + k * 2048, kBK * 128, 1024)
                                     : umma_desc_sw128(a_base + k * 32, 0, 1024);
#pragma unroll
            for (int h = 0; h < Cfg::NSPLIT; ++h) {
              const uint32_t bb = b_base + h * B_HALF;
              const uint64_t bd = B_MN ? umma_desc_sw128(bb + k * 2048, kBK * 128, 1024)
                                       : umma_desc_sw128(bb + k * 32, 0, 1024);
              umma_bf16(d_tmem + h * Cfg::MMA_N, ad, bd, IDESC, (kb | k) != 0 ? 1u : 0u);
            }
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[as]);
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    // warp w: TMEM lane quadrant q = w % 4 (rows 32q..32q+31), column chunks c % 2 == half
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    float* stg = stg_all + (warp - 4) * kStg;
    uint32_t it = 0;
    const bool d_f32 = p.d_f32 != 0, c_f32 = p.c_f32 != 0, vec = p.vec_ok != 0;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    constexpr int NCH = BN / 32;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      int mb, nb, z1, z2;
      decode_tile(p, t, mb, nb, z1, z2);
      const uint32_t as = it % ACC, aph = (it / ACC) & 1;
      mbar_wait(&tfull[as], aph);
      tc_fence_after();
      const uint32_t tacc = tmem_base + lane_base + as * BN;
      const int row = mb * kBM + q * 32 + lane;
      const bool row_ok = row < p.M;
      const size_t d_row = (size_t)z1 * p.sd1 + (size_t)z2 * p.sd2 + (size_t)row * p.ldd;
      const size_t c_row = (size_t)z1 * p.sc1 + (size_t)z2 * p.sc2 + (size_t)row * p.ldc;
      const size_t x_row = (size_t)z1 * p.sx1 + (size_t)z2 * p.sx2 + (size_t)row * p.ldx;
      const size_t o2_row = (size_t)z1 * p.s21 + (size_t)z2 * p.s22 + (size_t)row * p.ld2;
      if (p.mode == SG_EPI_NORMAL) {
#pragma unroll 1
        for (int c = half; c < NCH; c += 2) {
          uint32_t r[32];
          tmem_ld32(tacc + c * 32, r);
          tmem_wait_ld();
          if (c + 2 >= NCH) {  // this warp's last chunk of the tile
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[as]);
          }
          const int col0 = nb * BN + c * 32;
          if (col0 >= p.N) continue;  // warp-uniform
          const int ncols = min(32, p.N - col0);
          const bool vfull = vec && ncols == 32;
          float v[32];
          // issue every global load of the chunk before any store (C may alias D)
          float cv[32], xv[32];
          if (p.C && row_ok) {
            const void* cb = c_f32 ? static_cast<const void*>(static_cast<const float*>(p.C) + c_row + col0)
                                   : static_cast<const void*>(static_cast<const __nv_bfloat16*>(p.C) + c_row + col0);
            load_row32(cb, c_f32, vfull, ncols, cv);
          }
          if (p.act == SG_ACT_DGELU && row_ok)
            load_row32(static_cast<const __nv_bfloat16*>(p.aux) + x_row + col0, false, vfull, ncols, xv);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * p.alpha;
          if (p.bias) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += (j < ncols) ? __ldg(p.bias + col0 + j) : 0.f;
          }
          if (p.C) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += cv[j];
          }
          if (p.act == SG_ACT_GELU) {
            if (p.aux && row_ok) store_row32(static_cast<__nv_bfloat16*>(p.aux) + x_row + col0, false, vfull, ncols, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
          } else if (p.act == SG_ACT_DGELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= gelu_grad_fast(xv[j]);
          }
          if (row_ok) {
            void* db = d_f32 ? static_cast<void*>(static_cast<float*>(p.D) + d_row + col0)
                             : static_cast<void*>(static_cast<__nv_bfloat16*>(p.D) + d_row + col0);
            store_row32(db, d_f32, vfull, ncols, v);
            if (p.D2) store_row32(p.D2 + o2_row + col0, false, vfull, ncols, v);
          }
          if (p.colsum) {
            // column sums over this warp's 32 rows: transpose through smem, lane = column
#pragma unroll
            for (int j = 0; j < 32; ++j) stg[j * 32 + (lane ^ j)] = row_ok ? v[j] : 0.f;
            __syncwarp();
            float cs = 0.f;
#pragma unroll 8
            for (int i = 0; i < 32; ++i) cs += stg[lane * 32 + (i ^ lane)];
            if (lane < ncols) atomicAdd(p.colsum + (size_t)z1 * p.scs1 + (size_t)z2 * p.scs2 + col0 + lane, cs);
            __syncwarp();
          }
        }
      } else {
        // row-softmax modes: thread = row; the row's chunks are split between the
        // two warps of the quadrant, row partials combined through smem
        float* red = red_all + q * 32;  // [half][4 quadrants x 32]
        if (p.mode == SG_EPI_SOFTMAX) {
          const float sl2 = p.alpha * 1.4426950408889634f;  // alpha * log2(e)
          float m = -INFINITY;
#pragma unroll 1
          for (int c = half; c < NCH; c += 2) {
            uint32_t r[32];
            tmem_ld32(tacc + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c * 32 + j < p.N) m = fmaxf(m, __uint_as_float(r[j]));
          }
          red[half * 128 + lane] = m;
          quad_sync(q);
          m = fmaxf(red[lane], red[128 + lane]);
          const float ms = m * sl2;
          float z = 0.f;
#pragma unroll 1
          for (int c = half; c < NCH; c += 2) {
            uint32_t r[32];
            tmem_ld32(tacc + c * 32, r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (c * 32 + j < p.N) z += ex2_fast(fmaf(__uint_as_float(r[j]), sl2, -ms));
          }
          quad_sync(q);  // both warps have read the max slots
          red[half * 128 + lane] = z;
          quad_sync(q);
          const float inv = 1.f / (red[lane] + red[128 + lane]);
#pragma unroll 1
          for (int c = half; c < NCH; c += 2) {
            uint32_t r[32];
            tmem_ld32(tacc + c * 32, r);
            tmem_wait_ld();
            if (c + 2 >= NCH) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[as]);
            }
            const int col0 = c * 32;
            if (!row_ok || col0 >= p.N) continue;
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = ex2_fast(fmaf(__uint_as_float(r[j]), sl2, -ms)) * inv;
            store_row32(static_cast<__nv_bfloat16*>(p.D) + d_row + col0, false, vec && p.N - col0 >= 32,
                        min(32, p.N - col0), v);
          }
          quad_sync(q);  // smem partials free for the next tile
        } else {  // SG_EPI_SOFTMAX_BWD: D = P * (dP - sum(dP * P)) * alpha
          const __nv_bfloat16* pr = static_cast<const __nv_bfloat16*>(p.aux) + x_row;
          float acc = 0.f;
#pragma unroll 1
          for (int c = half; c < NCH; c += 2) {
            uint32_t r[32];
            tmem_ld32(tacc + c * 32, r);
            tmem_wait_ld();
            const int col0 = c * 32;
            if (!row_ok || col0 >= p.N) continue;
            float pv[32];
            load_row32(pr + col0, false, vec && p.N - col0 >= 32, min(32, p.N - col0), pv);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc = fmaf(__uint_as_float(r[j]), pv[j], acc);
          }
          red[half * 128 + lane] = acc;
          quad_sync(q);
          acc = red[lane] + red[128 + lane];
#pragma unroll 1
          for (int c = half; c < NCH; c += 2) {
            uint32_t r[32];
            tmem_ld32(tacc + c * 32, r);
            tmem_wait_ld();
            if (c + 2 >= NCH) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[as]);
            }
            const int col0 = c * 32;
            if (!row_ok || col0 >= p.N) continue;
            const bool v32 = vec && p.N - col0 >= 32;
            const int n = min(32, p.N - col0);
            float pv[32], v[32];
            load_row32(pr + col0, false, v32, n, pv);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = pv[j] * (__uint_as_float(r[j]) - acc) * p.alpha;
            store_row32(static_cast<__nv_bfloat16*>(p.D) + d_row + col0, false, v32, n, v);
          }
          quad_sync(q);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------ SIMT path
// CUDA-core fallback for operands the TMA unit cannot address (row pitches or
// batch strides that are not 16-byte multiples, e.g. head_dim 4 in the
// reference's unit-test configurations). NORMAL-mode semantics.
struct SimtParams {
  GemmParams p;
  const __nv_bfloat16* A;
  long long lda, sa1, sa2;
  int a_mn;
  const __nv_bfloat16* B;
  long long ldb, sb1, sb2;
  int b_mn;
  int nb1;
};

__global__ void gemm_simt_kernel(const __grid_constant__ SimtParams sp) {
  const GemmParams& p = sp.p;
  const long long total = (long long)sp.nb1 * p.nb2 * p.M * p.N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(idx % p.N);
    long long t = idx / p.N;
    const int m = (int)(t % p.M);
    t /= p.M;
    const int z2 = (int)(t % p.nb2);
    const int z1 = (int)(t / p.nb2);
    const __nv_bfloat16* a = sp.A + z1 * sp.sa1 + z2 * sp.sa2;
    const __nv_bfloat16* b = sp.B + z1 * sp.sb1 + z2 * sp.sb2;
    float acc = 0.f;
    for (int k = 0; k < p.K; ++k) {
      const float av = __bfloat162float(sp.a_mn ? a[(long long)k * sp.lda + m] : a[(long long)m * sp.lda + k]);
      const float bv = __bfloat162float(sp.b_mn ? b[(long long)k * sp.ldb + n] : b[(long long)n * sp.ldb + k]);
      acc = fmaf(av, bv, acc);
    }
    float v = acc * p.alpha;
    if (p.bias) v += p.bias[n];
    if (p.C) {
      const size_t ci = (size_t)z1 * p.sc1 + (size_t)z2 * p.sc2 + (size_t)m * p.ldc + n;
      v += p.c_f32 ? static_cast<const float*>(p.C)[ci] : __bfloat162float(static_cast<const __nv_bfloat16*>(p.C)[ci]);
    }
    const size_t xi = (size_t)z1 * p.sx1 + (size_t)z2 * p.sx2 + (size_t)m * p.ldx + n;
    if (p.act == SG_ACT_GELU) {
      if (p.aux) static_cast<__nv_bfloat16*>(p.aux)[xi] = __float2bfloat16_rn(v);
      v = gelu_f(v);
    } else if (p.act == SG_ACT_DGELU) {
      v *= gelu_grad_f(__bfloat162float(static_cast<const __nv_bfloat16*>(p.aux)[xi]));
    }
    const size_t di = (size_t)z1 * p.sd1 + (size_t)z2 * p.sd2 + (size_t)m * p.ldd + n;
    if (p.d_f32)
      static_cast<float*>(p.D)[di] = v;
    else
      static_cast<__nv_bfloat16*>(p.D)[di] = __float2bfloat16_rn(v);
    if (p.D2) p.D2[(size_t)z1 * p.s21 + (size_t)z2 * p.s22 + (size_t)m * p.ld2 + n] = __float2bfloat16_rn(v);
    if (p.colsum) atomicAdd(p.colsum + (size_t)z1 * p.scs1 + (size_t)z2 * p.scs2 + n, v);
  }
}

// ------------------------------------------------------------------ host side

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(ptr);
  });
  return fn;
}

// 4-D bf16 map over (inner, outer, b2, b1) with a box of 64 x box_outer.
static int make_operand_map(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long nb2,
                            long long nb1, long long ld, long long s2, long long s1, int box_outer, int* b2_first) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (!enc) return set_error(SG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (nb2 <= 1) s2 = ld * outer;
  if (nb1 <= 1) s1 = s2 * nb2;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * 2) % 16 || (s2 * 2) % 16 || (s1 * 2) % 16)
    return set_error(SG_ERR_SHAPE, "gemm operand: pointer/leading dims must be 16-byte aligned");
  const bool b2f = nb2 > 1 && s2 < ld;
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
  dims[0] = inner;
  if (b2f) {
    dims[1] = nb2; dims[2] = outer; dims[3] = nb1;
    strides[0] = s2 * 2; strides[1] = ld * 2; strides[2] = s1 * 2;
    box[0] = 64; box[1] = 1; box[2] = box_outer; box[3] = 1;
  } else {
    dims[1] = outer; dims[2] = nb2; dims[3] = nb1;
    strides[0] = ld * 2; strides[1] = s2 * 2; strides[2] = s1 * 2;
    box[0] = 64; box[1] = box_outer; box[2] = 1; box[3] = 1;
  }
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char msg[256];
    snprintf(msg, sizeof msg, "cuTensorMapEncodeTiled failed (%d): dims %lld,%lld,%lld,%lld ld=%lld s2=%lld s1=%lld",
             (int)r, inner, outer, nb2, nb1, ld, s2, s1);
    return set_error(SG_ERR_SHAPE, msg);
  }
  *b2_first = b2f ? 1 : 0;
  return SG_OK;
}

template <int BN, bool A_MN, bool B_MN>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, cudaStream_t stream,
                       int grid) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM) != cudaSuccess)
      return set_error(SG_ERR_CUDA, "cudaFuncSetAttribute(max smem) failed");
    attr_set = true;
  }
  kern<<<grid, kThreads, Cfg::SMEM, stream>>>(ta, tb, p);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SG_ERR_CUDA, cudaGetErrorString(e));
  return SG_OK;
}

template <int BN>
static int dispatch_major(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                          cudaStream_t s, int grid) {
  if (!amn && !bmn) return launch_gemm<BN, false, false>(ta, tb, p, s, grid);
  if (!amn && bmn) return launch_gemm<BN, false, true>(ta, tb, p, s, grid);
  if (amn && !bmn) return launch_gemm<BN, true, false>(ta, tb, p, s, grid);
  return launch_gemm<BN, true, true>(ta, tb, p, s, grid);
}

static int pick_bn(long long M, long long N, long long batch, int sms, int mode) {
  if (mode != SG_EPI_NORMAL) {  // the whole row in one tile
    for (int bn : {64, 128, 256, 512})
      if (N <= bn) return bn;
    return -1;
  }
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  // Largest tile unless it leaves the last wave badly underfilled.
  const long long mt = (M + kBM - 1) / kBM;
  double best_eff = -1.0;
  int best = 256;
  for (int bn : {256, 128}) {
    const long long tiles = mt * ((N + bn - 1) / bn) * batch;
    const long long waves = (tiles + sms - 1) / sms;
    const double work = (double)mt * kBM * ((N + bn - 1) / bn) * bn * batch;  // padded work
    const double eff = (double)M * N * batch / work * (double)tiles / (double)(waves * sms);
    if (eff > best_eff * 1.08) {
      best_eff = eff;
      best = bn;
    }
  }
  return best;
}

}  // namespace sg

using namespace sg;

extern "C" int sg_gemm(const sg_gemm_args* a, void* stream) {
  clear_error();
  if (!a) return set_error(SG_ERR_CONFIG, "null args");
  if (a->M < 1 || a->N < 1 || a->K < 1 || a->nb1 < 1 || a->nb2 < 1)
    return set_error(SG_ERR_SHAPE, "gemm: M, N, K and batch counts must be >= 1");
  if (a->M > INT32_MAX || a->N > INT32_MAX || a->K > INT32_MAX)
    return set_error(SG_ERR_SHAPE, "gemm: dimension exceeds int32");
  if (!a->A || !a->B || !a->D) return set_error(SG_ERR_CONFIG, "gemm: null operand");
  if ((a->act == SG_ACT_DGELU) && !a->aux) return set_error(SG_ERR_CONFIG, "gemm: DGELU needs aux");
  if (a->d_dtype != SG_DTYPE_BF16 && a->d_dtype != SG_DTYPE_F32) return set_error(SG_ERR_CONFIG, "gemm: d_dtype");
  if (a->mode != SG_EPI_NORMAL) {
    if (a->mode != SG_EPI_SOFTMAX && a->mode != SG_EPI_SOFTMAX_BWD) return set_error(SG_ERR_CONFIG, "gemm: mode");
    if (a->N > 512) return set_error(SG_ERR_SHAPE, "gemm: softmax epilogues need N <= 512");
    if (a->d_dtype != SG_DTYPE_BF16 || a->C || a->bias || a->act || a->D2 || a->colsum)
      return set_error(SG_ERR_CONFIG, "gemm: softmax epilogues write bf16 D only");
    if (a->mode == SG_EPI_SOFTMAX_BWD && !a->aux) return set_error(SG_ERR_CONFIG, "gemm: softmax bwd needs P");
    if (a->mode == SG_EPI_SOFTMAX && a->alpha <= 0.f) return set_error(SG_ERR_CONFIG, "gemm: softmax alpha > 0");
  }
  const int sms = sg_device_sm_count();
  if (sms <= 0) return set_error(SG_ERR_CUDA, "no CUDA device");

  GemmParams p{};
  p.M = (int)a->M;
  p.N = (int)a->N;
  p.K = (int)a->K;
  p.nb2 = (int)a->nb2;
  p.mode = a->mode;
  const long long batch = a->nb1 * a->nb2;
  const int bn = pick_bn(a->M, a->N, batch, sms, a->mode);
  p.m_tiles = (int)((a->M + kBM - 1) / kBM);
  p.n_tiles = (int)((a->N + bn - 1) / bn);
  p.k_blocks = (int)((a->K + kBK - 1) / kBK);
  const long long tiles = (long long)p.m_tiles * p.n_tiles * batch;
  if (tiles > INT32_MAX) return set_error(SG_ERR_SHAPE, "gemm: too many tiles");
  p.num_tiles = (int)tiles;
  p.D = a->D; p.ldd = a->ldd; p.sd1 = a->sd1; p.sd2 = a->sd2; p.d_f32 = a->d_dtype == SG_DTYPE_F32;
  p.C = a->C; p.ldc = a->ldc; p.sc1 = a->sc1; p.sc2 = a->sc2; p.c_f32 = a->c_dtype == SG_DTYPE_F32;
  p.bias = a->bias;
  p.aux = a->aux; p.ldx = a->ldx; p.sx1 = a->sx1; p.sx2 = a->sx2;
  p.D2 = static_cast<__nv_bfloat16*>(a->D2); p.ld2 = a->ld2; p.s21 = a->s21; p.s22 = a->s22;
  p.colsum = a->colsum; p.scs1 = a->scs1; p.scs2 = a->scs2;
  p.act = a->act;
  p.alpha = a->alpha;
  // 16-byte vector row access (softmax modes) when every row start of D / aux is 16-byte aligned.
  auto al = [](const void* ptr, long long ld, long long s1, long long s2, int esz) {
    if (!ptr) return true;
    return (reinterpret_cast<uintptr_t>(ptr) % 16) == 0 && (ld * esz) % 16 == 0 && (s1 * esz) % 16 == 0 &&
           (s2 * esz) % 16 == 0;
  };
  p.vec_ok = al(a->D, a->ldd, a->sd1, a->sd2, p.d_f32 ? 4 : 2) && al(a->aux, a->ldx, a->sx1, a->sx2, 2);

  // TMA needs 16-byte aligned bases, row pitches and batch strides; otherwise
  // take the CUDA-core path (tiny / odd-shaped operands only).
  auto tma_ok = [](const void* ptr, long long ld, long long n1, long long s1, long long n2, long long s2) {
    return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (ld * 2) % 16 == 0 && (n1 <= 1 || (s1 * 2) % 16 == 0) &&
           (n2 <= 1 || (s2 * 2) % 16 == 0);
  };
  if (!tma_ok(a->A, a->lda, a->nb1, a->sa1, a->nb2, a->sa2) || !tma_ok(a->B, a->ldb, a->nb1, a->sb1, a->nb2, a->sb2)) {
    if (a->mode != SG_EPI_NORMAL) return set_error(SG_ERR_SHAPE, "gemm: softmax epilogues need TMA-aligned operands");
    SimtParams sp;
    sp.p = p;
    sp.A = static_cast<const __nv_bfloat16*>(a->A);
    sp.lda = a->lda; sp.sa1 = a->sa1; sp.sa2 = a->sa2; sp.a_mn = a->a_mn_major;
    sp.B = static_cast<const __nv_bfloat16*>(a->B);
    sp.ldb = a->ldb; sp.sb1 = a->sb1; sp.sb2 = a->sb2; sp.b_mn = a->b_mn_major;
    sp.nb1 = (int)a->nb1;
    const long long total = a->nb1 * a->nb2 * a->M * a->N;
    const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)sms * 16);
    gemm_simt_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(sp);
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
  }
  CUtensorMap ta, tb;
  int rc;
  // A: K-major -> (K, M); MN-major -> (M, K)
  if (!a->a_mn_major)
    rc = make_operand_map(&ta, a->A, a->K, a->M, a->nb2, a->nb1, a->lda, a->sa2, a->sa1, kBM, &p.a_b2_first);
  else
    rc = make_operand_map(&ta, a->A, a->M, a->K, a->nb2, a->nb1, a->lda, a->sa2, a->sa1, kBK, &p.a_b2_first);
  if (rc) return rc;
  const int b_box = std::min(bn, 256);
  if (!a->b_mn_major)
    rc = make_operand_map(&tb, a->B, a->K, a->N, a->nb2, a->nb1, a->ldb, a->sb2, a->sb1, b_box, &p.b_b2_first);
  else
    rc = make_operand_map(&tb, a->B, a->N, a->K, a->nb2, a->nb1, a->ldb, a->sb2, a->sb1, kBK, &p.b_b2_first);
  if (rc) return rc;

  const int grid = (int)std::min<long long>(tiles, sms);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool amn = a->a_mn_major != 0, bmn = a->b_mn_major != 0;
  switch (bn) {
    case 64: return dispatch_major<64>(amn, bmn, ta, tb, p, s, grid);
    case 128: return dispatch_major<128>(amn, bmn, ta, tb, p, s, grid);
    case 256: return dispatch_major<256>(amn, bmn, ta, tb, p, s, grid);
    default: return dispatch_major<512>(amn, bmn, ta, tb, p, s, grid);
  }
}
