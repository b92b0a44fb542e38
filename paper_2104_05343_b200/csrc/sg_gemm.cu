// Persistent, warp-specialised tcgen05 GEMM for sm_100a (bf16 in, fp32 TMEM
// accumulate) with a fused SUMMA epilogue. This is the local product of every
// SUMMA step of /root/reference/pkg/src/summagrid/summa.py:95-164 (there a numpy
// `a @ b` via mesh.py:349-361) and of the per-head attention products of
// layers.py:404-459.
//
// CTA layout (256 / 384 / 512 threads, 1 CTA per SM, grid = min(#tiles, #SMs), or
// CTA pairs (cluster of 2, cta_group::2) for 256 x {128, 256} tiles):
//   warp 0      TMA producer (one lane): A/B tiles -> SWIZZLE_128B smem ring
//   warp 1      MMA issuer (one lane, the pair's leader): tcgen05.mma into TMEM
//   warp 2      TMEM allocator
//   warps 4..   4, 8 or 12 epilogue warps; warp w owns TMEM lane quadrant (w % 4)
//               = 32 tile rows and every (EW / 4)-th 32-column chunk
// Two TMEM accumulator buffers (one when BN = 512) let the epilogue of tile i
// overlap the MMAs of tile i+1; the smem ring has STAGES slots guarded by
// full/empty mbarriers.
//
// Epilogue modes:
//   NORMAL       tcgen05.ld (thread = row, 32 columns) -> alpha, bias, +C, GELU
//                (saves the pre-activation) or GELU', LayerNorm-backward row
//                statistics, bf16/fp32 D, optional bf16 copy D2, optional column
//                sums (bias gradients, register butterfly); inputs (C / aux) and
//                outputs move through swizzled smem staging by TMA, C == D
//                accumulates in place by TMA reduce-add (split-K, fused SGD).
//   SOFTMAX      D = softmax_row(alpha * acc) over the whole row (N <= 512 fits
//                TMEM): attention probabilities without an fp32 score matrix.
//   SOFTMAX_BWD  D = aux * (acc - rowsum(acc * aux)) * alpha with aux = P:
//                dS straight from the dP = dO V^T product (layers.py:447-450).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "sg.h"
#include "sg_internal.h"
#include "sg_ptx.cuh"
#include "sg_tmap.h"

namespace sg {

// n / d for 0 <= n < 2^31 as (n * m) >> (32 + s), m = ceil(2^(32+s) / d), s = ceil(log2 d)
// (exact: the rounding error n e / (d 2^(32+s)) stays below 1/d), precomputed on the
// host: every role decodes a tile index per tile, cheaply only without divisions
struct FastDiv {
  unsigned long long m;
  uint32_t d, s;
  __host__ void set(uint32_t div) {
    d = div;
    s = 0;
    while ((1ull << s) < div) ++s;
    m = (((unsigned long long)1 << (32 + s)) + div - 1) / div;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((unsigned long long)n * m) >> (32 + s));
  }
};

struct GemmParams {
  FastDiv fd_tiles, fd_per, fd_span, fd_nb2;  // tiles per split, m x n tiles, group span, nb2
  int M, N, K;
  int nb2;
  int m_tiles, n_tiles, k_blocks, num_tiles;
  int k_splits, kb_per_split;   // split-K: work unit = (split, tile), partial sums reduce-added into D
  int full_units;               // units >= full_units are half-width (BN / 2) tiles of the last round
  int group_m, group_shift;     // rasterisation: groups of group_m (= 1 << group_shift) m-tiles
  // die-local tile streams (large pair-tile products): the CTA pairs of each of the two
  // dies take alternate 8-m-tile halves of every 16-m-tile group, so A rows are shared
  // by pairs of one die (whose L2 then fetches them once); pair c works on die die_of[c]
  // as its slot_of[c]-th pair (a bijection measured once per device, sg_gemm_die_table)
  int die_mode, die_pairs;
  uint8_t die_of[128], slot_of[128];
  int a_b2_first, b_b2_first, o_b2_first, x_b2_first, c_b2_first;
  int mode;
  int d_f32;
  void* D;                      // direct stores of the row-softmax modes
  long long ldd, sd1, sd2;
  int vec_d;
  const void* C;
  long long ldc, sc1, sc2;
  int c_f32;
  const float* bias;
  const __nv_bfloat16* aux_in;  // DGELU pre-activation / SOFTMAX_BWD probabilities
  long long ldx, sx1, sx2;
  int aux_out;                  // GELU: store the pre-activation through tmX
  int reduce_add;               // C == D (fp32): D += result by TMA reduce-add, no epilogue loads
  int has_d2;                   // bf16 copy of D through tmD2
  float* colsum;
  long long scs1, scs2;
  const float* rowvec;          // SOFTMAX_BWD: D_i = rowsum(dO * O) per row
  long long srv1, srv2;
  // LayerNorm-backward row statistics of the fp32 output (C = LayerNorm input x,
  // loaded but not added): ln_stats[2 r] += sum xhat g, ln_stats[2 r + 1] += sum g,
  // g = D * gamma, xhat = (x - mean) rstd
  const float* ln_gamma;
  const float* ln_mean;
  const float* ln_rstd;
  float* ln_stats;
  int act;
  float alpha;
};

constexpr int kBM = 128;
constexpr int kBK = 64;
// Epilogue kinds: GENERIC decides every feature from GemmParams at run time; the
// others fix the feature set at compile time for the step's hot products, so the
// epilogue loop is short and branch-free (measured: the generic loop's size and
// flag branches cost instruction-fetch and branch stalls at ~2 epilogue warps / SMSP)
enum EpiKind : int {
  EK_GENERIC = 0,
  EK_STORE = 1,     // D = alpha acc (bf16 / fp32), optional TMA reduce-add
  EK_BIAS = 2,      // D = alpha acc + bias, optional TMA reduce-add
  EK_CIN_BIAS = 3,  // fp32 D = acc + bias + fp32 C (residual)
  EK_GELU_BIAS = 4, // D = gelu(acc + bias), pre-activation stored through tmX
  EK_DGELU = 5,     // D = acc * gelu'(aux) [+ column sums]
  EK_LN = 6,        // fp32 D = acc, LayerNorm-backward row statistics (C = x)
};
// Epilogue warps: 4 (one per TMEM lane quadrant), 8 (two per quadrant, each taking
// every other 32-column chunk) where the epilogue otherwise paces the tensor pipe
// at small K, or 12 for the epilogue-bound GELU' + column-sum product.
template <int EW>
struct EpiCfg {
  static constexpr int kThreads = 128 + 32 * EW;
  static constexpr int CSTEP = EW / 4;
  // 12 epilogue warps (512 threads, 128 registers at launch): the producer / MMA
  // warpgroup gives registers up and the epilogue warpgroups take them (setmaxnreg)
  static constexpr bool kRealloc = EW == 12;
};
// Per epilogue warp 8 KB of staging: two 4 KB slots (main tile up to 4 KB, or a
// 2 KB bf16 main tile + 2 KB bf16 side tile) so chunk c+1 never waits for chunk
// c's TMA store, or one 8 KB slot when an fp32 main tile needs a side tile.
constexpr int kStgBytes = 8192;

// PAIR: a 2-CTA cluster computes a 256 x BN tile with tcgen05.mma.cta_group::2
// (each CTA holds 128 rows of A, BN/2 rows of B and its 128 x BN accumulator),
// halving the per-SM shared-memory operand traffic and B loads; the freed smem
// buys deeper rings.
template <int BN, int EW, bool PAIR = false>
struct GemmCfg {
  static constexpr int MMA_N = BN > 256 ? 256 : BN;
  static constexpr int NSPLIT = BN / MMA_N;
  static constexpr int ACC_BUFS = 2 * BN <= 512 ? 2 : 1;
  static constexpr uint32_t TMEM_COLS = ACC_BUFS * BN;
  static constexpr int TM = PAIR ? 2 * kBM : kBM;  // tile rows
  static constexpr int BNL = PAIR ? BN / 2 : BN;   // B rows (N) loaded per CTA
  static constexpr uint32_t A_BYTES = kBM * kBK * 2;
  static constexpr uint32_t B_BYTES = BNL * kBK * 2;
  static constexpr int STAGES =
      PAIR ? (EW == 12 ? (BN == 256 ? 4 : 5) : EW == 8 ? (BN == 256 ? 5 : 6) : (BN == 256 ? 6 : 8))
           : (EW == 8 ? (BN == 256 ? 3 : 4) : (BN == 512 ? 2 : (BN == 256 ? 4 : (BN == 128 ? 6 : 8))));
  static constexpr size_t SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + EW * (kStgBytes + 128) + 512;
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(!PAIR || BN == 128 || BN == 256, "pair tiles are 256 x 128 or 256 x 256");
};

__device__ __forceinline__ void load_box(const CUtensorMap* tm, void* dst, uint64_t* bar, int inner, int outer,
                                         int z2, int z1, int b2_first) {
  if (b2_first)
    tma_load_4d(dst, tm, bar, inner, z2, outer, z1);
  else
    tma_load_4d(dst, tm, bar, inner, outer, z2, z1);
}

// TMA load by either CTA of a pair, completing on the leader's barrier
__device__ __forceinline__ void load_box_pair(const CUtensorMap* tm, void* dst, uint32_t bar_cluster, int inner,
                                              int outer, int z2, int z1, int b2_first) {
  if (b2_first)
    tma_load_4d_pair(dst, tm, bar_cluster, inner, z2, outer, z1);
  else
    tma_load_4d_pair(dst, tm, bar_cluster, inner, outer, z2, z1);
}

__device__ __forceinline__ void store_box(const CUtensorMap* tm, const void* src, int inner, int outer, int z2, int z1,
                                          int b2_first) {
  if (b2_first)
    tma_store_4d(tm, src, inner, z2, outer, z1);
  else
    tma_store_4d(tm, src, inner, outer, z2, z1);
}
__device__ __forceinline__ void reduce_box(const CUtensorMap* tm, const void* src, int inner, int outer, int z2,
                                           int z1, int b2_first) {
  if (b2_first)
    tma_reduce_add_4d(tm, src, inner, z2, outer, z1);
  else
    tma_reduce_add_4d(tm, src, inner, outer, z2, z1);
}

// Grouped rasterisation: tiles run in groups of kGroupM m-tiles, n fastest
// inside a group, so the CTAs in flight share a few A row panels and sweep B;
// each operand is then streamed from HBM about once even when A exceeds L2.
constexpr int kGroupM = 16;
__device__ __forceinline__ void decode_tile(const GemmParams& p, int t, int& mb, int& nb, int& z1, int& z2) {
  t -= (int)p.fd_tiles.div((uint32_t)t) * (int)p.fd_tiles.d;  // split-K units share the output tile
  const int z = (int)p.fd_per.div((uint32_t)t);
  const int r = t - z * (int)p.fd_per.d;
  const int group = (int)p.fd_span.div((uint32_t)r);
  const int first_m = group * p.group_m;
  const int gm = min(p.group_m, p.m_tiles - first_m);
  const int rr = r - group * (int)p.fd_span.d;
  if (gm == p.group_m) {
    mb = first_m + (rr & (p.group_m - 1));
    nb = rr >> p.group_shift;
  } else {
    mb = first_m + rr % gm;
    nb = rr / gm;
  }
  z1 = (int)p.fd_nb2.div((uint32_t)z);
  z2 = z - z1 * p.nb2;
}

// Work unit t -> tile. The last partial round of a pair-tile product can be issued
// as twice as many half-width units (tile columns [0, BN/2) and [BN/2, BN)): the
// round then costs one narrow tile instead of one full tile on fewer pairs
// (N = 1024 products: 3.46 -> 3.73 tile times... measured in DESIGN.md).
// half = -1 for a full tile.
__device__ __forceinline__ void decode_unit(const GemmParams& p, int t, int& mb, int& nb, int& z1, int& z2, int& half) {
  if (t >= p.full_units) {
    const int h = t - p.full_units;
    half = h & 1;
    t = p.full_units + (h >> 1);
  } else {
    half = -1;
  }
  decode_tile(p, t, mb, nb, z1, z2);
}

// k-block range of work unit t (the whole K unless split-K)
__device__ __forceinline__ void unit_k_range(const GemmParams& p, int t, int& kb0, int& kb1) {
  const int split = t / (p.num_tiles / p.k_splits);
  kb0 = split * p.kb_per_split;
  kb1 = min(p.k_blocks, kb0 + p.kb_per_split);
}

// tanh-GELU of 32 values on the paired fp32 pipe: 0.5 x (1 + tanh(c x (1 + a x^2)))
__device__ __forceinline__ void gelu_row(float (&v)[32]) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  const uint64_t ca2 = f2_pack(c * a, c * a), c2 = f2_pack(c, c), h2 = f2_pack(0.5f, 0.5f);
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const uint64_t x = f2_pack(v[j], v[j + 1]);
    const uint64_t t = ffma2(fmul2(x, x), ca2, c2);  // c + c a x^2
    const uint64_t u = fmul2(x, t);                  // c (x + a x^3)
    const uint64_t hx = fmul2(x, h2);
    const uint64_t th = f2_pack(tanh_fast(f2_lo(u)), tanh_fast(f2_hi(u)));
    const uint64_t y = ffma2(hx, th, hx);
    v[j] = f2_lo(y);
    v[j + 1] = f2_hi(y);
  }
}

// v *= gelu'(x), paired: with t = tanh(c (x + a x^3)) and w = x (0.5 c + 1.5 a c x^2),
// gelu'(x) = 0.5 (1 + t) + w (1 - t^2) = (0.5 + w) + t (0.5 - w t)
__device__ __forceinline__ void dgelu_row(float (&v)[32], const float (&x)[32]) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  const uint64_t ca2 = f2_pack(c * a, c * a), c2 = f2_pack(c, c), h2 = f2_pack(0.5f, 0.5f),
                 m1 = f2_pack(-1.f, -1.f), k1 = f2_pack(-1.5f * a * c, -1.5f * a * c), k0 = f2_pack(-0.5f * c, -0.5f * c);
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const uint64_t xx = f2_pack(x[j], x[j + 1]);
    const uint64_t x2 = fmul2(xx, xx);
    const uint64_t u = fmul2(xx, ffma2(x2, ca2, c2));  // c (x + a x^3)
    const uint64_t wn = fmul2(xx, ffma2(x2, k1, k0));  // -w
    const uint64_t t = f2_pack(tanh_fast(f2_lo(u)), tanh_fast(f2_hi(u)));
    const uint64_t g = ffma2(t, ffma2(wn, t, h2), ffma2(wn, m1, h2));
    const uint64_t y = fmul2(f2_pack(v[j], v[j + 1]), g);
    v[j] = f2_lo(y);
    v[j + 1] = f2_hi(y);
  }
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
__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- swizzled 32 x 32 staging tiles (match the TMA SWIZZLE_128B / _64B maps)
// fp32: 128-byte rows, 16-byte chunk k of row r at ((k ^ (r & 7)) << 4)
// bf16:  64-byte rows, 16-byte chunk k of row r at ((k ^ ((r >> 1) & 3)) << 4)
__device__ __forceinline__ uint32_t swz_f32(int r, int col) {
  return r * 128 + ((((col >> 2) ^ (r & 7))) << 4) + ((col & 3) << 2);
}
__device__ __forceinline__ uint32_t swz_bf16(int r, int col) {
  return r * 64 + ((((col >> 3) ^ ((r >> 1) & 3))) << 4) + ((col & 7) << 1);
}
__device__ __forceinline__ void st_row_f32(uint8_t* buf, int r, const float (&v)[32]) {
#pragma unroll
  for (int k = 0; k < 8; ++k)
    *reinterpret_cast<float4*>(buf + r * 128 + ((k ^ (r & 7)) << 4)) =
        make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
}
__device__ __forceinline__ void ld_row_f32(const uint8_t* buf, int r, float (&v)[32]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float4 x = *reinterpret_cast<const float4*>(buf + r * 128 + ((k ^ (r & 7)) << 4));
    v[4 * k] = x.x; v[4 * k + 1] = x.y; v[4 * k + 2] = x.z; v[4 * k + 3] = x.w;
  }
}
__device__ __forceinline__ void st_row_bf16(uint8_t* buf, int r, const float (&v)[32]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint4 x;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * k + 2 * e], v[8 * k + 2 * e + 1]);
    *reinterpret_cast<uint4*>(buf + r * 64 + ((k ^ ((r >> 1) & 3)) << 4)) = x;
  }
}
__device__ __forceinline__ void ld_row_bf16(const uint8_t* buf, int r, float (&v)[32]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint4 x = *reinterpret_cast<const uint4*>(buf + r * 64 + ((k ^ ((r >> 1) & 3)) << 4));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(h[e]);
      v[8 * k + 2 * e] = f.x; v[8 * k + 2 * e + 1] = f.y;
    }
  }
}

// One thread's 32 consecutive bf16 outputs (row-softmax modes write rows directly).
__device__ __forceinline__ void store_bf16_row(__nv_bfloat16* d, bool vec, int n, const float (&v)[32]) {
  if (vec && n == 32) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint4 x;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
      for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * k + 2 * e], v[8 * k + 2 * e + 1]);
      *reinterpret_cast<uint4*>(d + 8 * k) = x;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < n) d[j] = __float2bfloat16_rn(v[j]);
  }
}

template <int BN, bool A_MN, bool B_MN, int EW, bool PAIR, int KIND>
__global__ void __launch_bounds__(EpiCfg<EW>::kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmD2, const __grid_constant__ CUtensorMap tmC,
                const __grid_constant__ GemmParams p) {
  using Cfg = GemmCfg<BN, EW, PAIR>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int ACC = Cfg::ACC_BUFS;
  constexpr int TM = Cfg::TM, BNL = Cfg::BNL;
  constexpr uint32_t A_BYTES = Cfg::A_BYTES, B_BYTES = Cfg::B_BYTES;
  // pair mode: both CTAs of the cluster walk the same tile sequence; rank 0 (the
  // leader) issues the MMAs and owns the smem-full / TMEM-empty barriers
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int unit0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nunits = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  // this pair's unit stream: units u0, u0 + ustep, ... < ucount, tile tile_of(u)
  const bool dm = PAIR && p.die_mode;
  const int udie = dm ? p.die_of[unit0] : 0;
  const int u0 = dm ? p.slot_of[unit0] : unit0, ustep = dm ? p.die_pairs : nunits;
  const int ucount = dm ? (p.num_tiles >> 1) : p.num_tiles;
  auto tile_of = [&](int u) -> int {
    if (!dm) return u;
    const int hs = p.group_shift - 1, hg = 1 << hs;  // this die's half of a group: hg m-tiles
    const int per_g = hg * p.n_tiles;
    const int g = u / per_g, r = u - g * per_g;
    return (g * p.n_tiles + (r >> hs)) * p.group_m + udie * hg + (r & (hg - 1));  // the standard grouped order's index
  };
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint8_t* stg_all = sB + STAGES * B_BYTES;  // 1024-aligned
  float* bias_all = reinterpret_cast<float*>(stg_all + EW * kStgBytes);  // [EW][32] bias chunk per warp
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg_all + EW * (kStgBytes + 128));
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint64_t* inbar = bars + 2 * STAGES + 4;  // [EW][2]: epilogue input tiles (C / aux) landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + 2 * EW);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmD);
    if (p.C && !p.reduce_add) tma_prefetch_desc(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], PAIR ? 2 * EW : EW);
    }
    for (int i = 0; i < 2 * EW; ++i) mbar_init(&inbar[i], 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    if (PAIR)
      tmem_alloc_pair<Cfg::TMEM_COLS>(tmem_slot);
    else
      tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if (PAIR)
    cluster_sync_all();  // barrier inits and the pair's TMEM allocation visible cluster-wide
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_begin();  // prologue above overlaps the previous kernel; inputs are read below

  if (warp == 0) {
    if constexpr (EpiCfg<EW>::kRealloc) reg_dealloc<40>();
    {
      // ------------------------------------------------------------ producer
      // whole warp walks the loop (warp-uniform coordinates); one elected lane issues
      uint32_t stage = 0, phase = 0;
      for (int u = u0; u < ucount; u += ustep) {
        const int t = tile_of(u);
        int mb, nb, z1, z2, half;
        decode_unit(p, t, mb, nb, z1, z2, half);
        int kb0, kb1;
        unit_k_range(p, t, kb0, kb1);
        const int m0 = mb * TM + (int)rank * kBM;  // this CTA's A rows
        // this CTA's B rows (N); a half-width pair unit uses the first BNL / 2 rows of each
        // CTA's B tile (the box still loads BNL rows: same transaction bytes)
        const int n0 = half < 0 ? nb * BN + (int)rank * BNL : nb * BN + half * (BN / 2) + (int)rank * (BNL / 2);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * B_BYTES;
          if (!elect_one()) {
          } else if (PAIR) {
            // both CTAs' bytes complete on the leader's barrier
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
            const uint32_t fb = mapa_smem(&full[stage], 0);
            if (!A_MN) {
              load_box_pair(&tmA, a_dst, fb, kb * kBK, m0, z2, z1, p.a_b2_first);
            } else {
#pragma unroll
              for (int i = 0; i < kBM / 64; ++i)
                load_box_pair(&tmA, a_dst + i * 64 * kBK * 2, fb, m0 + i * 64, kb * kBK, z2, z1, p.a_b2_first);
            }
            if (!B_MN) {
              load_box_pair(&tmB, b_dst, fb, kb * kBK, n0, z2, z1, p.b_b2_first);
            } else {
#pragma unroll
              for (int i = 0; i < BNL / 64; ++i)
                load_box_pair(&tmB, b_dst + i * 64 * kBK * 2, fb, n0 + i * 64, kb * kBK, z2, z1, p.b_b2_first);
            }
          } else {
            mbar_arrive_expect_tx(&full[stage], A_BYTES + B_BYTES);
            if (!A_MN) {
              load_box(&tmA, a_dst, &full[stage], kb * kBK, m0, z2, z1, p.a_b2_first);
            } else {
#pragma unroll
              for (int i = 0; i < kBM / 64; ++i)
                load_box(&tmA, a_dst + i * 64 * kBK * 2, &full[stage], m0 + i * 64, kb * kBK, z2, z1, p.a_b2_first);
            }
            if (!B_MN) {
#pragma unroll
              for (int h = 0; h < Cfg::NSPLIT; ++h)
                load_box(&tmB, b_dst + h * Cfg::MMA_N * kBK * 2, &full[stage], kb * kBK, n0 + h * Cfg::MMA_N, z2, z1,
                         p.b_b2_first);
            } else {
#pragma unroll
              for (int i = 0; i < BN / 64; ++i)
                load_box(&tmB, b_dst + i * 64 * kBK * 2, &full[stage], n0 + i * 64, kb * kBK, z2, z1, p.b_b2_first);
            }
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if constexpr (EpiCfg<EW>::kRealloc) reg_dealloc<40>();
    if (rank == 0) {
      // ------------------------------------------------------------ MMA issuer
      // The whole warp walks the loop with warp-uniform operands (descriptors in uniform
      // registers, advanced by adding (bytes >> 4) to the start-address field); one
      // elected lane issues. A single-lane issuer pays a per-MMA lane waterfall of ~12
      // instructions, and the epilogue warps sharing its SMSP starve it of issue slots
      // (the flash backward traces: tools/ftrace.py).
      constexpr uint32_t IDESC_FULL = umma_idesc_bf16(TM, Cfg::MMA_N, A_MN, B_MN);
      constexpr uint32_t IDESC_HALF = umma_idesc_bf16(TM, Cfg::MMA_N / 2, A_MN, B_MN);
      // K-major SW128: K step of 16 bf16 = 32 B inside the 128 B swizzle row, SBO = 1024 B
      //   between 8-row groups along M/N. MN-major SW128: K step of 16 rows = 2048 B,
      //   LBO = 64-wide MN chunk stride (kBK rows x 128 B), SBO = 1024 B between 8-row K groups.
      constexpr uint64_t A_KSTEP = A_MN ? (2048 >> 4) : (32 >> 4), B_KSTEP = B_MN ? (2048 >> 4) : (32 >> 4);
      constexpr uint64_t A_STAGE = A_BYTES >> 4, B_STAGE = B_BYTES >> 4;
      constexpr uint64_t B_HALF = (Cfg::MMA_N * kBK * 2) >> 4;  // second MMA_N-wide half of B
      const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA), A_MN ? kBK * 128 : 0, 1024);
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sB), B_MN ? kBK * 128 : 0, 1024);
      const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
      uint32_t stage = 0, phase = 0, it = 0;
      for (int u = u0; u < ucount; u += ustep, ++it) {
        const int t = tile_of(u);
        const uint32_t IDESC = (PAIR && t >= p.full_units) ? IDESC_HALF : IDESC_FULL;
        const uint32_t as = it % ACC, aph = (it / ACC) & 1;
        if (PAIR)
          mbar_wait_cluster(&tempty[as], aph ^ 1);  // both CTAs' epilogues drained this buffer
        else
          mbar_wait(&tempty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tbase + as * BN;
        int kb0, kb1;
        unit_k_range(p, t, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad0 = a_desc0 + stage * A_STAGE, bd0 = b_desc0 + stage * B_STAGE;
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
#pragma unroll
              for (int h = 0; h < Cfg::NSPLIT; ++h) {
                const uint64_t ad = ad0 + k * A_KSTEP, bd = bd0 + h * B_HALF + k * B_KSTEP;
                if (PAIR)
                  umma_bf16_pair(d_tmem + h * Cfg::MMA_N, ad, bd, IDESC, (kb != kb0 || k != 0) ? 1u : 0u);
                else
                  umma_bf16(d_tmem + h * Cfg::MMA_N, ad, bd, IDESC, (kb != kb0 || k != 0) ? 1u : 0u);
              }
            }
            if (PAIR)
              umma_commit_pair(&empty[stage], 0x3);  // frees the slot in both CTAs
            else
              umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) {
          if (PAIR)
            umma_commit_pair(&tfull[as], 0x3);
          else
            umma_commit(&tfull[as]);
        }
        __syncwarp();
      }
    }
  } else if (warp < 4) {
    if constexpr (EpiCfg<EW>::kRealloc) reg_dealloc<40>();
  } else {
    if constexpr (EpiCfg<EW>::kRealloc) reg_alloc<152>();
    // -------------------------------------------------------------- epilogue
    // epilogue warp e owns TMEM lane quadrant q = e % 4 (tile rows 32q .. 32q+31,
    // a hardware restriction: warp w reads lanes 32 (w % 4) ..) and the chunks
    // c = e / 4, e / 4 + CSTEP, ...
    const int e = warp - 4;
    const int q = e & 3;
    constexpr int CSTEP = EpiCfg<EW>::CSTEP;
    const int c_first = e >> 2;
    uint8_t* stg_w = stg_all + e * kStgBytes;
    uint32_t it = 0, slot = 0, inph = 0;
    // feature flags: compile-time constants unless KIND == EK_GENERIC
    constexpr bool G = KIND == EK_GENERIC;
    const bool f_bias = G ? p.bias != nullptr : (KIND == EK_BIAS || KIND == EK_CIN_BIAS || KIND == EK_GELU_BIAS);
    const bool f_ln = G ? p.ln_stats != nullptr : KIND == EK_LN;
    const int f_act = G ? p.act : (KIND == EK_GELU_BIAS ? SG_ACT_GELU : (KIND == EK_DGELU ? SG_ACT_DGELU : SG_ACT_NONE));
    const int f_mode = G ? p.mode : SG_EPI_NORMAL;
    const bool f_colsum = G ? p.colsum != nullptr : (KIND == EK_DGELU && p.colsum != nullptr);
    const bool f_d2 = G ? p.has_d2 != 0 : false;
    const bool f_aux_out = G ? p.aux_out != 0 : KIND == EK_GELU_BIAS;
    const bool f_reduce = G ? p.reduce_add != 0 : ((KIND == EK_STORE || KIND == EK_BIAS) && p.reduce_add != 0);
    const bool d_f32 = (KIND == EK_CIN_BIAS || KIND == EK_LN) ? true : p.d_f32 != 0;
    const bool c_f32 = G ? p.c_f32 != 0 : true;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    constexpr int NCH = BN / 32;
    const uint32_t tempty_leader = PAIR ? mapa_smem(&tempty[0], 0) : 0;
    // release the accumulator buffer: to the leader's barrier in pair mode
    auto release_acc = [&](uint32_t as) {
      if (PAIR)
        mbar_arrive_remote(tempty_leader + as * 8);
      else
        mbar_arrive(&tempty[as]);
    };
    // one global input per chunk at most (C, or the GELU' / softmax-backward aux),
    // brought into the chunk's staging slot by TMA in the same swizzled layout the
    // stores use (fp32 C -> main tile, bf16 aux / C -> side tile); with two slots
    // the next chunk's tile is requested before this chunk is processed, and the
    // next tile's first chunk before that tile's accumulator is waited for
    const int in_kind =
        G ? ((p.C && !p.reduce_add) ? 1 : ((p.act == SG_ACT_DGELU || p.mode == SG_EPI_SOFTMAX_BWD) ? 2 : 0))
          : ((KIND == EK_CIN_BIAS || KIND == EK_LN) ? 1 : (KIND == EK_DGELU ? 2 : 0));
    const bool c_side = in_kind == 1 && !c_f32;  // bf16 C: side tile
    // slot = main tile (fp32: 4 KB, bf16: 2 KB) [+ 2 KB bf16 side tile]; two 4 KB slots when it fits
    const bool side = f_aux_out || f_d2 || in_kind == 2 || c_side;
    const int main_bytes = (d_f32 || (in_kind == 1 && c_f32)) ? 4096 : 2048;
    const bool dual = main_bytes + (side ? 2048 : 0) <= 4096;
    auto issue_in = [&](int tncol, int trow0, int tz1, int tz2, int c, uint32_t si) {  // lane 0 only
      uint8_t* base = stg_w + (dual ? si * 4096 : 0);
      uint64_t* bar = &inbar[e * 2 + si];
      const int col0 = tncol + c * 32;
      if (in_kind == 1 && c_f32) {
        mbar_arrive_expect_tx(bar, 4096);
        load_box(&tmC, base, bar, col0, trow0, tz2, tz1, p.c_b2_first);
      } else if (in_kind == 1) {
        mbar_arrive_expect_tx(bar, 2048);
        load_box(&tmC, base + main_bytes, bar, col0, trow0, tz2, tz1, p.c_b2_first);
      } else {
        mbar_arrive_expect_tx(bar, 2048);
        load_box(&tmX, base + main_bytes, bar, col0, trow0, tz2, tz1, p.x_b2_first);
      }
    };
    bool pref_next = false;  // the next tile's first chunk input is in flight
    for (int u = u0; u < ucount; u += ustep, ++it) {
      const int t = tile_of(u);
      int mb, nb, z1, z2, half;
      decode_unit(p, t, mb, nb, z1, z2, half);
      const int ncol = half < 0 ? nb * BN : nb * BN + half * (BN / 2);  // first column of the unit
      const int nch = half < 0 ? NCH : NCH / 2;                          // 32-column chunks of the unit
      const uint32_t as = it % ACC, aph = (it / ACC) & 1;
      const int row0 = mb * TM + (int)rank * kBM + q * 32;
      const int nrows = min(32, p.M - row0);
      float rv = 0.f;
      if (G && p.rowvec && lane < nrows) rv = p.rowvec[(size_t)z1 * p.srv1 + (size_t)z2 * p.srv2 + row0 + lane];
      float ln_mu = 0.f, ln_rs = 0.f, ln_sxg = 0.f, ln_sg = 0.f;
      if (f_ln && lane < nrows) {
        ln_mu = p.ln_mean[row0 + lane];
        ln_rs = p.ln_rstd[row0 + lane];
      }
      mbar_wait_sleep(&tfull[as], aph);  // sleeping: a spinning epilogue warp steals issue slots from the producer / MMA warps
      tc_fence_after();
      const uint32_t tacc = tmem_base + lane_base + as * BN;

      if (EW == 4 && f_mode == SG_EPI_SOFTMAX) {
        // whole row in TMEM: max, sum of exponentials, then P chunks through smem + TMA
        const float sl2 = p.alpha * 1.4426950408889634f;
        float m = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          uint32_t r[32];
          tmem_ld32(tacc + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j < p.N) m = fmaxf(m, __uint_as_float(r[j]));
        }
        const float ms = m * sl2;
        float z = 0.f;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          uint32_t r[32];
          tmem_ld32(tacc + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j < p.N) z += ex2_fast(fmaf(__uint_as_float(r[j]), sl2, -ms));
        }
        const float inv = 1.f / z;
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          uint32_t r[32];
          tmem_ld32(tacc + c * 32, r);
          tmem_wait_ld();
          if (c == NCH - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(as);
          }
          const int row = row0 + lane;
          if (c * 32 >= p.N || row >= p.M) continue;
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = ex2_fast(fmaf(__uint_as_float(r[j]), sl2, -ms)) * inv;
          store_bf16_row(static_cast<__nv_bfloat16*>(p.D) + (size_t)z1 * p.sd1 + (size_t)z2 * p.sd2 +
                             (size_t)row * p.ldd + c * 32,
                         p.vec_d, min(32, p.N - c * 32), v);
        }
        continue;
      }

      bool pref = pref_next;  // the current chunk's input is already in flight
      pref_next = false;
      // bias (or the LayerNorm gamma): lane j holds column j of the chunk (one
      // coalesced load, prefetched a chunk ahead), broadcast to the row threads via smem
      const float* vecp = f_bias ? p.bias : (f_ln ? p.ln_gamma : nullptr);
      auto load_bias = [&](int c) -> float {
        const int col = ncol + c * 32 + lane;
        return (vecp && c < nch && col < p.N) ? __ldg(vecp + col) : 0.f;
      };
      float bias_cur = load_bias(c_first), bias_nxt = 0.f;
#pragma unroll 1
      for (int c = c_first; c < nch; c += CSTEP) {
        const int col0 = ncol + c * 32;
        const bool active = col0 < p.N && nrows > 0;  // warp-uniform
        if (vecp) bias_nxt = load_bias(c + CSTEP);
        // accumulator chunk, thread = row
        uint32_t r[32];
        tmem_ld32(tacc + c * 32, r);
        tmem_wait_ld();
        if (c + CSTEP >= nch) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc(as);
        }
        if (active) {
          const uint32_t si = dual ? slot : 0;
          uint8_t* s0 = stg_w + si * 4096;                             // main tile: D, fp32 C input
          uint8_t* s1 = s0 + main_bytes;                               // bf16 side tile (SW64)
          if (dual) slot ^= 1;
          if (lane == 0) {
            if (in_kind && !pref) {  // not prefetched (first chunk of the tile / one slot)
              bulk_wait_read<0>();
              issue_in(ncol, row0, z1, z2, c, si);
            }
            const int cn = c + CSTEP;
            if (in_kind && dual && cn < nch && ncol + cn * 32 < p.N) {
              bulk_wait_read<0>();  // the other slot's last store has read it
              issue_in(ncol, row0, z1, z2, cn, si ^ 1);
            } else if (dual) {
              bulk_wait_read<1>();  // this slot's previous TMA stores have read it
            } else {
              bulk_wait_read<0>();
            }
          }
          pref = in_kind && dual && c + CSTEP < nch && ncol + (c + CSTEP) * 32 < p.N;
          __syncwarp();
          if (in_kind) {
            mbar_wait(&inbar[e * 2 + si], (inph >> si) & 1);
            inph ^= 1u << si;
          }
          float v[32];
          if (p.alpha != 1.f) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * p.alpha;
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          }
          if (EW == 4 && f_mode == SG_EPI_SOFTMAX_BWD) {
            float pv[32];
            ld_row_bf16(s1, lane, pv);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = pv[j] * (v[j] - rv * p.alpha);
            const int row = row0 + lane;
            if (row < p.M)
              store_bf16_row(static_cast<__nv_bfloat16*>(p.D) + (size_t)z1 * p.sd1 + (size_t)z2 * p.sd2 +
                                 (size_t)row * p.ldd + col0,
                             p.vec_d, min(32, p.N - col0), v);
          } else {
            if (f_bias) {
              // lane j's coalesced bias value -> the warp's 128-byte slot -> every row thread
              float* bw = bias_all + e * 32;
              bw[lane] = bias_cur;
              __syncwarp();
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float4 b4 = reinterpret_cast<const float4*>(bw)[k];
                const uint64_t lo = fadd2(f2_pack(v[4 * k], v[4 * k + 1]), f2_pack(b4.x, b4.y));
                const uint64_t hi = fadd2(f2_pack(v[4 * k + 2], v[4 * k + 3]), f2_pack(b4.z, b4.w));
                v[4 * k] = f2_lo(lo); v[4 * k + 1] = f2_hi(lo); v[4 * k + 2] = f2_lo(hi); v[4 * k + 3] = f2_hi(hi);
              }
              __syncwarp();
            }
            if (f_ln) {
              // C holds the LayerNorm input x (fp32, main tile); g = dy gamma
              float xv[32];
              ld_row_f32(s0, lane, xv);
              float* bw = bias_all + e * 32;
              bw[lane] = bias_cur;
              __syncwarp();
              uint64_t a_sxg = 0, a_sg = 0;  // two f32x2 partial sums each
              const uint64_t nmu = f2_pack(-ln_mu, -ln_mu);
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                const float2 g2 = reinterpret_cast<const float2*>(bw)[k];
                const uint64_t g = fmul2(f2_pack(v[2 * k], v[2 * k + 1]), f2_pack(g2.x, g2.y));
                const uint64_t xc = fadd2(f2_pack(xv[2 * k], xv[2 * k + 1]), nmu);
                a_sxg = ffma2(xc, g, a_sxg);
                a_sg = fadd2(a_sg, g);
              }
              __syncwarp();
              ln_sxg += (f2_lo(a_sxg) + f2_hi(a_sxg)) * ln_rs;
              ln_sg += f2_lo(a_sg) + f2_hi(a_sg);
            } else if (in_kind == 1) {
              float cv[32];
              if (c_f32)
                ld_row_f32(s0, lane, cv);
              else
                ld_row_bf16(s1, lane, cv);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += cv[j];
            }
            if (f_act == SG_ACT_GELU) {
              if (f_aux_out) st_row_bf16(s1, lane, v);
              gelu_row(v);
            } else if (f_act == SG_ACT_DGELU) {
              float xv[32];
              ld_row_bf16(s1, lane, xv);
              dgelu_row(v, xv);
            }
            __syncwarp();  // every lane has consumed the staged inputs before D overwrites them
            if (d_f32)
              st_row_f32(s0, lane, v);
            else
              st_row_bf16(s0, lane, v);
            if (f_d2) st_row_bf16(s1, lane, v);
            __syncwarp();
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (f_reduce)
                reduce_box(&tmD, s0, col0, row0, z2, z1, p.o_b2_first);
              else
                store_box(&tmD, s0, col0, row0, z2, z1, p.o_b2_first);
              if (f_aux_out) store_box(&tmX, s1, col0, row0, z2, z1, p.o_b2_first);
              if (f_d2) store_box(&tmD2, s1, col0, row0, z2, z1, p.o_b2_first);
              bulk_commit();
            }
            if (f_colsum) {
              // column sums by a register butterfly (reduce-scatter over the 32 row lanes:
              // five xor-shuffle rounds halve the columns each lane carries, lane j ends
              // with column j), of the fp32 values, rows past M masked; one coalesced
              // 128-byte reduction per chunk
              const bool full_rows = nrows == 32;
              float w16[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float a = full_rows || lane < nrows ? v[j] : 0.f;
                const float b = full_rows || lane < nrows ? v[j + 16] : 0.f;
                const bool hi = lane & 16;
                w16[j] = (hi ? b : a) + __shfl_xor_sync(0xffffffffu, hi ? a : b, 16);
              }
              float w8[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const bool hi = lane & 8;
                w8[j] = (hi ? w16[j + 8] : w16[j]) + __shfl_xor_sync(0xffffffffu, hi ? w16[j] : w16[j + 8], 8);
              }
              float w4[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const bool hi = lane & 4;
                w4[j] = (hi ? w8[j + 4] : w8[j]) + __shfl_xor_sync(0xffffffffu, hi ? w8[j] : w8[j + 4], 4);
              }
              float w2[2];
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const bool hi = lane & 2;
                w2[j] = (hi ? w4[j + 2] : w4[j]) + __shfl_xor_sync(0xffffffffu, hi ? w4[j] : w4[j + 2], 2);
              }
              const bool hi = lane & 1;
              const float cs = (hi ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, hi ? w2[0] : w2[1], 1);
              if (col0 + lane < p.N) atomicAdd(p.colsum + (size_t)z1 * p.scs1 + (size_t)z2 * p.scs2 + col0 + lane, cs);
            }
          }
        }
        bias_cur = bias_nxt;
      }
      if (in_kind && dual && u + ustep < ucount) {
        int mb2, nb2, y1, y2, half2;
        decode_unit(p, tile_of(u + ustep), mb2, nb2, y1, y2, half2);
        const int ncol2 = half2 < 0 ? nb2 * BN : nb2 * BN + half2 * (BN / 2);
        const int row0n = mb2 * TM + (int)rank * kBM + q * 32;
        if (ncol2 + c_first * 32 < p.N && row0n < p.M) {
          if (lane == 0) {
            bulk_wait_read<0>();
            issue_in(ncol2, row0n, y1, y2, c_first, slot);
          }
          pref_next = true;
        }
      }
      if (f_ln && lane < nrows) {
        atomicAdd(p.ln_stats + 2 * (size_t)(row0 + lane), ln_sxg);
        atomicAdd(p.ln_stats + 2 * (size_t)(row0 + lane) + 1, ln_sg);
      }
    }
    if (lane == 0) bulk_wait_all();  // global writes complete before the CTA retires
  }

  tc_fence_before();
  if (PAIR) {
    cluster_sync_all();
    if (warp == 2) tmem_dealloc_pair<Cfg::TMEM_COLS>(tmem_base);
  } else {
    __syncthreads();
    if (warp == 2) tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------ SIMT path
// CUDA-core fallback for operands or outputs the TMA unit cannot address (row
// pitches or batch strides that are not 16-byte multiples, e.g. head_dim 4 in
// the reference's unit-test configurations). NORMAL-mode semantics.
__global__ void gemm_simt_kernel(const __grid_constant__ sg_gemm_args a) {
  pdl_begin();
  const long long total = a.nb1 * a.nb2 * a.M * a.N;
  const __nv_bfloat16* A = static_cast<const __nv_bfloat16*>(a.A);
  const __nv_bfloat16* B = static_cast<const __nv_bfloat16*>(a.B);
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long n = idx % a.N;
    long long t = idx / a.N;
    const long long m = t % a.M;
    t /= a.M;
    const long long z2 = t % a.nb2;
    const long long z1 = t / a.nb2;
    const __nv_bfloat16* pa = A + z1 * a.sa1 + z2 * a.sa2;
    const __nv_bfloat16* pb = B + z1 * a.sb1 + z2 * a.sb2;
    float acc = 0.f;
    for (long long k = 0; k < a.K; ++k) {
      const float av = __bfloat162float(a.a_mn_major ? pa[k * a.lda + m] : pa[m * a.lda + k]);
      const float bv = __bfloat162float(a.b_mn_major ? pb[k * a.ldb + n] : pb[n * a.ldb + k]);
      acc = fmaf(av, bv, acc);
    }
    float v = acc * a.alpha;
    if (a.bias) v += a.bias[n];
    if (a.ln_stats) {
      const float g = v * a.ln_gamma[n];
      const float xh = (static_cast<const float*>(a.C)[m * a.ldc + n] - a.ln_mean[m]) * a.ln_rstd[m];
      atomicAdd(a.ln_stats + 2 * m, xh * g);
      atomicAdd(a.ln_stats + 2 * m + 1, g);
    } else if (a.C) {
      const long long ci = z1 * a.sc1 + z2 * a.sc2 + m * a.ldc + n;
      v += a.c_dtype == SG_DTYPE_F32 ? static_cast<const float*>(a.C)[ci]
                                     : __bfloat162float(static_cast<const __nv_bfloat16*>(a.C)[ci]);
    }
    const long long xi = z1 * a.sx1 + z2 * a.sx2 + m * a.ldx + n;
    if (a.act == SG_ACT_GELU) {
      if (a.aux) static_cast<__nv_bfloat16*>(a.aux)[xi] = __float2bfloat16_rn(v);
      v = gelu_f(v);
    } else if (a.act == SG_ACT_DGELU) {
      v *= gelu_grad_f(__bfloat162float(static_cast<const __nv_bfloat16*>(a.aux)[xi]));
    }
    const long long di = z1 * a.sd1 + z2 * a.sd2 + m * a.ldd + n;
    if (a.d_dtype == SG_DTYPE_F32)
      static_cast<float*>(a.D)[di] = v;
    else
      static_cast<__nv_bfloat16*>(a.D)[di] = __float2bfloat16_rn(v);
    if (a.D2) static_cast<__nv_bfloat16*>(a.D2)[z1 * a.s21 + z2 * a.s22 + m * a.ld2 + n] = __float2bfloat16_rn(v);
    if (a.colsum) atomicAdd(a.colsum + z1 * a.scs1 + z2 * a.scs2 + n, v);
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

// 4-D tensor map over (inner, outer, b2, b1) (b2 moved before outer when its
// stride is the smaller one, e.g. heads inside a row) with a box_inner x
// box_outer box; fails with SG_ERR_SHAPE when TMA cannot address the tensor.
static int make_map(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, int esz, long long inner,
                    long long outer, long long nb2, long long nb1, long long ld, long long s2, long long s1,
                    int box_inner, int box_outer, CUtensorMapSwizzle swz, int* b2_first) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (!enc) return set_error(SG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (nb2 <= 1) s2 = ld * outer;
  if (nb1 <= 1) s1 = s2 * nb2;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * esz) % 16 || (s2 * esz) % 16 || (s1 * esz) % 16)
    return set_error(SG_ERR_SHAPE, "gemm: pointer / leading dims must be 16-byte aligned for TMA");
  const bool b2f = nb2 > 1 && s2 < ld;
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
  dims[0] = inner;
  box[0] = box_inner;
  if (b2f) {
    dims[1] = nb2; dims[2] = outer; dims[3] = nb1;
    strides[0] = s2 * esz; strides[1] = ld * esz; strides[2] = s1 * esz;
    box[1] = 1; box[2] = box_outer; box[3] = 1;
  } else {
    dims[1] = outer; dims[2] = nb2; dims[3] = nb1;
    strides[0] = ld * esz; strides[1] = s2 * esz; strides[2] = s1 * esz;
    box[1] = box_outer; box[2] = 1; box[3] = 1;
  }
  static const CUtensorMapL2promotion promo = [] {  // SG_TMA_L2_PROMOTION=0/64/128/256 (experiments)
    const char* e = getenv("SG_TMA_L2_PROMOTION");
    const int v = e ? atoi(e) : 256;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
           : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  CUresult r = enc(map, dt, 4, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char msg[256];
    snprintf(msg, sizeof msg, "cuTensorMapEncodeTiled failed (%d): dims %lld,%lld,%lld,%lld ld=%lld s2=%lld s1=%lld",
             (int)r, inner, outer, nb2, nb1, ld, s2, s1);
    return set_error(SG_ERR_SHAPE, msg);
  }
  *b2_first = b2f ? 1 : 0;
  return SG_OK;
}

int tmap_bf16_4d(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long nb2, long long nb1,
                 long long ld, long long s2, long long s1, int box_inner, int box_outer, int* b2_first) {
  return make_map(map, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, inner, outer, nb2, nb1, ld, s2, s1, box_inner,
                  box_outer, CU_TENSOR_MAP_SWIZZLE_128B, b2_first);
}

int tmap_f32_tile_4d(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long nb2,
                     long long nb1, long long ld, long long s2, long long s1, int* b2_first) {
  return make_map(map, ptr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, inner, outer, nb2, nb1, ld, s2, s1, 32, 32,
                  CU_TENSOR_MAP_SWIZZLE_128B, b2_first);
}

int tmap_bf16_tile_4d(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long nb2,
                      long long nb1, long long ld, long long s2, long long s1, int* b2_first) {
  return make_map(map, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, inner, outer, nb2, nb1, ld, s2, s1, 32, 32,
                  CU_TENSOR_MAP_SWIZZLE_64B, b2_first);
}

static int operand_map(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long nb2,
                       long long nb1, long long ld, long long s2, long long s1, int box_outer, int* b2_first) {
  return make_map(map, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, inner, outer, nb2, nb1, ld, s2, s1, 64, box_outer,
                  CU_TENSOR_MAP_SWIZZLE_128B, b2_first);
}

// 32 x 32 output tiles: fp32 rows of 128 B (SWIZZLE_128B), bf16 rows of 64 B (SWIZZLE_64B)
static int output_map(CUtensorMap* map, const void* ptr, bool f32, long long N, long long M, long long nb2,
                      long long nb1, long long ld, long long s2, long long s1, int* b2_first) {
  return make_map(map, ptr, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, f32 ? 4 : 2, N,
                  M, nb2, nb1, ld, s2, s1, 32, 32, f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  b2_first);
}

struct Maps {
  CUtensorMap a, b, d, x, d2, c;
};

template <int BN, bool A_MN, bool B_MN, int EW, bool PAIR, int KIND = EK_GENERIC>
static int launch_gemm(const Maps& m, const GemmParams& p, cudaStream_t stream, int grid) {
  using Cfg = GemmCfg<BN, EW, PAIR>;
  auto kern = gemm_kernel<BN, A_MN, B_MN, EW, PAIR, KIND>;
  if (!ensure_smem(reinterpret_cast<const void*>(kern), (int)Cfg::SMEM))
    return set_error(SG_ERR_CUDA, "cudaFuncSetAttribute(max smem) failed");
  if (PAIR) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(EpiCfg<EW>::kThreads);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, m.a, m.b, m.d, m.x, m.d2, m.c, p);
    if (e != cudaSuccess) return set_error(SG_ERR_CUDA, cudaGetErrorString(e));
  } else {
    cudaError_t e = launch_k(kern, dim3(grid), dim3(EpiCfg<EW>::kThreads), Cfg::SMEM, stream, m.a, m.b, m.d, m.x, m.d2,
                             m.c, p);
    if (e != cudaSuccess) return set_error(SG_ERR_CUDA, cudaGetErrorString(e));
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SG_ERR_CUDA, cudaGetErrorString(e));
  return SG_OK;
}

template <int BN, int EW, bool PAIR = false>
static int dispatch_major(bool amn, bool bmn, const Maps& m, const GemmParams& p, cudaStream_t s, int grid,
                          int kind = EK_GENERIC) {
  // specialised epilogues for the operand layouts the step uses them with:
  // forward products (K-major A, MN-major B), dX products (both K-major),
  // weight gradients (both MN-major)
  if (PAIR && kind != EK_GENERIC) {
    if (!amn && bmn) {
      switch (kind) {
        case EK_STORE: return launch_gemm<BN, false, true, EW, PAIR, EK_STORE>(m, p, s, grid);
        case EK_BIAS: return launch_gemm<BN, false, true, EW, PAIR, EK_BIAS>(m, p, s, grid);
        case EK_CIN_BIAS: return launch_gemm<BN, false, true, EW, PAIR, EK_CIN_BIAS>(m, p, s, grid);
        case EK_GELU_BIAS: return launch_gemm<BN, false, true, EW, PAIR, EK_GELU_BIAS>(m, p, s, grid);
        default: break;
      }
    } else if (!amn && !bmn) {
      switch (kind) {
        case EK_STORE: return launch_gemm<BN, false, false, EW, PAIR, EK_STORE>(m, p, s, grid);
        case EK_DGELU: return launch_gemm<BN, false, false, EW, PAIR, EK_DGELU>(m, p, s, grid);
        case EK_LN: return launch_gemm<BN, false, false, EW, PAIR, EK_LN>(m, p, s, grid);
        default: break;
      }
    } else if (amn && bmn && kind == EK_STORE) {
      return launch_gemm<BN, true, true, EW, PAIR, EK_STORE>(m, p, s, grid);
    }
  }
  if (!amn && !bmn) return launch_gemm<BN, false, false, EW, PAIR>(m, p, s, grid);
  if (!amn && bmn) return launch_gemm<BN, false, true, EW, PAIR>(m, p, s, grid);
  if (amn && !bmn) return launch_gemm<BN, true, false, EW, PAIR>(m, p, s, grid);
  return launch_gemm<BN, true, true, EW, PAIR>(m, p, s, grid);
}

static double wave_eff(long long units, int sms) {
  const long long waves = (units + sms - 1) / sms;
  return (double)units / (double)(waves * sms);
}

static int pick_bn(long long M, long long N, long long batch, int sms, int mode, int tm = kBM) {
  if (mode != SG_EPI_NORMAL) {  // the whole row in one tile
    for (int bn : {64, 128, 256, 512})
      if (N <= bn) return bn;
    return -1;
  }
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  // 128 x 256 tiles read 96 B/clk of operands from smem per SM, 128 x 128 tiles
  // 128 B/clk (the smem limit): take the wide tile unless its last wave is much
  // emptier (measured: 256 wins by ~17% at equal wave counts).
  const long long mt = (M + tm - 1) / tm;
  auto eff = [&](int bn) {
    const long long nt = (N + bn - 1) / bn;
    return (double)N / (double)(nt * bn) * wave_eff(mt * nt * batch, sms);
  };
  // under one wave even at 128: the product is split along K, where the wide tile
  // wins (measured: h x h weight gradient 35 us at 256 vs 46 us at 128)
  if (mt * ((N + 127) / 128) * batch < sms) return 256;
  return eff(128) > eff(256) * 1.15 ? 128 : 256;
}

// Split-K factor for tile-starved products (e.g. the weight gradients, M x N =
// h x h with K = b*s tokens, under 3/4 of a wave): the split count minimising
// waves x (k-blocks per unit x t_kb + t_epi), each split keeping >= 8 k-blocks. The
// per-unit epilogue (a 256 x 256 fp32 reduce-add, ~4 us) is what makes many short
// units lose to fewer long ones (measured h x h, K = 16k: 4 splits 33 us vs 9 splits 36 us).
static int pick_splits(long long tiles, int k_blocks, int sms) {
  if (4 * tiles >= 3LL * sms) return 1;  // (measured: splitting a ~0.9-wave product loses to the reduce traffic)
  constexpr double t_kb = 1.0, t_epi = 14.0;  // in units of one 256 x 256 x 64 pair MMA step (512 clocks)
  int best = 1;
  double best_cost = (double)((tiles + sms - 1) / sms) * (k_blocks * t_kb + t_epi);
  for (int s = 2; s <= 16 && k_blocks / s >= 8; ++s) {
    const int per = (k_blocks + s - 1) / s;
    const int real = (k_blocks + per - 1) / per;
    const double cost = (double)((tiles * real + sms - 1) / sms) * (per * t_kb + t_epi);
    if (cost < best_cost * 0.98) {
      best = real;
      best_cost = cost;
    }
  }
  return best;
}

// ------------------------------------------------------------------ die table
// Which die each CTA pair of a full-grid pair launch lands on: the pairs are placed
// deterministically on an idle GPU (cluster c on SMs 2c + const, one CTA per SM); the
// probe (same one-CTA-per-SM footprint) records the SM of every cluster once per
// device, die = SM id >= SMs / 2. The table only has to be a bijection onto the two
// dies' pair slots for correctness (each die-local unit then has exactly one owner);
// when the hardware places a launch differently only the L2 locality is lost.
__global__ void __cluster_dims__(2, 1, 1) die_probe_kernel(int* out) {
  extern __shared__ uint8_t probe_smem[];
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = (int)smid;
  if (threadIdx.x == 1) probe_smem[0] = 0;
}

struct DieTable {
  bool ok = false;
  int pairs = 0;
  uint8_t die_of[128], slot_of[128];
};

static const DieTable* die_table(int sms, cudaStream_t stream) {
  static std::mutex mu;
  static DieTable tabs[64];
  static bool done[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return &tabs[dev];
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  DieTable& t = tabs[dev];
  done[dev] = true;
  const int pairs = sms / 2;
  if (sms % 4 != 0 || pairs > 128) return &t;
  int* d = nullptr;
  if (cudaMalloc(&d, sms * sizeof(int)) != cudaSuccess) return &t;
  const int smem = 200 * 1024;  // one CTA per SM, as the pair GEMMs
  int host[256];
  bool ran = cudaFuncSetAttribute(die_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  if (ran) {
    die_probe_kernel<<<sms, 32, smem, stream>>>(d);
    ran = cudaStreamSynchronize(stream) == cudaSuccess &&
          cudaMemcpy(host, d, sms * sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  cudaFree(d);
  if (!ran) {
    cudaGetLastError();
    return &t;
  }
  int count[2] = {0, 0};
  for (int c = 0; c < pairs; ++c) {
    const int die = host[2 * c] >= sms / 2 ? 1 : 0;
    if (host[2 * c + 1] / (sms / 2) != die) return &t;  // a pair across the die boundary: no table
    t.die_of[c] = (uint8_t)die;
    t.slot_of[c] = (uint8_t)count[die]++;
  }
  if (count[0] != pairs / 2 || count[1] != pairs / 2) return &t;
  t.pairs = pairs;
  t.ok = true;
  return &t;
}

static int launch_simt(const sg_gemm_args* a, int sms, void* stream) {
  if (a->mode != SG_EPI_NORMAL) return set_error(SG_ERR_SHAPE, "gemm: softmax epilogues need TMA-aligned operands");
  const long long total = a->nb1 * a->nb2 * a->M * a->N;
  const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)sms * 16);
  launch_k(gemm_simt_kernel, dim3(blocks), dim3(256), 0, static_cast<cudaStream_t>(stream), *a);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
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
  if (a->D2 && a->act != SG_ACT_NONE) return set_error(SG_ERR_CONFIG, "gemm: D2 copy with GELU / GELU' epilogue");
  if (a->C && a->act == SG_ACT_DGELU) return set_error(SG_ERR_CONFIG, "gemm: C input together with GELU' input");
  if (a->C && a->C != a->D && a->c_dtype != SG_DTYPE_F32 && (a->D2 || (a->act == SG_ACT_GELU && a->aux)))
    return set_error(SG_ERR_CONFIG, "gemm: a bf16 C input shares the side tile with D2 / the GELU input copy");
  if (a->ln_stats && (!a->ln_gamma || !a->ln_mean || !a->ln_rstd || !a->C || a->C == a->D ||
                      a->c_dtype != SG_DTYPE_F32 || a->d_dtype != SG_DTYPE_F32 || a->bias || a->act ||
                      a->D2 || a->colsum || a->mode != SG_EPI_NORMAL || a->nb1 * a->nb2 != 1))
    return set_error(SG_ERR_CONFIG, "gemm: LayerNorm statistics need an unbatched fp32 product with x as C only");
  if (a->mode != SG_EPI_NORMAL) {
    if (a->mode != SG_EPI_SOFTMAX && a->mode != SG_EPI_SOFTMAX_BWD) return set_error(SG_ERR_CONFIG, "gemm: mode");
    if (a->N > 512) return set_error(SG_ERR_SHAPE, "gemm: softmax epilogues need N <= 512");
    if (a->d_dtype != SG_DTYPE_BF16 || a->C || a->bias || a->act || a->D2 || a->colsum)
      return set_error(SG_ERR_CONFIG, "gemm: softmax epilogues write bf16 D only");
    if (a->mode == SG_EPI_SOFTMAX_BWD && (!a->aux || !a->rowvec))
      return set_error(SG_ERR_CONFIG, "gemm: softmax bwd needs P (aux) and D_i (rowvec)");
    if (a->mode == SG_EPI_SOFTMAX && a->alpha <= 0.f) return set_error(SG_ERR_CONFIG, "gemm: softmax alpha > 0");
  }
  const int sms = sg_gemm_sm_budget();  // every SM unless a dist mesh reserves some for NCCL
  if (sms <= 0) return set_error(SG_ERR_CUDA, "no CUDA device");

  GemmParams p{};
  p.M = (int)a->M;
  p.N = (int)a->N;
  p.K = (int)a->K;
  p.nb2 = (int)a->nb2;
  p.mode = a->mode;
  const long long batch = a->nb1 * a->nb2;
  // 2-CTA pair tiles (256 x 128 / 256 x 256) for every plain product with more
  // than one 128-row block; single-CTA tiles for the row-softmax modes, narrow
  // N and M <= 128. SG_GEMM_PAIR=0 / SG_GEMM_BN=n override (experiments).
  static const int env_pair = [] {
    const char* e = getenv("SG_GEMM_PAIR");
    return e ? atoi(e) : 1;
  }();
  static const int force_bn = [] {
    const char* e = getenv("SG_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  const bool pair = env_pair != 0 && a->mode == SG_EPI_NORMAL && a->M > kBM && a->N > 64;
  const int units = pair ? sms / 2 : sms;  // concurrent tile workers (CTA pairs or CTAs)
  const int tm = pair ? 2 * kBM : kBM;
  int bn = pick_bn(a->M, a->N, batch, units, a->mode, tm);
  if (force_bn && a->mode == SG_EPI_NORMAL && a->N > 128 && (!pair || force_bn == 128 || force_bn == 256))
    bn = force_bn;
  p.m_tiles = (int)((a->M + tm - 1) / tm);
  p.n_tiles = (int)((a->N + bn - 1) / bn);
  p.k_blocks = (int)((a->K + kBK - 1) / kBK);
  long long tiles = (long long)p.m_tiles * p.n_tiles * batch;
  if (tiles > INT32_MAX / 16) return set_error(SG_ERR_SHAPE, "gemm: too many tiles");
  // split-K: only for plain fp32 products whose partials can be TMA-reduce-added
  // (D zeroed first, or D == C accumulated in place); SG_DETERMINISTIC=1 disables it
  static const bool deterministic = [] {
    const char* e = getenv("SG_DETERMINISTIC");
    return e && atoi(e) != 0;
  }();
  const bool in_place = a->C == a->D && a->c_dtype == SG_DTYPE_F32 && a->ldc == a->ldd;
  const bool split_ok = !deterministic && a->mode == SG_EPI_NORMAL && a->d_dtype == SG_DTYPE_F32 && !a->bias &&
                        a->act == SG_ACT_NONE && !a->D2 && !a->colsum && batch == 1 && (a->C == nullptr || in_place);
  static const int env_splits = [] {  // SG_GEMM_SPLITS=n forces n splits where allowed (experiments)
    const char* e = getenv("SG_GEMM_SPLITS");
    return e ? atoi(e) : 0;
  }();
  p.k_splits = split_ok ? (env_splits > 0 ? env_splits : pick_splits(tiles, p.k_blocks, units)) : 1;
  p.kb_per_split = (p.k_blocks + p.k_splits - 1) / p.k_splits;
  p.k_splits = (p.k_blocks + p.kb_per_split - 1) / p.kb_per_split;
  tiles *= p.k_splits;
  p.num_tiles = (int)tiles;
  p.full_units = p.num_tiles;
  p.fd_tiles.set((uint32_t)(tiles / p.k_splits));
  // last partial round as half-width units (pair tiles 256 x 256 only, no split-K):
  // when at most half the pairs would work in it, twice as many 256 x 128 units finish
  // it in about 0.7 of a tile time. SG_GEMM_HALF_TAIL=0 disables (experiments).
  static const int env_half_tail = [] {
    const char* e = getenv("SG_GEMM_HALF_TAIL");
    return e ? atoi(e) : 1;
  }();
  static const int env_group = [] {  // SG_GEMM_GROUP_M=g (power of two) overrides the group height (experiments)
    const char* e = getenv("SG_GEMM_GROUP_M");
    return e ? atoi(e) : 0;
  }();
  p.group_m = env_group > 0 ? env_group : kGroupM;
  p.group_shift = 0;
  while ((1 << p.group_shift) < p.group_m) ++p.group_shift;
  p.group_m = 1 << p.group_shift;
  // die-local tile streams for large, full-grid pair products (SG_GEMM_DIE=0 disables):
  // on two-die parts the A rows a group shares are then read by one die's pairs (the
  // die-local streams replace the half-width last round)
  p.die_mode = 0;
  static const int env_die = [] {
    const char* e = getenv("SG_GEMM_DIE");
    return e ? atoi(e) : 1;
  }();
  if (env_die && pair && bn == 256 && batch == 1 && p.k_splits == 1 && units * 2 == sms && p.group_m >= 2 &&
      p.m_tiles % p.group_m == 0 && tiles >= 4 * units && (double)a->M * (double)a->N * (double)a->K >= 4.0e11) {
    const DieTable* dt = die_table(sms, static_cast<cudaStream_t>(stream));
    if (dt && dt->ok && dt->pairs == units) {
      p.die_mode = 1;
      p.die_pairs = units / 2;
      memcpy(p.die_of, dt->die_of, sizeof p.die_of);
      memcpy(p.slot_of, dt->slot_of, sizeof p.slot_of);
    }
  }
  if (env_half_tail && pair && bn == 256 && p.k_splits == 1 && !p.die_mode) {
    const long long tail = tiles % units;
    if (tiles >= units && tail > 0 && 2 * tail <= units) {
      p.full_units = (int)(tiles - tail);
      p.num_tiles = (int)(tiles + tail);
    }
  }
  p.fd_per.set((uint32_t)(p.m_tiles * p.n_tiles));
  p.fd_span.set((uint32_t)(p.group_m * p.n_tiles));
  p.fd_nb2.set((uint32_t)p.nb2);
  p.d_f32 = a->d_dtype == SG_DTYPE_F32;
  p.D = a->D; p.ldd = a->ldd; p.sd1 = a->sd1; p.sd2 = a->sd2;
  p.vec_d = (reinterpret_cast<uintptr_t>(a->D) % 16) == 0 && (a->ldd * 2) % 16 == 0 && (a->sd1 * 2) % 16 == 0 &&
            (a->sd2 * 2) % 16 == 0;
  p.C = a->C; p.ldc = a->ldc; p.sc1 = a->sc1; p.sc2 = a->sc2; p.c_f32 = a->c_dtype == SG_DTYPE_F32;
  // D += A B in place: no epilogue loads, the TMA unit adds the tile in L2 (plain
  // stores would need C; colsum / activations need the full sum, so they disable it)
  p.reduce_add = (a->C == a->D && a->c_dtype == SG_DTYPE_F32 && a->d_dtype == SG_DTYPE_F32 && a->ldc == a->ldd &&
                  (a->nb1 <= 1 || a->sc1 == a->sd1) && (a->nb2 <= 1 || a->sc2 == a->sd2) && !a->colsum &&
                  a->act == SG_ACT_NONE && !a->D2 && a->mode == SG_EPI_NORMAL)
                     ? 1
                     : 0;
  if (p.k_splits > 1) {
    p.reduce_add = 1;
    if (a->C == nullptr &&
        cudaMemset2DAsync(a->D, (size_t)a->ldd * 4, 0, (size_t)a->N * 4, (size_t)a->M,
                          static_cast<cudaStream_t>(stream)) != cudaSuccess)
      return set_error(SG_ERR_CUDA, "gemm: split-K zero fill failed");
  }
  p.bias = a->bias;
  p.aux_in = (a->act == SG_ACT_DGELU || a->mode == SG_EPI_SOFTMAX_BWD) ? static_cast<const __nv_bfloat16*>(a->aux)
                                                                      : nullptr;
  p.ldx = a->ldx; p.sx1 = a->sx1; p.sx2 = a->sx2;
  p.aux_out = (a->act == SG_ACT_GELU && a->aux) ? 1 : 0;
  p.has_d2 = a->D2 ? 1 : 0;
  p.colsum = a->colsum; p.scs1 = a->scs1; p.scs2 = a->scs2;
  p.rowvec = a->rowvec; p.srv1 = a->srv1; p.srv2 = a->srv2;
  p.ln_gamma = a->ln_gamma; p.ln_mean = a->ln_mean; p.ln_rstd = a->ln_rstd; p.ln_stats = a->ln_stats;
  p.act = a->act;
  p.alpha = a->alpha;

  // Everything the tensor-core path touches through TMA must be 16-byte
  // addressable; otherwise (tiny / odd-shaped tensors only) run on CUDA cores.
  Maps m;
  memset(&m, 0, sizeof m);
  int rc, tmp = 0;
  if (!a->a_mn_major)
    rc = operand_map(&m.a, a->A, a->K, a->M, a->nb2, a->nb1, a->lda, a->sa2, a->sa1, kBM, &p.a_b2_first);
  else
    rc = operand_map(&m.a, a->A, a->M, a->K, a->nb2, a->nb1, a->lda, a->sa2, a->sa1, kBK, &p.a_b2_first);
  const int b_box = pair ? bn / 2 : std::min(bn, 256);
  if (rc == SG_OK) {
    if (!a->b_mn_major)
      rc = operand_map(&m.b, a->B, a->K, a->N, a->nb2, a->nb1, a->ldb, a->sb2, a->sb1, b_box, &p.b_b2_first);
    else
      rc = operand_map(&m.b, a->B, a->N, a->K, a->nb2, a->nb1, a->ldb, a->sb2, a->sb1, kBK, &p.b_b2_first);
  }
  if (rc == SG_OK)
    rc = output_map(&m.d, a->D, p.d_f32, a->N, a->M, a->nb2, a->nb1, a->ldd, a->sd2, a->sd1, &p.o_b2_first);
  if (rc == SG_OK && p.aux_out)
    rc = output_map(&m.x, a->aux, false, a->N, a->M, a->nb2, a->nb1, a->ldx, a->sx2, a->sx1, &p.x_b2_first);
  if (rc == SG_OK && !p.aux_out && p.aux_in)  // GELU' / softmax-backward input tile
    rc = output_map(&m.x, a->aux, false, a->N, a->M, a->nb2, a->nb1, a->ldx, a->sx2, a->sx1, &p.x_b2_first);
  if (rc == SG_OK && a->C && !p.reduce_add)
    rc = output_map(&m.c, a->C, a->c_dtype == SG_DTYPE_F32, a->N, a->M, a->nb2, a->nb1, a->ldc, a->sc2, a->sc1,
                    &p.c_b2_first);
  if (rc == SG_OK && p.has_d2)
    rc = output_map(&m.d2, a->D2, false, a->N, a->M, a->nb2, a->nb1, a->ld2, a->s22, a->s21, &tmp);
  if (rc != SG_OK) {
    if (rc != SG_ERR_SHAPE) return rc;
    clear_error();
    return launch_simt(a, sms, stream);
  }
  if (!p.aux_out && !p.aux_in) m.x = m.d;  // unused maps still need a valid encoding
  if (!(a->C && !p.reduce_add)) m.c = m.d;
  if (!p.has_d2) m.d2 = m.d;

  const int grid = (int)std::min<long long>(p.num_tiles, units) * (pair ? 2 : 1);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // die-local tile streams for large, full-grid pair products (SG_GEMM_DIE=0 disables):
  // on two-die parts the A rows a 16-m-tile group shares are then read by one die's pairs
  const bool amn = a->a_mn_major != 0, bmn = a->b_mn_major != 0;
  // 8 epilogue warps unless the epilogue needs whole rows (softmax modes)
  static const int force_ew = [] {
    const char* e = getenv("SG_GEMM_EPI_WARPS");
    return e ? atoi(e) : 0;
  }();
  // (measured: at K > ~1.5k the mainloop hides a 4-warp epilogue and the 8-warp
  // variant's shallower smem ring (3 stages at BN = 256) costs ~10%)
  const bool ew8 = force_ew != 4 && a->mode == SG_EPI_NORMAL && (bn == 128 || bn == 256) &&
                   (force_ew == 8 || p.kb_per_split <= 24);
  // compile-time epilogue kind for the step's feature combinations (else generic)
  static const bool generic_only = [] {
    const char* e = getenv("SG_GEMM_GENERIC_EPI");
    return e && atoi(e) != 0;
  }();
  int kind = EK_GENERIC;
  const bool c_in = a->C && !p.reduce_add;
  if (!generic_only && a->mode == SG_EPI_NORMAL && !a->D2) {
    if (a->ln_stats)
      kind = EK_LN;
    else if (a->act == SG_ACT_DGELU && !a->bias && !c_in)
      kind = EK_DGELU;
    else if (a->act == SG_ACT_GELU && a->aux && a->bias && !c_in && !a->colsum)
      kind = EK_GELU_BIAS;
    else if (a->act == SG_ACT_NONE && c_in && p.c_f32 && p.d_f32 && a->bias && !a->colsum && a->alpha == 1.f)
      kind = EK_CIN_BIAS;
    else if (a->act == SG_ACT_NONE && !c_in && !a->colsum)
      kind = a->bias ? EK_BIAS : EK_STORE;
  }
  // GELU' + column sums is the one epilogue-bound product at the step's shapes: 12
  // epilogue warps (3 per TMEM lane quadrant) for it; SG_GEMM_EW12=0 disables
  static const int env_ew12 = [] {
    const char* e = getenv("SG_GEMM_EW12");
    return e ? atoi(e) : 1;
  }();
  if (pair && bn == 256 && kind == EK_DGELU && !amn && !bmn && env_ew12 && force_ew != 4 && force_ew != 8)
    return launch_gemm<256, false, false, 12, true, EK_DGELU>(m, p, s, grid);
  if (pair) {
    if (bn == 128)
      return ew8 ? dispatch_major<128, 8, true>(amn, bmn, m, p, s, grid, kind)
                 : dispatch_major<128, 4, true>(amn, bmn, m, p, s, grid, kind);
    return ew8 ? dispatch_major<256, 8, true>(amn, bmn, m, p, s, grid, kind)
               : dispatch_major<256, 4, true>(amn, bmn, m, p, s, grid, kind);
  }
  switch (bn) {
    case 64: return dispatch_major<64, 4>(amn, bmn, m, p, s, grid);
    case 128:
      return ew8 ? dispatch_major<128, 8>(amn, bmn, m, p, s, grid) : dispatch_major<128, 4>(amn, bmn, m, p, s, grid);
    case 256:
      return ew8 ? dispatch_major<256, 8>(amn, bmn, m, p, s, grid) : dispatch_major<256, 4>(amn, bmn, m, p, s, grid);
    default: return dispatch_major<512, 4>(amn, bmn, m, p, s, grid);
  }
}
