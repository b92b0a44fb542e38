// Flash-style multi-head attention on the 5th-gen tensor cores (layers.py:404-459 of
// the reference: softmax(Q K^T / sqrt(d)) V per head and its backward, no mask),
// without materialising the [b, n, s, s] probability matrix.
//
// Forward (flash_fwd2_kernel, head_dim 64 and 128): persistent, two 128-row query
// tiles per CTA ping-ponging on the tensor core, P in TMEM as the A operand of PV,
// O accumulated in TMEM; outputs O (bf16) into the interleaved context block and the
// row log-sum-exp (fp32) for the backward. Backward: flash_bwd2_kernel (d = 64,
// transposed orientation) and flash_bwd3_kernel (d = 128, transposed). Q/K/V are read in place
// from the QKV block through 4-D TMA maps (no head split copies).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "sg.h"
#include "sg_internal.h"
#include "sg_ptx.cuh"
#include "sg_tmap.h"

namespace sg {

struct FlashFwdParams {
  int s;            // sequence length (keys = queries)
  int nh;           // heads in the block
  int q_b2_first, k_b2_first, v_b2_first;
  float scale_log2; // log2(e) / sqrt(d)
  __nv_bfloat16* O;
  long long ldo;    // row pitch of the context block
  float* lse;       // [b, nh, s] natural-log log-sum-exp of the scaled scores
  int o_b2_first;   // O tile map (32 x 32 bf16 boxes): heads before rows
};

constexpr int kQB = 128;   // query rows per CTA
constexpr int kKB = 128;   // keys per block

__device__ __forceinline__ void tma4(const CUtensorMap* tm, void* dst, uint64_t* bar, int inner, int outer, int z2,
                                     int z1, int b2f) {
  if (b2f)
    tma_load_4d(dst, tm, bar, inner, z2, outer, z1);
  else
    tma_load_4d(dst, tm, bar, inner, outer, z2, z1);
}

__device__ __forceinline__ void tma4_l2(const CUtensorMap* tm, int inner, int outer, int z2, int z1, int b2f) {
  if (b2f)
    tma_prefetch_l2_4d(tm, inner, z2, outer, z1);
  else
    tma_prefetch_l2_4d(tm, inner, outer, z2, z1);
}

__device__ __forceinline__ float ex2f_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ============================================================================
// Forward, two query tiles per CTA ("ping-pong"): 640 threads (d = 64; d = 128 below)
//   warp 0      TMA: Q0, Q1 once per item; K_j / V_j blocks (three slots)
//   warps 1, 3  MMA issuers of tile 0 / tile 1: S_i,G+1 = Q_i K_G+1^T as soon as the
//               softmax warps hold S_i,G in registers, PV_i,G = P_i,G V_G once P_i,G
//               is in TMEM
//   warp 2      TMEM allocator: S0 | S1 | O0 | O1 | P0 | P1
//   warps 4-11  softmax of tile 0, warps 12-19 softmax of tile 1
// P never touches shared memory: the softmax warps write it as packed bf16 pairs
// into TMEM (tcgen05.st) and PV reads A from TMEM ("TS" MMA), so per key block the
// CTA's shared-memory traffic is only the K / V tiles and the score products'
// operands. Each query tile has its own MMA-issuing thread (a shared issuer forces
// the tiles into lockstep) and 8 softmax warps: warp (tile, key half, lane
// quadrant) owns 64 keys of 32 rows, so two warps of a tile share an SMSP's MUFU
// and fill each other's dependency gaps; the two halves of a row exchange the row
// max per block and the row sum per item through shared memory + an mbarrier. The
// tiles take turns on the exponentials (named barriers). A share of the exponentials
// runs as a polynomial on the FMA pipe (ex2_poly2). O accumulates in TMEM; the row
// max used for the exponent only advances (O and l rescaled through tcgen05.ld/st)
// when it grows by more than 2^8. Measured (tools/ftrace.py): a key block costs
// ~3500 clocks against 2048 of MUFU and ~1250 of tensor-core time; the M=128, N=64
// PV products issue at ~46 clocks each (tools/micro/umma_rate.cu) and both tiles'
// products queue on one tensor core.
// ============================================================================
constexpr int kQT = 2;  // query tiles per CTA

// d = 128 uses the same structure with P written over the consumed scores of S_i (TMEM:
// S0 | S1 | O0 | O1, 4 x 128 columns), so S_i,G+1 is issued after PV_i,G has read P_i,G
// (the other tile's softmax covers the gap); one Q slot, two K / V slots, O rows stored
// straight from registers.
template <int HD>
struct Flash2Cfg {
  static constexpr uint32_t T64 = 128 * 64 * 2;    // one 128 x 64 bf16 atom tile
  static constexpr uint32_t T = 128 * HD * 2;      // one 128-row tile (HD / 64 atoms)
  static constexpr int KV_SLOTS = HD == 64 ? 3 : 2;
  static constexpr int Q_SLOTS = HD == 64 ? 2 : 1; // d = 64: Q of the next item prefetched
  static constexpr uint32_t O_STG = HD == 64 ? kQT * 8 * 2048 : 0;  // d = 64: per softmax warp one 32 x 32 bf16 output tile
  static constexpr uint32_t X_XCH = (kQT * 2 + kQT) * 256 * 4;  // row max (2 slots) / row sum exchange
  static constexpr size_t SMEM = Q_SLOTS * kQT * T + KV_SLOTS * 2 * T + O_STG + X_XCH + 512;
  static constexpr bool P_IN_S = HD == 128;
};

// 2^y for a pair of exponents on the FMA pipe (no MUFU): y = j + f with j = rint(y)
// by the 1.5 * 2^23 shifter, 2^f by a degree-3 minimax polynomial on [-1/2, 1/2]
// (relative error 7.5e-5, far under the bf16 rounding of P), j added to the
// exponent field. y is clamped at -126 (2^-126 vanishes in bf16 P and in the row sum;
// below it the 2^f factor < 1 would underflow the exponent field).
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t y) {
  const float lo = fmaxf(f2_lo(y), -126.f), hi = fmaxf(f2_hi(y), -126.f);
  const uint64_t yc = f2_pack(lo, hi);
  const uint64_t sh = f2_pack(12582912.f, 12582912.f);
  const uint64_t t = fadd2(yc, sh);                                   // j in the low mantissa bits
  const uint64_t f = fadd2(yc, fadd2(f2_pack(-12582912.f, -12582912.f), t) ^ 0x8000000080000000ull);  // y - j
  uint64_t q = ffma2(f, f2_pack(0.0551716687545781f, 0.0551716687545781f),
                     f2_pack(0.24261114787053215f, 0.24261114787053215f));
  q = ffma2(q, f, f2_pack(0.6932609877583421f, 0.6932609877583421f));
  q = ffma2(q, f, f2_pack(0.9999280720307991f, 0.9999280720307991f));
  const uint32_t rl = static_cast<uint32_t>(q) + (static_cast<uint32_t>(t) << 23);
  const uint32_t rh = static_cast<uint32_t>(q >> 32) + (static_cast<uint32_t>(t >> 32) << 23);
  return static_cast<uint64_t>(rl) | (static_cast<uint64_t>(rh) << 32);
}

// Persistent: CTA c processes work items t = c, c + grid, ... with t = (query-tile
// pair, head, batch), pair index fastest (neighbouring CTAs share K / V in L2).
// All per-block barriers run on a CTA-wide block counter G across items, so the
// next item's Q, first K / V block and first score products are in flight while
// the current item finishes. NPOLY of every 16 exponent pairs go to the FMA-pipe
// polynomial instead of MUFU.EX2 (the MUFU rate bounds the softmax warps).
template <int HD, int NPOLY>
__global__ void __launch_bounds__(640, 1)
    flash_fwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                      const __grid_constant__ FlashFwdParams p, int bsz) {
  using Cfg = Flash2Cfg<HD>;
  constexpr uint32_t T64 = Cfg::T64, T = Cfg::T;
  constexpr int NS = Cfg::KV_SLOTS, QS = Cfg::Q_SLOTS;
  constexpr bool P_IN_S = Cfg::P_IN_S;
  constexpr int ATOMS = HD / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();
  uint8_t* sQ = smem;                             // [Q_SLOTS][kQT] tiles
  uint8_t* sK = sQ + QS * kQT * T;                // [NS]
  uint8_t* sV = sK + NS * T;                      // [NS]
  uint8_t* sO = sV + NS * T;                      // d = 64: [kQT][4 warps] x 4 KB output staging
  float* sX = reinterpret_cast<float*>(sO + Cfg::O_STG);  // half-row exchange
  uint64_t* bars = reinterpret_cast<uint64_t*>(sO + Cfg::O_STG + Cfg::X_XCH);
  uint64_t* q_full = bars;                // [2]
  uint64_t* q_empty = bars + 2;           // [2]
  uint64_t* k_full = bars + 4;            // [NS]
  uint64_t* v_full = k_full + NS;         // [NS]
  uint64_t* kv_empty = v_full + NS;       // [NS]
  uint64_t* s_full = kv_empty + NS;       // [kQT]
  uint64_t* s_free = s_full + kQT;        // [kQT]
  uint64_t* p_full = s_free + kQT;        // [kQT]
  uint64_t* pv_done = p_full + kQT;       // [kQT]
  uint64_t* o_full = pv_done + kQT;       // [kQT]
  uint64_t* xbar = o_full + kQT;          // [kQT][4] half-row meeting per block (row max)
  uint64_t* lbar = xbar + kQT * 4;        // [kQT][4] half-row meeting per item (row sum)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lbar + kQT * 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = (p.s + kKB - 1) / kKB;
  const int npairs = (p.s + kQT * kQB - 1) / (kQT * kQB);
  const int n_items = npairs * p.nh * bsz;
  const int my_items = n_items > (int)blockIdx.x ? (n_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = my_items * nkb;  // this CTA's key blocks over all its items
  auto decode = [&](int t, int& qb, int& h, int& b) {
    qb = t % npairs;
    const int r = t / npairs;
    h = r % p.nh;
    b = r / p.nh;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmO);
    for (int i = 0; i < QS; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], kQT);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&kv_empty[i], kQT);  // one commit per tile issuer
    }
    for (int i = 0; i < kQT; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 8);
      mbar_init(&p_full[i], 8);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_full[i], 1);
    }
    for (int i = 0; i < kQT * 4; ++i) {
      mbar_init(&xbar[i], 2);
      mbar_init(&lbar[i], 2);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_begin();
  // TMEM columns: S_i at 128 i, O_i at 256 + HD i, P_i (packed bf16 pairs) at 384 + 64 i
  // (d = 64) or over the consumed scores of S_i (d = 128)
  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      for (int t = blockIdx.x, it = 0; t < n_items; t += gridDim.x, ++it) {
        int qb, h, b;
        decode(t, qb, h, b);
        const int qs = it % QS;
        mbar_wait_sleep(&q_empty[qs], ((it / QS) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qs], kQT * T);
#pragma unroll
        for (int i = 0; i < kQT; ++i)
#pragma unroll
          for (int a = 0; a < ATOMS; ++a)
            tma4(&tmQ, sQ + (qs * kQT + i) * T + a * T64, &q_full[qs], a * 64, (qb * kQT + i) * kQB, h, b,
                 p.q_b2_first);
        for (int j = 0; j < nkb; ++j, ++g) {
          const int slot = g % NS;
          mbar_wait_sleep(&kv_empty[slot], ((g / NS) & 1) ^ 1);
          mbar_arrive_expect_tx(&k_full[slot], T);
#pragma unroll
          for (int a = 0; a < ATOMS; ++a)
            tma4(&tmK, sK + slot * T + a * T64, &k_full[slot], a * 64, j * kKB, h, b, p.k_b2_first);
          mbar_arrive_expect_tx(&v_full[slot], T);
#pragma unroll
          for (int a = 0; a < ATOMS; ++a)
            tma4(&tmV, sV + slot * T + a * T64, &v_full[slot], a * 64, j * kKB, h, b, p.v_b2_first);
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    {
      // whole warp walks the loop with warp-uniform operands; one elected lane issues
      // ------------------------------------------------------------ MMA issuer of tile i
      // one issuing thread per query tile, so neither tile's products wait for the
      // other tile's softmax progress (a shared issuer forces the tiles into lockstep
      // and both softmax warpgroups then contend for MUFU at the same time)
      const int i = warp >> 1;
      constexpr uint32_t IDESC_S = umma_idesc_bf16(kQB, kKB, false, false);  // Q, K both K-major
      constexpr uint32_t IDESC_PV = umma_idesc_bf16(kQB, HD, false, true);   // P (TMEM), V MN-major
      const bool trm = blockIdx.x == 0 && i == 0 && lane == 0;
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint64_t q_desc0 = umma_desc_sw128(smem_u32(sQ), 0, 1024), k_desc0 = umma_desc_sw128(smem_u32(sK), 0, 1024);
      const uint64_t v_desc0 = umma_desc_sw128(smem_u32(sV), kKB * 128, 1024);
      constexpr uint64_t kTile = T >> 4, kAtom = T64 >> 4;
      const uint32_t t_o = tm + 256 + i * HD;
      int tri = 0;
      (void)trm; (void)tri;
      // S_i for global block G (item G / nkb, key block G % nkb)
      auto issue_s = [&](int G) {
        const int it = G / nkb;
        const uint64_t qd = q_desc0 + ((it % QS) * kQT + i) * kTile, kd = k_desc0 + (G % NS) * kTile;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {  // K-dim = d: 16-element steps, 64-wide atoms
            const uint64_t off = (kk >> 2) * kAtom + (kk & 3) * 2;
            umma_bf16(tm + i * 128, qd + off, kd + off, IDESC_S, kk > 0 ? 1u : 0u);
          }
          umma_commit(&s_full[i]);
          if (G % nkb == nkb - 1) umma_commit(&q_empty[(G / nkb) % QS]);  // the item's last score product
        }
        __syncwarp();
      };
      auto ready_s = [&](int G) {  // Q of G's item (at its first block) and K_G landed
        if (G % nkb == 0) mbar_wait(&q_full[(G / nkb) % QS], ((G / nkb) / QS) & 1);
        mbar_wait(&k_full[G % NS], (G / NS) & 1);
        tc_fence_after();
      };
      if (total > 0) {
        ready_s(0);
        issue_s(0);
      }
      for (int G = 0; G < total; ++G) {
        const int slot = G % NS, j = G % nkb;
        SG_TR(trm, 2, tri, 10);
        if constexpr (P_IN_S) {
          // PV_i,G reads P_i,G from S_i's columns, then S_i,G+1 overwrites them (in order)
          mbar_wait(&v_full[slot], (G / NS) & 1);
          mbar_wait(&p_full[i], G & 1);
          tc_fence_after();
          const uint64_t vd = v_desc0 + slot * kTile;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kKB / 16; ++kk)
              umma_bf16_ts(t_o, tm + i * 128 + (kk >> 2) * 64 + (kk & 3) * 8, vd + 128 * kk, IDESC_PV,
                           (j | kk) != 0 ? 1u : 0u);
            umma_commit(&pv_done[i]);
            if (j == nkb - 1) umma_commit(&o_full[i]);
            umma_commit(&kv_empty[slot]);  // this tile is done with K_G, V_G
          }
          __syncwarp();
          if (G + 1 < total) {
            ready_s(G + 1);
            issue_s(G + 1);
          }
          continue;
        }
        if (G + 1 < total) {
          ready_s(G + 1);
          SG_TR(trm, 2, tri, 14);
          mbar_wait(&s_free[i], G & 1);  // softmax i holds S_i,G in registers
          tc_fence_after();
          SG_TR(trm, 2, tri, 15);
          issue_s(G + 1);
        }
        SG_TR(trm, 2, tri, 11);
        mbar_wait(&v_full[slot], (G / NS) & 1);
        mbar_wait(&p_full[i], G & 1);  // P_i,G in TMEM, O_i corrected (or read out, first block)
        tc_fence_after();
        SG_TR(trm, 2, tri, 12);
        const uint64_t vd = v_desc0 + slot * kTile;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kKB / 16; ++kk)
            umma_bf16_ts(t_o, tm + 384 + i * 64 + kk * 8, vd + 128 * kk, IDESC_PV, (j | kk) != 0 ? 1u : 0u);
          umma_commit(&pv_done[i]);
          if (j == nkb - 1) umma_commit(&o_full[i]);
          umma_commit(&kv_empty[slot]);  // this tile is done with K_G, V_G
        }
        __syncwarp();
        SG_TR(trm, 2, tri, 13);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    // warp 4 + 8 i + 4 h + q: tile i, key half h (keys 64 h .. 64 h + 63 of a block,
    // O / P columns 32 h ..), TMEM lane quadrant q (rows 32 q ..). The two halves of a
    // row meet once per block (row max) and once per item (row sum) through a
    // shared-memory exchange and an mbarrier. The two tiles' warps of an SMSP take
    // turns on the exponentials (named barriers, 2 x 2 warps): tile 1's block G after
    // tile 0's block G, tile 0's block G + 1 after tile 1's block G, so one tile's MUFU
    // phase overlaps the other tile's TMEM loads, row max and tensor-core round trip.
    const int w = warp - 4;
    const int i = w >> 3, kh = (w >> 2) & 1, qd = warp & 3;
    const int r = qd * 32 + lane;                 // row inside the tile
    const uint32_t lane_base = static_cast<uint32_t>(qd * 32) << 16;
    // this warp's S_i columns (its 64 keys), O_i columns (its HD / 2) and packed P_i columns
    const uint32_t t_s = tmem + i * 128 + kh * 64 + lane_base, t_o = tmem + 256 + i * HD + kh * (HD / 2) + lane_base,
                   t_p = P_IN_S ? t_s : tmem + 384 + i * 64 + kh * 32 + lane_base;
    uint64_t* my_xbar = &xbar[i * 4 + qd];
    uint64_t* my_lbar = &lbar[i * 4 + qd];
    float* xm = sX + (i * 2) * 2 * 128;           // [2 slots][2 halves][128] row maxima
    const uint64_t scale2 = f2_pack(p.scale_log2, p.scale_log2);
    const bool trs = blockIdx.x == 0 && qd == 0 && kh == 0 && lane == 0;
    int tri = 0;
    (void)trs; (void)tri;
    int G = 0;
    for (int t = blockIdx.x, it = 0; t < n_items; t += gridDim.x, ++it) {
      int qb, h, b;
      decode(t, qb, h, b);
      const int qrow = (qb * kQT + i) * kQB + r;  // query position
      float m_use = -INFINITY, l = 0.f;
      for (int j = 0; j < nkb; ++j, ++G) {
        const int kvalid = min(kKB, p.s - j * kKB) - kh * 64;  // valid keys of this half
        SG_TR(trs, i, tri, 0);
        mbar_wait_sleep(&s_full[i], G & 1);
        tc_fence_after();
        SG_TR(trs, i, tri, 1);
        uint32_t sv[2][32];
#pragma unroll
        for (int c = 0; c < 2; ++c) tmem_ld32(t_s + c * 32, sv[c]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[i]);  // the MMA may overwrite S_i now
        if (kvalid < 64) {  // partial last block: keys past the end never contribute
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (c * 32 + e >= kvalid) sv[c][e] = __float_as_uint(-INFINITY);
        }
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            mx[(e >> 1) & 1] = fmax3f(mx[(e >> 1) & 1], __uint_as_float(sv[c][e]), __uint_as_float(sv[c][e + 1]));
        const float m_loc = fmaxf(mx[0], mx[1]) * p.scale_log2;
        float* slot = xm + (G & 1) * 256;  // double-buffered: a half rewrites a slot only after the next meeting
        slot[kh * 128 + r] = m_loc;
        __syncwarp();
        if (lane == 0) mbar_arrive(my_xbar);
        SG_TR(trs, i, tri, 2);
        // PV_i,G-1 has finished reading P_i (and writing O_i)
        if (G > 0) mbar_wait_sleep(&pv_done[i], (G - 1) & 1);
        // this tile's turn on MUFU
        if (i == 1 || G > 0) named_bar_sync(1 + (1 - i) * 4 + qd, 128);
        mbar_wait_sleep(my_xbar, G & 1);
        // (a volatile shared load after the barrier: no exponential is scheduled ahead of the turn)
        const float m_cand = fmax3f(m_use, m_loc, *static_cast<volatile float*>(&slot[(kh ^ 1) * 128 + r]));
        float alpha = 1.f;
        bool correct = false;
        if (j == 0) {
          m_use = m_cand;
        } else if (__any_sync(0xffffffffu, m_cand > m_use + 8.f)) {  // same rows, same vote in both halves
          alpha = ex2f_fast(m_use - m_cand);
          m_use = m_cand;
          correct = true;
        }
        const uint64_t neg2 = f2_pack(-m_use, -m_use);
        SG_TR(trs, i, tri, 3);
        uint64_t ps2 = 0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          // packed pairs overwrite the consumed scores in place (contiguous STTM source)
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint64_t y =
                ffma2(f2_pack(__uint_as_float(sv[c][2 * e]), __uint_as_float(sv[c][2 * e + 1])), scale2, neg2);
            float p0, p1;
            if ((e * NPOLY) % 16 < NPOLY) {  // NPOLY of 16 pairs, spread over the chunk
              const uint64_t pp = ex2_poly2(y);
              p0 = f2_lo(pp);
              p1 = f2_hi(pp);
            } else {
              p0 = ex2f_fast(f2_lo(y));
              p1 = ex2f_fast(f2_hi(y));
            }
            ps2 = fadd2(ps2, f2_pack(p0, p1));
            __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
            sv[c][e] = *reinterpret_cast<uint32_t*>(&hv);
          }
          tmem_st16(t_p + c * 16, *reinterpret_cast<const uint32_t(*)[16]>(&sv[c][0]));  // 32 keys, packed pairs
        }
        SG_TR(trs, i, tri, 4);
        if (i == 0 || G + 1 < total) named_bar_arrive(1 + i * 4 + qd, 128);
        l = l * alpha + (f2_lo(ps2) + f2_hi(ps2));
        if (correct) {
          // this half's O_i columns *= 2^(m_old - m_new) before PV_i,G accumulates into them
#pragma unroll 1
          for (int oc = 0; oc < HD / 64; ++oc) {
            uint32_t ov[32];
            tmem_ld32(t_o + oc * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            tmem_st32(t_o + oc * 32, ov);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[i]);
      }
      // O_i of this item complete: row sum of both halves, normalise, bf16 into the
      // context block, lse. The next item's first PV overwrites O_i only after this
      // warpgroup's next p_full.
      float* xl = sX + 4 * 256 + i * 256;  // [2 halves][128] row sums
      xl[kh * 128 + r] = l;
      __syncwarp();
      if (lane == 0) mbar_arrive(my_lbar);
      mbar_wait_sleep(my_lbar, it & 1);
      l += xl[(kh ^ 1) * 128 + r];
      mbar_wait_sleep(&o_full[i], it & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      if constexpr (HD == 128) {
        // normalised bf16 rows straight to the context block: 64 columns = 128 B per row
        // (the TMEM loads are warp-collective: every lane loads, rows past s do not store)
        uint4* dst = reinterpret_cast<uint4*>(p.O + ((size_t)b * p.s + qrow) * p.ldo + (size_t)h * HD + kh * 64);
#pragma unroll
        for (int oc = 0; oc < 2; ++oc) {
          uint32_t ov[32];
          tmem_ld32(t_o + oc * 32, ov);
          tmem_wait_ld();
          if (qrow < p.s) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint4 x;
              __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
              for (int e = 0; e < 4; ++e)
                hh[e] = __floats2bfloat162_rn(__uint_as_float(ov[8 * k + 2 * e]) * inv,
                                              __uint_as_float(ov[8 * k + 2 * e + 1]) * inv);
              dst[oc * 4 + k] = x;
            }
          }
        }
        __syncwarp();
        tc_fence_before();
        if (kh == 0 && qrow < p.s && p.lse)
          p.lse[((size_t)b * p.nh + h) * p.s + qrow] = (m_use + __log2f(l)) * 0.6931471805599453f;
        continue;
      }
      // normalised bf16 rows -> this warp's 32 x 32 SW64 staging tile -> TMA store
      // into the context block (rows past s clipped)
      uint8_t* ostg = sO + w * 2048;
      if (lane == 0) bulk_wait_read<0>();  // the previous item's store has read the staging
      __syncwarp();
      {
        uint32_t ov[32];
        tmem_ld32(t_o, ov);
        tmem_wait_ld();
        uint8_t* orow = ostg + lane * 64;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint4 x;
          __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            hh[e] = __floats2bfloat162_rn(__uint_as_float(ov[8 * k + 2 * e]) * inv,
                                          __uint_as_float(ov[8 * k + 2 * e + 1]) * inv);
          *reinterpret_cast<uint4*>(orow + ((k ^ ((lane >> 1) & 3)) << 4)) = x;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int row0 = (qb * kQT + i) * kQB + qd * 32;
        if (p.o_b2_first)
          tma_store_4d(&tmO, ostg, kh * 32, h, row0, b);
        else
          tma_store_4d(&tmO, ostg, kh * 32, row0, h, b);
        bulk_commit();
      }
      __syncwarp();
      tc_fence_before();
      if (kh == 0 && qrow < p.s && p.lse)
        p.lse[((size_t)b * p.nh + h) * p.s + qrow] = (m_use + __log2f(l)) * 0.6931471805599453f;
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

template <int HD, int NPOLY>
static void launch_fwd2_k(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& o,
                          const FlashFwdParams& p, int b, int grid, cudaStream_t stream) {
  launch_k(flash_fwd2_kernel<HD, NPOLY>, dim3(grid), dim3(640), Flash2Cfg<HD>::SMEM, stream, q, k, v, o, p, b);
}

template <int HD>
static int launch_fwd2(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& o,
                       const FlashFwdParams& p, int b, cudaStream_t stream) {
  // SG_FLASH_POLY = pairs of 16 on the FMA-pipe exp2 (experiments; default below)
  static const int npoly = [] {  // measured (d = 64) at b=32 s=512 / b=4 s=2048: 0 -> 63.6 / 115.9 us, 2 -> 62.7 / 113.0,
    const char* e = getenv("SG_FLASH_POLY");  // 4 -> 63.7 / 115.1, 6 -> 67.2 / 123.2
    return e ? atoi(e) : 2;
  }();
  const void* kern = npoly >= 4 ? (const void*)flash_fwd2_kernel<HD, 4>
                     : npoly >= 2 ? (const void*)flash_fwd2_kernel<HD, 2> : (const void*)flash_fwd2_kernel<HD, 0>;
  if (!ensure_smem(kern, (int)Flash2Cfg<HD>::SMEM)) return set_error(SG_ERR_CUDA, "flash fwd: smem attribute");
  const int items = (p.s + kQT * kQB - 1) / (kQT * kQB) * p.nh * b;
  const int sms = sg_device_sm_count();
  const int grid = std::min(items, sms > 0 ? sms : 148);
  if (npoly >= 4)
    launch_fwd2_k<HD, 4>(q, k, v, o, p, b, grid, stream);
  else if (npoly >= 2)
    launch_fwd2_k<HD, 2>(q, k, v, o, p, b, grid, stream);
  else
    launch_fwd2_k<HD, 0>(q, k, v, o, p, b, grid, stream);
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}

}  // namespace sg

using namespace sg;

#ifdef SG_TRACE
extern "C" int sg_debug_trace(void* host) {
  return cudaMemcpyFromSymbol(host, sg::g_sgtrace, sizeof(sg::g_sgtrace)) == cudaSuccess ? 0 : 1;
}
extern "C" int sg_debug_trace_clear(void) {
  static unsigned long long zero[4][8192];
  return cudaMemcpyToSymbol(sg::g_sgtrace, zero, sizeof zero) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int sg_flash_attn_fwd(const void* qkv, int64_t ldq, int64_t b, int64_t s, int64_t nh, int64_t d,
                                 void* out, int64_t ldo, float* lse, void* stream) {
  clear_error();
  if (b < 1 || s < 1 || nh < 1 || (d != 64 && d != 128)) return set_error(SG_ERR_SHAPE, "flash fwd: d must be 64 or 128");
  if (ldq < 3 * nh * d || ldo < nh * d) return set_error(SG_ERR_SHAPE, "flash fwd: leading dimensions");
  if ((reinterpret_cast<uintptr_t>(out) & 15) || (ldo * 2) % 16) return set_error(SG_ERR_SHAPE, "flash fwd: unaligned");
  const __nv_bfloat16* base = static_cast<const __nv_bfloat16*>(qkv);
  const long long hb = nh * d;
  CUtensorMap tq, tk, tv;
  FlashFwdParams p{};
  p.s = (int)s;
  p.nh = (int)nh;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)d);
  p.O = static_cast<__nv_bfloat16*>(out);
  p.ldo = ldo;
  p.lse = lse;
  // [b, s, nh, d] views of the Q / K / V column ranges of the QKV block, box 64 x 128 rows
  int rc = tmap_bf16_4d(&tq, base, d, s, nh, b, ldq, d, s * ldq, 64, kQB, &p.q_b2_first);
  if (!rc) rc = tmap_bf16_4d(&tk, base + hb, d, s, nh, b, ldq, d, s * ldq, 64, kKB, &p.k_b2_first);
  if (!rc) rc = tmap_bf16_4d(&tv, base + 2 * hb, d, s, nh, b, ldq, d, s * ldq, 64, kKB, &p.v_b2_first);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUtensorMap to;
  rc = tmap_bf16_tile_4d(&to, out, d, s, nh, b, ldo, d, s * ldo, &p.o_b2_first);
  if (rc) return rc;
  if (d == 64) return launch_fwd2<64>(tq, tk, tv, to, p, (int)b, st);
  return launch_fwd2<128>(tq, tk, tv, to, p, (int)b, st);
}

// ============================================================================
// Backward (d = 64): one CTA = (128-key block, head, batch), loop over query
// blocks (FlashAttention-2 order). Per query block:
//   S  = Q K^T,  dP = dO V^T                       (TMEM, M = queries)
//   P  = exp(S / sqrt(d) - lse),  dS = P (dP - D) / sqrt(d)   (warps 4-7 -> smem)
//   dV += P^T dO,  dK += dS^T Q                     (TMEM accumulators, M = keys)
//   dQ  = dS K  -> fp32 accumulator via TMA reduce-add (one CTA per key block adds)
// with D = rowsum(dO * O) precomputed (sg_attn_rowdot). P / dS are stored once,
// [queries x keys] in the SWIZZLE_128B layout that is both the K-major A
// operand of dS K and the MN-major A operand of P^T dO / dS^T Q.
// ============================================================================
namespace sg {

struct FlashBwdParams {
  int s, nh;
  int q_b2_first, k_b2_first, v_b2_first, do_b2_first, dq_b2_first;
  float scale, scale_log2;
  const float* lse;   // [b, nh, s]
  const float* drow;  // [b, nh, s]
  __nv_bfloat16* dK;  // [b*s, ldg] head columns h*64
  __nv_bfloat16* dV;
  long long ldg;
  int dkv_b2_first;   // dK / dV tile maps: heads before rows
  int b0;             // first sequence of this launch (batch chunks keep the item table bounded)
  float* kv_colsum;   // optional [2 nh 64]: += column sums of dK (then dV)
};

constexpr uint32_t kT64 = 128 * 64 * 2;  // one 128 x 64 bf16 tile (16 KB)
constexpr int kMaxItems = 256;           // per-CTA work items of the persistent backward (item table in smem)

// ----------------------------------------------------------------------------
// Backward (d = 64), persistent, transposed orientation: CTA c walks work items
// t = c, c + grid, ... with t = (key block, head, batch), key block fastest. Per
// query block G (128 queries) of an item (128 keys):
//   S^T  = K Q^T,  dP^T = V dO^T                  (TMEM, M = keys, N = queries)
//   P^T  = 2^(S^T scale log2e - lse log2e)        -> TMEM (packed bf16, own region)
//   dS^T = P^T (dP^T - D) scale                   -> TMEM (packed, in place over dP^T)
//                                                    and shared memory ([keys x queries])
//   dV  += P^T dO,  dK += dS^T Q                   ("TS" MMAs: A read from TMEM)
//   dQ   = dS K                                    (A = dS, MN-major from shared memory)
// so per block the tensor core reads only Q, dO, K, V tiles and one copy of dS from
// shared memory (the N = 64 products of the [queries x keys] orientation, with P / dS
// from shared memory, are shared-memory bound: tools/micro/umma_rate.cu). Rows of the
// softmax are keys, so the per-query statistics (lse; D = rowsum(dO * O) from
// sg_attn_rowdot) are staged per warp in shared memory and read as broadcasts;
// queries past s get lse = +inf (P = 0), keys past s are zeroed.
//   warp 0      TMA producer: K per item (2 slots), V per item (1 slot), Q / dO per
//               block (3 slots, the block after next prefetched into L2)
//   warp 1      MMA issuer, per block G: S^T_G+1 as soon as the softmax warps have read
//               S^T_G; dV_G as soon as P^T_G is in TMEM (before dS_G exists); dK_G,
//               dP^T_G+1 and dQ_G once dS_G is stored. Four commits per block (each
//               commit costs the tensor pipe ~70 clocks, tools/micro/bwd_seq.cu): the
//               softmax warps reuse the Q / dO slot barrier (dK_G-1 done => dV_G-1 has
//               read P^T) and the dQ barrier (dQ_G-1 has read the single dS buffer).
//   warp 2      TMEM allocator: S^T | dP^T (dS^T) | P^T | dV | dK | dQ
//   warps 4-11  softmax: warp e owns TMEM lane quadrant e % 4 (32 keys) and query
//               half e / 4 (64 queries); NPOLY of every 16 exponent pairs run on the
//               FMA pipe (ex2_poly2) instead of MUFU
//   warps 12-15 drain: dQ_G (TMEM -> two 4 KB staging boxes -> TMA reduce-add into the
//               fp32 accumulator) and, at an item's end, dK / dV (both read out of TMEM
//               before the accumulators are released, then staged and TMA-stored)
//   setmaxnreg: producer / MMA warpgroup 56 registers, softmax 160, drain 128.
// G counts query blocks over all of the CTA's items (barrier phases).
// ----------------------------------------------------------------------------
constexpr int kQD = 3;  // Q / dO slots of the d = 64 backward
#ifndef SG_BWD_POLY
#define SG_BWD_POLY 0
#endif
constexpr int kBwdPoly = SG_BWD_POLY;  // exponent pairs of every 16 on the FMA pipe
// the MMA warp of the d = 64 backward waits sleeping (SG_MMA_SPIN: spinning)
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t parity) {
#ifdef SG_MMA_SPIN
  mbar_wait(bar, parity);
#else
  mbar_wait_sleep(bar, parity);
#endif
}

template <int NPOLY>
__global__ void __launch_bounds__(512, 1)
    flash_bwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                      const __grid_constant__ CUtensorMap tmDQ, const __grid_constant__ CUtensorMap tmDK,
                      const __grid_constant__ CUtensorMap tmDV, const __grid_constant__ FlashBwdParams p, int bsz) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();
  uint8_t* sK = smem;                 // 2 slots (items)
  uint8_t* sV = sK + 2 * kT64;        // 1 slot
  uint8_t* sQ = sV + kT64;            // kQD slots (query blocks)
  uint8_t* sDO = sQ + kQD * kT64;     // kQD slots
  uint8_t* sDS = sDO + kQD * kT64;    // 32 KB: [keys x queries], 2 atoms of 64 queries
  uint8_t* sStg = sDS + 2 * kT64;     // 4 drain warps x 2 x 4 KB (dQ fp32 boxes)
  float* sStat = reinterpret_cast<float*>(sStg + 4 * 8192);  // 2 slots x [128 -lse log2e | 128 -D scale]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStat + 2 * 256);
  int* items_tab = reinterpret_cast<int*>(bars + 32);  // this CTA's items as packed (kb, h, b)
  uint64_t* k_full = bars;         // [2]
  uint64_t* k_empty = bars + 2;    // [2]
  uint64_t* v_full = bars + 4;
  uint64_t* v_empty = bars + 5;
  uint64_t* qd_full = bars + 6;    // [kQD]
  uint64_t* qd_empty = bars + 9;   // [kQD] dK_G done (Q_G, dO_G free; P^T_G read by dV_G)
  uint64_t* s_full = bars + 12;
  uint64_t* s_free = bars + 13;    // S^T_G read out of TMEM (8 softmax warps)
  uint64_t* p_full = bars + 14;    // P^T_G in TMEM (8 softmax warps)
  uint64_t* dp_full = bars + 15;
  uint64_t* ds_full = bars + 16;   // dS^T_G in TMEM and dS_G in smem (8 softmax warps)
  uint64_t* dq_full = bars + 17;   // dQ_G done (the dS buffer is free)
  uint64_t* dq_empty = bars + 18;  // 4 drain warps
  uint64_t* acc_full = bars + 19;
  uint64_t* acc_empty = bars + 20; // 4 drain warps
  uint64_t* st_full = bars + 21;   // [2] statistics of block G in slot G & 1 (warp 3)
  uint64_t* st_empty = bars + 23;  // [2] the 8 softmax warps have read them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (p.s + 127) / 128;
  const int nkb = nqb;
  const int n_items = nkb * p.nh * bsz;
  auto decode = [&](int t, int& kb, int& h, int& b) {
    kb = t % nkb;
    const int r = t / nkb;
    h = r % p.nh;
    b = r / p.nh + p.b0;
  };
  const int my_items = n_items > (int)blockIdx.x ? (n_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = my_items * nqb;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
    tma_prefetch_desc(&tmDQ);
    tma_prefetch_desc(&tmDK);
    tma_prefetch_desc(&tmDV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kQD; ++i) {
      mbar_init(&qd_full[i], 1);
      mbar_init(&qd_empty[i], 1);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(s_free, 8);
    mbar_init(p_full, 8);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 8);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 4);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&st_full[i], 32);
      mbar_init(&st_empty[i], 8);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  // item coordinates, decoded once: kb | h << 10 | b << 20 (kb < 1024, h < 1024 checked by the host)
  for (int it = threadIdx.x; it < my_items && it < kMaxItems; it += blockDim.x) {
    int kb, h, b;
    decode((int)blockIdx.x + it * (int)gridDim.x, kb, h, b);
    items_tab[it] = kb | (h << 10) | ((b - p.b0) << 20);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_begin();
  // TMEM columns: S^T 0..127 | dP^T (then dS^T packed in place) 128..255 | P^T packed
  // 256..319 | dV 320..383 | dK 384..447 | dQ 448..511
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_p = tmem + 256, t_dv = tmem + 320, t_dk = tmem + 384,
                 t_dq = tmem + 448;
  auto item = [&](int it, int& kb, int& h, int& b) {
    const int v = items_tab[it];
    kb = v & 1023;
    h = (v >> 10) & 1023;
    b = (v >> 20) + p.b0;
  };

  if (warp == 0) {
    reg_dealloc<56>();
    if (lane == 0) {
      int G = 0;
      for (int t = blockIdx.x, it = 0; t < n_items; t += gridDim.x, ++it) {
        int kb, h, b;
        decode(t, kb, h, b);
        const int ks = it & 1;
        mbar_wait_sleep(&k_empty[ks], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[ks], kT64);
        tma4(&tmK, sK + ks * kT64, &k_full[ks], 0, kb * 128, h, b, p.k_b2_first);
        mbar_wait_sleep(v_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(v_full, kT64);
        tma4(&tmV, sV, v_full, 0, kb * 128, h, b, p.v_b2_first);
        for (int i = 0; i < nqb; ++i, ++G) {
          const int slot = G % kQD, use = G / kQD;
          {
            // Q / dO of block G + kQD into L2 now (its smem slot frees only when block G's
            // dK is done)
            int i2 = i + kQD, t2 = t, kb2 = kb, h2 = h, b2 = b;
            while (i2 >= nqb) {
              i2 -= nqb;
              t2 += gridDim.x;
            }
            if (t2 != t && t2 < n_items) decode(t2, kb2, h2, b2);
            if (t2 < n_items) {
              tma4_l2(&tmQ, 0, i2 * 128, h2, b2, p.q_b2_first);
              tma4_l2(&tmDO, 0, i2 * 128, h2, b2, p.do_b2_first);
            }
          }
          mbar_wait_sleep(&qd_empty[slot], (use & 1) ^ 1);
          mbar_arrive_expect_tx(&qd_full[slot], 2 * kT64);
          tma4(&tmQ, sQ + slot * kT64, &qd_full[slot], 0, i * 128, h, b, p.q_b2_first);
          tma4(&tmDO, sDO + slot * kT64, &qd_full[slot], 0, i * 128, h, b, p.do_b2_first);
        }
      }
    }
  } else if (warp == 1) {
    reg_dealloc<56>();
    // the whole warp walks the loop (warp-uniform operands live in uniform registers);
    // one elected lane issues each MMA / commit
    {
      constexpr uint32_t ID_ST = umma_idesc_bf16(128, 128, false, false);  // S^T, dP^T: M = keys, N = queries
      constexpr uint32_t ID_KV = umma_idesc_bf16(128, 64, false, true);    // dV, dK: A = P^T / dS^T (TMEM), B = dO / Q
      constexpr uint32_t ID_DQ = umma_idesc_bf16(128, 64, true, true);     // dQ: A = dS (MN-major), B = K
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t ts = tm, tdp = tm + 128, tp = tm + 256, tdv = tm + 320, tdk = tm + 384, tdq = tm + 448;
      // descriptors: K-step advances add (bytes >> 4) to the start-address field
      const uint64_t d_k0 = umma_desc_sw128(smem_u32(sK), 0, 1024), d_v0 = umma_desc_sw128(smem_u32(sV), 0, 1024);
      const uint64_t d_q0 = umma_desc_sw128(smem_u32(sQ), 0, 1024), d_do0 = umma_desc_sw128(smem_u32(sDO), 0, 1024);
      const uint64_t m_q0 = umma_desc_sw128(smem_u32(sQ), kT64, 1024), m_do0 = umma_desc_sw128(smem_u32(sDO), kT64, 1024);
      const uint64_t m_k0 = umma_desc_sw128(smem_u32(sK), kT64, 1024), m_ds = umma_desc_sw128(smem_u32(sDS), kT64, 1024);
      constexpr uint64_t kTile = kT64 >> 4;  // one 16 KB tile in descriptor units
      const bool trm = blockIdx.x == 0 && lane == 0;
      int tri = 0;
      (void)trm; (void)tri;
      auto issue_s = [&](int G) {  // S^T_G = K Q_G^T
        const int it = G / nqb, slot = G % kQD;
        if (G % nqb == 0) mma_wait(&k_full[it & 1], (it >> 1) & 1);
        mma_wait(&qd_full[slot], (G / kQD) & 1);
        tc_fence_after();
        SG_TR(trm, 0, tri, 8);
        const uint64_t ak = d_k0 + (it & 1) * kTile, bq = d_q0 + slot * kTile;
        if (elect_one()) {
#ifndef SG_EXP_NOMMA
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // K-dim = d = 64: 4 x 16 inside one atom (32 B = 2 units)
            umma_bf16(ts, ak + 2 * kk, bq + 2 * kk, ID_ST, kk > 0 ? 1u : 0u);
#endif
          umma_commit(s_full);
        }
        __syncwarp();
      };
      auto issue_dp = [&](int G) {  // dP^T_G = V dO_G^T (Q_G / dO_G already waited for by issue_s(G))
        const int it = G / nqb, slot = G % kQD;
        if (G % nqb == 0) {
          mma_wait(v_full, it & 1);
          tc_fence_after();
        }
        const uint64_t bdo = d_do0 + slot * kTile;
        if (elect_one()) {
#ifndef SG_EXP_NOMMA
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_bf16(tdp, d_v0 + 2 * kk, bdo + 2 * kk, ID_ST, kk > 0 ? 1u : 0u);
#endif
          umma_commit(dp_full);
          if (G % nqb == nqb - 1) umma_commit(v_empty);  // the item's last dP^T: V may be reloaded
        }
        __syncwarp();
      };
      if (total > 0) {
        issue_s(0);
        issue_dp(0);
      }
      for (int G = 0; G < total; ++G) {
        const int slot = G % kQD, it = G / nqb, i = G % nqb;
        const uint64_t mk = m_k0 + (it & 1) * kTile, mq = m_q0 + slot * kTile, mdo = m_do0 + slot * kTile;
        SG_TR(trm, 0, tri, 0);
        // S^T_G+1 overwrites S^T_G as soon as the softmax warps have read it
        mma_wait(s_free, G & 1);
        tc_fence_after();
        SG_TR(trm, 0, tri, 1);
        // S^T_G+1 now if its Q tile (and, at an item start, K) has landed, else after dV_G
        bool s_next = G + 1 >= total;
        if (!s_next && mbar_test(&qd_full[(G + 1) % kQD], ((G + 1) / kQD) & 1) &&
            ((G + 1) % nqb != 0 || mbar_test(&k_full[((G + 1) / nqb) & 1], (((G + 1) / nqb) >> 1) & 1))) {
          issue_s(G + 1);
          s_next = true;
        }
        SG_TR(trm, 0, tri, 2);
        mma_wait(p_full, G & 1);  // P^T_G in TMEM
        tc_fence_after();
        // the previous item's dK / dV have been read out before this item's first products
        if (i == 0 && it > 0) {
          mma_wait(acc_empty, (it - 1) & 1);
          tc_fence_after();
        }
        SG_TR(trm, 0, tri, 3);
#if !defined(SG_EXP_NOMMA) && !defined(SG_EXP_NOKV)
        if (elect_one()) {
#pragma unroll
          for (int kq = 0; kq < 8; ++kq)  // dV += P^T dO, K-dim = 128 queries: 8 packed columns / 16 rows per step
            umma_bf16_ts(tdv, tp + kq * 8, mdo + 128 * kq, ID_KV, (i | kq) != 0 ? 1u : 0u);
        }
        __syncwarp();
#endif
        SG_TR(trm, 0, tri, 9);
        if (!s_next) issue_s(G + 1);
        mma_wait(ds_full, G & 1);  // dS^T_G in TMEM (over dP^T_G), dS_G in smem
        tc_fence_after();
        SG_TR(trm, 0, tri, 4);
        if (elect_one()) {
#if !defined(SG_EXP_NOMMA) && !defined(SG_EXP_NOKV)
#pragma unroll
          for (int kq = 0; kq < 8; ++kq)  // dK += dS^T Q: query half kq / 4 packed at column 64 (kq / 4)
            umma_bf16_ts(tdk, tdp + (kq >> 2) * 64 + (kq & 3) * 8, mq + 128 * kq, ID_KV, (i | kq) != 0 ? 1u : 0u);
#endif
          umma_commit(&qd_empty[slot]);  // Q_G / dO_G free; P^T_G read (dV_G issued before dK_G)
        }
        __syncwarp();
        SG_TR(trm, 0, tri, 10);
        // dP^T_G+1 overwrites dS^T_G once dK_G has read it (MMAs execute in issue order)
        if (G + 1 < total) issue_dp(G + 1);
        SG_TR(trm, 0, tri, 11);
        if (G >= 1) mma_wait(dq_empty, (G - 1) & 1);  // dQ_G-1 drained
        tc_fence_after();
        SG_TR(trm, 0, tri, 5);
        if (elect_one()) {
#if !defined(SG_EXP_NOMMA) && !defined(SG_EXP_NODQ)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // dQ = dS K, K-dim = 128 keys: 16 key rows (2048 B) per step
            umma_bf16(tdq, m_ds + 128 * kk, mk + 128 * kk, ID_DQ, kk > 0 ? 1u : 0u);
#endif
          SG_TR(trm, 0, tri, 12);
          umma_commit(dq_full);  // dQ_G in TMEM; the dS buffer is free
          if (i == nqb - 1) {
            umma_commit(acc_full);          // this item's dK / dV complete
            umma_commit(&k_empty[it & 1]);  // and its K no longer needed
          }
        }
        __syncwarp();
        SG_TR(trm, 0, tri, 13);
      }
    }
  } else if (warp == 3) {
    reg_dealloc<56>();
    // statistics of every block into the shared table: -lse log2e and -D scale of its 128
    // queries (queries past s: lse = +inf, so P = 0), prefetched a block ahead
    float v[8];
    auto load = [&](int G, float (&x)[8]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] = INFINITY;
        x[4 + u] = 0.f;
      }
      if (G >= total) return;
      int kb, h, b;
      item(G / nqb, kb, h, b);
      const size_t off = ((size_t)b * p.nh + h) * p.s;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int qrow = (G % nqb) * 128 + u * 32 + lane;
        if (qrow < p.s) {
          x[u] = __ldg(p.lse + off + qrow);
          x[4 + u] = __ldg(p.drow + off + qrow);
        }
      }
    };
    load(0, v);
    for (int G = 0; G < total; ++G) {
      float* t = sStat + (G & 1) * 256;
      if (G >= 2) mbar_wait_sleep(&st_empty[G & 1], ((G - 2) >> 1) & 1);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        t[u * 32 + lane] = -v[u] * 1.4426950408889634f;
        t[128 + u * 32 + lane] = -v[4 + u] * p.scale;
      }
      mbar_arrive(&st_full[G & 1]);
      load(G + 1, v);
    }
  } else if (warp < 4) {
    reg_dealloc<56>();
#ifdef SG_TRACE
    // observer (instrumented build): completion times of the tensor-pipe commits
    if (warp == 2 && lane == 0 && blockIdx.x == 0) {
      int tri = 0;
      for (int G = 0; G < total; ++G) {  // completion order: S^T_G+1, dK_G, dP^T_G+1, dQ_G
        if (G + 1 < total) mbar_wait_sleep(s_full, (G + 1) & 1);
        SG_TR(true, 3, tri, 0);
        mbar_wait_sleep(&qd_empty[G % kQD], (G / kQD) & 1);
        SG_TR(true, 3, tri, 1);
        if (G + 1 < total) mbar_wait_sleep(dp_full, (G + 1) & 1);
        SG_TR(true, 3, tri, 2);
        mbar_wait_sleep(dq_full, G & 1);
        SG_TR(true, 3, tri, 3);
      }
    }
#endif
  } else if (warp < 12) {
    reg_alloc<160>();
    // 8 softmax warps: warp e owns TMEM lane quadrant e % 4 (32 keys) and query half e / 4
    const int e = warp - 4;
    const int q = e & 3, hq = e >> 2;
    const int r = q * 32 + lane;  // key row of the block
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const float scale = p.scale;
    const bool trs = blockIdx.x == 0 && lane == 0 && e == 0;
    int tri = 0;
    (void)trs; (void)tri;
    int it = 0, i = 0;  // (item, query block) of G, advanced incrementally
    int kb = 0, h = 0, b = 0;
    if (my_items > 0) item(0, kb, h, b);
    const uint64_t sl2 = f2_pack(p.scale_log2, p.scale_log2), sc2 = f2_pack(scale, scale);
    for (int G = 0; G < total; ++G) {
      const int kvalid = min(128, p.s - kb * 128);
      const float* st = sStat + (G & 1) * 256 + hq * 64;  // this warp's 64 queries: [0, 64) lse, [128, 192) D
      SG_TR(trs, e == 0 ? 1 : 3, tri, 0);
      mbar_wait_sleep(s_full, G & 1);
      mbar_wait_sleep(&st_full[G & 1], (G >> 1) & 1);
      tc_fence_after();
      SG_TR(trs, e == 0 ? 1 : 3, tri, 1);
#ifdef SG_EXP_NOSM
      {
        __syncwarp();
        if (lane == 0) mbar_arrive(&st_empty[G & 1]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
        if (G > 0) mbar_wait_sleep(&qd_empty[(G - 1) % kQD], ((G - 1) / kQD) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        mbar_wait_sleep(dp_full, G & 1);
        if (G > 0) mbar_wait_sleep(dq_full, (G - 1) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_full);
        if (i == nqb - 1) {
          i = 0;
          ++it;
          if (it < my_items) item(it, kb, h, b);
        } else {
          ++i;
        }
        continue;
      }
#endif
      uint32_t sv[64];
      tmem_ld32(t_s + lane_base + hq * 64, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
      tmem_ld32(t_s + lane_base + hq * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);  // the next block's S^T may overwrite these columns
      SG_TR(trs, e == 0 ? 1 : 3, tri, 2);
      // P^T = 2^(s scale log2e - lse log2e), pairs of queries on the paired fp32 pipe;
      // fp32 P kept (in sv) for dS, packed bf16 pairs for TMEM
      uint32_t pk[32];
      const bool key_ok = r < kvalid;
#pragma unroll
      for (int j4 = 0; j4 < 16; ++j4) {
        const float4 nl = *reinterpret_cast<const float4*>(st + 4 * j4);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = 2 * j4 + u;
          const uint64_t y = ffma2(f2_pack(__uint_as_float(sv[2 * j]), __uint_as_float(sv[2 * j + 1])), sl2,
                                   u ? f2_pack(nl.z, nl.w) : f2_pack(nl.x, nl.y));
          float p0, p1;
          if ((j * NPOLY) % 16 < NPOLY) {  // NPOLY of 16 pairs, spread over the row
            const uint64_t pp = ex2_poly2(y);
            p0 = f2_lo(pp);
            p1 = f2_hi(pp);
          } else {
            p0 = ex2f_fast(f2_lo(y));
            p1 = ex2f_fast(f2_hi(y));
          }
          sv[2 * j] = __float_as_uint(p0);
          sv[2 * j + 1] = __float_as_uint(p1);
          __nv_bfloat162 hp = __floats2bfloat162_rn(p0, p1);
          pk[j] = *reinterpret_cast<uint32_t*>(&hp);
        }
      }
      if (kvalid < 128 && !key_ok) {  // keys past s (last key block only): P = 0
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          sv[2 * j] = sv[2 * j + 1] = 0u;
          pk[j] = 0u;
        }
      }
      SG_TR(trs, e == 0 ? 1 : 3, tri, 3);
      if (G > 0) mbar_wait_sleep(&qd_empty[(G - 1) % kQD], ((G - 1) / kQD) & 1);  // dV_G-1 has read P^T_G-1
      tc_fence_after();
      tmem_st32(t_p + lane_base + hq * 32, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      SG_TR(trs, e == 0 ? 1 : 3, tri, 4);
      // dS^T = P^T (dP^T scale - D scale)
      mbar_wait_sleep(dp_full, G & 1);
      tc_fence_after();
      SG_TR(trs, e == 0 ? 1 : 3, tri, 5);
      uint32_t dk[32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t dv[32];
        tmem_ld32(t_dp + lane_base + hq * 64 + c * 32, dv);
        tmem_wait_ld();
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 nd = *reinterpret_cast<const float4*>(st + 128 + c * 32 + 4 * j4);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = 2 * j4 + u;
            const uint64_t t = ffma2(f2_pack(__uint_as_float(dv[2 * j]), __uint_as_float(dv[2 * j + 1])), sc2,
                                     u ? f2_pack(nd.z, nd.w) : f2_pack(nd.x, nd.y));
            const uint64_t ds =
                fmul2(f2_pack(__uint_as_float(sv[c * 32 + 2 * j]), __uint_as_float(sv[c * 32 + 2 * j + 1])), t);
            __nv_bfloat162 hd = __floats2bfloat162_rn(f2_lo(ds), f2_hi(ds));
            dk[c * 16 + j] = *reinterpret_cast<uint32_t*>(&hd);
          }
        }
      }
      // dS^T packed over this thread's own (already read) dP^T columns; dS into the smem
      // buffer ([keys x queries] rows: the MN-major A operand of dQ) once dQ_G-1 has read it
      tmem_st32(t_dp + lane_base + hq * 64, dk);
      __syncwarp();
      if (lane == 0) mbar_arrive(&st_empty[G & 1]);  // this warp has read block G's statistics
      SG_TR(trs, e == 0 ? 1 : 3, tri, 6);
      if (G > 0) mbar_wait_sleep(dq_full, (G - 1) & 1);
      uint8_t* drow_ = sDS + hq * kT64 + r * 128;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        *reinterpret_cast<uint4*>(drow_ + ((k ^ (r & 7)) << 4)) =
            make_uint4(dk[4 * k], dk[4 * k + 1], dk[4 * k + 2], dk[4 * k + 3]);
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      SG_TR(trs, e == 0 ? 1 : 3, tri, 7);
      if (i == nqb - 1) {
        i = 0;
        ++it;
        if (it < my_items) item(it, kb, h, b);
      } else {
        ++i;
      }
    }
  } else {
    // 4 drain warps (lane quadrant q = warp % 4, 32 rows): dQ of every block and, at
    // each item's end, its dK / dV, off the softmax warps' critical path
    reg_alloc<128>();
    const int q = warp & 3;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    uint8_t* stg = sStg + (warp - 12) * 8192;
    int it = 0, i = 0, kb = 0, h = 0, b = 0;
    if (my_items > 0) item(0, kb, h, b);
    const bool trd = blockIdx.x == 0 && lane == 0 && warp == 12;
    int tri = 0;
    (void)trd; (void)tri;
    for (int G = 0; G < total; ++G) {
      SG_TR(trd, 2, tri, 0);
      mbar_wait_sleep(dq_full, G & 1);
      tc_fence_after();
      SG_TR(trd, 2, tri, 1);
#ifdef SG_EXP_NODRAIN
      {
        __syncwarp();
        if (lane == 0) mbar_arrive(dq_empty);
        if (i == nqb - 1) {
          mbar_wait_sleep(acc_full, it & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);
          i = 0;
          ++it;
          if (it < my_items) item(it, kb, h, b);
        } else {
          ++i;
        }
        continue;
      }
#endif
      {
        uint32_t v[2][32];
        tmem_ld32(t_dq + lane_base, v[0]);
        tmem_ld32(t_dq + lane_base + 32, v[1]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dq_empty);
        // two 32 x 32 fp32 boxes, each with its own staging slot: box hf of block G waits
        // only for box hf of block G-1 to have been read by its reduce-add
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint8_t* box = stg + hf * 4096;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          SG_TR(trd, 2, tri, 2 + hf);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<float4*>(box + lane * 128 + ((k ^ (lane & 7)) << 4)) =
                make_float4(__uint_as_float(v[hf][4 * k]), __uint_as_float(v[hf][4 * k + 1]),
                            __uint_as_float(v[hf][4 * k + 2]), __uint_as_float(v[hf][4 * k + 3]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (p.dq_b2_first)
              tma_reduce_add_4d(&tmDQ, box, hf * 32, h, i * 128 + q * 32, b);
            else
              tma_reduce_add_4d(&tmDQ, box, hf * 32, i * 128 + q * 32, h, b);
            bulk_commit();
          }
        }
      }
      SG_TR(trd, 2, tri, 4);
      if (i == nqb - 1) {
        // this item's dK and dV: TMEM -> registers (both read before the accumulators are
        // released), bf16 rows straight to global memory (thread = key row, 128 B each)
        mbar_wait_sleep(acc_full, it & 1);
        tc_fence_after();
        SG_TR(trd, 2, tri, 5);
        uint32_t kp[32];
        {
          uint32_t v2[2][32];
          tmem_ld32(t_dk + lane_base, v2[0]);
          tmem_ld32(t_dk + lane_base + 32, v2[1]);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(v2[j >> 4][(2 * j) & 31]),
                                                      __uint_as_float(v2[j >> 4][(2 * j + 1) & 31]));
            kp[j] = *reinterpret_cast<uint32_t*>(&hh);
          }
        }
        uint32_t vp[32];
        {
          uint32_t v2[2][32];
          tmem_ld32(t_dv + lane_base, v2[0]);
          tmem_ld32(t_dv + lane_base + 32, v2[1]);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);  // the next item's dK / dV may overwrite TMEM
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(v2[j >> 4][(2 * j) & 31]),
                                                      __uint_as_float(v2[j >> 4][(2 * j + 1) & 31]));
            vp[j] = *reinterpret_cast<uint32_t*>(&hh);
          }
        }
        // staging: dK into box 0, dV into box 1 (each two SW64 32 x 32 bf16 tiles), each
        // once the reduce-add before it has read the box; TMA stores; bias-gradient column
        // sums read back from the staged tiles (rows past s hold zeros)
        const int key0 = kb * 128 + q * 32;
#pragma unroll 1
        for (int which = 0; which < 2; ++which) {
          uint8_t* box = stg + which * 4096;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint8_t* row = box + hf * 2048 + lane * 64;
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) {
              const int j = hf * 16 + 4 * k2;
              const uint4 x = which == 0 ? make_uint4(kp[j], kp[j + 1], kp[j + 2], kp[j + 3])
                                         : make_uint4(vp[j], vp[j + 1], vp[j + 2], vp[j + 3]);
              *reinterpret_cast<uint4*>(row + ((k2 ^ ((lane >> 1) & 3)) << 4)) = x;
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const CUtensorMap* tm = which == 0 ? &tmDK : &tmDV;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              if (p.dkv_b2_first)
                tma_store_4d(tm, box + hf * 2048, hf * 32, h, key0, b);
              else
                tma_store_4d(tm, box + hf * 2048, hf * 32, key0, h, b);
            }
            bulk_commit();
          }
          if (p.kv_colsum) {
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const uint8_t* tile = box + hf * 2048;
              float acc2[2] = {0.f, 0.f};
#pragma unroll
              for (int i2 = 0; i2 < 32; ++i2) {
                const int off = i2 * 64 + ((((lane >> 3) ^ ((i2 >> 1) & 3))) << 4) + (lane & 7) * 2;
                acc2[i2 & 1] += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(tile + off));
              }
              atomicAdd(p.kv_colsum + which * p.nh * 64 + h * 64 + hf * 32 + lane, acc2[0] + acc2[1]);
            }
          }
        }
        SG_TR(trd, 2, tri, 6);
        i = 0;
        ++it;
        if (it < my_items) item(it, kb, h, b);
      } else {
        ++i;
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}


constexpr uint32_t kT128 = 128 * 128 * 2;  // one 128 x 128 bf16 tile (2 atoms, 32 KB)

// ----------------------------------------------------------------------------
// Backward (d = 128), transposed orientation (round 2): the d = 64 design with the
// shared-memory and TMEM budgets of 128-wide tiles. Per query block G of an item:
//   S^T = K Q^T, dP^T = V dO^T (M = keys); P^T packed over the consumed scores of S^T,
//   dS^T packed over dP^T (TS A operands of dV += P^T dO, dK += dS^T Q); dS once into
//   shared memory as the MN-major A operand of dQ = dS K, whose accumulator reuses the
//   dP^T columns after dK has read dS^T.
// TMEM: S^T 0..127 | dP^T (dS^T, then dQ) 128..255 | dV 256..383 | dK 384..511.
// Per block the MMA warp issues dV_G (as soon as P^T_G is in TMEM), S^T_G+1 (it
// overwrites P^T_G after dV_G, in issue order), dK_G and dQ_G (once dS_G exists) and
// dP^T_G+1 (once the drain warps have read dQ_G), so the exponentials of block G+1 run
// while dK_G / dQ_G / dP^T_G+1 execute. Shared memory (226.75 KB): K 2 x 32 KB
// (items), V 32 KB, Q 2 x 32 KB, dO 32 KB, dS 32 KB — the drain warps stage dQ and,
// at an item's end, dK / dV through the dS buffer once dQ_G has read it (the softmax
// warps write dS_G+1 after the drain released it).
// ----------------------------------------------------------------------------
constexpr int kMaxItems128 = 128;

__global__ void __launch_bounds__(512, 1)
    flash_bwd3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                      const __grid_constant__ CUtensorMap tmDQ, const __grid_constant__ CUtensorMap tmDK,
                      const __grid_constant__ CUtensorMap tmDV, const __grid_constant__ FlashBwdParams p, int bsz) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();
  uint8_t* sK = smem;                   // 2 slots (items) x 2 atoms
  uint8_t* sV = sK + 2 * kT128;         // 1 slot
  uint8_t* sQ = sV + kT128;             // 2 slots (query blocks)
  uint8_t* sDO = sQ + 2 * kT128;        // 1 slot
  uint8_t* sDS = sDO + kT128;           // [keys x queries] 2 atoms; drain staging between uses
  float* sStat = reinterpret_cast<float*>(sDS + kT128);  // 2 slots x [128 -lse log2e | 128 -D scale]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStat + 2 * 256);
  int* items_tab = reinterpret_cast<int*>(bars + 32);
  uint64_t* k_full = bars;          // [2]
  uint64_t* k_empty = bars + 2;     // [2]
  uint64_t* v_full = bars + 4;
  uint64_t* v_empty = bars + 5;
  uint64_t* q_full = bars + 6;      // [2]
  uint64_t* q_empty = bars + 8;     // [2] dK_G done
  uint64_t* do_full = bars + 10;
  uint64_t* do_empty = bars + 11;   // dV_G done (dO free, P^T read)
  uint64_t* s_full = bars + 12;
  uint64_t* p_full = bars + 13;     // P^T_G in TMEM (8 softmax warps)
  uint64_t* dp_full = bars + 14;
  uint64_t* ds_full = bars + 15;    // dS^T_G in TMEM, dS_G in smem (8 softmax warps)
  uint64_t* dq_full = bars + 16;    // dQ_G done (dS buffer no longer read by the MMA)
  uint64_t* dq_empty = bars + 17;   // 4 drain warps: dQ_G read out of TMEM
  uint64_t* stg_free = bars + 18;   // 4 drain warps: staging in the dS buffer read by the TMA
  uint64_t* acc_full = bars + 19;
  uint64_t* acc_empty = bars + 20;  // 4 drain warps
  uint64_t* st_full = bars + 21;    // [2] statistics of block G in slot G & 1 (warp 3)
  uint64_t* st_empty = bars + 23;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (p.s + 127) / 128;
  const int nkb = nqb;
  const int n_items = nkb * p.nh * bsz;
  auto decode = [&](int t, int& kb, int& h, int& b) {
    kb = t % nkb;
    const int r = t / nkb;
    h = r % p.nh;
    b = r / p.nh + p.b0;
  };
  const int my_items = n_items > (int)blockIdx.x ? (n_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = my_items * nqb;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
    tma_prefetch_desc(&tmDQ);
    tma_prefetch_desc(&tmDK);
    tma_prefetch_desc(&tmDV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&st_full[i], 32);
      mbar_init(&st_empty[i], 8);
    }
    mbar_init(v_full, 1);
    mbar_init(v_empty, 1);
    mbar_init(do_full, 1);
    mbar_init(do_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(p_full, 8);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 8);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 4);
    mbar_init(stg_free, 4);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  for (int it = threadIdx.x; it < my_items && it < kMaxItems128; it += blockDim.x) {
    int kb, h, b;
    decode((int)blockIdx.x + it * (int)gridDim.x, kb, h, b);
    items_tab[it] = kb | (h << 10) | ((b - p.b0) << 20);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_begin();
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 384, t_dq = tmem + 128;
  auto item = [&](int it, int& kb, int& h, int& b) {
    const int v = items_tab[it];
    kb = v & 1023;
    h = (v >> 10) & 1023;
    b = (v >> 20) + p.b0;
  };

  if (warp == 0) {
    reg_dealloc<56>();
    if (lane == 0) {
      int G = 0;
      for (int t = blockIdx.x, it = 0; t < n_items; t += gridDim.x, ++it) {
        int kb, h, b;
        decode(t, kb, h, b);
        const int ks = it & 1;
        mbar_wait_sleep(&k_empty[ks], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[ks], kT128);
#pragma unroll
        for (int a = 0; a < 2; ++a) tma4(&tmK, sK + ks * kT128 + a * kT64, &k_full[ks], a * 64, kb * 128, h, b, p.k_b2_first);
        for (int i = 0; i < nqb; ++i, ++G) {
          {
            // Q / dO of block G + 2 into L2 now
            int i2 = i + 2, t2 = t, kb2 = kb, h2 = h, b2 = b;
            while (i2 >= nqb) {
              i2 -= nqb;
              t2 += gridDim.x;
            }
            if (t2 != t && t2 < n_items) decode(t2, kb2, h2, b2);
            if (t2 < n_items) {
#pragma unroll
              for (int a = 0; a < 2; ++a) {
                tma4_l2(&tmQ, a * 64, i2 * 128, h2, b2, p.q_b2_first);
                tma4_l2(&tmDO, a * 64, i2 * 128, h2, b2, p.do_b2_first);
              }
            }
          }
          const int qs = G & 1;
          mbar_wait_sleep(&q_empty[qs], ((G >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[qs], kT128);
#pragma unroll
          for (int a = 0; a < 2; ++a) tma4(&tmQ, sQ + qs * kT128 + a * kT64, &q_full[qs], a * 64, i * 128, h, b, p.q_b2_first);
          if (i == 0) {
            // this item's V once the previous item's last dP^T has read the slot
            mbar_wait_sleep(v_empty, (it & 1) ^ 1);
            mbar_arrive_expect_tx(v_full, kT128);
#pragma unroll
            for (int a = 0; a < 2; ++a) tma4(&tmV, sV + a * kT64, v_full, a * 64, kb * 128, h, b, p.v_b2_first);
          }
          mbar_wait_sleep(do_empty, (G & 1) ^ 1);
          mbar_arrive_expect_tx(do_full, kT128);
#pragma unroll
          for (int a = 0; a < 2; ++a) tma4(&tmDO, sDO + a * kT64, do_full, a * 64, i * 128, h, b, p.do_b2_first);
        }
      }
    }
  } else if (warp == 1) {
    reg_dealloc<56>();
    {
      // whole warp walks the loop (warp-uniform operands); one elected lane issues
      constexpr uint32_t ID_ST = umma_idesc_bf16(128, 128, false, false);  // S^T, dP^T: K-major over d
      constexpr uint32_t ID_KV = umma_idesc_bf16(128, 128, false, true);   // dV, dK: A TMEM, B = dO / Q MN-major
      constexpr uint32_t ID_DQ = umma_idesc_bf16(128, 128, true, true);    // dQ: A = dS MN-major, B = K MN-major
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t ts = tm, tdp = tm + 128, tdv = tm + 256, tdk = tm + 384;
      constexpr uint64_t kAtom = kT64 >> 4, kTile = kT128 >> 4;
      const uint64_t k_k = umma_desc_sw128(smem_u32(sK), 0, 1024), v_k = umma_desc_sw128(smem_u32(sV), 0, 1024);
      const uint64_t q_k = umma_desc_sw128(smem_u32(sQ), 0, 1024), do_k = umma_desc_sw128(smem_u32(sDO), 0, 1024);
      const uint64_t q_m = umma_desc_sw128(smem_u32(sQ), kT64, 1024), do_m = umma_desc_sw128(smem_u32(sDO), kT64, 1024);
      const uint64_t k_m = umma_desc_sw128(smem_u32(sK), kT64, 1024), ds_m = umma_desc_sw128(smem_u32(sDS), kT64, 1024);
      auto issue_s = [&](int G) {  // S^T_G = K Q_G^T
        const int it = G / nqb;
        if (G % nqb == 0) mbar_wait(&k_full[it & 1], (it >> 1) & 1);
        mbar_wait(&q_full[G & 1], (G >> 1) & 1);
        tc_fence_after();
        const uint64_t kd = k_k + (it & 1) * kTile, qd = q_k + (G & 1) * kTile;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // K-dim = d = 128: two atoms of 4 x 16
            const uint64_t off = (kk >> 2) * kAtom + (kk & 3) * 2;
            umma_bf16(ts, kd + off, qd + off, ID_ST, kk > 0 ? 1u : 0u);
          }
          umma_commit(s_full);
        }
        __syncwarp();
      };
      auto issue_dp = [&](int G) {  // dP^T_G = V dO_G^T
        const int it = G / nqb;
        if (G % nqb == 0) mbar_wait(v_full, it & 1);
        mbar_wait(do_full, G & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t off = (kk >> 2) * kAtom + (kk & 3) * 2;
            umma_bf16(tdp, v_k + off, do_k + off, ID_ST, kk > 0 ? 1u : 0u);
          }
          umma_commit(dp_full);
          if (G % nqb == nqb - 1) umma_commit(v_empty);  // the item's last dP^T: V may be reloaded
        }
        __syncwarp();
      };
      if (total > 0) {
        issue_s(0);
        issue_dp(0);
      }
      for (int G = 0; G < total; ++G) {
        const int it = G / nqb, i = G % nqb;
        mbar_wait(p_full, G & 1);  // P^T_G in TMEM (S^T_G read)
        tc_fence_after();
        if (i == 0 && it > 0) {  // the previous item's dK / dV read out
          mbar_wait(acc_empty, (it - 1) & 1);
          tc_fence_after();
        }
        if (elect_one()) {
#pragma unroll
          for (int kq = 0; kq < 8; ++kq)  // dV += P^T dO: 16 queries = 8 packed columns / 16 rows per step
            umma_bf16_ts(tdv, ts + (kq >> 2) * 64 + (kq & 3) * 8, do_m + 128 * kq, ID_KV, (i | kq) != 0 ? 1u : 0u);
          umma_commit(do_empty);  // dO_G free, P^T_G read
        }
        __syncwarp();
        if (G + 1 < total) issue_s(G + 1);  // overwrites P^T_G after dV_G (issue order)
        mbar_wait(ds_full, G & 1);  // dS^T_G in TMEM, dS_G in smem
        tc_fence_after();
        const uint64_t qm = q_m + (G & 1) * kTile, km = k_m + (it & 1) * kTile;
        if (elect_one()) {
#pragma unroll
          for (int kq = 0; kq < 8; ++kq)  // dK += dS^T Q
            umma_bf16_ts(tdk, tdp + (kq >> 2) * 64 + (kq & 3) * 8, qm + 128 * kq, ID_KV, (i | kq) != 0 ? 1u : 0u);
          umma_commit(&q_empty[G & 1]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // dQ = dS K into the dP^T columns (after dK read dS^T)
            umma_bf16(tdp, ds_m + 128 * kk, km + 128 * kk, ID_DQ, kk > 0 ? 1u : 0u);
          umma_commit(dq_full);
          if (i == nqb - 1) {
            umma_commit(acc_full);
            umma_commit(&k_empty[it & 1]);
          }
        }
        __syncwarp();
        if (G + 1 < total) {
          mbar_wait(dq_empty, G & 1);  // dQ_G read out of the dP^T columns
          tc_fence_after();
          issue_dp(G + 1);
        }
      }
    }
  } else if (warp == 3) {
    reg_dealloc<56>();
    float v[8];
    auto load = [&](int G, float (&x)[8]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] = INFINITY;
        x[4 + u] = 0.f;
      }
      if (G >= total) return;
      int kb, h, b;
      item(G / nqb, kb, h, b);
      const size_t off = ((size_t)b * p.nh + h) * p.s;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int qrow = (G % nqb) * 128 + u * 32 + lane;
        if (qrow < p.s) {
          x[u] = __ldg(p.lse + off + qrow);
          x[4 + u] = __ldg(p.drow + off + qrow);
        }
      }
    };
    load(0, v);
    for (int G = 0; G < total; ++G) {
      float* t = sStat + (G & 1) * 256;
      if (G >= 2) mbar_wait_sleep(&st_empty[G & 1], ((G - 2) >> 1) & 1);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        t[u * 32 + lane] = -v[u] * 1.4426950408889634f;
        t[128 + u * 32 + lane] = -v[4 + u] * p.scale;
      }
      mbar_arrive(&st_full[G & 1]);
      load(G + 1, v);
    }
  } else if (warp < 4) {
    reg_dealloc<56>();
  } else if (warp < 12) {
    reg_alloc<160>();
    const int e = warp - 4;
    const int q = e & 3, hq = e >> 2;
    const int r = q * 32 + lane;  // key row of the block
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const float scale = p.scale;
    int it = 0, i = 0;
    int kb = 0, h = 0, b = 0;
    if (my_items > 0) item(0, kb, h, b);
    const uint64_t sl2 = f2_pack(p.scale_log2, p.scale_log2), sc2 = f2_pack(scale, scale);
    for (int G = 0; G < total; ++G) {
      const int kvalid = min(128, p.s - kb * 128);
      const float* st = sStat + (G & 1) * 256 + hq * 64;
      mbar_wait_sleep(s_full, G & 1);
      mbar_wait_sleep(&st_full[G & 1], (G >> 1) & 1);
      tc_fence_after();
      uint32_t sv[64];
      tmem_ld32(t_s + lane_base + hq * 64, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
      tmem_ld32(t_s + lane_base + hq * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
      tmem_wait_ld();
      uint32_t pk[32];
      const bool key_ok = r < kvalid;
#pragma unroll
      for (int j4 = 0; j4 < 16; ++j4) {
        const float4 nl = *reinterpret_cast<const float4*>(st + 4 * j4);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = 2 * j4 + u;
          const uint64_t y = ffma2(f2_pack(__uint_as_float(sv[2 * j]), __uint_as_float(sv[2 * j + 1])), sl2,
                                   u ? f2_pack(nl.z, nl.w) : f2_pack(nl.x, nl.y));
          const float p0 = ex2f_fast(f2_lo(y)), p1 = ex2f_fast(f2_hi(y));
          sv[2 * j] = __float_as_uint(p0);
          sv[2 * j + 1] = __float_as_uint(p1);
          __nv_bfloat162 hp = __floats2bfloat162_rn(p0, p1);
          pk[j] = *reinterpret_cast<uint32_t*>(&hp);
        }
      }
      if (kvalid < 128 && !key_ok) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          sv[2 * j] = sv[2 * j + 1] = 0u;
          pk[j] = 0u;
        }
      }
      // P^T packed over this thread's own (already read) score columns
      tmem_st32(t_s + lane_base + hq * 64, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      mbar_wait_sleep(dp_full, G & 1);
      tc_fence_after();
      uint32_t dk[32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t dv[32];
        tmem_ld32(t_dp + lane_base + hq * 64 + c * 32, dv);
        tmem_wait_ld();
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 nd = *reinterpret_cast<const float4*>(st + 128 + c * 32 + 4 * j4);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int j = 2 * j4 + u;
            const uint64_t t = ffma2(f2_pack(__uint_as_float(dv[2 * j]), __uint_as_float(dv[2 * j + 1])), sc2,
                                     u ? f2_pack(nd.z, nd.w) : f2_pack(nd.x, nd.y));
            const uint64_t ds =
                fmul2(f2_pack(__uint_as_float(sv[c * 32 + 2 * j]), __uint_as_float(sv[c * 32 + 2 * j + 1])), t);
            __nv_bfloat162 hd = __floats2bfloat162_rn(f2_lo(ds), f2_hi(ds));
            dk[c * 16 + j] = *reinterpret_cast<uint32_t*>(&hd);
          }
        }
      }
      tmem_st32(t_dp + lane_base + hq * 64, dk);
      __syncwarp();
      if (lane == 0) mbar_arrive(&st_empty[G & 1]);
      if (G > 0) mbar_wait_sleep(stg_free, (G - 1) & 1);  // the drain warps released the dS buffer
      uint8_t* drow_ = sDS + hq * kT64 + r * 128;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        *reinterpret_cast<uint4*>(drow_ + ((k ^ (r & 7)) << 4)) =
            make_uint4(dk[4 * k], dk[4 * k + 1], dk[4 * k + 2], dk[4 * k + 3]);
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      if (i == nqb - 1) {
        i = 0;
        ++it;
        if (it < my_items) item(it, kb, h, b);
      } else {
        ++i;
      }
    }
  } else {
    // 4 drain warps (lane quadrant q): dQ_G (TMEM dP^T columns -> fp32 boxes in this warp's
    // 8 KB of the dS buffer -> TMA reduce-add), at an item's end dK / dV (bf16 boxes ->
    // TMA stores, bias-gradient column sums); then the dS buffer is released
    reg_alloc<128>();
    const int q = warp & 3;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    uint8_t* stg = sDS + (warp - 12) * 8192;
    int it = 0, i = 0, kb = 0, h = 0, b = 0;
    if (my_items > 0) item(0, kb, h, b);
    for (int G = 0; G < total; ++G) {
      mbar_wait_sleep(dq_full, G & 1);  // dQ_G done: the MMA no longer reads dS_G
      tc_fence_after();
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        uint32_t v[2][32];
        tmem_ld32(t_dq + lane_base + half * 64, v[0]);
        tmem_ld32(t_dq + lane_base + half * 64 + 32, v[1]);
        tmem_wait_ld();
        if (half == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dq_empty);  // dP^T_G+1 may overwrite the columns
        }
        if (lane == 0) bulk_wait_read<0>();  // the boxes' previous reduce-adds have read them
        __syncwarp();
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint8_t* box = stg + hf * 4096;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<float4*>(box + lane * 128 + ((k ^ (lane & 7)) << 4)) =
                make_float4(__uint_as_float(v[hf][4 * k]), __uint_as_float(v[hf][4 * k + 1]),
                            __uint_as_float(v[hf][4 * k + 2]), __uint_as_float(v[hf][4 * k + 3]));
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            const int col = half * 64 + hf * 32;
            if (p.dq_b2_first)
              tma_reduce_add_4d(&tmDQ, stg + hf * 4096, col, h, i * 128 + q * 32, b);
            else
              tma_reduce_add_4d(&tmDQ, stg + hf * 4096, col, i * 128 + q * 32, h, b);
          }
          bulk_commit();
        }
      }
      if (i == nqb - 1) {
        mbar_wait_sleep(acc_full, it & 1);
        tc_fence_after();
        const int key0 = kb * 128 + q * 32;
#pragma unroll 1
        for (int which = 0; which < 2; ++which) {
          // 128 columns as four SW64 32 x 32 bf16 tiles (2 KB each) in this warp's 8 KB
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            uint32_t v2[2][32];
            tmem_ld32((which == 0 ? t_dk : t_dv) + lane_base + half * 64, v2[0]);
            tmem_ld32((which == 0 ? t_dk : t_dv) + lane_base + half * 64 + 32, v2[1]);
            tmem_wait_ld();
            if (which == 1 && half == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(acc_empty);  // the next item's dK / dV may overwrite TMEM
            }
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              uint8_t* row = stg + (half * 2 + hf) * 2048 + lane * 64;
#pragma unroll
              for (int k2 = 0; k2 < 4; ++k2) {
                uint4 x;
                __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&x);
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2)
                  hh[e2] = __floats2bfloat162_rn(__uint_as_float(v2[hf][8 * k2 + 2 * e2]),
                                                 __uint_as_float(v2[hf][8 * k2 + 2 * e2 + 1]));
                *reinterpret_cast<uint4*>(row + ((k2 ^ ((lane >> 1) & 3)) << 4)) = x;
              }
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const CUtensorMap* tmap = which == 0 ? &tmDK : &tmDV;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if (p.dkv_b2_first)
                tma_store_4d(tmap, stg + c * 2048, c * 32, h, key0, b);
              else
                tma_store_4d(tmap, stg + c * 2048, c * 32, key0, h, b);
            }
            bulk_commit();
          }
          if (p.kv_colsum) {
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              const uint8_t* tile = stg + c * 2048;
              float acc2[2] = {0.f, 0.f};
#pragma unroll
              for (int i2 = 0; i2 < 32; ++i2) {
                const int off = i2 * 64 + ((((lane >> 3) ^ ((i2 >> 1) & 3))) << 4) + (lane & 7) * 2;
                acc2[i2 & 1] += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(tile + off));
              }
              atomicAdd(p.kv_colsum + which * p.nh * 128 + h * 128 + c * 32 + lane, acc2[0] + acc2[1]);
            }
          }
        }
      }
      // release the dS buffer once every staged box has been read by its TMA operation
      if (lane == 0) bulk_wait_read<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(stg_free);
      if (i == nqb - 1) {
        i = 0;
        ++it;
        if (it < my_items) item(it, kb, h, b);
      } else {
        ++i;
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}


}  // namespace sg

extern "C" int sg_flash_attn_bwd(const void* qkv, int64_t ldq, const void* dout, int64_t lddo, const float* lse,
                                 const float* drow, int64_t b, int64_t s, int64_t nh, int64_t d, float* dq_acc,
                                 int64_t lddq, void* dqkv, int64_t ldg, float* kv_colsum, void* stream) {
  using namespace sg;
  clear_error();
  if (b < 1 || s < 1 || nh < 1 || (d != 64 && d != 128)) return set_error(SG_ERR_SHAPE, "flash bwd: d must be 64 or 128");
  if (ldq < 3 * nh * d || lddo < nh * d || lddq < nh * d || ldg < 3 * nh * d)
    return set_error(SG_ERR_SHAPE, "flash bwd: leading dimensions");
  if ((reinterpret_cast<uintptr_t>(dqkv) & 15) || (ldg * 2) % 16) return set_error(SG_ERR_SHAPE, "flash bwd: unaligned");
  const __nv_bfloat16* base = static_cast<const __nv_bfloat16*>(qkv);
  const long long hb = nh * d;
  CUtensorMap tq, tk, tv, tdo, tdq, tdk, tdv;
  FlashBwdParams p{};
  p.s = (int)s;
  p.nh = (int)nh;
  p.scale = 1.f / sqrtf((float)d);
  p.scale_log2 = 1.4426950408889634f * p.scale;
  p.lse = lse;
  p.drow = drow;
  p.dK = static_cast<__nv_bfloat16*>(dqkv) + hb;
  p.dV = static_cast<__nv_bfloat16*>(dqkv) + 2 * hb;
  p.ldg = ldg;
  p.kv_colsum = kv_colsum;
  int rc = tmap_bf16_4d(&tq, base, d, s, nh, b, ldq, d, s * ldq, 64, 128, &p.q_b2_first);
  if (!rc) rc = tmap_bf16_4d(&tk, base + hb, d, s, nh, b, ldq, d, s * ldq, 64, 128, &p.k_b2_first);
  if (!rc) rc = tmap_bf16_4d(&tv, base + 2 * hb, d, s, nh, b, ldq, d, s * ldq, 64, 128, &p.v_b2_first);
  if (!rc) rc = tmap_bf16_4d(&tdo, dout, d, s, nh, b, lddo, d, s * lddo, 64, 128, &p.do_b2_first);
  if (!rc) rc = tmap_f32_tile_4d(&tdq, dq_acc, d, s, nh, b, lddq, d, s * lddq, &p.dq_b2_first);
  if (!rc) rc = tmap_bf16_tile_4d(&tdk, p.dK, d, s, nh, b, ldg, d, s * ldg, &p.dkv_b2_first);
  if (!rc) rc = tmap_bf16_tile_4d(&tdv, p.dV, d, s, nh, b, ldg, d, s * ldg, &p.dkv_b2_first);
  if (rc) return rc;
  // d = 64: 2 K, V, kQD Q, kQD dO, dS (2 atoms), 4 x 8 KB staging, 8 x 512 B statistics;
  // d = 128: K, V, Q, dO, P, dS as 32 KB tiles, 4 x 8 KB staging
  constexpr size_t SMEM64 = (3 + 2 * kQD + 2) * kT64 + 4 * 8192 + 2 * 1024 + 256 + kMaxItems * 4;
  constexpr size_t SMEM128T = 7 * kT128 + 2 * 1024 + 256 + kMaxItems128 * 4;
  const bool t128 = d == 128;
  const int nkb = (int)((s + 127) / 128);
  const int sms = sg_device_sm_count() > 0 ? sg_device_sm_count() : 148;
  if (nkb > 1024 || nh > 1024) return set_error(SG_ERR_SHAPE, "flash bwd: more than 1024 key blocks / heads");
  // sequences per launch: every CTA's items must fit its item table (large batches run
  // as several back-to-back launches over batch chunks)
  const long long per_seq = (long long)nkb * nh;
  const long long table = t128 ? kMaxItems128 : kMaxItems;  // per-CTA item table entries
  long long max_items = table * sms;
  if (const char* e = getenv("SG_FLASH_ITEMS_MAX")) max_items = std::max(1LL, std::min(max_items, atoll(e)));  // tests
  const int chunk = (int)std::max<long long>(1, std::min<long long>(2047, max_items / per_seq));
  if (per_seq > table * sms) return set_error(SG_ERR_SHAPE, "flash bwd: one sequence exceeds the item table");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const void* kern = d == 64 ? reinterpret_cast<const void*>(flash_bwd2_kernel<kBwdPoly>)
                             : reinterpret_cast<const void*>(flash_bwd3_kernel);
  if (!ensure_smem(kern, (int)(d == 64 ? SMEM64 : SMEM128T)))
    return set_error(SG_ERR_CUDA, "flash bwd: smem attribute");
  for (long long b0 = 0; b0 < b; b0 += chunk) {
    const int bc = (int)std::min<long long>(chunk, b - b0);
    const int items = (int)(per_seq * bc);
    p.b0 = (int)b0;
    if (d == 64)
      launch_k(flash_bwd2_kernel<kBwdPoly>, dim3(std::min(items, sms)), dim3(512), SMEM64, st, tq, tk, tv, tdo, tdq,
               tdk, tdv, p, bc);
    else
      launch_k(flash_bwd3_kernel, dim3(std::min(items, sms)), dim3(512), SMEM128T, st, tq, tk, tv, tdo, tdq, tdk,
               tdv, p, bc);
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}
