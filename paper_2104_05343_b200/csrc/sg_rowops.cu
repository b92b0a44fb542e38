// HBM-bound per-device kernels of the 2D transformer: LayerNorm (two-phase,
// so only the per-row (sum, sumsq) / (sum x^ g, sum g) scalars cross the mesh
// row), attention softmax and its backward, vocab-parallel cross entropy,
// embedding gather / scatter-add, bias column sums, SGD and the ordered
// element-wise folds the single-GPU mesh simulation uses for its reduces.
//
// Row kernels map one warp to one row and move 8 elements per lane per step
// with 16-byte vector accesses (bf16) or 2x16-byte (fp32); grids are sized as
// multiples of the SM count. Reference math: layers.py:253-351 (LayerNorm),
// dense.py:67-75 + layers.py:444-452 (softmax fwd/bwd), layers.py:539-624
// (cross entropy), layers.py:151-211 (embedding), layers.py:218-246 (bias).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstdint>

#include "sg.h"
#include "sg_internal.h"
#include "sg_ptx.cuh"

namespace sg {

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- 8-wide element access (n = number of valid elements, <= 8) ----------
__device__ __forceinline__ void ld8(const float* p, int n, float (&v)[8]) {
  if (n == 8) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < n ? p[i] : 0.f;
  }
}
__device__ __forceinline__ void ld8(const bf16* p, int n, float (&v)[8]) {
  if (n == 8) {
    uint4 a = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x; v[2 * i + 1] = f.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < n ? __bfloat162float(p[i]) : 0.f;
  }
}
__device__ __forceinline__ void st8(float* p, int n, const float (&v)[8]) {
  if (n == 8) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < n) p[i] = v[i];
  }
}
__device__ __forceinline__ void st8(bf16* p, int n, const float (&v)[8]) {
  if (n == 8) {
    uint4 a;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = a;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < n) p[i] = __float2bfloat16_rn(v[i]);
  }
}

// Raw 8-element vectors: the load is one (bf16) or two (fp32) 16-byte accesses
// into registers and the conversion to float happens later, so a kernel can
// issue every load of a row group before the first one is consumed (a
// conversion right after each load, as in ld8's mixed vector / scalar path,
// serialises the loads on the scoreboard).
template <typename T>
struct Vec8;
template <>
struct Vec8<float> {
  float4 a, b;
  __device__ __forceinline__ void load(const float* p) {
    a = *reinterpret_cast<const float4*>(p);
    b = *reinterpret_cast<const float4*>(p + 4);
  }
  __device__ __forceinline__ void to(float (&v)[8]) const {
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
};
template <>
struct Vec8<bf16> {
  uint4 a;
  __device__ __forceinline__ void load(const bf16* p) { a = *reinterpret_cast<const uint4*>(p); }
  __device__ __forceinline__ void to(float (&v)[8]) const {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x; v[2 * i + 1] = f.y;
    }
  }
};

template <typename T>
__device__ __forceinline__ float ld1(const T* p);
template <>
__device__ __forceinline__ float ld1<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld1<bf16>(const bf16* p) { return __bfloat162float(*p); }

static int g_sms = 0;
static int grid_for(long long work_items, int per_block, int waves = 8) {
  if (g_sms <= 0) g_sms = sg_device_sm_count();
  long long need = (work_items + per_block - 1) / per_block;
  long long cap = (long long)(g_sms > 0 ? g_sms : 148) * waves;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

static int launch_check() {
  count_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SG_OK : set_error(SG_ERR_CUDA, cudaGetErrorString(e));
}

static bool aligned16(const void* p, long long ld, int esz) {
  return p == nullptr || ((reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld * esz) % 16 == 0);
}

#define SG_DISPATCH_T(dt, T, ...)            \
  do {                                       \
    if ((dt) == SG_DTYPE_F32) {              \
      typedef float T;                       \
      __VA_ARGS__;                           \
    } else {                                 \
      typedef bf16 T;                        \
      __VA_ARGS__;                           \
    }                                        \
  } while (0)

// ============================================================ LayerNorm
// stats[row] = (sum x, sum x^2) over the local columns (layers.py:274-275)
template <typename TX>
__global__ void ln_stats_kernel(const TX* __restrict__ x, long long rows, int cols, long long ldx,
                                float* __restrict__ stats) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw) {
    const TX* xr = x + r * ldx;
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane * 8; c < cols; c += 256) {
      float v[8];
      ld8(xr + c, min(8, cols - c), v);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s1 += v[i];
        s2 += v[i] * v[i];
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      stats[2 * r] = s1;
      stats[2 * r + 1] = s2;
    }
  }
}

// y = (x - mu) * rstd * gamma + beta with mu, var from the (row all-reduced)
// stats or, when stats == nullptr, from this device's row (1 x c == 1 x 1).
template <typename TX, typename TY>
__global__ void ln_fwd_kernel(const TX* __restrict__ x, long long rows, int cols, long long ldx,
                              const float* __restrict__ stats, float inv_h, float eps,
                              const float* __restrict__ gamma, const float* __restrict__ beta, TY* __restrict__ y,
                              long long ldy, float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw) {
    const TX* xr = x + r * ldx;
    float s1, s2;
    if (stats) {
      s1 = stats[2 * r];
      s2 = stats[2 * r + 1];
    } else {
      s1 = 0.f;
      s2 = 0.f;
      for (int c = lane * 8; c < cols; c += 256) {
        float v[8];
        ld8(xr + c, min(8, cols - c), v);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          s1 += v[i];
          s2 += v[i] * v[i];
        }
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
    }
    const float mu = s1 * inv_h;
    const float var = fmaxf(s2 * inv_h - mu * mu, 0.f);  // one-pass variance (layers.py:296-297), clamped: fp32 cancellation on near-constant rows
    const float rs = rsqrtf(var + eps)  /* MUFU.RSQ: no IEEE-division slow-path call */;
    for (int c = lane * 8; c < cols; c += 256) {
      const int n = min(8, cols - c);
      float v[8], g[8], b[8];
      ld8(xr + c, n, v);
      ld8(gamma + c, n, g);
      ld8(beta + c, n, b);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = (v[i] - mu) * rs * g[i] + b[i];
      st8(y + r * ldy + c, n, v);
    }
    if (lane == 0) {
      if (mean_out) mean_out[r] = mu;
      if (rstd_out) rstd_out[r] = rs;
    }
  }
}

// stats[row] = (sum x^ g, sum g), g = dy * gamma (layers.py:319-321)
template <typename TD, typename TX>
__global__ void ln_bwd_stats_kernel(const TD* __restrict__ dy, long long lddy, const TX* __restrict__ x,
                                    long long ldx, const float* __restrict__ mean, const float* __restrict__ rstd,
                                    const float* __restrict__ gamma, long long rows, int cols,
                                    float* __restrict__ stats) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw) {
    const float mu = mean[r], rs = rstd[r];
    float sxg = 0.f, sg = 0.f;
    for (int c = lane * 8; c < cols; c += 256) {
      const int n = min(8, cols - c);
      float d[8], v[8], g[8];
      ld8(dy + r * lddy + c, n, d);
      ld8(x + r * ldx + c, n, v);
      ld8(gamma + c, n, g);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float gg = d[i] * g[i];
        sxg += (v[i] - mu) * rs * gg;
        sg += gg;
      }
    }
    sxg = warp_sum(sxg);
    sg = warp_sum(sg);
    if (lane == 0) {
      stats[2 * r] = sxg;
      stats[2 * r + 1] = sg;
    }
  }
}

// ---- column-segment row kernels -------------------------------------------
// Kernels that also produce column sums (LayerNorm backward, GELU', bias
// gradients) use one layout: a block is 8 warps, blockIdx.y selects a
// 256-column segment, each lane owns 8 consecutive columns of it, and the warps
// sweep the rows RU at a time with every load of the RU rows issued before
// any use (memory-level parallelism without a huge per-thread footprint).
// Per-column partials stay in registers (8 per quantity) and are folded once
// per block through shared memory, then one atomic per column per block.
constexpr int kSegCols = 256;
constexpr int kSegWarps = 8;

template <int NQ>
__device__ __forceinline__ void seg_flush(float (&acc)[NQ][8], float* const (&dst)[NQ], int c0, int cols,
                                          float* sm /* [NQ][8 warps][256] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    float4* p = reinterpret_cast<float4*>(sm + (q * kSegWarps + warp) * kSegCols + lane * 8);
    p[0] = make_float4(acc[q][0], acc[q][1], acc[q][2], acc[q][3]);
    p[1] = make_float4(acc[q][4], acc[q][5], acc[q][6], acc[q][7]);
  }
  __syncthreads();
  const int t = threadIdx.x;  // one column per thread
  if (c0 + t < cols) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (!dst[q]) continue;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kSegWarps; ++w) s += sm[(q * kSegWarps + w) * kSegCols + t];
      atomicAdd(dst[q] + c0 + t, s);
    }
  }
}

static dim3 seg_grid(long long rows, long long cols, int ru, int blocks_per_sm) {
  if (g_sms <= 0) g_sms = sg_device_sm_count();
  const int segs = (int)((cols + kSegCols - 1) / kSegCols);
  const long long row_groups = (rows + (long long)kSegWarps * ru - 1) / ((long long)kSegWarps * ru);
  long long gx = std::max(1LL, (long long)(g_sms > 0 ? g_sms : 148) * blocks_per_sm / segs);
  gx = std::min(gx, std::max(1LL, row_groups));
  return dim3((unsigned)gx, (unsigned)segs);
}

// dx = rstd * (g - sum_g/h - x^ * sum_xg/h) [+ resid], g = dy * gamma; dgamma +=
// column sums of dy x^, dbeta += column sums of dy (layers.py:329-342) and dsum +=
// column sums of dx (the upstream bias gradient, layers.py:238).
template <typename TD, typename TX, typename TR, int RU, bool FULL>
__global__ void __launch_bounds__(256) ln_bwd_kernel(
    const TD* __restrict__ dy, long long lddy, const TX* __restrict__ x, long long ldx,
    const float* __restrict__ mean, const float* __restrict__ rstd, const float* __restrict__ gamma, long long rows,
    int cols, const float* __restrict__ stats, float inv_h, const TR* __restrict__ resid, long long ldr,
    float* __restrict__ dx, long long lddx, bf16* __restrict__ dx2, long long lddx2, float* __restrict__ dgamma,
    float* __restrict__ dbeta, float* __restrict__ dsum) {
  pdl_begin();
  __shared__ __align__(16) float sm[3 * kSegWarps * kSegCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.y * kSegCols;
  const int c = c0 + lane * 8;
  const int n = max(0, min(8, cols - c));
  // FULL (cols % 8 == 0): every lane loads unconditionally (idle lanes / rows past
  // the end read a clamped in-bounds address and discard it)
  const int cl = FULL ? min(c, cols - 8) : c;
  float g[8];
  if (FULL) {
    Vec8<float> gv;
    gv.load(gamma + cl);
    gv.to(g);
  } else if (n > 0) {
    ld8(gamma + c, n, g);
  }
  float acc[3][8];
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[q][i] = 0.f;
  const long long step = (long long)gridDim.x * kSegWarps * RU;
  for (long long r0 = ((long long)blockIdx.x * kSegWarps + warp) * RU; r0 < rows; r0 += step) {
    float d[RU][8], v[RU][8], o[RU][8];
    if (FULL) {
      Vec8<TD> rd[RU];
      Vec8<TX> rx[RU];
      Vec8<TR> ro[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const long long r = min(r0 + u, rows - 1);
        rd[u].load(dy + r * lddy + cl);
        rx[u].load(x + r * ldx + cl);
        if (resid) ro[u].load(resid + r * ldr + cl);
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        rd[u].to(d[u]);
        rx[u].to(v[u]);
        if (resid) {
          ro[u].to(o[u]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) o[u][i] = 0.f;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const long long r = r0 + u;
        if (r < rows && n > 0) {
          ld8(dy + r * lddy + c, n, d[u]);
          ld8(x + r * ldx + c, n, v[u]);
          if (resid) {
            ld8(resid + r * ldr + c, n, o[u]);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) o[u][i] = 0.f;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const long long r = r0 + u;
      if (r >= rows || n <= 0) continue;
      const float mu = mean[r], rs = rstd[r];
      const float m_xg = stats[2 * r] * inv_h, m_g = stats[2 * r + 1] * inv_h;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (v[u][i] - mu) * rs;
        o[u][i] += rs * (d[u][i] * g[i] - m_g - xh * m_xg);
        acc[0][i] += d[u][i] * xh;
        acc[1][i] += d[u][i];
        acc[2][i] += o[u][i];
      }
      st8(dx + r * lddx + c, n, o[u]);
      if (dx2) st8(dx2 + r * lddx2 + c, n, o[u]);
    }
  }
  if (dgamma || dsum) {
    float* const dst[3] = {dgamma, dbeta, dsum};
    seg_flush<3>(acc, dst, c0, cols, sm);
  }
}

// out[c] += sum_r x[r, c]  (bias gradient before the column reduce, layers.py:238)
template <typename TX, int RU, bool FULL>
__global__ void __launch_bounds__(256) colsum_kernel(const TX* __restrict__ x, long long rows, int cols, long long ldx,
                                                     float* __restrict__ out) {
  pdl_begin();
  __shared__ __align__(16) float sm[kSegWarps * kSegCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.y * kSegCols;
  const int c = c0 + lane * 8;
  const int n = max(0, min(8, cols - c));
  const int cl = FULL ? min(c, cols - 8) : c;
  float acc[1][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[0][i] = 0.f;
  const long long step = (long long)gridDim.x * kSegWarps * RU;
  for (long long r0 = ((long long)blockIdx.x * kSegWarps + warp) * RU; r0 < rows; r0 += step) {
    float v[RU][8];
    if (FULL) {
      Vec8<TX> rv[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) rv[u].load(x + min(r0 + u, rows - 1) * ldx + cl);
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        rv[u].to(v[u]);
        if (r0 + u >= rows || n <= 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i) v[u][i] = 0.f;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (r0 + u < rows && n > 0) {
          ld8(x + (r0 + u) * ldx + c, n, v[u]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) v[u][i] = 0.f;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < RU; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[0][i] += v[u][i];
  }
  float* const dst[1] = {out};
  seg_flush<1>(acc, dst, c0, cols, sm);
}

// x[r, c] += bias[c]  (layers.py:228)
template <typename TX>
__global__ void bias_add_kernel(TX* __restrict__ x, long long rows, int cols, long long ldx,
                                const float* __restrict__ bias) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw)
    for (int c = lane * 8; c < cols; c += 256) {
      const int n = min(8, cols - c);
      float v[8], b[8];
      ld8(x + r * ldx + c, n, v);
      ld8(bias + c, n, b);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] += b[i];
      st8(x + r * ldx + c, n, v);
    }
}

// ============================================================ softmax
// P = softmax(S) row-wise with max subtraction (dense.py:67-75)
template <typename TS, typename TP>
__global__ void softmax_kernel(const TS* __restrict__ S, long long rows, int cols, long long lds, TP* __restrict__ P,
                               long long ldp) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw) {
    const TS* sr = S + r * lds;
    float m = -FLT_MAX;
    for (int c = lane * 8; c < cols; c += 256) {
      float v[8];
      const int n = min(8, cols - c);
      ld8(sr + c, n, v);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < n) m = fmaxf(m, v[i]);
    }
    m = warp_max(m);
    float z = 0.f;
    for (int c = lane * 8; c < cols; c += 256) {
      float v[8];
      const int n = min(8, cols - c);
      ld8(sr + c, n, v);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < n) z += __expf(v[i] - m);
    }
    const float inv = 1.0f / warp_sum(z);
    for (int c = lane * 8; c < cols; c += 256) {
      float v[8];
      const int n = min(8, cols - c);
      ld8(sr + c, n, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __expf(v[i] - m) * inv;
      st8(P + r * ldp + c, n, v);
    }
  }
}

// dS = P * (dP - sum(dP * P)) * scale  (layers.py:449-450)
template <typename TD, typename TP, typename TO>
__global__ void softmax_bwd_kernel(const TD* __restrict__ dP, long long lddp, const TP* __restrict__ P, long long ldp,
                                   long long rows, int cols, float scale, TO* __restrict__ dS, long long ldds) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw) {
    float acc = 0.f;
    for (int c = lane * 8; c < cols; c += 256) {
      float a[8], p[8];
      const int n = min(8, cols - c);
      ld8(dP + r * lddp + c, n, a);
      ld8(P + r * ldp + c, n, p);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc += a[i] * p[i];
    }
    acc = warp_sum(acc);
    for (int c = lane * 8; c < cols; c += 256) {
      float a[8], p[8];
      const int n = min(8, cols - c);
      ld8(dP + r * lddp + c, n, a);
      ld8(P + r * ldp + c, n, p);
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = p[i] * (a[i] - acc) * scale;
      st8(dS + r * ldds + c, n, a);
    }
  }
}

// ============================================================ cross entropy
// Local pass over this device's vocabulary block (layers.py:557-584): online
// (max, sum e^{x-max}) over the n_real valid columns and the label logit when
// the label falls in [col_lo, col_lo + ncols). Writes lmax[r], gmax[r]
// (= lmax, to be max-all-reduced in place) and packed[r] = (sum, x_label).
template <typename TL>
__global__ void xent_local_kernel(const TL* __restrict__ logits, long long rows, long long ldl, int n_real,
                                  const int64_t* __restrict__ labels, long long col_lo, float* __restrict__ lmax,
                                  float* __restrict__ gmax, float* __restrict__ packed) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw) {
    const TL* lr = logits + r * ldl;
    float m = -INFINITY, s = 0.f;
    int c = lane * 8;
    // interior: four 8-wide chunks per lane in flight, then one online update
    for (; c + 3 * 256 + 8 <= n_real; c += 1024) {
      Vec8<TL> raw[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) raw[k].load(lr + c + k * 256);
      float v[4][8];
      float cm = -INFINITY;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        raw[k].to(v[k]);
#pragma unroll
        for (int i = 0; i < 8; ++i) cm = fmaxf(cm, v[k][i]);
      }
      if (cm > m) {
        s *= __expf(m - cm);
        m = cm;
      }
      const float l2e = 1.4426950408889634f, ml = -m * l2e;
      float sp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float e;
          asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(v[k][i], l2e, ml)));
          sp[k] += e;
        }
      s += (sp[0] + sp[1]) + (sp[2] + sp[3]);
    }
    for (; c < n_real; c += 256) {
      float v[8];
      const int n = min(8, n_real - c);
      ld8(lr + c, n, v);
      float cm = -INFINITY;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < n) cm = fmaxf(cm, v[i]);
      if (cm > m) {
        s *= __expf(m - cm);
        m = cm;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < n) s += __expf(v[i] - m);
    }
    // combine (m, s) across lanes
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
      const float nm = fmaxf(m, om);
      s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
      m = nm;
    }
    if (lane == 0) {
      const long long lab = labels[r] - col_lo;
      const float xl = (lab >= 0 && lab < n_real) ? ld1(lr + lab) : 0.f;
      lmax[r] = m;
      gmax[r] = m;
      packed[2 * r] = s;
      packed[2 * r + 1] = xl;
    }
  }
}

// packed[r].sum *= e^{lmax - gmax} so the row all-reduce sums share one max.
__global__ void xent_rescale_kernel(long long rows, const float* __restrict__ lmax, const float* __restrict__ gmax,
                                    float* __restrict__ packed) {
  pdl_begin();
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += gridDim.x * (long long)blockDim.x) {
    const float lm = lmax[r];
    packed[2 * r] = lm == -INFINITY ? 0.f : packed[2 * r] * __expf(lm - gmax[r]);
  }
}

// loss[r] = log(sum) + max - x_label; *partial (+)= sum_r loss[r]  (layers.py:597-599)
__global__ void xent_loss_kernel(long long rows, const float* __restrict__ gmax, const float* __restrict__ packed,
                                 float* __restrict__ loss_rows, float* __restrict__ partial) {
  pdl_begin();
  float acc = 0.f;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += gridDim.x * (long long)blockDim.x) {
    const float l = logf(packed[2 * r]) + gmax[r] - packed[2 * r + 1];
    if (loss_rows) loss_rows[r] = l;
    acc += l;
  }
  acc = warp_sum(acc);
  __shared__ float sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) atomicAdd(partial, v);
  }
}

// dlogits = (e^{x - max} / sum - [col == label]) * scale; padded columns -> 0
// (layers.py:611-624). In place (dl == logits) is allowed.
template <typename TL, typename TO>
__global__ void xent_bwd_kernel(const TL* logits, long long rows, long long ldl, int n_real, int ncols,
                                const int64_t* __restrict__ labels, long long col_lo, const float* __restrict__ gmax,
                                const float* __restrict__ packed, float scale, TO* dl, long long lddl) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw) {
    const float m = gmax[r];
    const float inv = 1.0f / packed[2 * r];
    const long long lab = labels[r] - col_lo;
    // g = 2^(x log2e - m log2e) (scale / sum), the label column then - scale
    const float l2e = 1.4426950408889634f, ml = -m * l2e, sc = inv * scale;
    int c = lane * 8;
    for (; c + 3 * 256 + 8 <= n_real; c += 1024) {  // interior (all columns real), four chunks in flight
      Vec8<TL> raw[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) raw[k].load(logits + r * ldl + c + k * 256);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float v[8];
        raw[k].to(v);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float e;
          asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(v[i], l2e, ml)));
          v[i] = e * sc;
        }
        const long long off = lab - (c + k * 256);
        if (off >= 0 && off < 8) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (i == off) v[i] -= scale;
        }
        st8(dl + r * lddl + c + k * 256, 8, v);
      }
    }
    for (; c < ncols; c += 256) {
      float v[8];
      const int n = min(8, ncols - c);
      ld8(logits + r * ldl + c, n, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int cc = c + i;
        float g = cc < n_real ? __expf(v[i] - m) * inv : 0.f;
        if (cc == lab) g -= 1.f;
        v[i] = g * scale;
      }
      st8(dl + r * lddl + c, n, v);
    }
  }
}

// ============================================================ embedding
// out[t, :] = table[ids[t] - lo, :] for ids in [lo, lo + vb)  (layers.py:178-181)
template <typename TT, typename TO>
__global__ void embed_fwd_kernel(const int64_t* __restrict__ ids, long long n, long long lo, long long vb,
                                 const TT* __restrict__ table, long long ldt, int hc, TO* __restrict__ out,
                                 long long ldo) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long t = wid; t < n; t += nw) {
    const long long row = ids[t] - lo;
    if (row < 0 || row >= vb) continue;
    for (int c = lane * 8; c < hc; c += 256) {
      float v[8];
      const int k = min(8, hc - c);
      ld8(table + row * ldt + c, k, v);
      st8(out + t * ldo + c, k, v);
    }
  }
}

// *flag |= 1 when any id lies outside [0, v): the device-side form of the reference's
// range checks (layers.py:164-165 token ids, layers.py:552-553 labels), read back by
// the host at the next synchronisation point instead of stalling the step.
__global__ void check_ids_kernel(const int64_t* __restrict__ ids, long long n, long long v, int* flag) {
  pdl_begin();
  bool bad = false;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long id = ids[t];
    bad |= (id < 0) | (id >= v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// grad[ids[t] - lo, :] += dout[t, :] for ids in the block; repeated ids accumulate (layers.py:202-205)
template <typename TD>
__global__ void embed_bwd_kernel(const int64_t* __restrict__ ids, long long n, long long lo, long long vb,
                                 const TD* __restrict__ dout, long long ldd, int hc, float* __restrict__ grad,
                                 long long ldg) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long t = wid; t < n; t += nw) {
    const long long row = ids[t] - lo;
    if (row < 0 || row >= vb) continue;
    for (int c = lane * 8; c < hc; c += 256) {
      float v[8];
      const int k = min(8, hc - c);
      ld8(dout + t * ldd + c, k, v);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < k) atomicAdd(grad + row * ldg + c + i, v[i]);
    }
  }
}

// Deterministic variant (SG_DETERMINISTIC=1): one warp per table row scans the ids in
// order, collects the matching token positions into a shared-memory list (ballot order =
// token order) and folds their rows into the gradient row in that order, flushing every
// kDetList tokens; a single writer per row, so the sums are bit-reproducible (the
// atomic scatter-add above adds in arrival order).
constexpr int kDetList = 128;
template <typename TD>
__global__ void __launch_bounds__(256) embed_bwd_det_kernel(const int64_t* __restrict__ ids, long long n, long long lo,
                                                            long long vb, const TD* __restrict__ dout, long long ldd,
                                                            int hc, float* __restrict__ grad, long long ldg) {
  pdl_begin();
  __shared__ int list[8][kDetList];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  int* lst = list[wl];
  for (long long row = wid; row < vb; row += nw) {
    const long long id = row + lo;
    int cnt = 0;
    auto flush = [&]() {
      __syncwarp();
      for (int c = lane * 8; c < hc; c += 256) {
        const int k = min(8, hc - c);
        float acc[8];
        ld8(grad + row * ldg + c, k, acc);
        for (int m = 0; m < cnt; ++m) {
          float v[8];
          ld8(dout + (long long)lst[m] * ldd + c, k, v);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += v[i];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i < k) grad[row * ldg + c + i] = acc[i];
      }
      __syncwarp();
      cnt = 0;
    };
    for (long long t0 = 0; t0 < n; t0 += 32) {
      const long long t = t0 + lane;
      const bool hit = t < n && ids[t] == id;
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (m == 0) continue;
      const int nm = __popc(m);
      if (cnt + nm > kDetList) flush();
      if (hit) lst[cnt + __popc(m & ((1u << lane) - 1))] = (int)t;
      cnt += nm;
    }
    if (cnt > 0) flush();
  }
}

// ============================================================ element-wise
template <typename TS, typename TD>
__global__ void cast_kernel(const TS* __restrict__ s, TD* __restrict__ d, long long n) {
  pdl_begin();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x) {
    if constexpr (sizeof(TD) == 4)
      d[i] = ld1(s + i);
    else
      d[i] = __float2bfloat16_rn(ld1(s + i));
  }
}

struct SrcList {
  const void* p[8];
};
// dst = [dst (op)] src0 (op) src1 ... in list order: the rank-ordered fold of
// the reference's reduce / all-reduce (mesh.py:464-466, 490-497).
template <typename T>
__global__ void fold_kernel(T* __restrict__ dst, SrcList srcs, int nsrc, long long n, int accumulate, int op_max) {
  pdl_begin();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (long long)blockDim.x) {
    float acc = accumulate ? ld1(dst + i) : ld1(static_cast<const T*>(srcs.p[0]) + i);
    for (int k = accumulate ? 0 : 1; k < nsrc; ++k) {
      const float v = ld1(static_cast<const T*>(srcs.p[k]) + i);
      acc = op_max ? fmaxf(acc, v) : acc + v;
    }
    if constexpr (sizeof(T) == 4)
      dst[i] = acc;
    else
      dst[i] = __float2bfloat16_rn(acc);
  }
}

// ============================================================ epilogue
// out = act(alpha * x + bias + C) — the sg_gemm epilogue applied to fp32 partial
// sums that were reduced over the mesh before it could run (dist AB^T forms).
__device__ __forceinline__ float gelu_tanh(float x) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  return 0.5f * x * (1.f + tanhf(c * (x + a * x * x * x)));
}
__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  const float t = tanhf(c * (x + a * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * a * x * x);
}
template <typename TC, typename TO>
__global__ void epilogue_kernel(const float* __restrict__ x, long long rows, int cols, long long ldx, float alpha,
                                const float* __restrict__ bias, const TC* __restrict__ cin, long long ldc, int act,
                                bf16* __restrict__ aux, long long ldaux, TO* __restrict__ out, long long ldo) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r = wid; r < rows; r += nw)
    for (int c = lane * 8; c < cols; c += 256) {
      const int n = min(8, cols - c);
      float v[8], t[8];
      ld8(x + r * ldx + c, n, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] *= alpha;
      if (bias) {
        ld8(bias + c, n, t);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] += t[i];
      }
      if (cin) {
        ld8(cin + r * ldc + c, n, t);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] += t[i];
      }
      if (act == SG_ACT_GELU) {
        if (aux) st8(aux + r * ldaux + c, n, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gelu_tanh(v[i]);
      } else if (act == SG_ACT_DGELU) {
        ld8(aux + r * ldaux + c, n, t);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] *= gelu_tanh_grad(t[i]);
      }
      st8(out + r * ldo + c, n, v);
    }
}

// D[b, h, t] = sum_j dO[row, h*d + j] * O[row, h*d + j] with row = b*s + t: the
// rowsum(dP * P) term of the softmax backward, computed as rowsum(dO * O)
// (P V = O), one thread per (token row, head).
template <typename T>
__global__ void attn_rowdot_kernel(const T* __restrict__ dO, long long ldo, const T* __restrict__ O, long long ldO,
                                   long long rows, int nh, int d, int s, float* __restrict__ out) {
  pdl_begin();
  const long long total = rows * nh;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += gridDim.x * (long long)blockDim.x) {
    const long long row = i / nh;
    const int h = (int)(i - row * nh);
    const T* a = dO + row * ldo + (long long)h * d;
    const T* b = O + row * ldO + (long long)h * d;
    float acc = 0.f;
    for (int j = 0; j < d; j += 8) {
      float x[8], y[8];
      const int n = min(8, d - j);
      ld8(a + j, n, x);
      ld8(b + j, n, y);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(x[e], y[e], acc);
    }
    const long long bb = row / s, t = row - bb * s;
    out[(bb * nh + h) * (long long)s + t] = acc;
  }
}

// out = dact * gelu'(mid) (bf16 in / out, out may alias dact) and colsum += column
// sums of out: the h->4h GELU backward and its bias gradient in one pass
// (layers.py:502-504). Column-segment layout (see ln_bwd_kernel).
__device__ __forceinline__ float gelu_grad_approx(float x) {
  const float c = 0.7978845608028654f, a = 0.044715f;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(c * (x + a * x * x * x)));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * c * (1.f + 3.f * a * x * x);
}
template <typename TO, int RU, bool FULL>
__global__ void __launch_bounds__(256) dgelu_kernel(const bf16* dact, long long lda, const bf16* __restrict__ mid,
                                                    long long ldm, long long rows, int cols, TO* out, long long ldo,
                                                    float* __restrict__ colsum) {
  pdl_begin();
  __shared__ __align__(16) float sm[kSegWarps * kSegCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.y * kSegCols;
  const int c = c0 + lane * 8;
  const int n = max(0, min(8, cols - c));
  const int cl = FULL ? min(c, cols - 8) : c;
  float acc[1][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[0][i] = 0.f;
  const long long step = (long long)gridDim.x * kSegWarps * RU;
  for (long long r0 = ((long long)blockIdx.x * kSegWarps + warp) * RU; r0 < rows; r0 += step) {
    float g[RU][8], xm[RU][8];
    if (FULL) {
      Vec8<bf16> rg[RU], rm[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const long long r = min(r0 + u, rows - 1);
        rg[u].load(dact + r * lda + cl);
        rm[u].load(mid + r * ldm + cl);
      }
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        rg[u].to(g[u]);
        rm[u].to(xm[u]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (r0 + u < rows && n > 0) {
          ld8(dact + (r0 + u) * lda + c, n, g[u]);
          ld8(mid + (r0 + u) * ldm + c, n, xm[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      if (r0 + u >= rows || n <= 0) continue;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        g[u][i] *= gelu_grad_approx(xm[u][i]);
        acc[0][i] += g[u][i];
      }
      st8(out + (r0 + u) * ldo + c, n, g[u]);
    }
  }
  if (colsum) {
    float* const dst[1] = {colsum};
    seg_flush<1>(acc, dst, c0, cols, sm);
  }
}

// y = LayerNorm(x) with the whole row held in registers (cols = 256 * NV): one HBM
// read of x; the (sum, sumsq) row statistics come from the mesh all-reduce
// (stats != nullptr) or, on a 1-column mesh, from the registers themselves.
template <typename TX, typename TY, int NV>
__global__ void __launch_bounds__(256, NV <= 2 ? 4 : (NV == 4 ? 2 : 1)) ln_fwd_rows_kernel(
    const TX* __restrict__ x, long long rows, long long ldx, const float* __restrict__ stats, float inv_h, float eps,
    const float* __restrict__ gamma, const float* __restrict__ beta, TY* __restrict__ y, long long ldy,
    float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  pdl_begin();
  // RU rows per warp iteration (their loads in flight together, each gamma / beta
  // load serving RU rows); measured: RU = 2 at h = 1024 loses to the occupancy it costs
  constexpr int RU = 1;
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long r0 = wid * RU; r0 < rows; r0 += nw * RU) {
    Vec8<TX> raw[RU][NV];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const long long r = min(r0 + u, rows - 1);  // clamped: a duplicate row is computed, not stored
#pragma unroll
      for (int k = 0; k < NV; ++k) raw[u][k].load(x + r * ldx + k * 256 + lane * 8);
    }
    float mu[RU], rs[RU];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const long long r = min(r0 + u, rows - 1);
      float s1, s2;
      if (stats) {
        s1 = stats[2 * r];
        s2 = stats[2 * r + 1];
      } else {
        s1 = 0.f;
        s2 = 0.f;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          float v[8];
          raw[u][k].to(v);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            s1 += v[i];
            s2 = fmaf(v[i], v[i], s2);
          }
        }
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
      }
      mu[u] = s1 * inv_h;
      const float var = fmaxf(s2 * inv_h - mu[u] * mu[u], 0.f);  // one-pass variance (layers.py:296-297), clamped
      rs[u] = rsqrtf(var + eps);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int c = k * 256 + lane * 8;
      float g[8], bb[8];
      Vec8<float> gv, bv;
      gv.load(gamma + c);
      bv.load(beta + c);
      gv.to(g);
      bv.to(bb);
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        if (r0 + u >= rows) break;
        float v[8];
        raw[u][k].to(v);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = fmaf((v[i] - mu[u]) * rs[u], g[i], bb[i]);
        st8(y + (r0 + u) * ldy + c, 8, v);
      }
    }
    if (lane < RU && r0 + lane < rows) {
      float m = mu[0], q = rs[0];
#pragma unroll
      for (int u = 1; u < RU; ++u)
        if (lane == u) m = mu[u], q = rs[u];
      if (mean_out) mean_out[r0 + lane] = m;
      if (rstd_out) rstd_out[r0 + lane] = q;
    }
  }
}

// The dQKV block after the flash backward: dq (fp32 accumulator) -> bf16 columns
// [0, hb) of dqkv, and colsum += column sums of the whole [rows, 3 hb] gradient
// (the b_qkv gradient, layers.py:238) in the same pass. Column-segment layout;
// hb % 256 == 0 so every 256-column segment is all dQ or all dK / dV.
template <int RU>
__global__ void __launch_bounds__(256) qkv_grad_finish_kernel(const float* __restrict__ dq, long long lddq,
                                                              bf16* __restrict__ dqkv, long long ldg, long long rows,
                                                              int hb, float* __restrict__ colsum) {
  pdl_begin();
  __shared__ __align__(16) float sm[kSegWarps * kSegCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.y * kSegCols;
  const int c = c0 + lane * 8;
  const bool is_q = c0 < hb;
  float acc[1][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[0][i] = 0.f;
  const long long step = (long long)gridDim.x * kSegWarps * RU;
  for (long long r0 = ((long long)blockIdx.x * kSegWarps + warp) * RU; r0 < rows; r0 += step) {
    float v[RU][8];
    if (is_q) {
      Vec8<float> raw[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) raw[u].load(dq + min(r0 + u, rows - 1) * lddq + c);
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        raw[u].to(v[u]);
        if (r0 + u < rows) st8(dqkv + (r0 + u) * ldg + c, 8, v[u]);
      }
    } else {
      Vec8<bf16> raw[RU];
#pragma unroll
      for (int u = 0; u < RU; ++u) raw[u].load(dqkv + min(r0 + u, rows - 1) * ldg + c);
#pragma unroll
      for (int u = 0; u < RU; ++u) raw[u].to(v[u]);
    }
#pragma unroll
    for (int u = 0; u < RU; ++u)
      if (r0 + u < rows)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[0][i] += v[u][i];
  }
  if (colsum) {
    float* const dst[1] = {colsum};
    seg_flush<1>(acc, dst, c0, 3 * hb, sm);
  }
}

// D[b, h, t] = rowsum(dO * O) over each 64-wide head, a warp per token row: lane
// l holds elements 8l .. 8l+7 of each 256-column chunk, 8 lanes make a head.
template <int NV>
__global__ void __launch_bounds__(256) attn_rowdot64_kernel(const bf16* __restrict__ dO, long long ldo,
                                                            const bf16* __restrict__ O, long long ldO, long long rows,
                                                            int nh, int s, float* __restrict__ out) {
  pdl_begin();
  const int lane = threadIdx.x & 31;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  for (long long row = wid; row < rows; row += nw) {
    Vec8<bf16> a[NV], b[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      a[k].load(dO + row * ldo + k * 256 + lane * 8);
      b[k].load(O + row * ldO + k * 256 + lane * 8);
    }
    const long long bb = row / s, t = row - bb * s;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float x[8], y[8];
      a[k].to(x);
      b[k].to(y);
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(x[e], y[e], acc);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      const int h = k * 4 + (lane >> 3);
      if ((lane & 7) == 0) out[(bb * nh + h) * (long long)s + t] = acc;
    }
  }
}

// Multi-tensor SGD: w -= lr * g on fp32 masters (2-D, own row pitches) with the
// bf16 GEMM twin refreshed in the same pass (layers.py:761-772, model.py:356-364).
// Blocks are dealt out over fixed 4096-element chunks of all tensors.
constexpr int kSgdChunk = 4096;
constexpr int kSgdMax = 96;
struct SgdBatch {
  float* w[kSgdMax];
  bf16* wl[kSgdMax];
  const float* g[kSgdMax];
  long long ldw[kSgdMax], ldl[kSgdMax], ldg[kSgdMax], cols[kSgdMax];
  long long first_chunk[kSgdMax + 1];
  long long total[kSgdMax];
  int n;
  int vec4[kSgdMax];
  float lr;
};
__global__ void __launch_bounds__(256) sgd_multi_kernel(const __grid_constant__ SgdBatch b) {
  pdl_begin();
  for (long long ch = blockIdx.x; ch < b.first_chunk[b.n]; ch += gridDim.x) {
    int t = 0;
    while (t + 1 < b.n && b.first_chunk[t + 1] <= ch) ++t;
    const long long e0 = (ch - b.first_chunk[t]) * kSgdChunk;
    const long long e1 = min(e0 + kSgdChunk, b.total[t]);
    const long long cols = b.cols[t];
    float* w = b.w[t];
    bf16* wl = b.wl[t];
    const float* g = b.g[t];
    if (b.vec4[t]) {
      for (long long e = e0 + threadIdx.x * 4; e < e1; e += 1024) {
        const long long r = e / cols, cc = e - r * cols;
        float4 wv = *reinterpret_cast<float4*>(w + r * b.ldw[t] + cc);
        if (g) {  // (g == nullptr: w already updated, refresh its bf16 copy only)
          const float4 gv = *reinterpret_cast<const float4*>(g + r * b.ldg[t] + cc);
          wv.x -= b.lr * gv.x; wv.y -= b.lr * gv.y; wv.z -= b.lr * gv.z; wv.w -= b.lr * gv.w;
          *reinterpret_cast<float4*>(w + r * b.ldw[t] + cc) = wv;
        }
        if (wl) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(wv.x, wv.y), hi = __floats2bfloat162_rn(wv.z, wv.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(wl + r * b.ldl[t] + cc) = pk;
        }
      }
    } else {
      for (long long e = e0 + threadIdx.x; e < e1; e += 256) {
        const long long r = e / cols, cc = e - r * cols;
        const float v = g ? w[r * b.ldw[t] + cc] - b.lr * g[r * b.ldg[t] + cc] : w[r * b.ldw[t] + cc];
        if (g) w[r * b.ldw[t] + cc] = v;
        if (wl) wl[r * b.ldl[t] + cc] = __float2bfloat16_rn(v);
      }
    }
  }
}

}  // namespace sg

using namespace sg;



static cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" int sg_zero(void* ptr, int64_t bytes, void* stream) {
  clear_error();
  if (bytes <= 0) return SG_OK;
  if (cudaMemsetAsync(ptr, 0, (size_t)bytes, S(stream)) != cudaSuccess) return set_error(SG_ERR_CUDA, "memset");
  return SG_OK;
}

extern "C" int sg_ln_stats(const void* x, int xdt, int64_t rows, int64_t cols, int64_t ldx, float* stats,
                           void* stream) {
  clear_error();
  if (rows < 0 || cols < 1) return set_error(SG_ERR_SHAPE, "ln_stats: bad extents");
  if (!aligned16(x, ldx, xdt == SG_DTYPE_F32 ? 4 : 2)) return set_error(SG_ERR_SHAPE, "ln_stats: unaligned");
  if (rows == 0) return SG_OK;
  const int grid = grid_for(rows, 8);
  SG_DISPATCH_T(xdt, TX, (launch_k(ln_stats_kernel<TX>, dim3(grid), dim3(256), 0, S(stream), static_cast<const TX*>(x), rows, (int)cols, ldx, stats)));
  return launch_check();
}

extern "C" int sg_ln_fwd(const void* x, int xdt, int64_t rows, int64_t cols, int64_t ldx, const float* stats,
                         int64_t h_total, float eps, const float* gamma, const float* beta, void* y, int ydt,
                         int64_t ldy, float* mean, float* rstd, void* stream) {
  clear_error();
  if (rows < 0 || cols < 1 || h_total < cols) return set_error(SG_ERR_SHAPE, "ln_fwd: bad extents");
  if (!aligned16(x, ldx, xdt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(y, ldy, ydt == SG_DTYPE_F32 ? 4 : 2) ||
      !aligned16(gamma, 0, 4) || !aligned16(beta, 0, 4))
    return set_error(SG_ERR_SHAPE, "ln_fwd: unaligned");
  if (!stats && h_total != cols) return set_error(SG_ERR_CONFIG, "ln_fwd: sharded row needs all-reduced stats");
  if (rows == 0) return SG_OK;
  const int grid = grid_for(rows, 8);
  const float inv_h = 1.0f / (float)h_total;
  const int nv = cols % 256 == 0 ? (int)(cols / 256) : 0;
  if (nv == 1 || nv == 2 || nv == 4 || nv == 8) {
    // whole row in registers: a warp per row, grid = one wave of resident warps
    const int g2 = grid_for(rows, 8, nv <= 4 ? 8 : 4);
#define SG_LN_ROWS(NV) SG_DISPATCH_T(xdt, TX, SG_DISPATCH_T(ydt, TY, (launch_k(ln_fwd_rows_kernel<TX, TY, NV>, dim3(g2), dim3(256), 0, S(stream), static_cast<const TX*>(x), rows, ldx, stats, inv_h, eps, gamma, beta, static_cast<TY*>(y), ldy, mean, rstd))))
    switch (nv) {
      case 1: SG_LN_ROWS(1); break;
      case 2: SG_LN_ROWS(2); break;
      case 4: SG_LN_ROWS(4); break;
      default: SG_LN_ROWS(8); break;
    }
#undef SG_LN_ROWS
    return launch_check();
  }
  SG_DISPATCH_T(xdt, TX, SG_DISPATCH_T(ydt, TY, (launch_k(ln_fwd_kernel<TX, TY>, dim3(grid), dim3(256), 0, S(stream), static_cast<const TX*>(x), rows, (int)cols, ldx, stats, inv_h, eps, gamma, beta, static_cast<TY*>(y), ldy, mean, rstd))));
  return launch_check();
}

extern "C" int sg_ln_bwd_stats(const void* dy, int dydt, int64_t lddy, const void* x, int xdt, int64_t ldx,
                               const float* mean, const float* rstd, const float* gamma, int64_t rows, int64_t cols,
                               float* stats, void* stream) {
  clear_error();
  if (rows < 0 || cols < 1) return set_error(SG_ERR_SHAPE, "ln_bwd_stats: bad extents");
  if (!aligned16(dy, lddy, dydt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(x, ldx, xdt == SG_DTYPE_F32 ? 4 : 2))
    return set_error(SG_ERR_SHAPE, "ln_bwd_stats: unaligned");
  if (rows == 0) return SG_OK;
  const int grid = grid_for(rows, 8);
  SG_DISPATCH_T(dydt, TD, SG_DISPATCH_T(xdt, TX, (launch_k(ln_bwd_stats_kernel<TD, TX>, dim3(grid), dim3(256), 0, S(stream), static_cast<const TD*>(dy), lddy, static_cast<const TX*>(x), ldx, mean, rstd, gamma, rows, (int)cols, stats))));
  return launch_check();
}

extern "C" int sg_ln_bwd(const void* dy, int dydt, int64_t lddy, const void* x, int xdt, int64_t ldx,
                         const float* mean, const float* rstd, const float* gamma, int64_t rows, int64_t cols,
                         const float* stats, int64_t h_total, const void* resid, int rdt, int64_t ldr, void* dx,
                         int dxdt, int64_t lddx, void* dx2, int64_t lddx2, float* dgamma, float* dbeta,
                         float* dsum, void* stream) {
  clear_error();
  if (rows < 0 || cols < 1 || h_total < cols || !stats) return set_error(SG_ERR_SHAPE, "ln_bwd: bad arguments");
  if ((dgamma == nullptr) != (dbeta == nullptr)) return set_error(SG_ERR_CONFIG, "ln_bwd: dgamma/dbeta pair");
  if (!aligned16(dy, lddy, dydt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(x, ldx, xdt == SG_DTYPE_F32 ? 4 : 2) ||
      !aligned16(resid, ldr, rdt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(dx, lddx, dxdt == SG_DTYPE_F32 ? 4 : 2) ||
      !aligned16(dx2, lddx2, 2))
    return set_error(SG_ERR_SHAPE, "ln_bwd: unaligned");
  if (rows == 0) return SG_OK;
  const dim3 grid = seg_grid(rows, cols, 2, 2);
  const float inv_h = 1.0f / (float)h_total;
  if (rdt != SG_DTYPE_BF16) rdt = SG_DTYPE_F32;
  // dx is fp32 (residual-stream gradient); the optional dx2 is its bf16 GEMM operand copy
  if (dxdt != SG_DTYPE_F32) return set_error(SG_ERR_CONFIG, "ln_bwd: dx must be fp32");
#define SG_LN_BWD(FULL) SG_DISPATCH_T(dydt, TD, SG_DISPATCH_T(xdt, TX, SG_DISPATCH_T(rdt, TR, (launch_k(ln_bwd_kernel<TD, TX, TR, 2, FULL>, dim3(grid), dim3(256), 0, S(stream), static_cast<const TD*>(dy), lddy, static_cast<const TX*>(x), ldx, mean, rstd, gamma, rows, (int)cols, stats, inv_h, static_cast<const TR*>(resid), ldr, static_cast<float*>(dx), lddx, static_cast<bf16*>(dx2), lddx2, dgamma, dbeta, dsum)))))
  if (cols % 8 == 0)
    SG_LN_BWD(true);
  else
    SG_LN_BWD(false);
#undef SG_LN_BWD
  return launch_check();
}

extern "C" int sg_colsum(const void* x, int xdt, int64_t rows, int64_t cols, int64_t ldx, float* out,
                         int accumulate, void* stream) {
  clear_error();
  if (rows < 0 || cols < 1) return set_error(SG_ERR_SHAPE, "colsum: bad extents");
  if (!aligned16(x, ldx, xdt == SG_DTYPE_F32 ? 4 : 2)) return set_error(SG_ERR_SHAPE, "colsum: unaligned");
  if (!accumulate && cudaMemsetAsync(out, 0, cols * sizeof(float), S(stream)) != cudaSuccess)
    return set_error(SG_ERR_CUDA, "memset");
  if (rows == 0) return SG_OK;
  if (cols % 8 == 0)
    SG_DISPATCH_T(xdt, TX, (launch_k(colsum_kernel<TX, 4, true>, dim3(seg_grid(rows, cols, 4, 4)), dim3(256), 0, S(stream), static_cast<const TX*>(x), rows, (int)cols, ldx, out)));
  else
    SG_DISPATCH_T(xdt, TX, (launch_k(colsum_kernel<TX, 4, false>, dim3(seg_grid(rows, cols, 4, 2)), dim3(256), 0, S(stream), static_cast<const TX*>(x), rows, (int)cols, ldx, out)));
  return launch_check();
}

extern "C" int sg_bias_add(void* x, int xdt, int64_t rows, int64_t cols, int64_t ldx, const float* bias,
                           void* stream) {
  clear_error();
  if (rows < 0 || cols < 1) return set_error(SG_ERR_SHAPE, "bias_add: bad extents");
  if (!aligned16(x, ldx, xdt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(bias, 0, 4))
    return set_error(SG_ERR_SHAPE, "bias_add: unaligned");
  if (rows == 0) return SG_OK;
  SG_DISPATCH_T(xdt, TX, (launch_k(bias_add_kernel<TX>, dim3(grid_for(rows, 8)), dim3(256), 0, S(stream), static_cast<TX*>(x), rows, (int)cols, ldx, bias)));
  return launch_check();
}

extern "C" int sg_softmax_rows(const void* s, int sdt, int64_t rows, int64_t cols, int64_t lds, void* p, int pdt,
                               int64_t ldp, void* stream) {
  clear_error();
  if (rows < 0 || cols < 1) return set_error(SG_ERR_SHAPE, "softmax: bad extents");
  if (!aligned16(s, lds, sdt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(p, ldp, pdt == SG_DTYPE_F32 ? 4 : 2))
    return set_error(SG_ERR_SHAPE, "softmax: unaligned");
  if (rows == 0) return SG_OK;
  SG_DISPATCH_T(sdt, TS, SG_DISPATCH_T(pdt, TP, (launch_k(softmax_kernel<TS, TP>, dim3(grid_for(rows, 8)), dim3(256), 0, S(stream), static_cast<const TS*>(s), rows, (int)cols, lds, static_cast<TP*>(p), ldp))));
  return launch_check();
}

extern "C" int sg_softmax_bwd(const void* dp, int dpdt, int64_t lddp, const void* p, int pdt, int64_t ldp,
                              int64_t rows, int64_t cols, float scale, void* ds, int dsdt, int64_t ldds,
                              void* stream) {
  clear_error();
  if (rows < 0 || cols < 1) return set_error(SG_ERR_SHAPE, "softmax_bwd: bad extents");
  if (!aligned16(dp, lddp, dpdt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(p, ldp, pdt == SG_DTYPE_F32 ? 4 : 2) ||
      !aligned16(ds, ldds, dsdt == SG_DTYPE_F32 ? 4 : 2))
    return set_error(SG_ERR_SHAPE, "softmax_bwd: unaligned");
  if (rows == 0) return SG_OK;
  SG_DISPATCH_T(dpdt, TD, SG_DISPATCH_T(pdt, TP, SG_DISPATCH_T(dsdt, TO, (launch_k(softmax_bwd_kernel<TD, TP, TO>, dim3(grid_for(rows, 8)), dim3(256), 0, S(stream), static_cast<const TD*>(dp), lddp, static_cast<const TP*>(p), ldp, rows, (int)cols, scale, static_cast<TO*>(ds), ldds)))));
  return launch_check();
}

extern "C" int sg_xent_local(const void* logits, int ldt, int64_t rows, int64_t ldl, int64_t n_real,
                             const int64_t* labels, int64_t col_lo, float* lmax, float* gmax, float* packed,
                             void* stream) {
  clear_error();
  if (rows < 0 || n_real < 0) return set_error(SG_ERR_SHAPE, "xent_local: bad extents");
  if (!aligned16(logits, ldl, ldt == SG_DTYPE_F32 ? 4 : 2)) return set_error(SG_ERR_SHAPE, "xent_local: unaligned");
  if (rows == 0) return SG_OK;
  SG_DISPATCH_T(ldt, TL, (launch_k(xent_local_kernel<TL>, dim3(grid_for(rows, 8)), dim3(256), 0, S(stream), static_cast<const TL*>(logits), rows, ldl, (int)n_real, labels, col_lo, lmax, gmax, packed)));
  return launch_check();
}

extern "C" int sg_xent_rescale(int64_t rows, const float* lmax, const float* gmax, float* packed, void* stream) {
  clear_error();
  if (rows <= 0) return SG_OK;
  launch_k(xent_rescale_kernel, dim3(grid_for(rows, 256)), dim3(256), 0, S(stream), rows, lmax, gmax, packed);
  return launch_check();
}

extern "C" int sg_xent_loss(int64_t rows, const float* gmax, const float* packed, float* loss_rows, float* partial,
                            void* stream) {
  clear_error();
  if (cudaMemsetAsync(partial, 0, sizeof(float), S(stream)) != cudaSuccess) return set_error(SG_ERR_CUDA, "memset");
  if (rows <= 0) return SG_OK;
  launch_k(xent_loss_kernel, dim3(grid_for(rows, 256, 2)), dim3(256), 0, S(stream), rows, gmax, packed, loss_rows, partial);
  return launch_check();
}

extern "C" int sg_xent_bwd(const void* logits, int ldt, int64_t rows, int64_t ldl, int64_t n_real, int64_t ncols,
                           const int64_t* labels, int64_t col_lo, const float* gmax, const float* packed, float scale,
                           void* dl, int dldt, int64_t lddl, void* stream) {
  clear_error();
  if (rows < 0 || n_real < 0 || ncols < n_real) return set_error(SG_ERR_SHAPE, "xent_bwd: bad extents");
  if (!aligned16(logits, ldl, ldt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(dl, lddl, dldt == SG_DTYPE_F32 ? 4 : 2))
    return set_error(SG_ERR_SHAPE, "xent_bwd: unaligned");
  if (rows == 0 || ncols == 0) return SG_OK;
  SG_DISPATCH_T(ldt, TL, SG_DISPATCH_T(dldt, TO, (launch_k(xent_bwd_kernel<TL, TO>, dim3(grid_for(rows, 8)), dim3(256), 0, S(stream), static_cast<const TL*>(logits), rows, ldl, (int)n_real, (int)ncols, labels, col_lo, gmax, packed, scale, static_cast<TO*>(dl), lddl))));
  return launch_check();
}

extern "C" int sg_embed_fwd(const int64_t* ids, int64_t n, int64_t lo, int64_t vb, const void* table, int tdt,
                            int64_t ldt, int64_t hc, void* out, int odt, int64_t ldo, void* stream) {
  clear_error();
  if (n < 0 || hc < 1 || vb < 0) return set_error(SG_ERR_SHAPE, "embed_fwd: bad extents");
  if (!aligned16(table, ldt, tdt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(out, ldo, odt == SG_DTYPE_F32 ? 4 : 2))
    return set_error(SG_ERR_SHAPE, "embed_fwd: unaligned");
  if (n == 0) return SG_OK;
  SG_DISPATCH_T(tdt, TT, SG_DISPATCH_T(odt, TO, (launch_k(embed_fwd_kernel<TT, TO>, dim3(grid_for(n, 8)), dim3(256), 0, S(stream), ids, n, lo, vb, static_cast<const TT*>(table), ldt, (int)hc, static_cast<TO*>(out), ldo))));
  return launch_check();
}

extern "C" int sg_check_ids(const int64_t* ids, int64_t n, int64_t v, int* flag, void* stream) {
  clear_error();
  if (n < 0 || v < 1 || !flag) return set_error(SG_ERR_CONFIG, "check_ids: bad arguments");
  if (n == 0) return SG_OK;
  launch_k(check_ids_kernel, dim3((unsigned)std::min<long long>((n + 255) / 256, 1184)), dim3(256), 0, S(stream), ids,
           (long long)n, (long long)v, flag);
  return launch_check();
}

extern "C" int sg_embed_bwd(const int64_t* ids, int64_t n, int64_t lo, int64_t vb, const void* dout, int ddt,
                            int64_t ldd, int64_t hc, float* grad, int64_t ldg, void* stream) {
  clear_error();
  if (n < 0 || hc < 1 || vb < 0) return set_error(SG_ERR_SHAPE, "embed_bwd: bad extents");
  if (!aligned16(dout, ldd, ddt == SG_DTYPE_F32 ? 4 : 2)) return set_error(SG_ERR_SHAPE, "embed_bwd: unaligned");
  if (n == 0) return SG_OK;
  static const bool deterministic = [] {
    const char* e = getenv("SG_DETERMINISTIC");
    return e && atoi(e) != 0;
  }();
  if (deterministic) {
    if (n > INT32_MAX) return set_error(SG_ERR_SHAPE, "embed_bwd: too many tokens for the deterministic path");
    const unsigned blocks = (unsigned)std::max<long long>(1, std::min<long long>((vb + 7) / 8, 148LL * 16));
    SG_DISPATCH_T(ddt, TD, (launch_k(embed_bwd_det_kernel<TD>, dim3(blocks), dim3(256), 0, S(stream), ids, n, lo, vb, static_cast<const TD*>(dout), ldd, (int)hc, grad, ldg)));
  } else {
    SG_DISPATCH_T(ddt, TD, (launch_k(embed_bwd_kernel<TD>, dim3(grid_for(n, 8)), dim3(256), 0, S(stream), ids, n, lo, vb, static_cast<const TD*>(dout), ldd, (int)hc, grad, ldg)));
  }
  return launch_check();
}

extern "C" int sg_sgd_multi(const sg_sgd_item* items, int n, float lr, void* stream) {
  clear_error();
  if (n < 0 || (n > 0 && !items)) return set_error(SG_ERR_CONFIG, "sgd: bad item list");
  for (int base = 0; base < n; base += kSgdMax) {
    SgdBatch bt{};
    bt.lr = lr;
    long long chunks = 0;
    for (int i = base; i < n && bt.n < kSgdMax; ++i) {
      const sg_sgd_item& it = items[i];
      if (it.rows < 0 || it.cols < 0 || !it.w || (!it.g && !it.w_bf16)) return set_error(SG_ERR_SHAPE, "sgd: bad item");
      if (it.rows == 0 || it.cols == 0) continue;
      const int k = bt.n++;
      bt.w[k] = it.w;
      bt.wl[k] = static_cast<bf16*>(it.w_bf16);
      bt.g[k] = it.g;
      bt.ldw[k] = it.ldw; bt.ldl[k] = it.ldl; bt.ldg[k] = it.ldg; bt.cols[k] = it.cols;
      bt.total[k] = it.rows * it.cols;
      bt.vec4[k] = it.cols % 4 == 0 && it.ldw % 4 == 0 && (!it.g || it.ldg % 4 == 0) && (!it.w_bf16 || it.ldl % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(it.w) & 15) == 0 && (reinterpret_cast<uintptr_t>(it.g) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(it.w_bf16) & 7) == 0;
      bt.first_chunk[k] = chunks;
      chunks += (bt.total[k] + kSgdChunk - 1) / kSgdChunk;
    }
    bt.first_chunk[bt.n] = chunks;
    if (chunks == 0) continue;
    if (g_sms <= 0) g_sms = sg_device_sm_count();
    const long long grid = std::min<long long>(chunks, (long long)(g_sms > 0 ? g_sms : 148) * 8);
    launch_k(sgd_multi_kernel, dim3((int)grid), dim3(256), 0, S(stream), bt);
    const int rc = launch_check();
    if (rc != SG_OK) return rc;
  }
  return SG_OK;
}

extern "C" int sg_sgd(float* w, int64_t ldw, void* w_bf16, int64_t ldl, const float* g, int64_t ldg, float lr,
                      int64_t rows, int64_t cols, void* stream) {
  sg_sgd_item it{w, w_bf16, g, ldw, ldl, ldg, rows, cols};
  return sg_sgd_multi(&it, 1, lr, stream);
}

extern "C" int sg_cast(const void* src, int sdt, void* dst, int ddt, int64_t n, void* stream) {
  clear_error();
  if (n <= 0) return SG_OK;
  SG_DISPATCH_T(sdt, TS, SG_DISPATCH_T(ddt, TD, (launch_k(cast_kernel<TS, TD>, dim3(grid_for(n, 256, 4)), dim3(256), 0, S(stream), static_cast<const TS*>(src), static_cast<TD*>(dst), n))));
  return launch_check();
}

extern "C" int sg_fold(void* dst, int dt, const void* const* srcs, int nsrc, int64_t n, int accumulate, int op_max,
                       void* stream) {
  clear_error();
  if (nsrc < 0 || nsrc > 8 || (nsrc == 0 && !accumulate)) return set_error(SG_ERR_CONFIG, "fold: 1..8 sources");
  if (n <= 0 || nsrc == 0) return SG_OK;
  SrcList l{};
  for (int i = 0; i < nsrc; ++i) l.p[i] = srcs[i];
  SG_DISPATCH_T(dt, T, (launch_k(fold_kernel<T>, dim3(grid_for(n, 256, 4)), dim3(256), 0, S(stream), static_cast<T*>(dst), l, nsrc, n, accumulate, op_max)));
  return launch_check();
}

extern "C" int sg_epilogue(const float* x, int64_t rows, int64_t cols, int64_t ldx, float alpha, const float* bias,
                           const void* cin, int cdt, int64_t ldc, int act, void* aux, int64_t ldaux, void* out,
                           int odt, int64_t ldo, void* stream) {
  clear_error();
  if (rows < 0 || cols < 1) return set_error(SG_ERR_SHAPE, "epilogue: bad extents");
  if (act == SG_ACT_DGELU && !aux) return set_error(SG_ERR_CONFIG, "epilogue: DGELU needs aux");
  if (!aligned16(x, ldx, 4) || !aligned16(cin, ldc, cdt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(aux, ldaux, 2) ||
      !aligned16(out, ldo, odt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(bias, 0, 4))
    return set_error(SG_ERR_SHAPE, "epilogue: unaligned");
  if (rows == 0) return SG_OK;
  SG_DISPATCH_T(cdt, TC, SG_DISPATCH_T(odt, TO, (launch_k(epilogue_kernel<TC, TO>, dim3(grid_for(rows, 8)), dim3(256), 0, S(stream), x, rows, (int)cols, ldx, alpha, bias, static_cast<const TC*>(cin), ldc, act, static_cast<bf16*>(aux), ldaux, static_cast<TO*>(out), ldo))));
  return launch_check();
}

extern "C" int sg_attn_rowdot(const void* dO, int dt, int64_t ldo, const void* O, int64_t ldO, int64_t rows, int64_t nh,
                              int64_t d, int64_t s, float* out, void* stream) {
  clear_error();
  if (rows < 0 || nh < 1 || d < 1 || s < 1 || rows % s) return set_error(SG_ERR_SHAPE, "attn_rowdot: bad extents");
  if (!aligned16(dO, ldo, dt == SG_DTYPE_F32 ? 4 : 2) || !aligned16(O, ldO, dt == SG_DTYPE_F32 ? 4 : 2) ||
      (d * (dt == SG_DTYPE_F32 ? 4 : 2)) % 16)
    return set_error(SG_ERR_SHAPE, "attn_rowdot: unaligned");
  if (rows == 0) return SG_OK;
  const int64_t nv_rd = nh * 64 / 256;
  if (dt == SG_DTYPE_BF16 && d == 64 && (nh * 64) % 256 == 0 && (nv_rd <= 4 || nv_rd == 8)) {
    const int nv = (int)(nh * 64 / 256);
    const dim3 g2(grid_for(rows, 8, 8));
#define SG_ROWDOT(NV) launch_k(attn_rowdot64_kernel<NV>, g2, dim3(256), 0, S(stream), static_cast<const bf16*>(dO), ldo, static_cast<const bf16*>(O), ldO, rows, (int)nh, (int)s, out)
    switch (nv) {
      case 1: SG_ROWDOT(1); break;
      case 2: SG_ROWDOT(2); break;
      case 3: SG_ROWDOT(3); break;
      case 4: SG_ROWDOT(4); break;
      default: SG_ROWDOT(8); break;
    }
#undef SG_ROWDOT
    return launch_check();
  }
  SG_DISPATCH_T(dt, T, (launch_k(attn_rowdot_kernel<T>, dim3(grid_for(rows * nh, 256, 8)), dim3(256), 0, S(stream), static_cast<const T*>(dO), ldo, static_cast<const T*>(O), ldO, rows, (int)nh, (int)d, (int)s, out)));
  return launch_check();
}

extern "C" int sg_dgelu(const void* dact, int64_t lda, const void* mid, int64_t ldm, int64_t rows, int64_t cols,
                        void* out, int odt, int64_t ldo, float* colsum, void* stream) {
  clear_error();
  if (rows < 0 || cols < 1) return set_error(SG_ERR_SHAPE, "dgelu: bad extents");
  if (!aligned16(dact, lda, 2) || !aligned16(mid, ldm, 2) || !aligned16(out, ldo, odt == SG_DTYPE_F32 ? 4 : 2))
    return set_error(SG_ERR_SHAPE, "dgelu: unaligned");
  if (rows == 0) return SG_OK;
#define SG_DGELU(FULL) SG_DISPATCH_T(odt, TO, (launch_k(dgelu_kernel<TO, 4, FULL>, dim3(seg_grid(rows, cols, 4, 2)), dim3(256), 0, S(stream), static_cast<const bf16*>(dact), lda, static_cast<const bf16*>(mid), ldm, rows, (int)cols, static_cast<TO*>(out), ldo, colsum)))
  if (cols % 8 == 0)
    SG_DGELU(true);
  else
    SG_DGELU(false);
#undef SG_DGELU
  return launch_check();
}

extern "C" int sg_qkv_grad_finish(const float* dq, int64_t lddq, void* dqkv, int64_t ldg, int64_t rows, int64_t hb,
                                  float* colsum, int64_t cols, void* stream) {
  clear_error();
  if (rows < 0 || hb < 1 || hb % 256 != 0) return set_error(SG_ERR_SHAPE, "qkv_grad_finish: hb must be a multiple of 256");
  if (cols != hb && cols != 3 * hb) return set_error(SG_ERR_SHAPE, "qkv_grad_finish: cols must be hb or 3 hb");
  if (!aligned16(dq, lddq, 4) || !aligned16(dqkv, ldg, 2)) return set_error(SG_ERR_SHAPE, "qkv_grad_finish: unaligned");
  if (rows == 0) return SG_OK;
  // cols = hb: only the dQ segments (their bf16 conversion and column sums)
  launch_k(qkv_grad_finish_kernel<2>, seg_grid(rows, cols, 2, 3), dim3(256), 0, S(stream), dq,
           lddq, static_cast<bf16*>(dqkv), ldg, rows, (int)hb, colsum);
  return launch_check();
}
