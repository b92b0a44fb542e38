// Shared TMA tensor-map construction (implemented in sg_gemm.cu).
#pragma once
#include <cuda.h>

namespace sg {
// 4-D bf16 map over (inner, outer, b2, b1), SWIZZLE_128B, box box_inner x box_outer;
// b2 moves before outer when its stride is smaller (e.g. heads inside a row).
int tmap_bf16_4d(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long nb2, long long nb1,
                 long long ld, long long s2, long long s1, int box_inner, int box_outer, int* b2_first);
}  // namespace sg

namespace sg {
// 4-D fp32 map with a 32 x 32 box, SWIZZLE_128B (128-byte rows): epilogue tiles
// for TMA stores / reduce-adds of fp32 results.
int tmap_f32_tile_4d(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long nb2,
                     long long nb1, long long ld, long long s2, long long s1, int* b2_first);
}  // namespace sg

namespace sg {
// 4-D bf16 map with a 32 x 32 box, SWIZZLE_64B (64-byte rows): bf16 epilogue tiles.
int tmap_bf16_tile_4d(CUtensorMap* map, const void* ptr, long long inner, long long outer, long long nb2,
                      long long nb1, long long ld, long long s2, long long s1, int* b2_first);
}  // namespace sg
