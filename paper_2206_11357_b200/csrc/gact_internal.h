// gact_internal.h — parameter blocks shared by the host launchers and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gact {

constexpr int kMaxBatch = 256;  // == GACT_MAX_BATCH

// One tensor of a quantize launch.
struct QTensor {
  const void* x;
  uint32_t* packed;
  float* group_min;
  float* group_scale;
  int64_t n;
  int64_t nwords;
  uint64_t seed;
  uint64_t ctr0;  // Philox block offset of x[0]: (element offset of x in its whole tensor, a multiple of 512) / 16
};

// Launch parameters (passed by value as __grid_constant__; MAXB = 1 for single calls).
// Tensors are concatenated in tile space: tensor i owns tiles [tile_start[i], tile_start[i+1]).
template <int MAXB>
struct QBatch {
  int32_t count;
  int32_t log2g;    // G = 2^log2g (5 <= log2g <= 12), or -1: G not a power of two (`group`)
  int32_t group;    // G: a multiple of 32 in [32, 4096]
  float Lf;         // 2^bits - 1 (used by the stats-only kernel; BITS is a template param otherwise)
  int64_t tiles_total;
  int64_t tile_start[MAXB + 1];
  QTensor t[MAXB];
};

struct DTensor {
  void* y;
  const uint32_t* packed;
  const float* group_min;
  const float* group_scale;
  int64_t n;
};

template <int MAXB>
struct DBatch {
  int32_t count;
  int32_t log2g;       // as in QBatch; -1: G not a power of two
  int32_t lane_elems;  // 16: 256-bit stores (y 32-B, packed 16-B aligned); 8: 128-bit stores
  uint64_t gdiv;       // G not a power of two: ceil(2^64 / (G / 8)), the group of the 8-element
                       // chunk c is umul64hi(c, gdiv) (exact for c < 2^55)
  int64_t tiles_total;
  int64_t tile_start[MAXB + 1];
  DTensor t[MAXB];
};

// One tensor (or piece of a tensor) of a multi-class enqueue (gact_host.cu).
struct QItem {
  QTensor t;
  int32_t dtype, bits;
};
struct DItem {
  DTensor t;
  int32_t dtype, bits;
};
// Enqueue quantize / dequantize launches for `count` items (any mix of dtypes and bits):
// one launch per (dtype, bits) class and per <= kMaxBatch items, in input order. Items with
// n == 0 are skipped. Arguments are assumed validated. Returns the first launch error.
cudaError_t enqueue_quantize(const QItem* items, int32_t count, int32_t G, cudaStream_t s);
cudaError_t enqueue_dequantize(const DItem* items, int32_t count, int32_t G, cudaStream_t s);

// Group sizes: a multiple of 32 in [32, 4096]. group_log2 gives log2 G for powers of two, -1
// for the others (valid; the generic kernels), and -2 for invalid G.
inline int group_log2(int32_t G) {
  if (G < 32 || G > 4096 || (G & 31) != 0) return -2;
  if ((G & (G - 1)) != 0) return -1;
  int l = 0;
  while ((1 << l) < G) ++l;
  return l;
}
// M = ceil(2^64 / d), d = G / 8 in [4, 512] (G not a power of two): floor((2^64 - 1) / d) + 1
// equals ceil(2^64 / d) for every d > 1 that is not a power of two. Then for a chunk index
// c < 2^55, umul64hi(c, M) = floor(c M / 2^64) = floor(c / d): c M / 2^64 - c / d < c 2^-64
// < 2^-9 <= 1 / d, and frac(c / d) <= 1 - 1 / d.
inline uint64_t chunk_group_divisor(int32_t G) {
  const uint64_t d = (uint64_t)(G / 8);
  return ~0ull / d + 1;
}

// Host-side launchers (gact_quantize.cu / gact_dequant.cu). Return cudaError_t of the launch.
// `dtype` in {0,1,2}; `bits` in {1,2,4,8}. Tile sizes: quantize_tile_elems(G, dtype), dequant 256.
template <int MAXB>
cudaError_t launch_quantize(const QBatch<MAXB>& p, int dtype, int bits, cudaStream_t s);
template <int MAXB>
cudaError_t launch_group_stats(const QBatch<MAXB>& p, int dtype, cudaStream_t s);
template <int MAXB>
cudaError_t launch_dequantize(const DBatch<MAXB>& p, int dtype, int bits, cudaStream_t s);

// Quantize tile: max(G, 256) elements for powers of two (a tile holds 256 / G groups below
// 256); for other G, a super-tile of lcm(G, 256) elements = P = lcm / 256 warp passes holding
// lcm / G whole groups below 256 (and below 512 for 2-byte inputs), else one group (a warp per
// group). `dtype`: GACT_F32 / GACT_BF16 / GACT_F16 (0 / 1 / 2).
inline int64_t quantize_tile_elems(int32_t G, int32_t dtype) {
  if (group_log2(G) >= 0) return G >= 256 ? G : 256;
  if (G > 256 && (dtype == 0 || G > 512)) return G;
  int64_t a = G, b = 256;
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return (int64_t)G / a * 256;
}
// Each tensor's quantize tile count is rounded up to this, so that a CTA unit (8 warps x up
// to 8 consecutive tiles) never straddles two tensors of a batch.
#ifndef GACT_TILE_ALIGN
#define GACT_TILE_ALIGN 128
#endif
constexpr int64_t kTileAlign = GACT_TILE_ALIGN;
inline int64_t quantize_tiles(int64_t n, int32_t G, int32_t dtype) {
  const int64_t te = quantize_tile_elems(G, dtype);
  const int64_t t = (n + te - 1) / te;
  return (t + kTileAlign - 1) / kTileAlign * kTileAlign;
}
constexpr int64_t kDequantTileElems = 256;  // the narrow (8-element lane) tile
// Dequantize tile counts are rounded up to this (CTA units never straddle tensors).
constexpr int64_t kDequantAlign = 32;
inline int64_t dequant_tiles(int64_t n, int lane_elems) {
  const int64_t te = 32 * lane_elems;
  const int64_t t = (n + te - 1) / te;
  return (t + kDequantAlign - 1) / kDequantAlign * kDequantAlign;
}

}  // namespace gact
