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
  int32_t log2g;    // group size G = 2^log2g, 5 <= log2g <= 12
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
  int32_t log2g;
  int32_t lane_elems;  // 16: 256-bit stores (y 32-B, packed 16-B aligned); 8: 128-bit stores
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
cudaError_t enqueue_quantize(const QItem* items, int32_t count, int log2g, cudaStream_t s);
cudaError_t enqueue_dequantize(const DItem* items, int32_t count, int log2g, cudaStream_t s);

// Host-side launchers (gact_quantize.cu / gact_dequant.cu). Return cudaError_t of the launch.
// `dtype` in {0,1,2}; `bits` in {1,2,4,8}. Tile sizes: quantize max(G, 256), dequant 256.
template <int MAXB>
cudaError_t launch_quantize(const QBatch<MAXB>& p, int dtype, int bits, cudaStream_t s);
template <int MAXB>
cudaError_t launch_group_stats(const QBatch<MAXB>& p, int dtype, cudaStream_t s);
template <int MAXB>
cudaError_t launch_dequantize(const DBatch<MAXB>& p, int dtype, int bits, cudaStream_t s);

inline int64_t quantize_tile_elems(int log2g) { return log2g >= 8 ? (int64_t(1) << log2g) : 256; }
// Each tensor's quantize tile count is rounded up to this, so that a CTA unit (8 warps x up
// to 8 consecutive tiles) never straddles two tensors of a batch.
constexpr int64_t kTileAlign = 64;
inline int64_t quantize_tiles(int64_t n, int log2g) {
  const int64_t te = quantize_tile_elems(log2g);
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
