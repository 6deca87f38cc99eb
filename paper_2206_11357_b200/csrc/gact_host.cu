// gact_host.cu — the C ABI of include/gact.h: argument validation, launch parameter
// blocks, and the host-side bit allocator (eqn:ilp P:471-475, greedy P:534).
//
// No allocation, no synchronisation, no state: every call validates its arguments, fills
// a parameter block that travels by value into the kernel (__grid_constant__) and enqueues
// one launch per (dtype, bits) class on the caller's stream.
#include <cmath>
#include <cstring>
#include <queue>
#include <vector>

#include "gact.h"
#include "gact_internal.h"

namespace {

using gact::DBatch;
using gact::DTensor;
using gact::QBatch;
using gact::QTensor;

bool valid_bits(int32_t b) { return b == 1 || b == 2 || b == 4 || b == 8; }
bool valid_dtype(int32_t d) { return d == GACT_F32 || d == GACT_BF16 || d == GACT_F16; }

// Group sizes: multiples of 32 in [32, 4096]; powers of two take the specialised kernels.
bool valid_group(int32_t G) { return gact::group_log2(G) >= -1; }

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Validation of one quantize-side tensor (x, packed, stats) — header rules.
gact_status check_q(const void* x, int32_t dtype, int64_t n, int32_t bits, const uint32_t* packed,
                    const float* mn, const float* sc, bool need_packed) {
  if (!valid_bits(bits)) return GACT_ERR_UNSUPPORTED_BITS;
  if (n < 0 || !valid_dtype(dtype)) return GACT_ERR_INVALID_ARG;
  if (n == 0) return GACT_OK;
  if (!x || !mn || !sc || (need_packed && !packed)) return GACT_ERR_INVALID_ARG;
  if (!aligned(x, 16) || !aligned(mn, 4) || !aligned(sc, 4) || (need_packed && !aligned(packed, 8)))
    return GACT_ERR_ALIGNMENT;
  return GACT_OK;
}

gact_status check_d(const uint32_t* packed, const float* mn, const float* sc, int64_t n,
                    int32_t bits, const void* y, int32_t y_dtype) {
  if (!valid_bits(bits)) return GACT_ERR_UNSUPPORTED_BITS;
  if (n < 0 || !valid_dtype(y_dtype)) return GACT_ERR_INVALID_ARG;
  if (n == 0) return GACT_OK;
  if (!packed || !mn || !sc || !y) return GACT_ERR_INVALID_ARG;
  if (!aligned(y, 16) || !aligned(packed, 8) || !aligned(mn, 4) || !aligned(sc, 4))
    return GACT_ERR_ALIGNMENT;
  return GACT_OK;
}

QTensor make_q(const void* x, int64_t n, int32_t bits, uint64_t seed, uint32_t* packed, float* mn,
               float* sc) {
  QTensor t;
  t.x = x;
  t.packed = packed;
  t.group_min = mn;
  t.group_scale = sc;
  t.n = n;
  t.nwords = ceil_div(n * bits, 32);
  t.seed = seed;
  t.ctr0 = 0;
  return t;
}

DTensor make_d(void* y, int64_t n, const uint32_t* packed, const float* mn, const float* sc) {
  DTensor t;
  t.y = y;
  t.packed = packed;
  t.group_min = mn;
  t.group_scale = sc;
  t.n = n;
  return t;
}

gact_status from_cuda(cudaError_t e) { return e == cudaSuccess ? GACT_OK : GACT_ERR_CUDA; }

// 256-bit stores / 128-bit code loads of the wide dequantize path need y 32-byte and packed
// 16-byte aligned (PyTorch allocations are); otherwise the 16-byte path of the ABI is used.
bool wide_ok(const void* y, const void* packed) { return aligned(y, 32) && aligned(packed, 16); }

}  // namespace

namespace gact {

// A launch of one tensor takes the single-tensor kernels (QBatch<1> / DBatch<1>): a 64-byte
// instead of an 18 KB parameter block, and CTA-uniform bookkeeping. Measured on a 2^27-element
// bf16 tensor, back to back (tools/launch_cost.py): quantize 65.5 -> 61.7 us at b = 1.
template <template <int> class PB>
PB<1> single_of(const PB<kMaxBatch>& p) {
  static_assert(offsetof(PB<1>, tile_start) == offsetof(PB<kMaxBatch>, tile_start),
                "the scalar prefix of the parameter block does not depend on MAXB");
  PB<1> q;
  std::memset(&q, 0, sizeof(q));
  std::memcpy(&q, &p, offsetof(PB<1>, tile_start));
  q.tile_start[0] = p.tile_start[0];
  q.tile_start[1] = p.tile_start[1];
  q.t[0] = p.t[0];
  return q;
}

// Items are grouped by (dtype, bits); each class is launched in chunks of <= kMaxBatch
// items, in input order (the parameter blocks are 16 KB: kept off the stack).
cudaError_t enqueue_quantize(const QItem* items, int32_t count, int32_t G, cudaStream_t s) {
  static thread_local QBatch<kMaxBatch> p;
  bool seen[3][9] = {};
  for (int32_t c = 0; c < count; ++c) {
    const int32_t dt = items[c].dtype, bits = items[c].bits;
    if (items[c].t.n == 0 || seen[dt][bits]) continue;
    seen[dt][bits] = true;
    int32_t i = c;
    while (i < count) {
      std::memset(&p, 0, offsetof(QBatch<kMaxBatch>, tile_start));
      p.log2g = group_log2(G);
      p.group = G;
      p.Lf = (float)((1 << bits) - 1);
      int32_t m = 0;
      int64_t tiles = 0;
      for (; i < count && m < kMaxBatch; ++i) {
        const QItem& it = items[i];
        if (it.t.n == 0 || it.dtype != dt || it.bits != bits) continue;
        p.tile_start[m] = tiles;
        p.t[m] = it.t;
        tiles += quantize_tiles(it.t.n, G, dt);
        ++m;
      }
      if (m == 0) break;
      p.count = m;
      p.tile_start[m] = tiles;
      p.tiles_total = tiles;
      const cudaError_t e = m == 1 ? launch_quantize<1>(single_of(p), dt, bits, s)
                                   : launch_quantize<kMaxBatch>(p, dt, bits, s);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

cudaError_t enqueue_dequantize(const DItem* items, int32_t count, int32_t G, cudaStream_t s) {
  static thread_local DBatch<kMaxBatch> p;
  bool seen[3][9] = {};
  for (int32_t c = 0; c < count; ++c) {
    const int32_t dt = items[c].dtype, bits = items[c].bits;
    if (items[c].t.n == 0 || seen[dt][bits]) continue;
    seen[dt][bits] = true;
    int32_t i = c;
    while (i < count) {
      std::memset(&p, 0, offsetof(DBatch<kMaxBatch>, tile_start));
      p.log2g = group_log2(G);
      p.gdiv = p.log2g < 0 ? chunk_group_divisor(G) : 0;
      // the items this launch covers decide the lane width: wide if all are aligned for it
      int32_t m = 0;
      bool wide = true;
      for (int32_t j = i; j < count && m < kMaxBatch; ++j) {
        const DItem& it = items[j];
        if (it.t.n == 0 || it.dtype != dt || it.bits != bits) continue;
        wide = wide && wide_ok(it.t.y, it.t.packed);
        ++m;
      }
      p.lane_elems = wide ? 16 : 8;
      m = 0;
      int64_t tiles = 0;
      for (; i < count && m < kMaxBatch; ++i) {
        const DItem& it = items[i];
        if (it.t.n == 0 || it.dtype != dt || it.bits != bits) continue;
        p.tile_start[m] = tiles;
        p.t[m] = it.t;
        tiles += dequant_tiles(it.t.n, p.lane_elems);
        ++m;
      }
      if (m == 0) break;
      p.count = m;
      p.tile_start[m] = tiles;
      p.tiles_total = tiles;
      const cudaError_t e = m == 1 ? launch_dequantize<1>(single_of(p), dt, bits, s)
                                   : launch_dequantize<kMaxBatch>(p, dt, bits, s);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace gact

// ===================================================================================== ABI
extern "C" {

int32_t gact_version(void) { return (1 << 16) | 0; }

const char* gact_status_string(int32_t s) {
  switch (s) {
    case GACT_OK: return "GACT_OK";
    case GACT_ERR_INVALID_ARG: return "GACT_ERR_INVALID_ARG";
    case GACT_ERR_UNSUPPORTED_BITS: return "GACT_ERR_UNSUPPORTED_BITS";
    case GACT_ERR_GROUP_SIZE: return "GACT_ERR_GROUP_SIZE";
    case GACT_ERR_ALIGNMENT: return "GACT_ERR_ALIGNMENT";
    case GACT_ERR_INFEASIBLE: return "GACT_ERR_INFEASIBLE";
    case GACT_ERR_CUDA: return "GACT_ERR_CUDA";
    default: return "GACT_ERR_UNKNOWN";
  }
}

int64_t gact_num_groups(int64_t n, int32_t group_size) {
  if (n < 0 || group_size < 1) return -1;
  return ceil_div(n, group_size);
}

int64_t gact_packed_words(int64_t n, int32_t bits) {
  if (n < 0 || bits < 1) return -1;
  return ceil_div(n * bits, 32);
}

gact_status gact_group_stats(const void* x, int32_t dtype, int64_t n, int32_t group_size,
                             int32_t bits, float* group_min, float* group_scale, void* stream) {
  gact_status st = check_q(x, dtype, n, bits, nullptr, group_min, group_scale, false);
  if (st != GACT_OK) return st;
  if (!valid_group(group_size)) return GACT_ERR_GROUP_SIZE;
  if (n == 0) return GACT_OK;
  QBatch<1> p;
  std::memset(&p, 0, sizeof(p));
  p.count = 1;
  p.log2g = gact::group_log2(group_size);
  p.group = group_size;
  p.Lf = (float)((1 << bits) - 1);
  p.t[0] = make_q(x, n, bits, 0, nullptr, group_min, group_scale);
  p.tile_start[0] = 0;
  p.tiles_total = p.tile_start[1] = gact::quantize_tiles(n, group_size, dtype);
  return from_cuda(gact::launch_group_stats<1>(p, dtype, static_cast<cudaStream_t>(stream)));
}

gact_status gact_quantize_pack(const void* x, int32_t dtype, int64_t n, int32_t group_size,
                               int32_t bits, uint64_t seed, uint32_t* packed, float* group_min,
                               float* group_scale, void* stream) {
  gact_status st = check_q(x, dtype, n, bits, packed, group_min, group_scale, true);
  if (st != GACT_OK) return st;
  if (!valid_group(group_size)) return GACT_ERR_GROUP_SIZE;
  if (n == 0) return GACT_OK;
  QBatch<1> p;
  std::memset(&p, 0, sizeof(p));
  p.count = 1;
  p.log2g = gact::group_log2(group_size);
  p.group = group_size;
  p.Lf = (float)((1 << bits) - 1);
  p.t[0] = make_q(x, n, bits, seed, packed, group_min, group_scale);
  p.tile_start[0] = 0;
  p.tiles_total = p.tile_start[1] = gact::quantize_tiles(n, group_size, dtype);
  return from_cuda(gact::launch_quantize<1>(p, dtype, bits, static_cast<cudaStream_t>(stream)));
}

gact_status gact_unpack_dequantize(const uint32_t* packed, const float* group_min,
                                   const float* group_scale, int64_t n, int32_t group_size,
                                   int32_t bits, void* y, int32_t y_dtype, void* stream) {
  gact_status st = check_d(packed, group_min, group_scale, n, bits, y, y_dtype);
  if (st != GACT_OK) return st;
  if (!valid_group(group_size)) return GACT_ERR_GROUP_SIZE;
  if (n == 0) return GACT_OK;
  DBatch<1> p;
  std::memset(&p, 0, sizeof(p));
  p.count = 1;
  p.log2g = gact::group_log2(group_size);
  p.gdiv = p.log2g < 0 ? gact::chunk_group_divisor(group_size) : 0;
  p.lane_elems = wide_ok(y, packed) ? 16 : 8;
  p.t[0] = make_d(y, n, packed, group_min, group_scale);
  p.tile_start[0] = 0;
  p.tiles_total = p.tile_start[1] = gact::dequant_tiles(n, p.lane_elems);
  return from_cuda(gact::launch_dequantize<1>(p, y_dtype, bits, static_cast<cudaStream_t>(stream)));
}

gact_status gact_quantize_pack_batch(const gact_tensor_desc* descs, int32_t count,
                                     int32_t group_size, void* stream) {
  if (count < 0 || (count > 0 && !descs)) return GACT_ERR_INVALID_ARG;
  for (int32_t i = 0; i < count; ++i) {
    const gact_tensor_desc& d = descs[i];
    gact_status st = check_q(d.data, d.dtype, d.n, d.bits, d.packed, d.group_min, d.group_scale, true);
    if (st != GACT_OK) return st;
  }
  if (!valid_group(group_size)) return GACT_ERR_GROUP_SIZE;
  static thread_local std::vector<gact::QItem> items;
  items.clear();
  for (int32_t i = 0; i < count; ++i) {
    const gact_tensor_desc& d = descs[i];
    items.push_back({make_q(d.data, d.n, d.bits, d.seed, d.packed, d.group_min, d.group_scale), d.dtype, d.bits});
  }
  return from_cuda(gact::enqueue_quantize(items.data(), count, group_size, static_cast<cudaStream_t>(stream)));
}

gact_status gact_unpack_dequantize_batch(const gact_tensor_desc* descs, int32_t count,
                                         int32_t group_size, void* stream) {
  if (count < 0 || (count > 0 && !descs)) return GACT_ERR_INVALID_ARG;
  for (int32_t i = 0; i < count; ++i) {
    const gact_tensor_desc& d = descs[i];
    gact_status st = check_d(d.packed, d.group_min, d.group_scale, d.n, d.bits, d.data, d.dtype);
    if (st != GACT_OK) return st;
  }
  if (!valid_group(group_size)) return GACT_ERR_GROUP_SIZE;
  static thread_local std::vector<gact::DItem> items;
  items.clear();
  for (int32_t i = 0; i < count; ++i) {
    const gact_tensor_desc& d = descs[i];
    items.push_back({make_d(d.data, d.n, d.packed, d.group_min, d.group_scale), d.dtype, d.bits});
  }
  return from_cuda(gact::enqueue_dequantize(items.data(), count, group_size, static_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------------------- allocator
// S(b) = (2^b - 1)^-2, S(32) = 0.
static double S_of(int32_t b) {
  if (b == 32) return 0.0;
  const double m = (double)((1ull << b) - 1ull);
  return 1.0 / (m * m);
}

extern "C" double gact_variance_factor(int32_t bits) {
  if (bits == 32 || (bits >= 1 && bits <= 16)) return S_of(bits);
  return -1.0;
}

gact_status gact_allocate_bits(const double* c, const int64_t* D, int32_t L,
                               const int32_t* ladder, int32_t n_ladder, uint64_t budget_bits,
                               int32_t* bits_out) {
  if (L < 0 || n_ladder < 1 || !ladder) return GACT_ERR_INVALID_ARG;
  if (L > 0 && (!c || !D || !bits_out)) return GACT_ERR_INVALID_ARG;
  for (int32_t k = 0; k < n_ladder; ++k) {
    if (!((ladder[k] >= 1 && ladder[k] <= 16) || ladder[k] == 32)) return GACT_ERR_INVALID_ARG;
    if (k > 0 && ladder[k] <= ladder[k - 1]) return GACT_ERR_INVALID_ARG;
  }
  for (int32_t l = 0; l < L; ++l)
    if (std::isnan(c[l]) || c[l] < 0.0 || D[l] < 1) return GACT_ERR_INVALID_ARG;
  unsigned __int128 need_min = 0, total = 0;
  for (int32_t l = 0; l < L; ++l) {
    need_min += (unsigned __int128)ladder[0] * (uint64_t)D[l];
    total += (unsigned __int128)ladder[n_ladder - 1] * (uint64_t)D[l];
  }
  if (need_min > budget_bits) return GACT_ERR_INFEASIBLE;

  // Min-heap of (ratio of the next step down, tensor index), ordered lexicographically:
  // it holds exactly one entry per tensor (its current ratio), so every pop is the global
  // minimum with ties to the smaller index — the step a full scan would take.
  std::vector<int32_t> level(L, n_ladder - 1);
  auto ratio = [&](int32_t l) {
    const int32_t hi = ladder[level[l]], lo = ladder[level[l] - 1];
    const double num = c[l] * (S_of(lo) - S_of(hi));
    const double den = (double)(hi - lo) * (double)D[l];
    return num / den;
  };
  struct Item {
    double r;
    int32_t l;
  };
  auto worse = [](const Item& a, const Item& b) { return a.r > b.r || (a.r == b.r && a.l > b.l); };
  std::priority_queue<Item, std::vector<Item>, decltype(worse)> heap(worse);
  if (n_ladder > 1)
    for (int32_t l = 0; l < L; ++l) heap.push(Item{ratio(l), l});
  while (total > budget_bits && !heap.empty()) {
    const Item it = heap.top();
    heap.pop();
    const int32_t l = it.l;
    const int32_t hi = ladder[level[l]], lo = ladder[level[l] - 1];
    total -= (unsigned __int128)(hi - lo) * (uint64_t)D[l];
    level[l] -= 1;
    if (level[l] > 0) heap.push(Item{ratio(l), l});
  }
  for (int32_t l = 0; l < L; ++l) bits_out[l] = ladder[level[l]];
  return GACT_OK;
}

}  // extern "C"
