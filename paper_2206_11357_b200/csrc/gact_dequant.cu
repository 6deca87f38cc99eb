// gact_dequant.cu — fused unpack + dequantize kernels (steps a4-a5 of DESIGN.md §1;
// T^{-1}_{h,b} of App. Prop. 3; "Decompressor dequantizes context tensors",
// §5.2), sm_100a.
//
// A warp owns a 256-element tile at a time; each lane decodes a chunk of 8 elements:
// one 1/2/4/8-byte load of its packed unit, one broadcast load of (mn, scale) of its group,
// then per element  q = field(unit) ; qf = float(q) via the 2^23 magic number (FADD2) ;
// y = fma(qf, scale, mn) (FFMA2, one rounding) ; RNE to the output dtype (F2FP pack) ;
// one 16- or 32-byte store. U tiles are decoded per iteration for memory-level parallelism.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gact_device.cuh"
#include "gact_internal.h"


namespace gact {

namespace {

template <int MAXB>
__device__ __forceinline__ int advance_cursor(const DBatch<MAXB>& P, int cur, int64_t tile) {
  if constexpr (MAXB > 1) {
    while (cur + 1 < P.count && tile >= P.tile_start[cur + 1]) ++cur;
  }
  return cur;
}

// The chunk's unit; for b < 8 it lies inside one word (index < nwords since e0 < n), for
// b = 8 its second word exists only if e0 + 4 < n.
template <int BITS>
__device__ __forceinline__ uint2 load_unit(const uint32_t* packed, int64_t e0, int64_t n) {
  const unsigned char* bytes = reinterpret_cast<const unsigned char*>(packed) + (e0 * BITS) / 8;
  if constexpr (BITS == 1) {
    return make_uint2(__ldg(reinterpret_cast<const uint8_t*>(bytes)), 0u);
  } else if constexpr (BITS == 2) {
    return make_uint2(__ldg(reinterpret_cast<const uint16_t*>(bytes)), 0u);
  } else if constexpr (BITS == 4) {
    return make_uint2(__ldg(reinterpret_cast<const uint32_t*>(bytes)), 0u);
  } else {
    if (e0 + kChunk <= n) return __ldg(reinterpret_cast<const uint2*>(bytes));
    const uint32_t* w = reinterpret_cast<const uint32_t*>(bytes);
    return make_uint2(__ldg(w), e0 + 4 < n ? __ldg(w + 1) : 0u);
  }
}

// The 8 bit patterns 0x4B00_0000 | q_j (the floats 2^23 + q_j) of a chunk's unit.
//   b = 8: one byte permute per element (PRMT with the 0x4B byte);
//   b = 4: even / odd nibbles split into bytes with two masks, then byte permutes;
//   b = 1, 2: shift + mask-or per element.
template <int BITS>
__device__ __forceinline__ void magic_codes(uint2 u, uint32_t m[8]) {
  if constexpr (BITS == 8) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      m[j] = __byte_perm(u.x, 0x4B000000u, 0x7540 | j);
      m[4 + j] = __byte_perm(u.y, 0x4B000000u, 0x7540 | j);
    }
  } else if constexpr (BITS == 4) {
    const uint32_t ev = u.x & 0x0F0F0F0Fu;         // bytes: q0 q2 q4 q6
    const uint32_t od = (u.x >> 4) & 0x0F0F0F0Fu;  // bytes: q1 q3 q5 q7
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      m[2 * j] = __byte_perm(ev, 0x4B000000u, 0x7540 | j);
      m[2 * j + 1] = __byte_perm(od, 0x4B000000u, 0x7540 | j);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = ((u.x >> (j * BITS)) & ((1u << BITS) - 1u)) | 0x4B000000u;
  }
}

// y_j = fma(q_j, scale, mn) for the 8 elements of a unit, as 4 packed pairs.
template <int BITS>
__device__ __forceinline__ void decode8(uint2 u, float mn, float scale, float y[8]) {
  const f2_t mn2 = f2_make(mn, mn), sc2 = f2_make(scale, scale);
  const f2_t magic = f2_make(8388608.0f, 8388608.0f);
  uint32_t m[8];
  magic_codes<BITS>(u, m);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const f2_t q2 = f2_sub_rn(f2_bits(m[2 * p], m[2 * p + 1]), magic);  // exact: q_j as float
    f2_split(f2_fma_rn(q2, sc2, mn2), y[2 * p], y[2 * p + 1]);
  }
}

template <int DT>
__device__ __forceinline__ void store8(void* ybase, int64_t e0, const float y[8]) {
  if constexpr (DT == DT_F32) {
    float* p = static_cast<float*>(ybase) + e0;
    __stcs(reinterpret_cast<float4*>(p), make_float4(y[0], y[1], y[2], y[3]));
    __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(y[4], y[5], y[6], y[7]));
  } else {
    uint32_t w[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      if constexpr (DT == DT_BF16) {
        __nv_bfloat162 h = __floats2bfloat162_rn(y[2 * p], y[2 * p + 1]);
        w[p] = *reinterpret_cast<uint32_t*>(&h);
      } else {
        __half2 h = __floats2half2_rn(y[2 * p], y[2 * p + 1]);
        w[p] = *reinterpret_cast<uint32_t*>(&h);
      }
    }
    uint4* p = reinterpret_cast<uint4*>(static_cast<uint16_t*>(ybase) + e0);
    __stcs(p, make_uint4(w[0], w[1], w[2], w[3]));
  }
}

// 16 elements of one lane with 256-bit streaming stores (y 32-byte aligned): 32 bytes of
// bf16 / f16 or 2 x 32 bytes of f32. Wide stores reach a markedly higher write bandwidth
// than 128-bit ones on B200.
__device__ __forceinline__ void st256(void* p, const uint32_t w[8]) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]),
               "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
}

template <int DT>
__device__ __forceinline__ void store16(void* ybase, int64_t e0, const float y[16]) {
  if constexpr (DT == DT_F32) {
    float* p = static_cast<float*>(ybase) + e0;
    st256(p, reinterpret_cast<const uint32_t*>(y));
    st256(p + 8, reinterpret_cast<const uint32_t*>(y) + 8);
  } else {
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if constexpr (DT == DT_BF16) {
        __nv_bfloat162 h = __floats2bfloat162_rn(y[2 * q], y[2 * q + 1]);
        w[q] = *reinterpret_cast<uint32_t*>(&h);
      } else {
        __half2 h = __floats2half2_rn(y[2 * q], y[2 * q + 1]);
        w[q] = *reinterpret_cast<uint32_t*>(&h);
      }
    }
    st256(static_cast<uint16_t*>(ybase) + e0, w);
  }
}

// The packed codes of 16 consecutive elements (2*BITS bytes; packed 16-byte aligned) as the
// units of their two 8-element halves.
template <int BITS>
__device__ __forceinline__ void load_unit16(const unsigned char* p, uint2& u0, uint2& u1) {
  if constexpr (BITS == 1) {
    const uint32_t v = __ldg(reinterpret_cast<const uint16_t*>(p));
    u0 = make_uint2(v & 0xFFu, 0u);
    u1 = make_uint2(v >> 8, 0u);
  } else if constexpr (BITS == 2) {
    const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(p));
    u0 = make_uint2(v & 0xFFFFu, 0u);
    u1 = make_uint2(v >> 16, 0u);
  } else if constexpr (BITS == 4) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    u0 = make_uint2(v.x, 0u);
    u1 = make_uint2(v.y, 0u);
  } else {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    u0 = make_uint2(v.x, v.y);
    u1 = make_uint2(v.z, v.w);
  }
}

template <int DT>
__device__ __forceinline__ void store1(void* ybase, int64_t e, float y) {
  if constexpr (DT == DT_F32) {
    static_cast<float*>(ybase)[e] = y;
  } else if constexpr (DT == DT_BF16) {
    static_cast<__nv_bfloat16*>(ybase)[e] = __float2bfloat16_rn(y);
  } else {
    static_cast<__half*>(ybase)[e] = __float2half_rn(y);
  }
}

// The group of element e (a multiple of 8): e >> log2g for G = 2^log2g; otherwise the
// quotient of its 8-element chunk index by G / 8 through the precomputed reciprocal
// (DBatch::gdiv; exact for chunk indices < 2^55).
template <bool POW2>
__device__ __forceinline__ int64_t group_of(int64_t e, int log2g, uint64_t gdiv) {
  if constexpr (POW2) return e >> log2g;
  else return (int64_t)__umul64hi((uint64_t)e >> 3, gdiv);
}

// The tail of a tensor (its last, partial unit): chunk by chunk, guarded. Out of line.
template <int DT, int BITS>
__device__ __noinline__ void dequant_generic(const DTensor T, int64_t e_first, int chunks,
                                             int log2g, uint64_t gdiv, int lane) {
  for (int k = 0; k < chunks; ++k) {
    const int64_t e = e_first + (int64_t)k * kDequantTileElems + lane * kChunk;
    if (e >= T.n) continue;
    const uint2 unit = load_unit<BITS>(T.packed, e, T.n);
    const int64_t g = log2g >= 0 ? group_of<true>(e, log2g, gdiv) : group_of<false>(e, log2g, gdiv);
    float y[8];
    decode8<BITS>(unit, __ldg(T.group_min + g), __ldg(T.group_scale + g), y);
    if (e + kChunk <= T.n) {
      store8<DT>(T.y, e, y);
    } else {
      for (int j = 0; j < 8; ++j)
        if (e + j < T.n) store1<DT>(T.y, e + j, y[j]);
    }
  }
}

// Grid = waves x resident CTAs: many waves (CTAs take units dynamically) reach a far higher
// write bandwidth than a persistent grid (bf16 ResNet-50 set: 5.8 -> 6.6 TB/s).
#ifndef GACT_D_WAVES
#define GACT_D_WAVES 32
#endif
#ifndef GACT_D_UNIT
#define GACT_D_UNIT 4
#endif
// 5 resident CTAs per SM (48 registers, no spills; 6 would spill): more stores in flight.
// Single 2^28-element bf16 tensors, b = 1: 108 -> 92 us; 2^27, b = 2: 60 -> 52 us; BERT
// layer dequantize -3.5%; fp32 output within 1%.
#ifndef GACT_D_MINB
#define GACT_D_MINB 5
#endif
constexpr int kDequantUnit = GACT_D_UNIT;  // tiles per warp per unit
static_assert(kDequantAlign % (kWarps * kDequantUnit) == 0, "CTA unit must divide the alignment");

// CTAs walk units of 8 warps x U tiles (tensors padded to kDequantAlign tiles), so the
// unit's tensor bookkeeping is CTA-uniform; a warp decodes U consecutive tiles of 32 x LE
// elements (LE = 16: 256-bit stores, needs y 32-byte and packed 16-byte aligned; LE = 8:
// 128-bit stores, the ABI's 16-byte alignment).
template <int DT, int BITS, int MAXB, int LE, bool POW2 = true>
__global__ void __launch_bounds__(kThreads, GACT_D_MINB)
    dequantize_kernel(const __grid_constant__ DBatch<MAXB> P) {
  constexpr int U = kDequantUnit;
  constexpr int CU = kWarps * U;
  constexpr int TE = 32 * LE;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  int cur = 0;
  for (int64_t cu = blockIdx.x; cu < P.tiles_total / CU; cu += gridDim.x) {
    cur = advance_cursor(P, cur, cu * CU);
    const DTensor& T = P.t[cur];
    const int64_t e_base = (cu * CU - P.tile_start[cur] + (int64_t)warp * U) * TE;
    if (e_base + U * TE > T.n) {
      if (e_base < T.n) dequant_generic<DT, BITS>(T, e_base, U * TE / (int)kDequantTileElems, P.log2g, P.gdiv, lane);
      continue;
    }
    const int64_t e_lane = e_base + lane * LE;
    const unsigned char* src = reinterpret_cast<const unsigned char*>(T.packed) + (e_lane * BITS) / 8;
    uint2 unit[U][LE / 8];
    float mn[U], sc[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const unsigned char* p = src + (k * TE * BITS) / 8;
      if constexpr (LE == 16) {
        load_unit16<BITS>(p, unit[k][0], unit[k][1]);
      } else {
        if constexpr (BITS == 1) unit[k][0] = make_uint2(__ldg(p), 0u);
        else if constexpr (BITS == 2) unit[k][0] = make_uint2(__ldg(reinterpret_cast<const uint16_t*>(p)), 0u);
        else if constexpr (BITS == 4) unit[k][0] = make_uint2(__ldg(reinterpret_cast<const uint32_t*>(p)), 0u);
        else unit[k][0] = __ldg(reinterpret_cast<const uint2*>(p));
      }
      const int64_t g = group_of<POW2>(e_lane + k * TE, P.log2g, P.gdiv);  // LE | G: one group per lane
      mn[k] = __ldg(T.group_min + g);
      sc[k] = __ldg(T.group_scale + g);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      float y[LE];
#pragma unroll
      for (int h = 0; h < LE / 8; ++h) decode8<BITS>(unit[k][h], mn[k], sc[k], y + 8 * h);
      if constexpr (LE == 16) store16<DT>(T.y, e_lane + k * TE, y);
      else store8<DT>(T.y, e_lane + k * TE, y);
    }
  }
}

template <typename K>
int max_blocks_per_sm(K kernel) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess || b < 1) b = 1;
  return b;
}

template <auto Kernel, typename PB>
cudaError_t launch_dk(const PB& p, cudaStream_t s) {
  static const int per_sm = max_blocks_per_sm(Kernel);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = p.tiles_total / (kWarps * kDequantUnit);
  const int64_t cap = (int64_t)sms * per_sm * GACT_D_WAVES;
  const int grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  Kernel<<<grid, kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

#ifndef GACT_D_WIDE16
#define GACT_D_WIDE16 1  // 256-bit stores also for 2-byte outputs
#endif

template <int DT, int BITS, int MAXB>
cudaError_t launch_d(const DBatch<MAXB>& p, cudaStream_t s) {
  if (p.log2g < 0) {  // G not a power of two (16 | G): the same kernels with the division
    if (p.lane_elems == 16) return launch_dk<dequantize_kernel<DT, BITS, MAXB, 16, false>>(p, s);
    return launch_dk<dequantize_kernel<DT, BITS, MAXB, 8, false>>(p, s);
  }
  if (p.lane_elems == 16 && (DT == DT_F32 || GACT_D_WIDE16)) {
    return launch_dk<dequantize_kernel<DT, BITS, MAXB, 16>>(p, s);
  }
  if (p.lane_elems == 16) {  // narrow kernel over a tile space counted for 16-element lanes
    DBatch<MAXB> q = p;
    q.lane_elems = 8;
    for (int i = 0; i <= q.count; ++i) q.tile_start[i] *= 2;
    q.tiles_total *= 2;
    return launch_dk<dequantize_kernel<DT, BITS, MAXB, 8>>(q, s);
  }
  return launch_dk<dequantize_kernel<DT, BITS, MAXB, 8>>(p, s);
}

template <int DT, int MAXB>
cudaError_t launch_d_bits(const DBatch<MAXB>& p, int bits, cudaStream_t s) {
  switch (bits) {
    case 1: return launch_d<DT, 1, MAXB>(p, s);
    case 2: return launch_d<DT, 2, MAXB>(p, s);
    case 4: return launch_d<DT, 4, MAXB>(p, s);
    default: return launch_d<DT, 8, MAXB>(p, s);
  }
}

}  // namespace

template <int MAXB>
cudaError_t launch_dequantize(const DBatch<MAXB>& p, int dtype, int bits, cudaStream_t s) {
  if (p.tiles_total == 0) return cudaSuccess;
  switch (dtype) {
    case DT_F32: return launch_d_bits<DT_F32, MAXB>(p, bits, s);
    case DT_BF16: return launch_d_bits<DT_BF16, MAXB>(p, bits, s);
    default: return launch_d_bits<DT_F16, MAXB>(p, bits, s);
  }
}

template cudaError_t launch_dequantize<1>(const DBatch<1>&, int, int, cudaStream_t);
template cudaError_t launch_dequantize<kMaxBatch>(const DBatch<kMaxBatch>&, int, int, cudaStream_t);

}  // namespace gact
