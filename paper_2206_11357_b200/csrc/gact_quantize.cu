// gact_quantize.cu — fused group-reduce + stochastic-rounding quantize + bit-pack kernels
// (steps a1-a3 of DESIGN.md §1; the quantizer of App. Prop. 3), sm_100a.
//
// Work decomposition. A tensor of n elements is cut into tiles of TE = max(G, 256)
// elements; a warp owns a tile at a time and each lane a chunk of 8 consecutive elements
// (8 random bytes = half a Philox4x32-10 block, R3: a lane's chunks in 256-element
// sub-tiles 2m and 2m + 1 share one block; one 16- or 32-byte coalesced load).
// Tensors of a batch are concatenated in tile space (QBatch::tile_start), each tensor's
// tile count rounded up to kTileAlign = 128, so that a CTA UNIT (8 warps x U consecutive
// tiles) never straddles two tensors. CTAs walk units grid-stride: the active window of a
// launch is compact in memory, each warp streams U * TE contiguous elements per step, and
// the unit's bookkeeping (tensor, seed, pointers) is CTA-uniform (single-tensor launches
// keep it in the uniform datapath; batched launches index the descriptor table per unit).
//  * G in {256, ..., 4096} (2048 and 4096: 2-byte inputs only): one tile == one group, reduced
//    in registers, coded from the same registers, written once: x is read exactly once. A
//    lane holds 16 chunks per unit for 2-byte inputs (U = 16 / CPL tiles; 8 chunks for
//    G = 2048 and for single-tensor b = 1 launches), 4 for fp32. The lane's Philox blocks (two
//    chunks per block) are computed while the unit's loads are in flight (they depend only on
//    (seed, element index)), with their rounds 0-1 shared (philox4x32_10_xn). Min / max:
//    2-byte units of U >= 2 groups fold packed (min, -max) pairs and reduce all U groups with
//    one recursive-halving butterfly (GACT_Q_XRED), each lane computes one group's division,
//    and the groups' (mn, inv) reach the lanes through shared memory; otherwise FMNMX3
//    in-thread, one CREDUX per group for min and max, divisions on U lanes, shuffles.
//  * G in {32, 64, 128}: a tile holds 256/G groups of G/8 lanes. 2-byte inputs: units of
//    G / 8 tiles (16 at G = 32) reduced by one butterfly over the lane bits of a group's
//    segment (quantize_smallx_kernel); fp32: segmented shuffles per tile.
//  * G in {2048, 4096}, fp32: the group spans the CTA's registers (one HBM read).
//  * G not a power of two: a warp per group, two passes (the second from L1 / L2).
// A tensor's last tile may be partial (n % TE != 0): it takes the guarded generic path.
#include <cfloat>

#include "gact_device.cuh"
#include "gact_internal.h"

namespace gact {

namespace {

constexpr unsigned kFull = 0xffffffffu;

template <int MAXB>
__device__ __forceinline__ int advance_cursor(const QBatch<MAXB>& P, int cur, int64_t tile) {
  if constexpr (MAXB > 1) {
    while (cur + 1 < P.count && tile >= P.tile_start[cur + 1]) ++cur;
  }
  return cur;
}

// The tensor holding tile `tile` (the last i with tile_start[i] <= tile), by binary search:
// a CTA's first unit may lie anywhere in a launch of up to 256 tensors.
template <int MAXB>
__device__ __forceinline__ int first_cursor(const QBatch<MAXB>& P, int64_t tile) {
  if constexpr (MAXB == 1) {
    return 0;
  } else {
    int lo = 0, hi = P.count - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.tile_start[mid] <= tile) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  }
}

// Random bytes (R3, include/gact.h). The chunk of 8 elements starting at element e (a multiple
// of 8) takes half of Philox block 32 (e / 512) + (e / 8 mod 32) (+ the tensor piece's block
// offset ctr0): words 0-1 in the first 256 elements of its 512-element span, 2-3 in the second.
__device__ __forceinline__ uint64_t rand_block(const QTensor& T, int64_t e) {
  return (((uint64_t)e >> 9) << 5) + (((uint64_t)e >> 3) & 31u) + T.ctr0;
}
__device__ __forceinline__ uint2 rand_half(uint4 r, int64_t e) {
  return ((e >> 8) & 1) ? make_uint2(r.z, r.w) : make_uint2(r.x, r.y);
}
__device__ __forceinline__ uint2 chunk_rand(const QTensor& T, int64_t e) {
  return rand_half(philox4x32_10(rand_block(T, e), (uint32_t)T.seed, (uint32_t)(T.seed >> 32)), e);
}

template <int DT>
__device__ __forceinline__ void load8_guarded(float v[8], const void* x, int64_t e, int64_t n,
                                              float fill) {
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = (e + j < n) ? load1<DT>(x, e + j) : fill;
}

// Codes of a chunk whose elements >= n were replaced by mn (t = 0 -> q = 0, the zero
// padding of the last word).
template <int DT, int BITS>
__device__ __forceinline__ void code_chunk_guarded(const QTensor& T, int64_t e, float mn,
                                                   float inv) {
  float v[8];
  load8_guarded<DT>(v, T.x, e, T.n, mn);
  store_unit_guarded<BITS>(T.packed, e, T.nwords, quantize_chunk<BITS>(v, mn, inv, chunk_rand(T, e)));
}

// One tile of a tensor with G >= 256, full or partial (the group may be short): warp
// reduction, per-lane division, codes; chunks inside the tensor by 16/32-byte loads (the coding
// pass re-reads them from L1 / L2), the tensor's last chunk element by element. Each chunk's
// random bytes from its own Philox block (chunk_rand). The slow generic path, out of line.
template <int DT, int BITS, bool STATS>
__device__ __noinline__ void tile_generic(const QTensor T, int64_t e0, int log2g, float Lf,
                                          int lane) {
  const int cpl = 1 << (log2g - 8);
  float lmn = FLT_MAX, lmx = -FLT_MAX;  // neutral; the tile has at least one element
  for (int c = 0; c < cpl; ++c) {
    const int64_t e = e0 + c * kWarpTile + lane * kChunk;
    if (e + kChunk <= T.n) {
      Raw8<DT> raw;
      load8<DT>(raw, T.x, e);
      chunk_minmax_raw<DT>(raw, lmn, lmx);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (e + j < T.n) {
          const float x = load1<DT>(T.x, e + j);
          lmn = fminf(lmn, x);
          lmx = fmaxf(lmx, x);
        }
      }
    }
  }
  const GroupParams gp = group_params(warp_min(lmn), warp_max(lmx), Lf);
  const int64_t g = e0 >> log2g;
  if (lane == 0) {
    T.group_min[g] = gp.mn;
    T.group_scale[g] = gp.scale;
  }
  if constexpr (!STATS) {
    for (int c = 0; c < cpl; ++c) {
      const int64_t e = e0 + c * kWarpTile + lane * kChunk;
      if (e + kChunk <= T.n) {
        Raw8<DT> raw;
        load8<DT>(raw, T.x, e);
        store_unit<BITS>(T.packed, e, quantize_chunk_raw<DT, BITS>(raw, gp.mn, gp.inv, chunk_rand(T, e)));
      } else if ((e * BITS) / 32 < T.nwords) {
        code_chunk_guarded<DT, BITS>(T, e, gp.mn, gp.inv);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// G in {256, 512, 1024} (2048 for 2-byte inputs): CPL = G/256 chunks per lane, U = quant_unit()/CPL tiles per unit,
// all in registers.
// Grid = waves x resident CTAs. Several waves (CTAs pick up units dynamically as others
// retire) beat a persistent grid for the FMA-bound 2-byte inputs (+6% at bf16); fp32 inputs
// (HBM-bound) keep the persistent grid. Measured on B200: DESIGN.md §4.
#ifndef GACT_Q_WAVES_F32
#define GACT_Q_WAVES_F32 1
#endif
#ifndef GACT_Q_WAVES
#define GACT_Q_WAVES 8
#endif
#ifndef GACT_QS_MINB
#define GACT_QS_MINB 3  // small-G kernel: minimum resident CTAs per SM (register cap)
#endif
#ifndef GACT_BYTE2_CPL
#define GACT_BYTE2_CPL 2  // byte-2 codes (code_and_pack) for G <= 256 * this: G = 512 +1.5-3% at every b; G = 1024 mixed (-0.7% .. +1%), not taken
#endif
#ifndef GACT_BYTE2_MIX
#define GACT_BYTE2_MIX 4  // G = 256: every 4th chunk packs by shift-add (0: every chunk byte-2)
#endif
#ifndef GACT_ANYG_K3
#define GACT_ANYG_K3 4  // G = 96 / 192, 2-byte: super-tiles per warp iteration (at 2 CTAs per SM; 2 / 4: +9% / +17% over 1)
#endif
#ifndef GACT_ANYG_K5
#define GACT_ANYG_K5 2  // G = 160 / 320, 2-byte (at 2 CTAs per SM: +22% over 1)
#endif
#ifndef GACT_ANYG_MG2
#define GACT_ANYG_MG2 1  // G > 256 not a power of two: two groups per warp iteration where they fit (G = 288 +57%, 800 +6-22%)
#endif
#ifndef GACT_ANYG_SMALL_PK2
#define GACT_ANYG_SMALL_PK2 6  // super-tile kernel: 2 CTAs per SM (128 registers) from this many passes (G = 224: +9%)
#endif
#ifndef GACT_Q_ANYG_REG
#define GACT_Q_ANYG_REG 1  // G not a power of two: the register-resident one-pass kernel
#endif
#ifndef GACT_Q_SMEMBC
// 2-byte units: the groups' (mn, inv) reach the lanes through shared memory (one 8-byte
// broadcast load per tile) instead of two shuffles per tile. A/B: single 2^28 bf16 G = 256
// b = 2 / 8 +2% / +1%, b = 4 -0.6%; ResNet-50 bench quantize 0.885 -> 0.892.
#define GACT_Q_SMEMBC 1
#endif
#ifndef GACT_Q_XRED
#define GACT_Q_XRED 1  // 2-byte units of U >= 2 groups: butterfly reduction of packed (min, -max)
#endif
// Chunks (Philox blocks) per lane per CTA unit. 2-byte inputs (issue-bound): 16 -- the unit's
// 8 Philox blocks share rounds 0-1, and the per-unit work (tensor lookup, key schedule, loop,
// addresses, the division of each lane's group) is amortised over 16 tiles; 128 registers
// (12-40 bytes of spills), 2 CTAs per SM. Measured against 8-chunk units at 3 CTAs per SM
// (80 registers), A/B on one box: ResNet-50 bench quantize 0.845 -> 0.883, BERT-large 24
// layers 0.771 -> 0.797; single 2^28 bf16 tensors b = 2 / 4 -2.5 / -3% time, b = 8 equal,
// b = 1 +0.8% -- so single-tensor b = 1 launches keep 8-chunk units (GACT_Q_UNIT_B1S), and
// so does G = 2048 (16 chunks = 2 groups per warp: b = 2 / 4 / 8 2% / 2% / 1.5% slower).
// G = 4096 (2-byte): 16 chunks = one group per warp; replaced a warp-pair kernel (8 chunks
// per lane, the pair's min / max through shared memory behind a named barrier): bf16 2^28
// b = 1 / 2 / 4 117.2 / 116.9 / 119.8 -> 112.0 / 111.9 / 113.2 us, b = 8 equal.
// fp32 (HBM-bound): 4 (8 would spill).
#ifndef GACT_Q_UNIT
#define GACT_Q_UNIT 16
#endif
#ifndef GACT_Q_UNIT_B1S
#define GACT_Q_UNIT_B1S 8
#endif
#ifndef GACT_Q_UNIT_F32
#define GACT_Q_UNIT_F32 4
#endif
#ifndef GACT_Q_MINB
#define GACT_Q_MINB 3  // 8-chunk 2-byte units and the fp32 CTA-wide kernel: 3 CTAs per SM
#endif
#ifndef GACT_Q_MINB_U16
#define GACT_Q_MINB_U16 2  // 16-chunk 2-byte units: 2 CTAs per SM (128 registers)
#endif
#ifndef GACT_Q_MINB_F32
#define GACT_Q_MINB_F32 2
#endif
#ifndef GACT_Q_MINB_LOWB
// 8-chunk units, b = 1, single-tensor launches: 2 CTAs per SM (+2-3% at G <= 1024 against 3).
#define GACT_Q_MINB_LOWB 2
#endif
// chunks per lane per unit for group size 256 CPL
template <int DT, int BITS, int MAXB, int CPL>
__host__ __device__ constexpr int quant_unit() {
  return DT == DT_F32 ? GACT_Q_UNIT_F32
         : CPL == 16 ? 16                                            // G = 4096: one group per warp
         : (CPL == 8 || (BITS == 1 && MAXB == 1)) ? GACT_Q_UNIT_B1S  // G = 2048: one group per warp
                                                  : GACT_Q_UNIT;
}
// tiles per warp per unit
template <int DT, int BITS, int MAXB, int CPL>
__host__ __device__ constexpr int unit_tiles() {
  return quant_unit<DT, BITS, MAXB, CPL>() / CPL > 0 ? quant_unit<DT, BITS, MAXB, CPL>() / CPL : 1;
}
template <int DT, int BITS, int MAXB, int CPL>
__host__ __device__ constexpr int quant_minb() {
  return DT == DT_F32 ? GACT_Q_MINB_F32
         : quant_unit<DT, BITS, MAXB, CPL>() >= 16 ? GACT_Q_MINB_U16
         : (BITS == 1 && MAXB == 1) ? GACT_Q_MINB_LOWB : GACT_Q_MINB;
}
static_assert(kWarps * GACT_Q_UNIT <= kTileAlign && kTileAlign % (kWarps * GACT_Q_UNIT) == 0 &&
              kTileAlign % (kWarps * GACT_Q_UNIT_B1S) == 0 &&
              kWarps * GACT_Q_UNIT_F32 <= kTileAlign && kTileAlign % (kWarps * GACT_Q_UNIT_F32) == 0,
              "a CTA unit must divide the tile alignment");

template <int DT, int BITS, int CPL, int MAXB, bool STATS>
__global__ void __launch_bounds__(kThreads, quant_minb<DT, BITS, MAXB, CPL>())
    quantize_big_kernel(const __grid_constant__ QBatch<MAXB> P) {
  constexpr int U = unit_tiles<DT, BITS, MAXB, CPL>();
  constexpr int TE = CPL * kWarpTile;  // == G
#if GACT_Q_SMEMBC
  __shared__ float2 bc[kWarps][U];  // per warp: (mn, inv) of the unit's U groups
#endif
  constexpr int CU = kWarps * U;       // tiles per CTA unit (divides kTileAlign)
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float Lf = STATS ? P.Lf : (float)((1 << BITS) - 1);
  const int64_t cunits = P.tiles_total / CU;
  int cur = first_cursor(P, (int64_t)blockIdx.x * CU);
  // CTA-unit bookkeeping (tensor, seed, base pointers) depends only on blockIdx and the
  // loop counter: it lives in uniform registers.
  for (int64_t cu = blockIdx.x; cu < cunits; cu += gridDim.x) {
    cur = advance_cursor(P, cur, cu * CU);
    const QTensor& T = P.t[cur];
    const int64_t e_base = (cu * CU - P.tile_start[cur]) * TE + (int64_t)warp * U * TE;
    if (e_base + U * TE > T.n) {  // the tensor's last units: guarded, one tile at a time
      for (int k = 0; k < U; ++k)
        if (e_base + k * TE < T.n) tile_generic<DT, BITS, STATS>(T, e_base + k * TE, P.log2g, Lf, lane);
      continue;
    }
    const int64_t e_lane = e_base + lane * kChunk;
    Raw8<DT> raw[U][CPL];
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int c = 0; c < CPL; ++c) load8<DT>(raw[k][c], T.x, e_lane + k * TE + c * kWarpTile);
    // The unit's Philox blocks depend only on the seed and the element index, so they are
    // computed while the loads are in flight. (Computing the NEXT unit's blocks one
    // iteration ahead, or in separate producer warps fed by TMA bulk copies, were both
    // measured slower on B200: DESIGN.md §4.)
    // The lane's chunks sit in the unit's U * CPL consecutive 256-element sub-tiles (chunk
    // kc = k CPL + c in sub-tile kc); sub-tiles 2m and 2m + 1 take the two halves of Philox
    // block blk0 + 32 m (R3: e_base is a multiple of 512, so blk0 = rand_block(T, e_lane)),
    // computed with their rounds 0-1 shared (philox4x32_10_xn).
    static_assert((U * CPL) % 2 == 0, "a unit covers whole 512-element spans");
    uint2 rnd[U][CPL];
    if constexpr (!STATS) {
      uint4 r4[(U * CPL) / 2];
      philox4x32_10_xn<(U * CPL) / 2>(rand_block(T, e_lane), (uint32_t)T.seed, (uint32_t)(T.seed >> 32), r4);
#pragma unroll
      for (int k = 0; k < U; ++k)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const uint4 q = r4[(k * CPL + c) >> 1];
          rnd[k][c] = ((k * CPL + c) & 1) ? make_uint2(q.z, q.w) : make_uint2(q.x, q.y);
        }
    }
#if GACT_Q_XRED
    if constexpr (DT != DT_F32 && !STATS && U >= 2) {
      // (U = 1, G = 2048: one CREDUX pair per unit measured 1% faster than 5 shuffle levels.)
      // 2-byte inputs: every lane folds each of the unit's U tiles (groups) into one packed
      // (min, -max) pair (bf16x2 / f16x2: exact), then a recursive-halving butterfly reduces
      // the U groups across the warp at once. The first log2(U) levels (xor 16, 8, ...) halve
      // the tiles a lane keeps (the lane with bit `mask` set keeps the upper half and sends the
      // lower), the remaining levels finish the reduction of the one left: lane l ends with
      // group t(l) = (l >> (5 - log2 U)) & (U - 1), computes its parameters, and group k's
      // (mn, inv) reach every lane through shared memory (GACT_Q_SMEMBC; else two shuffles
      // from lane k << (5 - log2 U)). For U = 16 (G = 256): 16 shuffles + 16 HMNMX2 for all 16
      // groups, where one CREDUX pair per group needs 32 CREDUX + 32 uniform-to-vector moves
      // + 30 selects.
      constexpr int LU = U == 16 ? 4 : U == 8 ? 3 : U == 4 ? 2 : U == 2 ? 1 : 0;
      static_assert((1 << LU) == U, "U is a power of two <= 16");
      constexpr int SH = 5 - LU;
      uint32_t p[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        p[k] = chunk_minnegmax_packed<DT>(raw[k][0]);
#pragma unroll
        for (int c = 1; c < CPL; ++c) p[k] = min2_packed<DT>(p[k], chunk_minnegmax_packed<DT>(raw[k][c]));
      }
#pragma unroll
      for (int lvl = 0; lvl < LU; ++lvl) {
        const int mask = 16 >> lvl, half = U >> (lvl + 1);
        const bool upper = lane & mask;
#pragma unroll
        for (int j = 0; j < half; ++j) {
          const uint32_t send = upper ? p[j] : p[j + half], keep = upper ? p[j + half] : p[j];
          p[j] = min2_packed<DT>(keep, __shfl_xor_sync(kFull, send, mask));
        }
      }
#pragma unroll
      for (int mask = 16 >> LU; mask >= 1; mask >>= 1) p[0] = min2_packed<DT>(p[0], __shfl_xor_sync(kFull, p[0], mask));
      float a, b;
      unpack_minmax<DT>(p[0], a, b);
      const GroupParams gp = group_params(a, b, Lf);
      if ((lane & ((1 << SH) - 1)) == 0) {
        const int64_t g = e_base / TE + ((lane >> SH) & (U - 1));  // t(l)
        T.group_min[g] = gp.mn;
        T.group_scale[g] = gp.scale;
      }
      unsigned char* out = reinterpret_cast<unsigned char*>(T.packed) + (e_lane * BITS) / 8;
#if GACT_Q_SMEMBC
      // (mn, inv) of the U groups through shared memory: one 8-byte store per group, one
      // broadcast 8-byte load per tile (instead of two shuffles per tile)
      if ((lane & ((1 << SH) - 1)) == 0) bc[warp][(lane >> SH) & (U - 1)] = make_float2(gp.mn, gp.inv);
      __syncwarp();
#endif
#pragma unroll
      for (int k = 0; k < U; ++k) {
#if GACT_Q_SMEMBC
        const float2 pk = bc[warp][k];
        const float mn = pk.x, inv = pk.y;
#else
        const int src = k << SH;  // a lane l with t(l) = k
        const float inv = __shfl_sync(kFull, gp.inv, src);
        const float mn = __shfl_sync(kFull, gp.mn, src);
#endif
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          // G = 256: every GACT_BYTE2_MIX-th chunk takes the shift-add packing (FMA pipes)
          // instead of the byte-2 gather (ALU pipe), balancing the two (A/B, 1 in 4: b = 1
          // +1.5%, ResNet-50 quantize +1%; 1 in 2 slower; at G = 512 the mix measured slower)
          constexpr int MIX = CPL == 1 ? GACT_BYTE2_MIX : 0;
          const bool b2 = CPL <= GACT_BYTE2_CPL && (MIX == 0 || (k * CPL + c) % (MIX > 0 ? MIX : 1) != MIX - 1);
          unsigned char* o = out + ((k * TE + c * kWarpTile) * BITS) / 8;
          if (b2) store_unit_at<BITS>(o, quantize_chunk_raw<DT, BITS, true>(raw[k][c], mn, inv, rnd[k][c]));
          else store_unit_at<BITS>(o, quantize_chunk_raw<DT, BITS, false>(raw[k][c], mn, inv, rnd[k][c]));
        }
      }
#if GACT_Q_SMEMBC
      __syncwarp();  // every lane has read bc[warp] before the next unit writes it
#endif
      continue;
    }
#endif
    float mnk[U], mxk[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      float lmn = FLT_MAX, lmx = -FLT_MAX;
#pragma unroll
      for (int c = 0; c < CPL; ++c) chunk_minmax_raw<DT>(raw[k][c], lmn, lmx);
      mnk[k] = warp_min(lmn);
      mxk[k] = warp_max(lmx);
    }
    // The U groups' divisions run on lanes 0..U-1 (lane l computes group l % U).
    const int sel = lane & (U - 1);
    float a = mnk[0], b = mxk[0];
#pragma unroll
    for (int k = 1; k < U; ++k) {
      a = (sel == k) ? mnk[k] : a;
      b = (sel == k) ? mxk[k] : b;
    }
    const GroupParams gp = group_params(a, b, Lf);
    if (lane < U) {
      const int64_t g = e_base / TE + lane;
      T.group_min[g] = gp.mn;
      T.group_scale[g] = gp.scale;
    }
    if constexpr (!STATS) {
      unsigned char* out = reinterpret_cast<unsigned char*>(T.packed) + (e_lane * BITS) / 8;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const float inv = __shfl_sync(kFull, gp.inv, k);
        const float mn = __fadd_rn(mnk[k], 0.0f);
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          store_unit_at<BITS>(out + ((k * TE + c * kWarpTile) * BITS) / 8,
                              quantize_chunk_raw<DT, BITS>(raw[k][c], mn, inv, rnd[k][c]));
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// G in {2048, 4096}, fp32 inputs: a group spans the CTA (8 warps x CPW chunks per lane), all in
// registers; U = 4/CPW groups per CTA unit. Per group each warp reduces its share with
// CREDUX, parks it in shared memory (double-buffered by unit parity: one barrier per unit),
// and re-reduces the 8 warp partials with CREDUX; the U divisions run on U lanes.
template <int DT, int BITS, int CPW, int MAXB, bool STATS>
__global__ void __launch_bounds__(kThreads, GACT_Q_MINB)
    quantize_cta_kernel(const __grid_constant__ QBatch<MAXB> P) {
  constexpr int U = 4 / CPW;                  // groups per CTA unit
  constexpr int WE = CPW * kWarpTile;         // elements of a group per warp
  constexpr int TE = kWarps * WE;             // == G
  __shared__ float red[2][U][2][kWarps];      // [parity][group][min, max][warp]
  // CPW = 1: the random half a warp's partner computed for it ([parity][group][warp][lane])
  __shared__ uint2 xr[2][CPW == 1 ? U : 1][kWarps][32];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float Lf = STATS ? P.Lf : (float)((1 << BITS) - 1);
  const int64_t cunits = P.tiles_total / U;   // a quantize tile is one group here
  int cur = 0, par = 0;
  // `par` selects the half of red[] a unit uses. It flips only on units that pass the
  // barrier: a guarded unit (no barrier) between two full units must not flip it, or the
  // second full unit would write the half the first one's warps may still be reading.
  for (int64_t cu = blockIdx.x; cu < cunits; cu += gridDim.x) {
    cur = advance_cursor(P, cur, cu * U);
    const QTensor& T = P.t[cur];
    const int64_t e_unit = (cu * U - P.tile_start[cur]) * TE;
    if (e_unit + U * TE > T.n) {  // CTA-uniform: the tensor's last unit, warp k codes group k
      if (warp < U && e_unit + warp * TE < T.n)
        tile_generic<DT, BITS, STATS>(T, e_unit + warp * TE, P.log2g, Lf, lane);
      continue;
    }
    const int64_t e_lane = e_unit + warp * WE + lane * kChunk;
    Raw8<DT> raw[U][CPW];
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int c = 0; c < CPW; ++c) load8<DT>(raw[k][c], T.x, e_lane + k * TE + c * kWarpTile);
    // R3: with CPW = 2 a warp's two chunks of a group are sub-tiles 2m, 2m + 1 (one block);
    // with CPW = 1 the pair of sub-tiles belongs to warps 2m, 2m + 1: the even warp computes
    // the blocks of groups 0-1, the odd one those of groups 2-3, and each hands its partner
    // the other half through shared memory (read after the unit's barrier).
    uint2 rnd[U][CPW];
    const bool odd = warp & 1;
    if constexpr (!STATS) {
      const uint32_t k0 = (uint32_t)T.seed, k1 = (uint32_t)(T.seed >> 32);
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t e = e_lane + k * TE;
        if constexpr (CPW == 2) {
          const uint4 r = philox4x32_10(rand_block(T, e), k0, k1);
          rnd[k][0] = make_uint2(r.x, r.y);
          rnd[k][1] = make_uint2(r.z, r.w);
        } else if ((k >= U / 2) == odd) {
          const uint4 r = philox4x32_10(rand_block(T, e), k0, k1);
          rnd[k][0] = odd ? make_uint2(r.z, r.w) : make_uint2(r.x, r.y);
          xr[par][k][warp ^ 1][lane] = odd ? make_uint2(r.x, r.y) : make_uint2(r.z, r.w);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      float lmn = FLT_MAX, lmx = -FLT_MAX;
#pragma unroll
      for (int c = 0; c < CPW; ++c) chunk_minmax_raw<DT>(raw[k][c], lmn, lmx);
      lmn = warp_min(lmn);
      lmx = warp_max(lmx);
      if (lane == 0) {
        red[par][k][0][warp] = lmn;
        red[par][k][1][warp] = lmx;
      }
    }
    __syncthreads();
    float mnk[U], mxk[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      mnk[k] = warp_min(red[par][k][0][lane & (kWarps - 1)]);
      mxk[k] = warp_max(red[par][k][1][lane & (kWarps - 1)]);
    }
    if constexpr (!STATS && CPW == 1) {
#pragma unroll
      for (int k = 0; k < U; ++k)
        if ((k >= U / 2) != odd) rnd[k][0] = xr[par][k][warp][lane];
    }
    par ^= 1;
    const int sel = lane & (U - 1);
    float a = mnk[0], b = mxk[0];
#pragma unroll
    for (int k = 1; k < U; ++k) {
      a = (sel == k) ? mnk[k] : a;
      b = (sel == k) ? mxk[k] : b;
    }
    const GroupParams gp = group_params(a, b, Lf);
    if (warp == 0 && lane < U) {
      const int64_t g = (e_unit >> P.log2g) + lane;
      T.group_min[g] = gp.mn;
      T.group_scale[g] = gp.scale;
    }
    if constexpr (!STATS) {
      unsigned char* out = reinterpret_cast<unsigned char*>(T.packed) + (e_lane * BITS) / 8;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const float inv = __shfl_sync(kFull, gp.inv, k);
        const float mn = __fadd_rn(mnk[k], 0.0f);
#pragma unroll
        for (int c = 0; c < CPW; ++c)
          store_unit_at<BITS>(out + ((k * TE + c * kWarpTile) * BITS) / 8,
                              quantize_chunk_raw<DT, BITS>(raw[k][c], mn, inv, rnd[k][c]));
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// G in {32, 64, 128}: a 256-element tile holds 256/G groups of lpg = G/8 lanes each;
// units of U tiles (U <= lpg: a group's U divisions run on U lanes of its segment).
#ifndef GACT_QS_XRED
#define GACT_QS_XRED 1  // 2-byte G = 32 / 64 / 128: quantize_smallx_kernel (butterfly over whole units)
#endif
#ifndef GACT_QSX_MIX
#define GACT_QSX_MIX 4  // quantize_smallx_kernel: byte-2 codes for all but every 4th tile (A/B: b <= 2 +1%)
#endif
#ifndef GACT_QS_UNIT
#define GACT_QS_UNIT 8  // 2-byte inputs, G = 64 / 128: tiles per unit (G = 32 and fp32 keep 4)
#endif
template <int DT, int LOG2G>
__host__ __device__ constexpr int small_unit() { return (DT != DT_F32 && LOG2G >= 6) ? GACT_QS_UNIT : 4; }
template <int DT, int BITS, bool STATS>
__device__ __forceinline__ void small_tile(const QTensor& T, int64_t e, bool full, const Raw8<DT>& raw,
                                           uint2 rnd, int log2g, int lpg, float Lf, int lane) {
  float v[8];
  float lmn = FLT_MAX, lmx = -FLT_MAX;
  if (full) {
    chunk_minmax_raw<DT>(raw, lmn, lmx);
  } else {
    load8_guarded<DT>(v, T.x, e, T.n, FLT_MAX);
    lmn = min3f(min3f(v[0], v[1], v[2]), min3f(v[3], v[4], v[5]), fminf(v[6], v[7]));
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (e + j < T.n) lmx = fmaxf(lmx, v[j]);
  }
  for (int o = 1; o < lpg; o <<= 1) {
    lmn = fminf(lmn, __shfl_xor_sync(kFull, lmn, o));
    lmx = fmaxf(lmx, __shfl_xor_sync(kFull, lmx, o));
  }
  const int64_t g = e >> log2g;
  if ((g << log2g) >= T.n) return;  // group entirely beyond the tensor
  const GroupParams gp = group_params(lmn, lmx, Lf);
  if ((lane & (lpg - 1)) == 0) {
    T.group_min[g] = gp.mn;
    T.group_scale[g] = gp.scale;
  }
  if constexpr (!STATS) {
    if (full) {
      store_unit<BITS>(T.packed, e, quantize_chunk_raw<DT, BITS>(raw, gp.mn, gp.inv, rnd));
    } else if ((e * BITS) / 32 < T.nwords) {
      code_chunk_guarded<DT, BITS>(T, e, gp.mn, gp.inv);
    }
  }
}

template <int DT, int BITS, int MAXB, bool STATS, int LOG2G>
__global__ void __launch_bounds__(kThreads, GACT_QS_MINB)
    quantize_small_kernel(const __grid_constant__ QBatch<MAXB> P) {
  constexpr int U = small_unit<DT, LOG2G>();
  const int lane = threadIdx.x & 31;
  const float Lf = STATS ? P.Lf : (float)((1 << BITS) - 1);
  constexpr int lpg = 1 << (LOG2G - 3);  // lanes per group
  const int warp = threadIdx.x >> 5;
  constexpr int CU = kWarps * U;
  int cur = 0;
  for (int64_t cu = blockIdx.x; cu < P.tiles_total / CU; cu += gridDim.x) {
    cur = advance_cursor(P, cur, cu * CU);
    const QTensor& T = P.t[cur];
    const int64_t e_lane = (cu * CU - P.tile_start[cur] + warp * U) * kWarpTile + lane * kChunk;
    const int64_t e_warp = e_lane - lane * kChunk;
    Raw8<DT> raw[U];
    uint2 rnd[U];
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (e_warp + (k + 1) * kWarpTile <= T.n) load8<DT>(raw[k], T.x, e_lane + k * kWarpTile);
    if constexpr (!STATS) {
      // the unit's 4 tiles are 2 whole 512-element spans (tile_start is a multiple of 64):
      // blocks blk0, blk0 + 32 (R3), rounds 0-1 shared (philox4x32_10_xn)
      uint4 r2[U / 2];
      philox4x32_10_xn<U / 2>(rand_block(T, e_lane), (uint32_t)T.seed, (uint32_t)(T.seed >> 32), r2);
#pragma unroll
      for (int k = 0; k < U; ++k)
        rnd[k] = (k & 1) ? make_uint2(r2[k >> 1].z, r2[k >> 1].w) : make_uint2(r2[k >> 1].x, r2[k >> 1].y);
    }
    if (e_warp + U * kWarpTile > T.n) {  // the tensor's last unit: tile by tile, guarded
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t t0 = e_warp + k * kWarpTile;
        if (t0 >= T.n) break;  // warp-uniform: the rest of the unit is padding
        small_tile<DT, BITS, STATS>(T, e_lane + k * kWarpTile, t0 + kWarpTile <= T.n, raw[k], rnd[k],
                                    P.log2g, lpg, Lf, lane);
      }
      continue;
    }
    // Full unit: segmented butterflies give every lane its group's (min, max) for the U tiles;
    // the U divisions of a group run on U different lanes of its segment (lpg >= 4 = U) and
    // are broadcast back with one shuffle per tile.
    float mnk[U], mxk[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if constexpr (DT == DT_F32) {
        float lmn = FLT_MAX, lmx = -FLT_MAX;
        chunk_minmax_raw<DT>(raw[k], lmn, lmx);
#pragma unroll
        for (int o = 1; o < lpg; o <<= 1) {
          lmn = fminf(lmn, __shfl_xor_sync(kFull, lmn, o));
          lmx = fmaxf(lmx, __shfl_xor_sync(kFull, lmx, o));
        }
        mnk[k] = lmn;
        mxk[k] = lmx;
      } else {  // (min, -max) packed in one register: one shuffle + one HMNMX2 per step
        uint32_t pm = chunk_minnegmax_packed<DT>(raw[k]);
#pragma unroll
        for (int o = 1; o < lpg; o <<= 1) pm = min2_packed<DT>(pm, __shfl_xor_sync(kFull, pm, o));
        unpack_minmax<DT>(pm, mnk[k], mxk[k]);
      }
    }
    const int sl = lane & (lpg - 1);  // lane within its group's segment
    const int sel = sl & (U - 1);
    float a = mnk[0], b = mxk[0];
#pragma unroll
    for (int k = 1; k < U; ++k) {
      a = (sel == k) ? mnk[k] : a;
      b = (sel == k) ? mxk[k] : b;
    }
    const GroupParams gp = group_params(a, b, Lf);
    if (sl < U) {  // segment lane k stores tile k's group
      const int64_t g = (e_lane + sl * kWarpTile) >> P.log2g;
      T.group_min[g] = gp.mn;
      T.group_scale[g] = gp.scale;
    }
    if constexpr (!STATS) {
      unsigned char* out = reinterpret_cast<unsigned char*>(T.packed) + (e_lane * BITS) / 8;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const float inv = __shfl_sync(kFull, gp.inv, (lane & ~(lpg - 1)) + k);
        const float mn = __fadd_rn(mnk[k], 0.0f);
        store_unit_at<BITS>(out + (k * kWarpTile * BITS) / 8, quantize_chunk_raw<DT, BITS>(raw[k], mn, inv, rnd[k]));
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// G in {32, 64, 128}, 2-byte inputs: the G = 256 kernel's structure with a tile holding 256 / G
// groups of lpg = G / 8 lanes. A warp unit is U = R lpg tiles (R = 2 at G = 32, else 1); every
// lane folds its chunk of each tile into a packed (min, -max) pair, and a recursive-halving
// butterfly over the lane bits inside a group's segment (xor lpg / 2, ..., 1) leaves lane l
// with the groups of tiles R (l & (lpg - 1)) + r, r < R, in its own segment: U - R shuffles
// per unit for all of the unit's groups (the segmented kernel above: log2(lpg) per tile).
// Each lane computes R divisions; (mn, inv) reach the lanes through shared memory. A tensor's
// last unit takes small_tile per tile. (G = 64 / 128 against the segmented kernel: bf16 2^28
// b = 1-8 +9-10% / +13-19%.)
template <int DT, int BITS, int MAXB, bool STATS, int LOG2G>
__global__ void __launch_bounds__(kThreads, LOG2G >= 7 ? 2 : 3)
    quantize_smallx_kernel(const __grid_constant__ QBatch<MAXB> P) {
  static_assert(DT != DT_F32 && LOG2G >= 5 && LOG2G <= 7, "2-byte inputs, G = 32 / 64 / 128");
  constexpr int lpg = 1 << (LOG2G - 3);  // lanes per group
  constexpr int R = LOG2G == 5 ? 2 : 1;  // groups per lane per unit
  constexpr int U = R * lpg;             // tiles per warp unit
  constexpr int CU = kWarps * U;
  constexpr int GPT = 32 / lpg;          // groups per tile
  constexpr int LU = LOG2G - 3;          // butterfly levels
  __shared__ float2 bc[kWarps][U][GPT];  // (mn, inv) of the unit's groups
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int seg = lane >> LU;            // the lane's group within a tile
  const float Lf = STATS ? P.Lf : (float)((1 << BITS) - 1);
  const int64_t cunits = P.tiles_total / CU;
  int cur = first_cursor(P, (int64_t)blockIdx.x * CU);
  for (int64_t cu = blockIdx.x; cu < cunits; cu += gridDim.x) {
    cur = advance_cursor(P, cur, cu * CU);
    const QTensor& T = P.t[cur];
    const int64_t e_warp = (cu * CU - P.tile_start[cur] + (int64_t)warp * U) * kWarpTile;
    const int64_t e_lane = e_warp + lane * kChunk;
    if (e_warp + U * kWarpTile > T.n) {  // the tensor's last units: tile by tile, guarded
      for (int k = 0; k < U; ++k) {
        const int64_t t0 = e_warp + k * kWarpTile;
        if (t0 >= T.n) break;  // warp-uniform: the rest of the unit is padding
        const int64_t e = e_lane + k * kWarpTile;
        Raw8<DT> raw;
        const bool full = t0 + kWarpTile <= T.n;
        if (full) load8<DT>(raw, T.x, e);
        small_tile<DT, BITS, STATS>(T, e, full, raw, STATS ? make_uint2(0, 0) : chunk_rand(T, e), LOG2G, lpg, Lf, lane);
      }
      continue;
    }
    Raw8<DT> raw[U];
#pragma unroll
    for (int k = 0; k < U; ++k) load8<DT>(raw[k], T.x, e_lane + k * kWarpTile);
    uint2 rnd[U];
    if constexpr (!STATS) {
      uint4 r4[U / 2];
      philox4x32_10_xn<U / 2>(rand_block(T, e_lane), (uint32_t)T.seed, (uint32_t)(T.seed >> 32), r4);
#pragma unroll
      for (int k = 0; k < U; ++k) rnd[k] = (k & 1) ? make_uint2(r4[k >> 1].z, r4[k >> 1].w) : make_uint2(r4[k >> 1].x, r4[k >> 1].y);
    }
    uint32_t p[U];
#pragma unroll
    for (int k = 0; k < U; ++k) p[k] = chunk_minnegmax_packed<DT>(raw[k]);
#pragma unroll
    for (int lvl = 0; lvl < LU; ++lvl) {
      const int mask = (lpg >> 1) >> lvl, half = U >> (lvl + 1);
      const bool upper = lane & mask;
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const uint32_t send = upper ? p[j] : p[j + half], keep = upper ? p[j + half] : p[j];
        p[j] = min2_packed<DT>(keep, __shfl_xor_sync(kFull, send, mask));
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float a, b;
      unpack_minmax<DT>(p[r], a, b);
      const GroupParams gp = group_params(a, b, Lf);
      const int t = R * (lane & (lpg - 1)) + r;  // tile of the lane's r-th group
      const int64_t g = (e_warp + t * kWarpTile) / (lpg * kChunk) + seg;
      T.group_min[g] = gp.mn;
      T.group_scale[g] = gp.scale;
      if constexpr (!STATS) bc[warp][t][seg] = make_float2(gp.mn, gp.inv);
    }
    if constexpr (!STATS) {
      __syncwarp();
      unsigned char* out = reinterpret_cast<unsigned char*>(T.packed) + (e_lane * BITS) / 8;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const float2 pk = bc[warp][k][seg];
        unsigned char* o = out + (k * kWarpTile * BITS) / 8;
        if (GACT_QSX_MIX > 0 && k % (GACT_QSX_MIX > 0 ? GACT_QSX_MIX : 1) != GACT_QSX_MIX - 1)
          store_unit_at<BITS>(o, quantize_chunk_raw<DT, BITS, true>(raw[k], pk.x, pk.y, rnd[k]));
        else
          store_unit_at<BITS>(o, quantize_chunk_raw<DT, BITS, false>(raw[k], pk.x, pk.y, rnd[k]));
      }
      __syncwarp();  // every lane has read bc[warp] before the next unit writes it
    }
  }
}

// ---------------------------------------------------------------------------------------
// G a multiple of 32 that is not a power of two (include/gact.h): one warp per group, the
// group's G / 8 chunks strided over the lanes; min / max by CREDUX, then a second pass codes
// the chunks (re-read: the group's <= 16 KB sit in L1 / L2). Each chunk's random bytes come
// from its own Philox block (chunk_rand: half of the block used). Tiles = groups, 8 per CTA
// unit (tensors padded to kTileAlign tiles). The generic path; powers of two are specialised.
template <int DT, int BITS, int MAXB, bool STATS>
__global__ void __launch_bounds__(kThreads)
    quantize_anyg_kernel(const __grid_constant__ QBatch<MAXB> P) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float Lf = STATS ? P.Lf : (float)((1 << BITS) - 1);
  const int64_t G = P.group;
  const int64_t cunits = P.tiles_total / kWarps;
  int cur = first_cursor(P, (int64_t)blockIdx.x * kWarps);
  for (int64_t cu = blockIdx.x; cu < cunits; cu += gridDim.x) {
    cur = advance_cursor(P, cur, cu * kWarps);
    const QTensor& T = P.t[cur];
    const int64_t g = cu * kWarps - P.tile_start[cur] + warp;
    const int64_t e0 = g * G;
    if (e0 >= T.n) continue;  // alignment padding of the tile space
    const int64_t e1 = e0 + G < T.n ? e0 + G : T.n;
    float lmn = FLT_MAX, lmx = -FLT_MAX;  // neutral; the group has at least one element
    for (int64_t e = e0 + lane * kChunk; e < e1; e += 32 * kChunk) {
      if (e + kChunk <= e1) {
        Raw8<DT> raw;
        load8<DT>(raw, T.x, e);
        chunk_minmax_raw<DT>(raw, lmn, lmx);
      } else {
        for (int j = 0; j < kChunk; ++j) {
          if (e + j < e1) {
            const float x = load1<DT>(T.x, e + j);
            lmn = fminf(lmn, x);
            lmx = fmaxf(lmx, x);
          }
        }
      }
    }
    const GroupParams gp = group_params(warp_min(lmn), warp_max(lmx), Lf);
    if (lane == 0) {
      T.group_min[g] = gp.mn;
      T.group_scale[g] = gp.scale;
    }
    if constexpr (!STATS) {
      // every chunk of the group's span up to the tensor's last word: chunks past n code as
      // zeros, which writes the zero padding of the last word (G b / 32 words per group)
      for (int64_t e = e0 + lane * kChunk; e < e0 + G; e += 32 * kChunk) {
        if (e + kChunk <= e1) {  // a partial chunk only ends the tensor
          Raw8<DT> raw;
          load8<DT>(raw, T.x, e);
          store_unit<BITS>(T.packed, e, quantize_chunk_raw<DT, BITS>(raw, gp.mn, gp.inv, chunk_rand(T, e)));
        } else if ((e * BITS) / 32 < T.nwords) {
          code_chunk_guarded<DT, BITS>(T, e, gp.mn, gp.inv);
        }
      }
    }
  }
}

// The tensor's last group (short, or followed by the zero padding of the last word): the
// two-pass generic path, out of line.
template <int DT, int BITS, bool STATS>
__device__ __noinline__ void group_generic(const QTensor T, int64_t g, int64_t G, float Lf, int lane) {
  const int64_t e0 = g * G;
  const int64_t e1 = e0 + G < T.n ? e0 + G : T.n;
  float lmn = FLT_MAX, lmx = -FLT_MAX;
  for (int64_t e = e0 + lane * kChunk; e < e1; e += 32 * kChunk) {
    if (e + kChunk <= e1) {
      Raw8<DT> raw;
      load8<DT>(raw, T.x, e);
      chunk_minmax_raw<DT>(raw, lmn, lmx);
    } else {
      for (int j = 0; j < kChunk; ++j) {
        if (e + j < e1) {
          const float x = load1<DT>(T.x, e + j);
          lmn = fminf(lmn, x);
          lmx = fmaxf(lmx, x);
        }
      }
    }
  }
  const GroupParams gp = group_params(warp_min(lmn), warp_max(lmx), Lf);
  if (lane == 0) {
    T.group_min[g] = gp.mn;
    T.group_scale[g] = gp.scale;
  }
  if constexpr (!STATS) {
    for (int64_t e = e0 + lane * kChunk; e < e0 + G; e += 32 * kChunk) {
      if (e + kChunk <= e1) {
        Raw8<DT> raw;
        load8<DT>(raw, T.x, e);
        store_unit<BITS>(T.packed, e, quantize_chunk_raw<DT, BITS>(raw, gp.mn, gp.inv, chunk_rand(T, e)));
      } else if ((e * BITS) / 32 < T.nwords) {
        code_chunk_guarded<DT, BITS>(T, e, gp.mn, gp.inv);
      }
    }
  }
}

// G a multiple of 32 that is not a power of two, one group per warp held in registers: lane l
// owns the group's chunks l, l + 32, ... (at most NC of them, G <= 256 NC), loaded once; min /
// max by CREDUX; codes from the same registers. Random bytes (R3): a lane's chunks sit 256
// elements apart, so they pair up inside 512-element spans as the big kernel's do, except that
// the first chunk may be the second half of its span (sh = 1): chunk i takes half (i + sh) & 1
// of block slot (i + sh) >> 1, the slots being blk(e_first - 256 sh) + 32 j, computed with
// their rounds 0-1 shared (philox4x32_10_xn). One pass over x (the two-pass kernel above is
// kept for fp32 at G > 2048). A tensor's last group takes group_generic.
// MG = 2: a warp takes two consecutive groups as one span of 2 G elements (chunk j of the span
// belongs to group j >= cpg; lanes stay busy across the groups' boundary); two CREDUX pairs,
// the two divisions on lanes 0 / 1, (mn, inv) broadcast by shuffles.
template <int DT, int BITS, int MAXB, bool STATS, int NC, int MG>
__global__ void __launch_bounds__(kThreads, (NC >= 12 || (DT == DT_F32 && NC >= 8)) ? 2 : 3)
    quantize_anyg_reg_kernel(const __grid_constant__ QBatch<MAXB> P) {
  static_assert(MG == 1 || MG == 2, "one or two groups per warp iteration");
  constexpr int NB = NC / 2 + 1;  // block slots per lane
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float Lf = STATS ? P.Lf : (float)((1 << BITS) - 1);
  const int64_t G = P.group;
  const int cpg = P.group / kChunk;  // chunks per group
  constexpr int CU = kWarps * MG;
  const int64_t cunits = P.tiles_total / CU;
  int cur = first_cursor(P, (int64_t)blockIdx.x * CU);
  for (int64_t cu = blockIdx.x; cu < cunits; cu += gridDim.x) {
    cur = advance_cursor(P, cur, cu * CU);
    const QTensor& T = P.t[cur];
    const int64_t g = cu * CU - P.tile_start[cur] + (int64_t)warp * MG;
    const int64_t e0 = g * G;
    if (e0 >= T.n) continue;  // alignment padding of the tile space
    if (e0 + MG * G >= T.n) {  // the tensor's last group(s)
      for (int q = 0; q < MG; ++q)
        if ((g + q) * G < T.n) group_generic<DT, BITS, STATS>(T, g + q, G, Lf, lane);
      continue;
    }
    const int span = MG * cpg;  // chunks of the warp's groups
    const int64_t e_lane = e0 + lane * kChunk;
    Raw8<DT> raw[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i)
      if (lane + 32 * i < span) load8<DT>(raw[i], T.x, e_lane + i * kWarpTile);
    uint4 r4[NB];
    const int sh = (int)((e_lane >> 8) & 1);  // the lane's first chunk is the second half of its block
    if constexpr (!STATS)
      philox4x32_10_xn<NB>(rand_block(T, e_lane - 256 * sh), (uint32_t)T.seed, (uint32_t)(T.seed >> 32), r4);
    float mn0 = FLT_MAX, mx0 = -FLT_MAX, mn1 = FLT_MAX, mx1 = -FLT_MAX;  // neutral
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int j = lane + 32 * i;
      if (j < span) {
        if (MG == 1 || j < cpg) chunk_minmax_raw<DT>(raw[i], mn0, mx0);
        else chunk_minmax_raw<DT>(raw[i], mn1, mx1);
      }
    }
    GroupParams gp0, gp1;
    if constexpr (MG == 1) {
      gp0 = group_params(warp_min(mn0), warp_max(mx0), Lf);
      if (lane == 0) {
        T.group_min[g] = gp0.mn;
        T.group_scale[g] = gp0.scale;
      }
    } else {
      const float a0 = warp_min(mn0), b0 = warp_max(mx0), a1 = warp_min(mn1), b1 = warp_max(mx1);
      const GroupParams gq = group_params(lane & 1 ? a1 : a0, lane & 1 ? b1 : b0, Lf);  // lane q: group q
      if (lane < 2) {
        T.group_min[g + lane] = gq.mn;
        T.group_scale[g + lane] = gq.scale;
      }
      gp0.mn = __shfl_sync(kFull, gq.mn, 0);
      gp0.inv = __shfl_sync(kFull, gq.inv, 0);
      gp1.mn = __shfl_sync(kFull, gq.mn, 1);
      gp1.inv = __shfl_sync(kFull, gq.inv, 1);
    }
    if constexpr (!STATS) {
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int j = lane + 32 * i;
        if (j < span) {
          const uint4 q = sh ? r4[(i + 1) >> 1] : r4[i >> 1];  // half (i + sh) & 1 of slot (i + sh) >> 1
          const uint2 rnd = ((i + sh) & 1) ? make_uint2(q.z, q.w) : make_uint2(q.x, q.y);
          const bool second = MG == 2 && j >= cpg;
          store_unit<BITS>(T.packed, e_lane + i * kWarpTile,
                           quantize_chunk_raw<DT, BITS>(raw[i], second ? gp1.mn : gp0.mn, second ? gp1.inv : gp0.inv, rnd));
        }
      }
    }
  }
}

// G < 256 not a power of two (96, 160, 192, 224; for 2-byte inputs also 288 ... 480): a warp
// per super-tile of lcm(G, 256) = 256 P elements (P = 3 ... 15 passes), which holds Q = 256 P / G
// whole groups of cpg = G / 8 chunks. Lane l loads its chunk of every pass (all 32 lanes busy, x read once); a group spans
// whole aligned 4-lane blocks (cpg is a multiple of 4 and groups start at multiples of cpg), so
// two butterfly steps give each block's (min, max); the 8 P block values go through shared
// memory, lane q < Q folds its group's cpg / 4 blocks and computes the division, and each lane
// reads its chunk's (mn, inv) back. Random bytes as in quantize_anyg_reg_kernel (the lane's
// chunks 256 elements apart, first chunk possibly the second half of its block). A tensor's
// last super-tile takes group_generic group by group.
template <int DT, int BITS, int MAXB, bool STATS, int P, int K>
__global__ void __launch_bounds__(kThreads, P * K >= GACT_ANYG_SMALL_PK2 ? 2 : 3)
    quantize_anyg_small_kernel(const __grid_constant__ QBatch<MAXB> Pb) {
  constexpr int PK = P * K;             // passes per warp iteration (K super-tiles)
  constexpr int NB = (PK + 1) / 2 + 1;  // block slots per lane
  __shared__ float2 blk[kWarps][8 * PK];  // (min, max) of the 4-lane blocks
  __shared__ float2 gpar[kWarps][32];     // (mn, inv) of the groups
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float Lf = STATS ? Pb.Lf : (float)((1 << BITS) - 1);
  const int64_t G = Pb.group;
  const int cpg = Pb.group / kChunk;           // chunks per group (12, 20, 24, 28)
  const int bpg = cpg / 4;                     // 4-lane blocks per group
  const int Q = K * (32 * P / cpg);            // groups per warp iteration (<= 32)
  const uint32_t rcp = (65536u + cpg - 1) / cpg;  // chunk c -> group (c rcp) >> 16, exact for c < 32 PK
  constexpr int64_t S = 256 * P;               // one super-tile (the host's quantize tile)
  constexpr int CU = kWarps * K;
  const int64_t cunits = Pb.tiles_total / CU;
  int cur = first_cursor(Pb, (int64_t)blockIdx.x * CU);
  for (int64_t cu = blockIdx.x; cu < cunits; cu += gridDim.x) {
    cur = advance_cursor(Pb, cur, cu * CU);
    const QTensor& T = Pb.t[cur];
    const int64_t e_tile = (cu * CU - Pb.tile_start[cur] + (int64_t)warp * K) * S;
    if (e_tile >= T.n) continue;  // alignment padding of the tile space
    const int64_t g0 = e_tile / G;
    if (e_tile + K * S > T.n) {  // the tensor's last super-tiles: group by group
      for (int q = 0; q < Q; ++q)
        if ((g0 + q) * G < T.n) group_generic<DT, BITS, STATS>(T, g0 + q, G, Lf, lane);
      continue;
    }
    const int64_t e_lane = e_tile + lane * kChunk;
    Raw8<DT> raw[PK];
#pragma unroll
    for (int p = 0; p < PK; ++p) load8<DT>(raw[p], T.x, e_lane + p * kWarpTile);
    uint4 r4[NB];
    const int sh = (int)((e_lane >> 8) & 1);
    if constexpr (!STATS)
      philox4x32_10_xn<NB>(rand_block(T, e_lane - 256 * sh), (uint32_t)T.seed, (uint32_t)(T.seed >> 32), r4);
#pragma unroll
    for (int p = 0; p < PK; ++p) {
      float lmn = FLT_MAX, lmx = -FLT_MAX;
      if constexpr (DT != DT_F32) {  // packed (min, -max): one shuffle + one HMNMX2 per step
        uint32_t pm = chunk_minnegmax_packed<DT>(raw[p]);
        pm = min2_packed<DT>(pm, __shfl_xor_sync(kFull, pm, 1));
        pm = min2_packed<DT>(pm, __shfl_xor_sync(kFull, pm, 2));
        unpack_minmax<DT>(pm, lmn, lmx);
      } else {
        chunk_minmax_raw<DT>(raw[p], lmn, lmx);
        lmn = fminf(lmn, __shfl_xor_sync(kFull, lmn, 1));
        lmx = fmaxf(lmx, __shfl_xor_sync(kFull, lmx, 1));
        lmn = fminf(lmn, __shfl_xor_sync(kFull, lmn, 2));
        lmx = fmaxf(lmx, __shfl_xor_sync(kFull, lmx, 2));
      }
      if ((lane & 3) == 0) blk[warp][8 * p + (lane >> 2)] = make_float2(lmn, lmx);
    }
    __syncwarp();
    if (lane < Q) {
      float a = FLT_MAX, b = -FLT_MAX;
      for (int k = 0; k < bpg; ++k) {
        const float2 v = blk[warp][lane * bpg + k];
        a = fminf(a, v.x);
        b = fmaxf(b, v.y);
      }
      const GroupParams gp = group_params(a, b, Lf);
      T.group_min[g0 + lane] = gp.mn;
      T.group_scale[g0 + lane] = gp.scale;
      gpar[warp][lane] = make_float2(gp.mn, gp.inv);
    }
    __syncwarp();
    if constexpr (!STATS) {
#pragma unroll
      for (int p = 0; p < PK; ++p) {
        const float2 pq = gpar[warp][((uint32_t)(32 * p + lane) * rcp) >> 16];
        const uint4 q = sh ? r4[(p + 1) >> 1] : r4[p >> 1];  // half (p + sh) & 1 of slot (p + sh) >> 1
        const uint2 rnd = ((p + sh) & 1) ? make_uint2(q.z, q.w) : make_uint2(q.x, q.y);
        if (DT != DT_F32 && p % 4 != 3)  // byte-2 codes, one pass in four on shift-add (pipe balance)
          store_unit<BITS>(T.packed, e_lane + p * kWarpTile, quantize_chunk_raw<DT, BITS, true>(raw[p], pq.x, pq.y, rnd));
        else
          store_unit<BITS>(T.packed, e_lane + p * kWarpTile, quantize_chunk_raw<DT, BITS, false>(raw[p], pq.x, pq.y, rnd));
      }
    }
    __syncwarp();  // every lane has read blk / gpar before the next super-tile writes them
  }
}

// ------------------------------------------------------------------------- launching
template <typename K>
int max_blocks_per_sm(K kernel) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess || b < 1) b = 1;
  return b;
}

inline int sm_count() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

template <auto Kernel, typename PB>
cudaError_t launch_persistent(const PB& p, int64_t tiles_per_warp_iter, cudaStream_t s, int waves = 1) {
  // (One CTA per unit for launches of <= 2 / 4 x this grid -- finer balancing of the last
  // wave of a 2^27-element tensor -- measured neutral / 3% slower: DESIGN.md §4a.)
  static const int per_sm = max_blocks_per_sm(Kernel);  // one cache per kernel
  const int64_t want = (p.tiles_total + (int64_t)kWarps * tiles_per_warp_iter - 1) /
                       ((int64_t)kWarps * tiles_per_warp_iter);
  const int64_t cap = (int64_t)sm_count() * per_sm * waves;
  const int grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  Kernel<<<grid, kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

// One CTA per unit of `tiles_per_unit` tiles, up to `waves` x resident CTAs.
template <auto Kernel, typename PB>
cudaError_t launch_units(const PB& p, int64_t tiles_per_unit, cudaStream_t s, int waves = 1) {
  static const int per_sm = max_blocks_per_sm(Kernel);
  const int64_t want = (p.tiles_total + tiles_per_unit - 1) / tiles_per_unit;
  const int64_t cap = (int64_t)sm_count() * per_sm * waves;
  const int grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  Kernel<<<grid, kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

template <int DT, int BITS, int MAXB, bool STATS>
cudaError_t launch_q(const QBatch<MAXB>& p, cudaStream_t s) {
  if (p.log2g < 0) {  // G not a power of two: a warp per group in registers (fp32: G <= 2048)
    const int P = (int)(quantize_tile_elems(p.group, DT) / kWarpTile);
    if (p.group < 256 || (DT != DT_F32 && p.group < 512)) {  // a warp per super-tile of lcm(G, 256)
      // K super-tiles per warp iteration (2-byte G = 96 / 192: 4, i.e. 12 passes; fp32: 1)
      constexpr int K3 = DT == DT_F32 ? 1 : GACT_ANYG_K3, K5 = DT == DT_F32 ? 1 : GACT_ANYG_K5;
      if (P == 3) return launch_units<quantize_anyg_small_kernel<DT, BITS, MAXB, STATS, 3, K3>>(p, kWarps * K3, s, 8);
      if (P == 5) return launch_units<quantize_anyg_small_kernel<DT, BITS, MAXB, STATS, 5, K5>>(p, kWarps * K5, s, 8);
      if (P == 7) return launch_units<quantize_anyg_small_kernel<DT, BITS, MAXB, STATS, 7, 1>>(p, kWarps, s, 8);
      if constexpr (DT != DT_F32) {  // 2-byte, 256 < G < 512: P = 9, 11, 13, 15
        if (P == 9) return launch_units<quantize_anyg_small_kernel<DT, BITS, MAXB, STATS, 9, 1>>(p, kWarps, s, 8);
        if (P == 11) return launch_units<quantize_anyg_small_kernel<DT, BITS, MAXB, STATS, 11, 1>>(p, kWarps, s, 8);
        if (P == 13) return launch_units<quantize_anyg_small_kernel<DT, BITS, MAXB, STATS, 13, 1>>(p, kWarps, s, 8);
        return launch_units<quantize_anyg_small_kernel<DT, BITS, MAXB, STATS, 15, 1>>(p, kWarps, s, 8);
      }
    }
#if GACT_Q_ANYG_REG
    // chunks per lane for one / two groups per warp iteration (two where they fit in 16 / 8)
    const int nc1 = (p.group + kWarpTile - 1) / kWarpTile, nc2 = (2 * p.group + kWarpTile - 1) / kWarpTile;
    constexpr int NCMAX = DT == DT_F32 ? 8 : 16;
    if (GACT_ANYG_MG2 && nc2 <= 4) return launch_units<quantize_anyg_reg_kernel<DT, BITS, MAXB, STATS, 4, 2>>(p, kWarps * 2, s, 8);
    if (GACT_ANYG_MG2 && nc2 <= 8) return launch_units<quantize_anyg_reg_kernel<DT, BITS, MAXB, STATS, 8, 2>>(p, kWarps * 2, s, 8);
    if constexpr (DT != DT_F32)
      if (GACT_ANYG_MG2 && nc2 <= 12) return launch_units<quantize_anyg_reg_kernel<DT, BITS, MAXB, STATS, 12, 2>>(p, kWarps * 2, s, 8);
    if (GACT_ANYG_MG2 && nc2 <= NCMAX) return launch_units<quantize_anyg_reg_kernel<DT, BITS, MAXB, STATS, NCMAX, 2>>(p, kWarps * 2, s, 8);
    if (nc1 <= 4) return launch_units<quantize_anyg_reg_kernel<DT, BITS, MAXB, STATS, 4, 1>>(p, kWarps, s, 8);
    if (nc1 <= 8) return launch_units<quantize_anyg_reg_kernel<DT, BITS, MAXB, STATS, 8, 1>>(p, kWarps, s, 8);
    if constexpr (DT != DT_F32)
      if (nc1 <= 12) return launch_units<quantize_anyg_reg_kernel<DT, BITS, MAXB, STATS, 12, 1>>(p, kWarps, s, 8);
    if constexpr (DT != DT_F32) return launch_units<quantize_anyg_reg_kernel<DT, BITS, MAXB, STATS, 16, 1>>(p, kWarps, s, 8);
#endif
    return launch_units<quantize_anyg_kernel<DT, BITS, MAXB, STATS>>(p, kWarps, s, 8);
  }
  const int waves = DT == DT_F32 ? GACT_Q_WAVES_F32 : GACT_Q_WAVES;
  switch (p.log2g) {
    case 5:
#if GACT_QS_XRED
      if constexpr (DT != DT_F32) return launch_persistent<quantize_smallx_kernel<DT, BITS, MAXB, STATS, 5>>(p, 8, s, waves);
#endif
      return launch_persistent<quantize_small_kernel<DT, BITS, MAXB, STATS, 5>>(p, small_unit<DT, 5>(), s, waves);
    case 6:
#if GACT_QS_XRED
      if constexpr (DT != DT_F32) return launch_persistent<quantize_smallx_kernel<DT, BITS, MAXB, STATS, 6>>(p, 8, s, waves);
#endif
      return launch_persistent<quantize_small_kernel<DT, BITS, MAXB, STATS, 6>>(p, small_unit<DT, 6>(), s, waves);
    case 7:
#if GACT_QS_XRED
      if constexpr (DT != DT_F32) return launch_persistent<quantize_smallx_kernel<DT, BITS, MAXB, STATS, 7>>(p, 16, s, waves);
#endif
      return launch_persistent<quantize_small_kernel<DT, BITS, MAXB, STATS, 7>>(p, small_unit<DT, 7>(), s, waves);
    case 8:
      return launch_persistent<quantize_big_kernel<DT, BITS, 1, MAXB, STATS>>(p, unit_tiles<DT, BITS, MAXB, 1>(), s, waves);
    case 9:
      return launch_persistent<quantize_big_kernel<DT, BITS, 2, MAXB, STATS>>(p, unit_tiles<DT, BITS, MAXB, 2>(), s, waves);
    case 10:
      return launch_persistent<quantize_big_kernel<DT, BITS, 4, MAXB, STATS>>(p, unit_tiles<DT, BITS, MAXB, 4>(), s, waves);
    case 11:
      if constexpr (DT != DT_F32) {
        // 2-byte inputs: one group per warp, 8 chunks per lane, all in registers (the 8-chunk
        // unit of G = 256 with U = 1 tile), read once.
        return launch_persistent<quantize_big_kernel<DT, BITS, 8, MAXB, STATS>>(p, unit_tiles<DT, BITS, MAXB, 8>(), s, waves);
      } else {
        // fp32 (HBM-bound): the group spread over the CTA in registers
        return launch_units<quantize_cta_kernel<DT, BITS, 1, MAXB, STATS>>(p, 4, s, waves);
      }
    default:  // G = 4096
      if constexpr (DT != DT_F32) {
        // 2-byte inputs: one group per warp, 16 chunks per lane in registers, read once
        return launch_persistent<quantize_big_kernel<DT, BITS, 16, MAXB, STATS>>(p, unit_tiles<DT, BITS, MAXB, 16>(), s, waves);
      } else {
        return launch_units<quantize_cta_kernel<DT, BITS, 2, MAXB, STATS>>(p, 2, s, waves);
      }
  }
}

template <int DT, int MAXB>
cudaError_t launch_q_bits(const QBatch<MAXB>& p, int bits, cudaStream_t s) {
  switch (bits) {
    case 1: return launch_q<DT, 1, MAXB, false>(p, s);
    case 2: return launch_q<DT, 2, MAXB, false>(p, s);
    case 4: return launch_q<DT, 4, MAXB, false>(p, s);
    default: return launch_q<DT, 8, MAXB, false>(p, s);
  }
}

}  // namespace

template <int MAXB>
cudaError_t launch_quantize(const QBatch<MAXB>& p, int dtype, int bits, cudaStream_t s) {
  if (p.tiles_total == 0) return cudaSuccess;
  switch (dtype) {
    case DT_F32: return launch_q_bits<DT_F32, MAXB>(p, bits, s);
    case DT_BF16: return launch_q_bits<DT_BF16, MAXB>(p, bits, s);
    default: return launch_q_bits<DT_F16, MAXB>(p, bits, s);
  }
}

template <int MAXB>
cudaError_t launch_group_stats(const QBatch<MAXB>& p, int dtype, cudaStream_t s) {
  if (p.tiles_total == 0) return cudaSuccess;
  switch (dtype) {
    case DT_F32: return launch_q<DT_F32, 1, MAXB, true>(p, s);
    case DT_BF16: return launch_q<DT_BF16, 1, MAXB, true>(p, s);
    default: return launch_q<DT_F16, 1, MAXB, true>(p, s);
  }
}

template cudaError_t launch_quantize<1>(const QBatch<1>&, int, int, cudaStream_t);
template cudaError_t launch_quantize<kMaxBatch>(const QBatch<kMaxBatch>&, int, int, cudaStream_t);
template cudaError_t launch_group_stats<1>(const QBatch<1>&, int, cudaStream_t);

}  // namespace gact
