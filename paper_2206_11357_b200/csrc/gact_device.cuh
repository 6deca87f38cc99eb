// gact_device.cuh — device building blocks of the GACT compressor kernels (sm_100a).
//
// Product code. Implements the quantizer defined in include/gact.h (App. Prop. 3 of the
// paper) with IEEE binary32 operations issued explicitly (no contraction):
// the oracle/ directory is an independent CPU implementation used only by the tests.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gact {

constexpr int kChunk = 8;       // elements per lane chunk (8 random bytes: half a Philox block)
constexpr int kWarpTile = 256;  // 32 lanes x 8 elements: one coalesced warp pass
constexpr int kWarps = 8;       // warps per CTA
constexpr int kThreads = kWarps * 32;

enum : int { DT_F32 = 0, DT_BF16 = 1, DT_F16 = 2 };

// ------------------------------------------------------------------------ Philox4x32-10
// Salmon et al., SC'11 (Random123 constants). key = seed, counter = (block lo, hi, 0, 0).
// Written with explicit PTX (mul.wide.u32 -> one IMAD.WIDE.U32, lop3 -> one LOP3 for the
// 3-way xor) so that a round costs 2 + 2 instructions; the key schedule is the same for
// every call with the same seed and is shared (CSE) across the calls of an iteration.
__device__ __forceinline__ void mul_wide(uint32_t a, uint32_t m, uint32_t& lo, uint32_t& hi) {
  asm("{\n\t.reg .b64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}"
      : "=r"(lo), "=r"(hi)
      : "r"(a), "r"(m));
}
__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

#ifndef GACT_EXP_ROUNDS
#define GACT_EXP_ROUNDS 10  // experiments only (DESIGN.md §4a table): Philox4x32-10 is the generator
#endif
// (Round 1 also measured the upper product halves on the FP64 pipe -- fma.rm.f64 on
// {a, 0x43300000}, bit-exact: fewer FMA-heavy cycles but more instructions, slower.)
__device__ __forceinline__ uint4 philox4x32_10(uint64_t block, uint32_t k0, uint32_t k1) {
  uint32_t c0 = (uint32_t)block, c1 = (uint32_t)(block >> 32), c2 = 0u, c3 = 0u;
#pragma unroll
  for (int r = 0; r < GACT_EXP_ROUNDS; ++r) {
    uint32_t lo0, hi0, lo1, hi1;
    mul_wide(c0, 0xD2511F53u, lo0, hi0);
    mul_wide(c2, 0xCD9E8D57u, lo1, hi1);
    const uint32_t n0 = xor3(hi1, c1, k0);
    const uint32_t n2 = xor3(hi0, c3, k1);
    c1 = lo1;
    c3 = lo0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

// Philox4x32-10 of the N blocks blk + 32 m, m = 0..N-1 (a lane's blocks in one quantize
// unit), bit-identical to N philox4x32_10 calls, with the work they share done once. When
// lo32(blk) + 32 (N - 1) does not wrap, every counter is (c0 + 32 m, c1, 0, 0), so
//   round 0: M0 (c0 + 32 m) = P_0 + m (32 M0) as 64-bit sums (one multiply, N - 1 adds); the
//            outputs are (c1 ^ k0, 0, hi P_m ^ k1, lo P_m): word 0 is common to all N;
//   round 1: M0 (c1 ^ k0) is common (one multiply instead of N);
// rounds 2-9 run per block. A wrapping lo32 (tensors past 2^35 elements) takes N calls.
template <int N>
__device__ __forceinline__ void philox4x32_10_xn(uint64_t blk, uint32_t k0, uint32_t k1, uint4 r[N]) {
  const uint32_t c0 = (uint32_t)blk, c1 = (uint32_t)(blk >> 32);
  if (c0 > 0xFFFFFFFFu - 32u * (N - 1)) {
#pragma unroll
    for (int m = 0; m < N; ++m) r[m] = philox4x32_10(blk + 32u * m, k0, k1);
    return;
  }
  constexpr uint64_t kD = 32ull * 0xD2511F53ull;
  const uint32_t x0 = c1 ^ k0;  // round-0 word 0, common
  uint32_t L, H;                // round 1: M0 * x0, common
  mul_wide(x0, 0xD2511F53u, L, H);
  const uint32_t k0r1 = k0 + 0x9E3779B9u, k1r1 = k1 + 0xBB67AE85u;
  uint64_t P = (uint64_t)c0 * 0xD2511F53u;
#pragma unroll
  for (int m = 0; m < N; ++m, P += kD) {
    const uint32_t p_lo = (uint32_t)P, p_hi = (uint32_t)(P >> 32);
    // after round 0: (x0, 0, p_hi ^ k1, p_lo); round 1:
    uint32_t lo1, hi1;
    mul_wide(p_hi ^ k1, 0xCD9E8D57u, lo1, hi1);
    uint32_t a0 = hi1 ^ k0r1, a1 = lo1, a2 = xor3(H, p_lo, k1r1), a3 = L;
    uint32_t q0 = k0r1, q1 = k1r1;
#pragma unroll
    for (int rd = 2; rd < GACT_EXP_ROUNDS; ++rd) {
      q0 += 0x9E3779B9u;
      q1 += 0xBB67AE85u;
      uint32_t l0, h0, l1, h1;
      mul_wide(a0, 0xD2511F53u, l0, h0);
      mul_wide(a2, 0xCD9E8D57u, l1, h1);
      const uint32_t n0 = xor3(h1, a1, q0);
      const uint32_t n2 = xor3(h0, a3, q1);
      a1 = l1;
      a3 = l0;
      a0 = n0;
      a2 = n2;
    }
    r[m] = make_uint4(a0, a1, a2, a3);
  }
}
// ------------------------------------------------------------------- packed f32x2 math
// sm_100a executes these as FADD2 / FMUL2 / FFMA2 (two lanes of fp32 per instruction),
// each lane correctly rounded in the stated mode — identical to two scalar IEEE ops.
typedef unsigned long long f2_t;

__device__ __forceinline__ f2_t f2_make(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_split(f2_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_bits(uint32_t lo, uint32_t hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ void f2_split_bits(f2_t v, uint32_t& lo, uint32_t& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_sub_rn(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_add_rm(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_fma_rm(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t f2_fma_rn(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ float min3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// Warp-wide fp32 min / max in one instruction (CREDUX on sm_100a).
__device__ __forceinline__ float warp_min(float v) {
  float r;
  asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float warp_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// ------------------------------------------------------------------- global memory I/O
// Inputs are streamed once: read-only path, no L1 allocation.
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// 8 raw elements of one lane chunk: 32 bytes (f32) or 16 bytes (bf16 / f16).
template <int DT>
struct Raw8 {
  uint4 a, b;
};
template <>
struct Raw8<DT_BF16> {
  uint4 a;
};
template <>
struct Raw8<DT_F16> {
  uint4 a;
};


template <int DT>
__device__ __forceinline__ void load8(Raw8<DT>& r, const void* base, int64_t e) {
  if constexpr (DT == DT_F32) {
    const float* p = static_cast<const float*>(base) + e;
    r.a = ldg_stream(p);
    r.b = ldg_stream(p + 4);
  } else {
    const uint16_t* p = static_cast<const uint16_t*>(base) + e;
    r.a = ldg_stream(p);
  }
}

__device__ __forceinline__ float f16_bits_to_f32(uint32_t h) {
  float f;
  asm("{ .reg .f16 t; mov.b16 t, %1; cvt.f32.f16 %0, t; }" : "=f"(f) : "h"((unsigned short)h));
  return f;
}

// Widen to binary32 (exact for every dtype). Element j of the chunk -> v[j].
template <int DT>
__device__ __forceinline__ void widen8(const Raw8<DT>& r, float v[8]) {
  if constexpr (DT == DT_F32) {
    v[0] = __uint_as_float(r.a.x); v[1] = __uint_as_float(r.a.y);
    v[2] = __uint_as_float(r.a.z); v[3] = __uint_as_float(r.a.w);
    v[4] = __uint_as_float(r.b.x); v[5] = __uint_as_float(r.b.y);
    v[6] = __uint_as_float(r.b.z); v[7] = __uint_as_float(r.b.w);
  } else if constexpr (DT == DT_BF16) {
    const uint32_t w[4] = {r.a.x, r.a.y, r.a.z, r.a.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);             // element 2i: low half
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u); // element 2i+1: high half
    }
  } else {
    const uint32_t w[4] = {r.a.x, r.a.y, r.a.z, r.a.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = f16_bits_to_f32(w[i] & 0xFFFFu);
      v[2 * i + 1] = f16_bits_to_f32(w[i] >> 16);
    }
  }
}

// One element with bounds handling (partial tiles only).
template <int DT>
__device__ __forceinline__ float load1(const void* base, int64_t e) {
  if constexpr (DT == DT_F32) {
    return static_cast<const float*>(base)[e];
  } else if constexpr (DT == DT_BF16) {
    return __uint_as_float((uint32_t)static_cast<const uint16_t*>(base)[e] << 16);
  } else {
    return f16_bits_to_f32(static_cast<const uint16_t*>(base)[e]);
  }
}

// ------------------------------------------------------------------ group parameters
// mn, scale = range / L (RN), inv = L / range (RZ; 0 for a constant group).
struct GroupParams {
  float mn, scale, inv;
};

// RZ(a / b) for finite a > 0, b > 0: q = RN(a / b), then one step toward zero if q
// overshoots (the residual a - q b of a correctly rounded quotient is exact, so its sign
// decides); RN overflow (a / b > FLT_MAX) gives FLT_MAX, the RZ result. Avoids the
// out-of-line __fdiv_rz path.
__device__ __forceinline__ float div_rz_pos(float a, float b) {
  const float q = __fdiv_rn(a, b);
  if (q == __int_as_float(0x7f800000)) return __int_as_float(0x7f7fffff);
  const float r = __fmaf_rn(-q, b, a);
  return (r < 0.0f) ? __int_as_float(__float_as_int(q) - 1) : q;
}

__device__ __forceinline__ GroupParams group_params(float mn, float mx, float Lf) {
  GroupParams p;
  mn = __fadd_rn(mn, 0.0f);  // -0 -> +0
  mx = __fadd_rn(mx, 0.0f);
  const float range = __fsub_rn(mx, mn);
  p.mn = mn;
  // range / 1 == range exactly (b = 1: the constant folds and the division disappears)
  p.scale = (Lf == 1.0f) ? range : __fdiv_rn(range, Lf);
  p.inv = (range > 0.0f) ? div_rz_pos(Lf, range) : 0.0f;
  return p;
}

// ----------------------------------------------------------- stochastic rounding + pack
// Codes of 8 consecutive elements (chunk), packed LSB-first into BITS*8 bits:
//   q_j = floor(d_j * inv + (2 k_j + 1) 2^-9),  d_j = RN(v_j - mn)     (include/gact.h)
// with the product and the sum exact; k_j is the element's random byte (R3: a chunk of 8
// elements takes 8 consecutive bytes of its Philox block, words r.x (elements 0-3) and r.y
// (4-7), least significant byte first). Per pair of elements (j = 2p, 2p+1), for every b:
//   c = 128 + (2k+1) 2^-9                 one PRMT: 0x4300_0000 | k << 8 | 0x80 (exact)
//   v = fma.rm(d, inv, c)                 FFMA2.RM: RD(d*inv + c), one rounding, downward
//   w = add.rm(v, 2^23 - 128)             FADD2.RM: bits(w) = 0x4B00_0000 + floor(v) - 128
// Every integer below 2^24 is a binary32 value, so rounding down never crosses one:
// floor(RD(s)) = floor(s) whatever the binade of s (v < 128 + 2^b + 1 <= 385 spans
// [128, 512) for b = 8), hence floor(v) = 128 + floor(T + u) = 128 + q; and [2^23, 2^24) is
// the integer grid, so bits(w) - 0x4B00_0000 = q_j exactly. The low byte of bits(w) is q_j.
// (With round 1's 16-bit lanes 128 + (2k+1) 2^-17 was not a binary32 value; the 8-bit
// lattice point is, which saves the extra add b = 8 needed then.)

template <int BITS>
struct PackedUnit {
  uint32_t lo, hi;  // hi used only for BITS == 8 (64-bit unit)
};

#ifndef GACT_BYTE2_MAXB
#define GACT_BYTE2_MAXB 4  // byte-2 codes up to this b (G = 256 kernel; b = 8 packs by byte permutes anyway)
#endif
static_assert(GACT_BYTE2_MAXB <= 4, "byte 2 of bits(v) holds q only while v < 256, i.e. b <= 4");
#ifndef GACT_MAGIC_OFFSETS
#define GACT_MAGIC_OFFSETS 1
#endif
// Integer offset m_j added to element j's magic (2^23 - 128 + m_j: bits(w_j) = 0x4B00_0000 + m_j
// + q_j, still on the integer grid of [2^23, 2^24) and below 2^24), chosen so that the offsets
// cancel in the packed sum: sum_j (0x4B00_0000 + m_j) << (b j) == 0 (mod 2^32), which saves the
// correction add per chunk. Each m_j is a multiple of 2^16, so m_j << (b j) lies above the code
// bits. b = 4: 0x4B00_0000 + 0xB500_0000; b = 2: 0xE700_0000 + (0x64_0000 << 6); b = 1:
// 0xB500_0000 + (0x2E_0000 << 6) + (0x7F_0000 << 7).
template <int BITS>
__host__ __device__ constexpr uint32_t magic_off(int j) {
  if (!GACT_MAGIC_OFFSETS) return 0;
  return BITS == 4 ? (j == 1 ? 0x500000u : 0u)
       : BITS == 2 ? (j == 3 ? 0x640000u : 0u)
       : BITS == 1 ? (j == 6 ? 0x2E0000u : j == 7 ? 0x7F0000u : 0u) : 0u;
}
template <int BITS>
__host__ __device__ constexpr uint32_t magic_sum(int first, int count) {
  uint32_t s = 0;
  for (int j = first; j < first + count; ++j) s += (0x4B000000u + magic_off<BITS>(j)) << (j * BITS);
  return s;
}
static_assert(!GACT_MAGIC_OFFSETS || (magic_sum<1>(0, 8) == 0 && magic_sum<2>(0, 8) == 0 && magic_sum<4>(0, 8) == 0),
              "the magic offsets cancel in the packed sum");

// w_j (= 0x4B00_0000 + q_j) of the pair (d_lo, d_hi) whose random bytes are bytes SEL and
// SEL + 1 of Philox word rw. (Building c in the integer pipe instead -- funnel shift + lop3
// -- was measured slower in round 1: it overloads the ALU pipe that the Philox xors and byte
// permutes use.)
template <int SEL, int BITS, int J>
__device__ __forceinline__ void code_pair(f2_t d2, f2_t inv2, uint32_t rw, uint32_t& w_lo,
                                          uint32_t& w_hi) {
  static_assert(SEL == 0 || SEL == 2, "a pair's bytes are 0-1 or 2-3 of its word");
  const uint32_t clo = __byte_perm(rw, 0x43000080u, 0x7604 | (SEL << 4));        // 128 + (2k+1) 2^-9
  const uint32_t chi = __byte_perm(rw, 0x43000080u, 0x7604 | ((SEL + 1) << 4));
  // elements J, J + 1 of the chunk: 2^23 - 128 + m_j (exact: integers below 2^24)
  const f2_t magic = f2_make(8388608.0f - 128.0f + (float)magic_off<BITS>(J),
                             8388608.0f - 128.0f + (float)magic_off<BITS>(J + 1));
  f2_split_bits(f2_add_rm(f2_fma_rm(d2, inv2, f2_bits(clo, chi)), magic), w_lo, w_hi);
}

// Pack the low bytes q_j of w_j (= 0x4B00_0000 + q_j) into the chunk's 8*BITS-bit unit:
// b = 8 by byte permutes; b < 8 by one IMAD per code (acc + (w_j << b j), mod 2^32), minus
// the constant sum of the 0x4B00_0000 terms. Integer-pipe alternatives were measured slower
// or equal (2^28 bf16): gathering the even / odd low bytes with 6 PRMT and
// merging them, pairwise IMAD + 3 PRMT, and gathering byte 2 of the FFMA2.RN results (no
// FADD2.RM) with byte permutes + LEA.HI: the integer pipe is as busy as the FMA-heavy pipe.
// Round 2, with the 8-bit lattice (byte 2 of bits(fma.rm(d, inv, c)) is q for b <= 4): 6 PRMT
// + 1 LEA (b = 4) or 6 PRMT + 2 IMAD + 1 PRMT / SHF (b = 2 / 1, a multiply moving four byte
// values to bits 24-31) per chunk, 40 fewer instructions per 8-tile unit, measured neutral
// to 3% slower at G = 64-4096 (b = 4 +1% at G = 1024 only): the ALU pipe becomes the limit.
template <int BITS>
__device__ __forceinline__ PackedUnit<BITS> pack_codes(const uint32_t w[8]) {
  PackedUnit<BITS> out;
  if constexpr (BITS == 8) {
    out.lo = __byte_perm(__byte_perm(w[0], w[1], 0x0040), __byte_perm(w[2], w[3], 0x0040), 0x5410);
    out.hi = __byte_perm(__byte_perm(w[4], w[5], 0x0040), __byte_perm(w[6], w[7], 0x0040), 0x5410);
  } else {
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += w[j] << (BITS * j);  // mod 2^32
    out.lo = acc - magic_sum<BITS>(0, 8);
    out.hi = 0;
  }
  return out;
}

// Codes of the chunk's 8 elements from the 4 pairs d2[p] = (d_2p, d_2p+1) and the chunk's
// 8 random bytes r (r.x: elements 0-3, r.y: 4-7), packed.
// (Coding each pair's odd element at scale 2^b and packing by two exact fp32 adds per pair
// plus 3 byte permutes -- moving the packing off the FMA-heavy pipe -- was measured slower
// in round 1: bf16 2^28, b = 1 / 2 / 4: 195 / 200 / 183 us vs 175 / 179 / 171.)
// BYTE2 (b <= 4): codes from byte 2 of the FFMA2.RM result, gathered by byte permutes and
// packed by one or two multiplies -- taken by the G = 256 2-byte kernel (A/B: b = 4 +2.7%, b = 2
// +0.7%, b = 1 +1%, ResNet-50 quantize +1-2%); at G = 64 / 1024 / 4096 it measured 1-2.5%
// slower (b <= 2), so the others keep the integerising add and the shift-add packing.
template <int BITS, bool BYTE2 = false>
__device__ __forceinline__ PackedUnit<BITS> code_and_pack(const f2_t d2[4], float inv, uint2 r) {
  const f2_t inv2 = f2_make(inv, inv);
  if constexpr (BYTE2 && BITS <= GACT_BYTE2_MAXB) {
    // v_j = fma.rm(d_j, inv, 128 + u_j) lies in [128, 128 + 2^b): bits(v_j) = 0x4300_0000 +
    // floor((v_j - 128) 2^16), so byte 2 of bits(v_j) is q_j (no integerising add). Gather the
    // eight byte-2 values into two words by 6 byte permutes. b = 4: A = [q0, q2, q4, q6],
    // B = [q1, q3, q5, q7], A + 16 B is the packed word. b <= 2: A = [q0, q1, q2, q3],
    // B = [q4, .., q7], and one multiply per word moves its four b-bit codes into byte 3, the
    // cross products landing below bit 24 in disjoint fields (b = 1: A * 0x01020408 puts q_i at
    // bit 24 + i, B * 0x10204080 at bit 28 + i, their sum is the code byte; b = 2:
    // A * 0x01041040 puts q_i at bits 24 + 2i, likewise B, and one permute joins the bytes).
    uint32_t v[8];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint32_t rw = p < 2 ? r.x : r.y;
      const int sel = (p & 1) * 2;
      const uint32_t clo = __byte_perm(rw, 0x43000080u, 0x7604 | (sel << 4));
      const uint32_t chi = __byte_perm(rw, 0x43000080u, 0x7604 | ((sel + 1) << 4));
      f2_split_bits(f2_fma_rm(d2[p], inv2, f2_bits(clo, chi)), v[2 * p], v[2 * p + 1]);
    }
    PackedUnit<BITS> out;
    out.hi = 0;
    if constexpr (BITS == 4) {  // even codes in A, odd codes in B: byte i = q_2i | q_2i+1 << 4
      const uint32_t A = __byte_perm(__byte_perm(v[0], v[2], 0x0062), __byte_perm(v[4], v[6], 0x0062), 0x5410);
      const uint32_t B = __byte_perm(__byte_perm(v[1], v[3], 0x0062), __byte_perm(v[5], v[7], 0x0062), 0x5410);
      out.lo = B * 16u + A;
      return out;
    }
    const uint32_t A = __byte_perm(__byte_perm(v[0], v[1], 0x0062), __byte_perm(v[2], v[3], 0x0062), 0x5410);
    const uint32_t B = __byte_perm(__byte_perm(v[4], v[5], 0x0062), __byte_perm(v[6], v[7], 0x0062), 0x5410);
    if constexpr (BITS == 1) {
      out.lo = (A * 0x01020408u + B * 0x10204080u) >> 24;
    } else {
      out.lo = __byte_perm(A * 0x01041040u, B * 0x01041040u, 0x0073);
    }
    return out;
  }
  uint32_t w[8];
  code_pair<0, BITS, 0>(d2[0], inv2, r.x, w[0], w[1]);
  code_pair<2, BITS, 2>(d2[1], inv2, r.x, w[2], w[3]);
  code_pair<0, BITS, 4>(d2[2], inv2, r.y, w[4], w[5]);
  code_pair<2, BITS, 6>(d2[3], inv2, r.y, w[6], w[7]);
  return pack_codes<BITS>(w);
}

// From binary32 values (any dtype widened, or the guarded paths).
template <int BITS>
__device__ __forceinline__ PackedUnit<BITS> quantize_chunk(const float v[8], float mn, float inv,
                                                           uint2 r) {
  const f2_t mn2 = f2_make(mn, mn);
  f2_t d2[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) d2[p] = f2_sub_rn(f2_make(v[2 * p], v[2 * p + 1]), mn2);
  return code_and_pack<BITS>(d2, inv, r);
}

// Straight from the loaded chunk. bf16 / f16: d = x - mn by the mixed-precision subtract
// (sub.rn.f32.bf16 / .f16: exact widening, one binary32 rounding) on each half-word.
template <int DT, int BITS, bool BYTE2 = false>
__device__ __forceinline__ PackedUnit<BITS> quantize_chunk_raw(const Raw8<DT>& raw, float mn,
                                                               float inv, uint2 r) {
  if constexpr (DT == DT_F32) {
    float v[8];
    widen8<DT>(raw, v);
    return quantize_chunk<BITS>(v, mn, inv, r);
  } else {
    const uint32_t xw[4] = {raw.a.x, raw.a.y, raw.a.z, raw.a.w};
    f2_t d2[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      float dlo, dhi;
      if constexpr (DT == DT_BF16) {
        asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\tsub.rn.f32.bf16 %0, l, %3;\n\t"
            "sub.rn.f32.bf16 %1, h, %3;\n\t}"
            : "=f"(dlo), "=f"(dhi) : "r"(xw[p]), "f"(mn));
      } else {
        asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\tsub.rn.f32.f16 %0, l, %3;\n\t"
            "sub.rn.f32.f16 %1, h, %3;\n\t}"
            : "=f"(dlo), "=f"(dhi) : "r"(xw[p]), "f"(mn));
      }
      d2[p] = f2_make(dlo, dhi);
    }
    return code_and_pack<BITS, BYTE2>(d2, inv, r);
  }
}

// Fold a loaded chunk's 8 values into running binary32 (mn, mx). bf16 / f16 reduce the
// four packed words with 2-wide min / max first (HMNMX2), then widen the two survivors.
template <int DT>
__device__ __forceinline__ void chunk_minmax_raw(const Raw8<DT>& raw, float& mn, float& mx) {
  if constexpr (DT == DT_F32) {
    float v[8];
    widen8<DT>(raw, v);
    mn = min3f(min3f(mn, v[0], v[1]), min3f(v[2], v[3], v[4]), min3f(v[5], v[6], v[7]));
    mx = max3f(max3f(mx, v[0], v[1]), max3f(v[2], v[3], v[4]), max3f(v[5], v[6], v[7]));
  } else {
    uint32_t m01, m23, m, M01, M23, M;
    if constexpr (DT == DT_BF16) {
      asm("min.bf16x2 %0, %1, %2;" : "=r"(m01) : "r"(raw.a.x), "r"(raw.a.y));
      asm("min.bf16x2 %0, %1, %2;" : "=r"(m23) : "r"(raw.a.z), "r"(raw.a.w));
      asm("min.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(m01), "r"(m23));
      asm("max.bf16x2 %0, %1, %2;" : "=r"(M01) : "r"(raw.a.x), "r"(raw.a.y));
      asm("max.bf16x2 %0, %1, %2;" : "=r"(M23) : "r"(raw.a.z), "r"(raw.a.w));
      asm("max.bf16x2 %0, %1, %2;" : "=r"(M) : "r"(M01), "r"(M23));
      mn = min3f(mn, __uint_as_float(__byte_perm(m, 0u, 0x1044)), __uint_as_float(m & 0xFFFF0000u));
      mx = max3f(mx, __uint_as_float(__byte_perm(M, 0u, 0x1044)), __uint_as_float(M & 0xFFFF0000u));
    } else {
      asm("min.f16x2 %0, %1, %2;" : "=r"(m01) : "r"(raw.a.x), "r"(raw.a.y));
      asm("min.f16x2 %0, %1, %2;" : "=r"(m23) : "r"(raw.a.z), "r"(raw.a.w));
      asm("min.f16x2 %0, %1, %2;" : "=r"(m) : "r"(m01), "r"(m23));
      asm("max.f16x2 %0, %1, %2;" : "=r"(M01) : "r"(raw.a.x), "r"(raw.a.y));
      asm("max.f16x2 %0, %1, %2;" : "=r"(M23) : "r"(raw.a.z), "r"(raw.a.w));
      asm("max.f16x2 %0, %1, %2;" : "=r"(M) : "r"(M01), "r"(M23));
      mn = min3f(mn, f16_bits_to_f32(m & 0xFFFFu), f16_bits_to_f32(m >> 16));
      mx = max3f(mx, f16_bits_to_f32(M & 0xFFFFu), f16_bits_to_f32(M >> 16));
    }
  }
}

template <int DT>
__device__ __forceinline__ uint32_t min2_packed(uint32_t a, uint32_t b) {
  uint32_t r;
  if constexpr (DT == DT_BF16) asm("min.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  else asm("min.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// 2-byte dtypes: the chunk's (min, -max) as one packed pair (low half: min, high half: the
// negated max), so that a segmented butterfly moves and reduces both with one shuffle and one
// 2-wide min (HMNMX2) per step. Exact: negation flips the sign bit, and min / max of bf16 /
// f16 values equal those of their (exact) binary32 widenings.
template <int DT>
__device__ __forceinline__ uint32_t chunk_minnegmax_packed(const Raw8<DT>& raw) {
  static_assert(DT != DT_F32, "2-byte dtypes only");
  uint32_t m01, m23, m, M01, M23, M;
  if constexpr (DT == DT_BF16) {
    asm("min.bf16x2 %0, %1, %2;" : "=r"(m01) : "r"(raw.a.x), "r"(raw.a.y));
    asm("min.bf16x2 %0, %1, %2;" : "=r"(m23) : "r"(raw.a.z), "r"(raw.a.w));
    asm("min.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(m01), "r"(m23));
    asm("max.bf16x2 %0, %1, %2;" : "=r"(M01) : "r"(raw.a.x), "r"(raw.a.y));
    asm("max.bf16x2 %0, %1, %2;" : "=r"(M23) : "r"(raw.a.z), "r"(raw.a.w));
    asm("max.bf16x2 %0, %1, %2;" : "=r"(M) : "r"(M01), "r"(M23));
  } else {
    asm("min.f16x2 %0, %1, %2;" : "=r"(m01) : "r"(raw.a.x), "r"(raw.a.y));
    asm("min.f16x2 %0, %1, %2;" : "=r"(m23) : "r"(raw.a.z), "r"(raw.a.w));
    asm("min.f16x2 %0, %1, %2;" : "=r"(m) : "r"(m01), "r"(m23));
    asm("max.f16x2 %0, %1, %2;" : "=r"(M01) : "r"(raw.a.x), "r"(raw.a.y));
    asm("max.f16x2 %0, %1, %2;" : "=r"(M23) : "r"(raw.a.z), "r"(raw.a.w));
    asm("max.f16x2 %0, %1, %2;" : "=r"(M) : "r"(M01), "r"(M23));
  }
  const uint32_t nM = M ^ 0x80008000u;
  return min2_packed<DT>(__byte_perm(m, nM, 0x5410), __byte_perm(m, nM, 0x7632));
}
// (min, -max) pair -> binary32 (mn, mx).
template <int DT>
__device__ __forceinline__ void unpack_minmax(uint32_t p, float& mn, float& mx) {
  if constexpr (DT == DT_BF16) {
    mn = __uint_as_float(p << 16);
    mx = __uint_as_float((p & 0xFFFF0000u) ^ 0x80000000u);
  } else {
    mn = f16_bits_to_f32(p & 0xFFFFu);
    mx = f16_bits_to_f32((p >> 16) ^ 0x8000u);
  }
}

// Store the chunk's packed unit at byte address p. Element e0 (multiple of 8) starts at
// bit e0*BITS, a byte boundary; the unit is 8*BITS bits: u8 / u16 / u32 / u64.
template <int BITS>
__device__ __forceinline__ void store_unit_at(unsigned char* p, PackedUnit<BITS> u) {
  if constexpr (BITS == 1) {
    *reinterpret_cast<uint8_t*>(p) = (uint8_t)u.lo;
  } else if constexpr (BITS == 2) {
    *reinterpret_cast<uint16_t*>(p) = (uint16_t)u.lo;
  } else if constexpr (BITS == 4) {
    *reinterpret_cast<uint32_t*>(p) = u.lo;
  } else {
    *reinterpret_cast<uint2*>(p) = make_uint2(u.lo, u.hi);
  }
}

template <int BITS>
__device__ __forceinline__ void store_unit(uint32_t* packed, int64_t e0, PackedUnit<BITS> u) {
  store_unit_at<BITS>(reinterpret_cast<unsigned char*>(packed) + (e0 * BITS) / 8, u);
}

// Guarded form for a tensor's last (partial) tile: only bytes of words < nwords.
template <int BITS>
__device__ __forceinline__ void store_unit_guarded(uint32_t* packed, int64_t e0, int64_t nwords,
                                                   PackedUnit<BITS> u) {
  const int64_t byte0 = (e0 * BITS) / 8;
  if constexpr (BITS == 8) {
    const int64_t w0 = byte0 / 4;
    if (w0 < nwords) packed[w0] = u.lo;
    if (w0 + 1 < nwords) packed[w0 + 1] = u.hi;
  } else {
    if (byte0 / 4 < nwords) store_unit<BITS>(packed, e0, u);
  }
}

}  // namespace gact
