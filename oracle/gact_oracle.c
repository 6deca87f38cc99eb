/*
 * gact_oracle.c — plain, slow, obviously-correct CPU oracle of the GACT compressor.
 *
 * TEST INFRASTRUCTURE ONLY (see gact_oracle.h). Single-threaded, element by element, in
 * the paper's order and notation. Shares no code, header, table or constant generator
 * with the CUDA path. Build: gcc -O2 -std=c11 -ffp-contract=off -frounding-math (the
 * Makefile): no FMA contraction, no fast-math, directed rounding honoured.
 *
 * Precision: the north_star fixes the code computation to "fixed-order IEEE fp32
 * arithmetic with FMA contraction disabled" (BASELINE.json), so group statistics and the
 * transform t are binary32 here, one rounding per operation (x86-64 SSE: FLT_EVAL_METHOD
 * is 0, no excess precision). The floor of t + u, the decompressed value, S(b) and the
 * allocator are evaluated in binary64 / exact integer arithmetic.
 *
 * Paper passages (P:n = /root/reference/PAPER.md line n):
 *   quantizer  App. Prop. 3 P:226-233 (T_{h,b}, stochastic rounding, T^{-1}),
 *              "per-group quantizer" P:547, R = 1/4 range^2 and S(b) P:479-480
 *   budget     eqn:ilp P:471-475; greedy P:534; eqn:var-decomposition P:485-487
 *   seeds      Alg. 1 P:512-521 ("seed Q^(l) with r_l")
 * Readings R1..R12 where the paper is silent are listed in DESIGN.md §3.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py to something
 * other than itself (KAT vectors, ATen's Philox, NumPy/torch dtype conversions, exact
 * rational arithmetic, exhaustive enumeration of the random byte, closed-form round trips, brute force).
 */
#include "gact_oracle.h"

#include <fenv.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------
 * R3  Counter-based random lanes: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11;
 * Random123 constants). The paper only says "seed Q^(l) with r_l"; a
 * counter-based generator makes the replay of Alg. 1 exact and order-independent.
 * ---------------------------------------------------------------------------------- */
#define PHILOX_M0 0xD2511F53u /* multiplier applied to counter word 0 */
#define PHILOX_M1 0xCD9E8D57u /* multiplier applied to counter word 2 */
#define PHILOX_W0 0x9E3779B9u /* key bump, word 0 (golden ratio) */
#define PHILOX_W1 0xBB67AE85u /* key bump, word 1 (sqrt(3) - 1) */

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0; /* 32x32 -> 64 product */
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += PHILOX_W0; /* the key is bumped after every round */
    k1 += PHILOX_W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Element i draws 8 random bits (R3, R4 as revised by DESIGN.md §4's ceiling table):
 *   block  beta(i) = 32 floor(i / 512) + (floor(i / 8) mod 32),
 *   byte   j(i)    = 8 (floor(i / 256) mod 2) + (i mod 8)
 * of the block's 16 output bytes (word j >> 2, byte j & 3, least significant first);
 * key = (lo32(seed), hi32(seed)), counter = (lo32(beta), hi32(beta), 0, 0). Every block
 * serves 16 elements: chunk l (8 consecutive elements) of the first and of the second
 * 256-element half of each 512-element span. */
uint32_t oracle_rand8(uint64_t seed, uint64_t i) {
  uint64_t block = ((i >> 9) << 5) + ((i >> 3) & 31u);
  uint32_t ctr[4] = {(uint32_t)block, (uint32_t)(block >> 32), 0u, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t r[4];
  oracle_philox4x32_10(ctr, key, r);
  uint32_t j = (uint32_t)(((i >> 8) & 1u) * 8u + (i & 7u));
  return (r[j >> 2] >> (8u * (j & 3u))) & 0xFFu;
}

/* ------------------------------------------------------------------------------------
 * Element access. bfloat16 is by definition the upper half of a binary32 pattern;
 * binary16 is decoded from its fields (IEEE 754-2008 §3.4): sign, 5-bit exponent with
 * bias 15, 10-bit fraction, subnormals at exponent field 0. Both widen exactly.
 * ---------------------------------------------------------------------------------- */
static float f32_from_bits(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t bits_from_f32(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

static double f16_value(uint16_t h) {
  int sign = (h >> 15) & 1;
  int e = (h >> 10) & 0x1F;
  int m = h & 0x3FF;
  double v;
  if (e == 0) v = ldexp((double)m, -24);                    /* subnormal: m * 2^-24 */
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = ldexp((double)(1024 + m), e - 25);                /* (1 + m/1024) * 2^(e-15) */
  return sign ? -v : v;
}

float oracle_widen(const void* x, int32_t dtype, int64_t i) {
  if (dtype == ORACLE_F32) return ((const float*)x)[i];
  if (dtype == ORACLE_BF16) return f32_from_bits((uint32_t)((const uint16_t*)x)[i] << 16);
  return (float)f16_value(((const uint16_t*)x)[i]);
}

/* Round-to-nearest-even of a real v into a binary format with p significand bits,
 * minimum normal exponent emin and largest finite value vmax (IEEE 754 §4.3.1). */
static double round_to_format(double v, int p, int emin, double vmax) {
  if (v == 0.0 || !isfinite(v)) return v;
  int e;
  frexp(fabs(v), &e);          /* |v| in [2^(e-1), 2^e) */
  int exp_v = e - 1;
  if (exp_v < emin) exp_v = emin; /* subnormal range shares the ulp of 2^emin */
  double ulp = ldexp(1.0, exp_v - (p - 1));
  double r = nearbyint(v / ulp) * ulp; /* v/ulp is exact (power of two); default mode RNE */
  /* overflow: values at or beyond vmax + ulp/2 round to infinity */
  if (fabs(r) > vmax) return v > 0 ? INFINITY : -INFINITY;
  return r;
}

/* The same for the exact real s + e, given as an unevaluated sum with |e| <= ulp64(s) / 2
 * (a TwoSum pair): rounded ONCE. s + e and s round alike unless s is exactly halfway
 * between two neighbours of the format, where the sign of e breaks the tie. */
static double round_to_format_sum(double s, double e, int p, int emin, double vmax) {
  if (s == 0.0 || !isfinite(s)) return s + e;
  int ex;
  frexp(fabs(s), &ex);
  int exp_v = ex - 1;
  if (exp_v < emin) exp_v = emin;
  double ulp = ldexp(1.0, exp_v - (p - 1));
  double t = s / ulp, f = floor(t), r;
  if (t - f == 0.5 && e != 0.0) r = (e > 0.0 ? f + 1.0 : f) * ulp;
  else r = nearbyint(t) * ulp;
  if (fabs(r) > vmax) return s > 0 ? INFINITY : -INFINITY;
  return r;
}

static uint32_t encode_dtype(double r, int32_t dtype);

uint32_t oracle_round_to_dtype(double v, int32_t dtype) {
  if (dtype == ORACLE_F32) return encode_dtype(round_to_format(v, 24, -126, 3.4028234663852886e38), dtype);
  if (dtype == ORACLE_BF16) return encode_dtype(round_to_format(v, 8, -126, 3.3895313892515355e38), dtype);
  return encode_dtype(round_to_format(v, 11, -14, 65504.0), dtype);
}

/* s + e (a TwoSum pair) rounded once to nearest-even into dtype, encoded. */
static uint32_t round_sum_to_dtype(double s, double e, int32_t dtype) {
  if (dtype == ORACLE_F32) return encode_dtype(round_to_format_sum(s, e, 24, -126, 3.4028234663852886e38), dtype);
  if (dtype == ORACLE_BF16) return encode_dtype(round_to_format_sum(s, e, 8, -126, 3.3895313892515355e38), dtype);
  return encode_dtype(round_to_format_sum(s, e, 11, -14, 65504.0), dtype);
}

/* Encoding of a value r representable in dtype. */
static uint32_t encode_dtype(double r, int32_t dtype) {
  if (dtype == ORACLE_F32) return bits_from_f32((float)r);           /* exact */
  if (dtype == ORACLE_BF16) return bits_from_f32((float)r) >> 16;    /* low half is zero */
  /* binary16: from its fields */
  uint16_t sign = signbit(r) ? 0x8000u : 0u;
  double a = fabs(r);
  if (isinf(a)) return sign | 0x7C00u;
  if (a == 0.0) return sign;
  if (a < ldexp(1.0, -14)) return sign | (uint16_t)(a / ldexp(1.0, -24)); /* subnormal */
  int e;
  double f = frexp(a, &e); /* a = f * 2^e, f in [0.5, 1) */
  uint16_t exp_field = (uint16_t)(e - 1 + 15);
  uint16_t frac = (uint16_t)((f * 2.0 - 1.0) * 1024.0);
  return sign | (uint16_t)(exp_field << 10) | frac;
}

/* ------------------------------------------------------------------------------------
 * R1, R2  Per-group statistics (App. Prop. 3: T_{h,b} uses min_j h and max_j h of
 * the group; "per-group quantizer" P:547). Groups are consecutive runs of G elements of
 * the flattened tensor; the last group may be short.
 * ---------------------------------------------------------------------------------- */

/* IEEE division a / b rounded toward zero (R2: inv uses RZ so that t <= L, proof in
 * DESIGN.md). The rounding mode is switched around the division (-frounding-math). */
static float div_toward_zero(float a, float b) {
  int old = fegetround();
  fesetround(FE_TOWARDZERO);
  volatile float va = a, vb = b;
  volatile float r = va / vb;
  fesetround(old);
  return r;
}

typedef struct { float mn, scale, inv; } group_params;

static group_params group_stats_one(const void* x, int32_t dtype, int64_t lo, int64_t hi,
                                    int32_t bits) {
  float mn = oracle_widen(x, dtype, lo), mx = mn;
  for (int64_t i = lo + 1; i < hi; ++i) {
    float v = oracle_widen(x, dtype, i);
    if (v < mn) mn = v;
    if (v > mx) mx = v;
  }
  mn = mn + 0.0f; /* -0 -> +0: the stored min never depends on which zero was seen */
  mx = mx + 0.0f;
  float Lf = (float)((1u << bits) - 1u); /* L = 2^b - 1, exact */
  float range = mx - mn;
  group_params p;
  p.mn = mn;
  p.scale = range / Lf;                                   /* the decode step, RN */
  p.inv = (range == 0.0f) ? 0.0f : div_toward_zero(Lf, range); /* constant group: t = 0 */
  return p;
}

static int valid_common(int64_t n, int32_t G, int32_t bits, int32_t dtype) {
  if (n < 0 || G < 1) return 0;
  if (!(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return 0;
  if (dtype < 0 || dtype > 2) return 0;
  return 1;
}

int32_t oracle_group_stats(const void* x, int32_t dtype, int64_t n, int32_t G, int32_t bits,
                           int64_t g0, int64_t g1, float* mn_out, float* scale_out) {
  if (!valid_common(n, G, bits, dtype)) return ORACLE_EINVAL;
  int64_t ng = (n + G - 1) / G;
  if (g0 < 0 || g1 > ng || g0 > g1) return ORACLE_EINVAL;
  for (int64_t g = g0; g < g1; ++g) {
    int64_t lo = g * G, hi = lo + G < n ? lo + G : n;
    group_params p = group_stats_one(x, dtype, lo, hi, bits);
    mn_out[g - g0] = p.mn;
    scale_out[g - g0] = p.scale;
  }
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------------------
 * R4, R5  Stochastic rounding (App. Prop. 3):
 *   Q(h)_j = T^{-1}(ceil(T(h_j)))  w.p. T(h_j) - floor(T(h_j)),  else T^{-1}(floor(T(h_j)))
 * realised as q = floor(T + u) with u = (2k+1) 2^-9, k uniform on [0, 2^8): the event
 * q = ceil(T) is {u >= 1 - frac(T)}, whose probability is frac(T) up to 2^-9 (R4).
 * T = d * inv with d = h_j - min rounded to binary32 (R5); the product and the sum with u
 * are EXACT reals (no rounding of T): q = floor(P) + [P - floor(P) >= 1 - u] with
 * P = d * inv held exactly in binary64 (24 x 24 significand bits <= 53), and
 * P - floor(P), 1 - u exact -- a comparison of exact values.
 * ---------------------------------------------------------------------------------- */
int32_t oracle_quantize_codes(const void* x, int32_t dtype, int64_t n, int32_t G, int32_t bits,
                              uint64_t seed, int64_t g0, int64_t g1, uint8_t* q_out,
                              float* mn_out, float* scale_out) {
  if (!valid_common(n, G, bits, dtype)) return ORACLE_EINVAL;
  int64_t ng = (n + G - 1) / G;
  if (g0 < 0 || g1 > ng || g0 > g1) return ORACLE_EINVAL;
  const double L = (double)((1u << bits) - 1u);
  for (int64_t g = g0; g < g1; ++g) {
    int64_t lo = g * G, hi = lo + G < n ? lo + G : n;
    group_params p = group_stats_one(x, dtype, lo, hi, bits);
    mn_out[g - g0] = p.mn;
    scale_out[g - g0] = p.scale;
    for (int64_t i = lo; i < hi; ++i) {
      float h = oracle_widen(x, dtype, i);
      float d = h - p.mn;                      /* h_j - min_j h   (binary32, RN) */
      double P = (double)d * (double)p.inv;    /* T = (2^b-1)(h_j - min)/(max - min), exact */
      if (!(P >= 0.0 && P <= L)) return ORACLE_EINVARIANT; /* proven in DESIGN.md R2 */
      uint32_t k = oracle_rand8(seed, (uint64_t)i);
      double one_minus_u = (512.0 - 2.0 * (double)k - 1.0) / 512.0; /* 1 - u, exact */
      double F = floor(P);
      double q = F + ((P - F) >= one_minus_u ? 1.0 : 0.0); /* floor(T + u), exact */
      if (q > L) return ORACLE_EINVARIANT;
      q_out[i - g0 * G] = (uint8_t)q;
    }
  }
  return ORACLE_OK;
}

/* R6  Packing: element i -> bits [(i b) mod 32, +b) of word floor(i b / 32), LSB first. */
int32_t oracle_pack(const uint8_t* q, int64_t n, int32_t bits, uint32_t* packed) {
  if (n < 0 || !(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return ORACLE_EINVAL;
  int64_t words = (n * bits + 31) / 32;
  memset(packed, 0, (size_t)words * 4);
  for (int64_t i = 0; i < n; ++i) {
    if (q[i] >> bits) return ORACLE_EINVARIANT;
    int64_t bit = i * bits;
    packed[bit >> 5] |= (uint32_t)q[i] << (bit & 31);
  }
  return ORACLE_OK;
}

int32_t oracle_unpack(const uint32_t* packed, int64_t n, int32_t bits, uint8_t* q) {
  if (n < 0 || !(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return ORACLE_EINVAL;
  uint32_t L = (1u << bits) - 1u;
  for (int64_t i = 0; i < n; ++i) {
    int64_t bit = i * bits;
    q[i] = (uint8_t)((packed[bit >> 5] >> (bit & 31)) & L);
  }
  return ORACLE_OK;
}

int32_t oracle_quantize_pack(const void* x, int32_t dtype, int64_t n, int32_t G, int32_t bits,
                             uint64_t seed, uint32_t* packed, float* mn, float* scale) {
  if (!valid_common(n, G, bits, dtype)) return ORACLE_EINVAL;
  int64_t ng = (n + G - 1) / G;
  uint8_t* q = (uint8_t*)malloc(n > 0 ? (size_t)n : 1);
  if (!q) return ORACLE_EINVAL;
  int32_t rc = oracle_quantize_codes(x, dtype, n, G, bits, seed, 0, ng, q, mn, scale);
  if (rc == ORACLE_OK) rc = oracle_pack(q, n, bits, packed);
  free(q);
  return rc;
}

/* ------------------------------------------------------------------------------------
 * R7  Decompression T^{-1}_{h,b}(q) = min + q (max - min)/(2^b - 1) = mn + q * scale
 * (App. Prop. 3; "Decompressor dequantizes"). oracle_dequantize_f64 gives
 * it in binary64 (q * scale is exact, 8 x 24 bits; the sum rounds once at 2^-53);
 * oracle_unpack_dequantize rounds the EXACT value once into the output dtype: the sum is
 * kept as the TwoSum pair (s, e), s + e = mn + q * scale exactly (Knuth), and only then
 * rounded (round_sum_to_dtype), so there is no double rounding through binary64.
 * ---------------------------------------------------------------------------------- */
int32_t oracle_dequantize_f64(const uint32_t* packed, const float* mn, const float* scale,
                              int64_t n, int32_t G, int32_t bits, double* y) {
  if (n < 0 || G < 1 || !(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return ORACLE_EINVAL;
  uint8_t* q = (uint8_t*)malloc(n > 0 ? (size_t)n : 1);
  if (!q) return ORACLE_EINVAL;
  oracle_unpack(packed, n, bits, q);
  for (int64_t i = 0; i < n; ++i) {
    int64_t g = i / G;
    y[i] = (double)mn[g] + (double)q[i] * (double)scale[g];
  }
  free(q);
  return ORACLE_OK;
}

int32_t oracle_unpack_dequantize(const uint32_t* packed, const float* mn, const float* scale,
                                 int64_t n, int32_t G, int32_t bits, void* y, int32_t y_dtype) {
  if (y_dtype < 0 || y_dtype > 2) return ORACLE_EINVAL;
  if (n < 0 || G < 1 || !(bits == 1 || bits == 2 || bits == 4 || bits == 8)) return ORACLE_EINVAL;
  uint8_t* q = (uint8_t*)malloc(n > 0 ? (size_t)n : 1);
  if (!q) return ORACLE_EINVAL;
  oracle_unpack(packed, n, bits, q);
  for (int64_t i = 0; i < n; ++i) {
    int64_t g = i / G;
    double a = (double)mn[g], b = (double)q[i] * (double)scale[g]; /* both exact */
    double s = a + b;                                               /* TwoSum (Knuth): */
    double bv = s - a, av = s - bv;
    double e = (a - av) + (b - bv);                                 /* s + e == a + b */
    uint32_t enc = round_sum_to_dtype(s, e, y_dtype);
    if (y_dtype == ORACLE_F32) ((uint32_t*)y)[i] = enc;
    else ((uint16_t*)y)[i] = (uint16_t)enc;
  }
  free(q);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------------------
 * R9, R10  Bit allocation. eqn:ilp:
 *     min_b  sum_l c_l S(b_l)  s.t.  sum_l b_l D_l <= B,   S(b) = (2^b - 1)^-2
 * S(32) = 0: 32 bits means the tensor is kept in full precision.
 * ---------------------------------------------------------------------------------- */
double oracle_S(int32_t b) {
  if (b == 32) return 0.0;
  double m = (double)((1ull << b) - 1ull); /* exact for b <= 16 */
  return 1.0 / (m * m);
}

double oracle_predicted_variance(const double* c, const int32_t* bits, int32_t L) {
  double v = 0.0;
  for (int32_t l = 0; l < L; ++l) v += c[l] * oracle_S(bits[l]);
  return v;
}

static int valid_alloc(const double* c, const int64_t* D, int32_t L, const int32_t* ladder,
                       int32_t n_ladder) {
  if (L < 0 || n_ladder < 1 || !ladder) return 0;
  if (L > 0 && (!c || !D)) return 0;
  for (int32_t k = 0; k < n_ladder; ++k) {
    if (!((ladder[k] >= 1 && ladder[k] <= 16) || ladder[k] == 32)) return 0;
    if (k > 0 && ladder[k] <= ladder[k - 1]) return 0;
  }
  for (int32_t l = 0; l < L; ++l) {
    if (isnan(c[l]) || c[l] < 0.0 || D[l] < 1) return 0;
  }
  return 1;
}

/* The greedy of P:534 in its plainest form: start at the top of the ladder; while over
 * budget, scan all tensors for the smallest variance increase per bit saved and lower that
 * one step (ties -> smaller l). O(L) per step. */
int32_t oracle_allocate_bits(const double* c, const int64_t* D, int32_t L, const int32_t* ladder,
                             int32_t n_ladder, uint64_t B, int32_t* bits_out) {
  if (!valid_alloc(c, D, L, ladder, n_ladder) || (L > 0 && !bits_out)) return ORACLE_EINVAL;
  unsigned __int128 need_min = 0, total = 0;
  for (int32_t l = 0; l < L; ++l) {
    need_min += (unsigned __int128)ladder[0] * (uint64_t)D[l];
    total += (unsigned __int128)ladder[n_ladder - 1] * (uint64_t)D[l];
  }
  if (need_min > B) return ORACLE_EINFEASIBLE;
  int32_t* level = (int32_t*)malloc(L > 0 ? (size_t)L * sizeof(int32_t) : 1);
  if (!level) return ORACLE_EINVAL;
  for (int32_t l = 0; l < L; ++l) level[l] = n_ladder - 1;
  while (total > B) {
    int32_t best = -1;
    double best_ratio = 0.0;
    for (int32_t l = 0; l < L; ++l) {
      if (level[l] == 0) continue;
      int32_t hi = ladder[level[l]], lo = ladder[level[l] - 1];
      double num = c[l] * (oracle_S(lo) - oracle_S(hi));
      double den = (double)(hi - lo) * (double)D[l];
      double ratio = num / den;
      if (best < 0 || ratio < best_ratio) { best = l; best_ratio = ratio; }
    }
    if (best < 0) break; /* unreachable: need_min <= B */
    int32_t hi = ladder[level[best]], lo = ladder[level[best] - 1];
    total -= (unsigned __int128)(hi - lo) * (uint64_t)D[best];
    level[best] -= 1;
  }
  for (int32_t l = 0; l < L; ++l) bits_out[l] = ladder[level[l]];
  free(level);
  return ORACLE_OK;
}

int32_t oracle_allocate_bruteforce(const double* c, const int64_t* D, int32_t L,
                                   const int32_t* ladder, int32_t n_ladder, uint64_t B,
                                   int32_t* bits_out, double* value_out) {
  if (!valid_alloc(c, D, L, ladder, n_ladder) || L > 12) return ORACLE_EINVAL;
  int32_t idx[12] = {0}, scheme[12] = {0};
  int found = 0;
  double best = 0.0;
  for (;;) {
    unsigned __int128 used = 0;
    for (int32_t l = 0; l < L; ++l) {
      scheme[l] = ladder[idx[l]];
      used += (unsigned __int128)scheme[l] * (uint64_t)D[l];
    }
    if (used <= B) {
      double v = oracle_predicted_variance(c, scheme, L);
      if (!found || v < best) {
        found = 1;
        best = v;
        for (int32_t l = 0; l < L; ++l) bits_out[l] = scheme[l];
      }
    }
    int32_t l = L - 1; /* next scheme in lexicographic order (last index fastest) */
    while (l >= 0 && idx[l] == n_ladder - 1) { idx[l] = 0; --l; }
    if (l < 0) break;
    idx[l] += 1;
  }
  if (!found) return ORACLE_EINFEASIBLE;
  if (value_out) *value_out = best;
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------------------
 * Alg. 1: c_l = 1/2 ||g0 - g1||^2 / S(b_l). The squared distance of the two
 * gradient evaluations, each element widened exactly, differences and squares in long
 * double, summed in index order.
 * ---------------------------------------------------------------------------------- */
double oracle_sq_diff_sum(const void* a, const void* b, int32_t dtype, int64_t n) {
  long double acc = 0.0L;
  for (int64_t i = 0; i < n; ++i) {
    long double d = (long double)oracle_widen(a, dtype, i) - (long double)oracle_widen(b, dtype, i);
    acc += d * d;
  }
  return (double)acc;
}
