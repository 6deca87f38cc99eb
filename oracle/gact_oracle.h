/*
 * gact_oracle.h — the CPU ORACLE of the GACT compressor hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product library
 * (paper_2206_11357_b200/, include/gact.h) never includes, links or calls it, and this
 * file includes nothing from the product. See oracle/gact_oracle.c for the definitions
 * and the paper passages each function follows.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; DESIGN.md §3 = the readings taken
 * where the paper is silent (R1..R12).
 */
#ifndef GACT_ORACLE_H_
#define GACT_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype tags of the oracle (independent of the product's enum; same numeric meaning
 * is fixed by DESIGN.md §2: 0 = binary32, 1 = bfloat16, 2 = binary16). */
enum { ORACLE_F32 = 0, ORACLE_BF16 = 1, ORACLE_F16 = 2 };

/* Error codes returned by the oracle (0 = ok). */
enum { ORACLE_OK = 0, ORACLE_EINVAL = 1, ORACLE_EINFEASIBLE = 5, ORACLE_EINVARIANT = 99 };

/* Philox4x32-10 block function (R3). */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* The 8-bit random number k_i of element i under `seed` (R3): byte 8 (i/256 mod 2) + i mod 8
 * of Philox block 32 (i / 512) + (i / 8 mod 32). */
uint32_t oracle_rand8(uint64_t seed, uint64_t i);

/* The value of element i of a dtype-tagged buffer, widened to binary32 (exact). */
float oracle_widen(const void* x, int32_t dtype, int64_t i);

/* Round a real (given as double) to the nearest value of `dtype`, ties to even,
 * and return the encoding (binary32: 32-bit pattern; bf16/f16: 16-bit pattern). */
uint32_t oracle_round_to_dtype(double v, int32_t dtype);

/* Group statistics of groups [g0, g1) of a tensor of n elements (R1, R2). */
int32_t oracle_group_stats(const void* x, int32_t dtype, int64_t n, int32_t G, int32_t bits,
                           int64_t g0, int64_t g1, float* mn_out, float* scale_out);

/* Codes of the elements of groups [g0, g1): q_out[i - g0*G] = q_i (R1-R5). Also writes the
 * groups' mn / scale. x is the WHOLE tensor (index i is the global element index). */
int32_t oracle_quantize_codes(const void* x, int32_t dtype, int64_t n, int32_t G, int32_t bits,
                              uint64_t seed, int64_t g0, int64_t g1, uint8_t* q_out,
                              float* mn_out, float* scale_out);

/* Pack / unpack codes q[0..n) at `bits` each (R6). packed has ceil(n*bits/32) words. */
int32_t oracle_pack(const uint8_t* q, int64_t n, int32_t bits, uint32_t* packed);
int32_t oracle_unpack(const uint32_t* packed, int64_t n, int32_t bits, uint8_t* q);

/* The whole compressor: codes + pack + group stats for a full tensor. */
int32_t oracle_quantize_pack(const void* x, int32_t dtype, int64_t n, int32_t G, int32_t bits,
                             uint64_t seed, uint32_t* packed, float* mn, float* scale);

/* Decompressor, exact value: y_i = mn_g + q_i * scale_g evaluated in binary64 (R7). */
int32_t oracle_dequantize_f64(const uint32_t* packed, const float* mn, const float* scale,
                              int64_t n, int32_t G, int32_t bits, double* y);

/* Decompressor into a dtype buffer: round_to_dtype(y_i) (R7). */
int32_t oracle_unpack_dequantize(const uint32_t* packed, const float* mn, const float* scale,
                                 int64_t n, int32_t G, int32_t bits, void* y, int32_t y_dtype);

/* S(b) of P:479-480 with S(32) = 0 (R9). */
double oracle_S(int32_t b);

/* sum_l c_l S(b_l), the bound of eqn:var-decomposition. */
double oracle_predicted_variance(const double* c, const int32_t* bits, int32_t L);

/* Greedy solver of eqn:ilp (R10). */
int32_t oracle_allocate_bits(const double* c, const int64_t* D, int32_t L, const int32_t* ladder,
                             int32_t n_ladder, uint64_t B, int32_t* bits_out);

/* Exhaustive solver of eqn:ilp: the minimum of sum c_l S(b_l) over ALL ladder^L schemes
 * with sum b_l D_l <= B (L <= 12). Returns the minimising scheme (first in lexicographic
 * order among equal minima) and its value. */
int32_t oracle_allocate_bruteforce(const double* c, const int64_t* D, int32_t L,
                                   const int32_t* ladder, int32_t n_ladder, uint64_t B,
                                   int32_t* bits_out, double* value_out);

/* sum_i (a_i - b_i)^2, the ||g0 - g1||^2 of Alg. 1, accumulated in long double
 * (x86 80-bit) in index order. */
double oracle_sq_diff_sum(const void* a, const void* b, int32_t dtype, int64_t n);

#ifdef __cplusplus
}
#endif

#endif
