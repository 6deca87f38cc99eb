/*
 * gact.h — C ABI of the GACT activation-compressor hot path, B200 (sm_100a).
 *
 * GACT (arXiv 2206.11357) compresses every saved context tensor h^(l) of a training
 * step with a per-group stochastic-rounding quantizer to b_l bits (PAPER.md App.
 * Prop. 3; "the same per-group quantizer in ActNN", §5), decompresses
 * it in backward (§5.2), and chooses the bits b = (b_l) by solving the budget
 * problem eqn:ilp with a greedy solver (§4.3).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (LaTeX source); DESIGN.md §3 lists
 * every reading taken where the paper is silent.
 *
 * ---------------------------------------------------------------------------------
 * The quantizer this library computes (DESIGN.md §3 "readings" R1-R9)
 * ---------------------------------------------------------------------------------
 * A tensor is its row-major flattened vector x[0..n) ("each tensor ... is
 * represented by a flattened D_l-dimensional vector"). It is cut into ng = ceil(n/G)
 * consecutive groups of G elements; the last group may be short (no padding).
 * With L = 2^b - 1, for group g (all arithmetic IEEE-754 binary32, one rounding per
 * operation, no FMA contraction):
 *     mn    = min_j x_j + 0.0f        mx = max_j x_j + 0.0f      (+0.0f maps -0 to +0)
 *     range = mx - mn                                           (round to nearest)
 *     scale = range / L                                          (round to nearest)
 *     inv   = range == 0 ? 0 : L / range                        (round toward ZERO)
 * and for every element i of the group
 *     d_i = x_i - mn                                             (round to nearest)
 *     T_i = d_i * inv                                            (EXACT real product)
 *     q_i = floor(T_i + (2 k_i + 1) 2^-9),  k_i = random byte of (seed, i)     (below)
 *                                     (exact real floor, no rounding of T_i; q_i in [0, L]
 *                                      because T_i <= range * RZ(L / range) <= L)
 * which is T_{h,b} of P:233 followed by the stochastic rounding of P:229-230:
 * q_i = ceil(T) with probability frac(T) rounded to the centred 2^-8 lattice of thresholds
 * u = (2k+1) 2^-9 (|P - frac T| <= 2^-9; R4, §4a), else floor(T); q_i = T_i when
 * T_i is an integer. (R2, R4, R5; the GPU evaluates it exactly, for every b, as
 * add.rm(fma.rm(d, inv, 128 + u), 2^23 - 128): 128 + u is a binary32 value and rounding
 * down never crosses an integer; the oracle as floor(P) + [P - floor(P) >= 1 - u] in
 * binary64.)
 * Decompression (T^{-1}):   y_i = fma(q_i, scale, mn) in binary32, then
 * rounded to nearest-even into the output dtype.
 *
 * Random bytes (counter-based; "seed Q^(l) with r_l" needs exact replay):
 *   Philox4x32-10 (Salmon et al. 2011, Random123 constants), key = (lo32(seed),
 *   hi32(seed)), counter = (lo32(beta), hi32(beta), 0, 0) -> words r[0..3], with
 *     beta(i) = 32 floor(i / 512) + (floor(i / 8) mod 32),
 *     j(i)    = 8 (floor(i / 256) mod 2) + (i mod 8),
 *     k_i     = (r[j >> 2] >> (8 (j & 3))) & 0xFF.
 *   Each block serves 16 elements (every byte once): the 8-element chunk at position
 *   l = floor(i / 8) mod 32 of both 256-element halves of a 512-element span.
 *   Use a distinct seed per tensor (Alg. 1 seeds r_1..r_L); equal seeds correlate tensors.
 *
 * Packing: code q_i occupies bits [(i*b) mod 32, +b) of uint32 word (i*b)/32, LSB first;
 * the unused high bits of the last word are zero. packed has ceil(n*b/32) words.
 *
 * ---------------------------------------------------------------------------------
 * Conventions for every call
 * ---------------------------------------------------------------------------------
 *  - Ownership: the caller owns and allocates every buffer (PyTorch's caching allocator
 *    in the binding). The library never allocates, frees, synchronises or keeps state
 *    (except the staged forms' streams and events, below); it is thread-safe. Sizes come
 *    from gact_num_groups / gact_packed_words.
 *  - Device calls (x, y, packed, group_min, group_scale are DEVICE pointers) enqueue on
 *    `stream` (a cudaStream_t passed as void*; NULL = legacy default stream) and return
 *    without waiting. gact_allocate_bits takes HOST pointers and runs on the host.
 *  - Validation happens before any launch; on any error nothing is written.
 *      bits not in {1,2,4,8}                          -> GACT_ERR_UNSUPPORTED_BITS
 *      group_size not a multiple of 32 in [32, 4096]  -> GACT_ERR_GROUP_SIZE
 *    (powers of two run specialised kernels; the other multiples of 32 a generic one: a
 *    warp per group)
 *      x / y not 16-byte aligned, packed not 8-byte,
 *      group_min / group_scale not 4-byte aligned     -> GACT_ERR_ALIGNMENT
 *      n < 0, NULL pointer with n > 0, bad dtype      -> GACT_ERR_INVALID_ARG
 *    n == 0 is valid and launches nothing.
 *  - Inputs must be finite; NaN/Inf input or a group whose range overflows binary32 is
 *    undefined behaviour (SPEC S:106-107 calls it an error; checking it would cost a
 *    device sync). No output is ever non-finite for finite input whose ranges are finite.
 *  - Determinism: every output is a pure function of (x, n, G, b, seed): independent of
 *    grid shape, stream and device. Alg. 1's seed replay relies on this.
 *  - A launch failure is returned as GACT_ERR_CUDA (cudaGetLastError after the launch).
 */
#ifndef GACT_H_
#define GACT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { GACT_F32 = 0, GACT_BF16 = 1, GACT_F16 = 2 } gact_dtype;

typedef enum {
  GACT_OK = 0,
  GACT_ERR_INVALID_ARG = 1,
  GACT_ERR_UNSUPPORTED_BITS = 2,
  GACT_ERR_GROUP_SIZE = 3,
  GACT_ERR_ALIGNMENT = 4,
  GACT_ERR_INFEASIBLE = 5,
  GACT_ERR_CUDA = 6
} gact_status;

/* Library ABI version, (major << 16) | minor. */
int32_t gact_version(void);

/* Human-readable name of a status code (static storage; never NULL). */
const char* gact_status_string(int32_t status);

/* ceil(n / group_size): number of groups, i.e. entries of group_min / group_scale.
 * Returns -1 if n < 0 or group_size < 1. */
int64_t gact_num_groups(int64_t n, int32_t group_size);

/* ceil(n * bits / 32): uint32 words of `packed`. Returns -1 if n < 0 or bits < 1. */
int64_t gact_packed_words(int64_t n, int32_t bits);

/* a1 — group statistics only (App. Prop. 3: min_j h, max_j h of each group).
 *   x            device, n elements of dtype `dtype` (gact_dtype), 16-byte aligned
 *   group_min    device, out, ng floats: mn of each group (as defined above)
 *   group_scale  device, out, ng floats: scale = range / (2^bits - 1)
 * Reads x once; writes exactly what gact_quantize_pack writes to the same two arrays. */
gact_status gact_group_stats(const void* x, int32_t dtype, int64_t n, int32_t group_size,
                             int32_t bits, float* group_min, float* group_scale,
                             void* stream);

/* a1+a2+a3 — fused group-reduce, stochastic-rounding quantize and bit-pack
 * (App. Prop. 3; eqn:ac P:360-362 applies Q to every context tensor).
 *   x            device, n elements of `dtype`, 16-byte aligned, finite
 *   seed         the Philox key for this tensor (Alg. 1's r_l)
 *   packed       device, out, gact_packed_words(n, bits) uint32 words, 8-byte aligned
 *   group_min    device, out, gact_num_groups(n, group_size) floats
 *   group_scale  device, out, gact_num_groups(n, group_size) floats
 * Reads x exactly once (single pass: the group is reduced in registers, then coded). */
gact_status gact_quantize_pack(const void* x, int32_t dtype, int64_t n, int32_t group_size,
                               int32_t bits, uint64_t seed, uint32_t* packed,
                               float* group_min, float* group_scale, void* stream);

/* a4+a5 — fused unpack and dequantize (T^{-1}_{h,b}; §5.2
 * "Decompressor dequantizes context tensors").
 *   packed, group_min, group_scale   device, in, as written by gact_quantize_pack
 *   y            device, out, n elements of `y_dtype`, 16-byte aligned
 * y_i = RNE_{y_dtype}( fma(q_i, scale_g, mn_g) ). */
gact_status gact_unpack_dequantize(const uint32_t* packed, const float* group_min,
                                   const float* group_scale, int64_t n, int32_t group_size,
                                   int32_t bits, void* y, int32_t y_dtype, void* stream);

/* One tensor of a batched call. All pointers are device pointers with the alignment
 * rules above; each tensor has its own n, bits, dtype and seed. */
typedef struct {
  void* data;           /* quantize: input x (read only) | dequantize: output y */
  uint32_t* packed;     /* quantize: output  | dequantize: input (const use)   */
  float* group_min;     /* quantize: output  | dequantize: input               */
  float* group_scale;   /* quantize: output  | dequantize: input               */
  int64_t n;            /* elements                                            */
  uint64_t seed;        /* Philox key (ignored by dequantize)                  */
  int32_t bits;         /* in {1,2,4,8}                                        */
  int32_t dtype;        /* dtype of x (quantize) or of y (dequantize)          */
} gact_tensor_desc;

/* Batched forms: one kernel launch (per <= GACT_MAX_BATCH tensors) compresses or
 * decompresses a whole context h = (h^(l))_{l=1..L} with per-tensor b_l.
 * `descs` is a HOST array; it is copied into the launch's parameter space, so it may be
 * reused as soon as the call returns. Results are bit-identical to calling the
 * single-tensor functions one tensor at a time. Any invalid descriptor -> its error code,
 * nothing launched. */
#define GACT_MAX_BATCH 256
gact_status gact_quantize_pack_batch(const gact_tensor_desc* descs, int32_t count,
                                     int32_t group_size, void* stream);
gact_status gact_unpack_dequantize_batch(const gact_tensor_desc* descs, int32_t count,
                                         int32_t group_size, void* stream);

/* Staged (host-buffer) forms — the compressor with its inputs and outputs in HOST memory,
 * i.e. the paper's "Parallel Swap and Prefetch" (compressed tensors offloaded to
 * the CPU and swapped back, "two new streams (swap in/out)" ordered by "the CUDA event") as
 * one call.
 * Each of data / packed / group_min / group_scale of each descriptor may be a host pointer
 * (page-locked: the copies overlap the kernels; pageable: correct, copies serialise) or a
 * device pointer; the library classifies it with cudaPointerGetAttributes. Host buffers
 * are staged through `workspace` in pieces of whole lcm(group_size, 4096)-element blocks:
 * GACT_STAGED_SLOTS slots of workspace_bytes / GACT_STAGED_SLOTS bytes rotate so that the
 * host->device copies of piece k+1 (internal stream), the batched kernels of piece k (on
 * `stream`) and the device->host copies of piece k-1 (second internal stream) overlap;
 * events order them. The Philox counter of every element stays its index in the whole
 * tensor, so results are bit-identical to the batch forms on the same descriptors.
 *   workspace        device, >= GACT_STAGED_MIN_WORKSPACE bytes, 256-byte aligned,
 *                    caller-owned (contents clobbered)
 *   stream           work is ordered after everything already enqueued on `stream`
 * Same validation and alignment rules as the batch forms, plus GACT_ERR_INVALID_ARG for a
 * NULL / small / misaligned workspace. Pieces are whole multiples of lcm(group_size, 4096)
 * elements (4096 for powers of two), so a slot must hold one such piece in the worst case
 * (fp32, b = 8): a group size such as 4064 needs ~3 MB per slot. BLOCKING: returns after every output is written
 * (host outputs readable, device outputs complete). The internal streams and events are
 * created once per host thread and device and reused (the only state the library keeps). */
#define GACT_STAGED_SLOTS 3
#define GACT_STAGED_MIN_WORKSPACE (3u * 65536u)
gact_status gact_quantize_pack_staged(const gact_tensor_desc* descs, int32_t count,
                                      int32_t group_size, void* workspace,
                                      uint64_t workspace_bytes, void* stream);
gact_status gact_unpack_dequantize_staged(const gact_tensor_desc* descs, int32_t count,
                                          int32_t group_size, void* workspace,
                                          uint64_t workspace_bytes, void* stream);

/* a6 — bit allocation: greedy solution of eqn:ilp (solver P:534)
 *     min_b  sum_l c_l S(b_l)   s.t.  sum_l b_l D_l <= B,   S(b) = (2^b - 1)^-2, S(32) = 0
 * (S from P:479-480; 32 bits = keep the tensor uncompressed).
 * Greedy (downgrade from the top): start every b_l at max(ladder); while
 * sum b_l D_l > B, lower the tensor whose next step down b -> b- has the smallest
 *     ratio_l = c_l * (S(b-) - S(b)) / ((b - b-) * D_l)       (IEEE double, this order)
 * (ties -> smaller l), until within budget.
 *   sensitivity  host, L doubles c_l >= 0 (may be +inf: never lowered before finite ones)
 *   numel        host, L int64 D_l >= 1
 *   ladder       host, n_ladder strictly ascending widths, each in [1,16] or == 32
 *   budget_bits  B, in bits of codes (the per-group sidecar is not counted, R8)
 *   bits_out     host, out, L int32
 * Errors: GACT_ERR_INFEASIBLE if sum_l min(ladder) D_l > B; GACT_ERR_INVALID_ARG on NaN
 * or negative c_l, D_l < 1, bad ladder, L < 0, NULL pointers. O(L log L). */
gact_status gact_allocate_bits(const double* sensitivity, const int64_t* numel, int32_t L,
                               const int32_t* ladder, int32_t n_ladder, uint64_t budget_bits,
                               int32_t* bits_out);

/* S(b) = (2^b - 1)^-2, the per-tensor variance factor of P:479-480 (Var of the b-bit
 * quantizer <= 1/4 range^2 S(b)), with S(32) = 0 (32 bits = uncompressed): the S the
 * allocator above uses, exposed so that callers of Alg. 1 (c_l = 1/2 ||g0 - g1||^2 / S(b_l),
 * P:524) and of the variance prediction sum_l c_l S(b_l) use the same
 * definition. Host function. bits in [1, 16] or 32; any other value returns -1.0. */
double gact_variance_factor(int32_t bits);

/* NEXT-3 — the reduction of Alg. 1: sum_i (a_i - b_i)^2 of two gradient
 * vectors g0, g1 (one fwd+bwd each, seeds differing only for tensor l), from which
 * c_l = 1/2 ||g0 - g1||^2 / S(b_l). Deterministic: a fixed grid of GACT_REDUCE_BLOCKS
 * blocks writes binary64 partial sums in a fixed order, one block adds them in order, so
 * the result is a pure function of (a, b, n) on any GPU.
 *   a, b       device, n elements of `dtype` (gact_dtype), 16-byte aligned
 *   partials   device, workspace of GACT_REDUCE_BLOCKS doubles (caller-owned)
 *   out        device, out, one double (overwritten, not accumulated)
 * Each element is widened exactly to binary64; (a - b)^2 accumulates in binary64. */
#define GACT_REDUCE_BLOCKS 512
gact_status gact_sq_diff_sum(const void* a, const void* b, int32_t dtype, int64_t n,
                             double* partials, double* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GACT_H_ */
