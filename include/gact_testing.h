/* gact_testing.h — test-only entry point of libgact (not part of the method's ABI).
 *
 * Exposes the device Philox4x32-10 generator of the quantize kernels (include/gact.h,
 * "Random lanes") at arbitrary block counters, so that tests can pin it against the CPU
 * oracle where the quantize kernels' shortcuts differ from the plain generator: the batched
 * kernels compute a lane's N blocks blk + 32 m (m < N; N = 8 for 2-byte inputs, 4 for fp32)
 * with rounds 0-1 shared, and fall back to N plain calls when
 * lo32(blk) + 32 (N - 1) wraps — which only tensors beyond 2^35 elements reach.
 */
#ifndef GACT_TESTING_H_
#define GACT_TESTING_H_

#include <stdint.h>

#include "gact.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Writes the n_blocks x 4 output words of Philox4x32-10 for counters (lo32, hi32, 0, 0) of
 * blk + 32 m, m < n_blocks, key = (lo32(seed), hi32(seed)), to out[4 m + j] (a DEVICE buffer
 * of 4 n_blocks uint32, caller-owned). n_blocks is 4 or 8. shared_form != 0: the quantize
 * kernels' shared-round form (including its wrap fallback); 0: plain generator calls. One
 * thread, enqueued on `stream`. Errors: GACT_ERR_INVALID_ARG for out == NULL or another
 * n_blocks, GACT_ERR_CUDA on launch failure. */
gact_status gact_test_philox_blocks(uint64_t blk, uint64_t seed, int32_t shared_form, int32_t n_blocks,
                                    uint32_t* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GACT_TESTING_H_ */
