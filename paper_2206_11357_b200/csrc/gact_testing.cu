// gact_testing.cu — the test-only entry point of include/gact_testing.h: the device Philox
// generator at arbitrary counters (plain and shared-round forms), for the parity tests.
#include "gact_device.cuh"
#include "gact_testing.h"

namespace {

__global__ void philox_blocks_kernel(uint64_t blk, uint64_t seed, int shared_form, uint32_t* out) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint4 r[4];
  if (shared_form) {
    gact::philox4x32_10_x4(blk, k0, k1, r);
  } else {
#pragma unroll
    for (int m = 0; m < 4; ++m) r[m] = gact::philox4x32_10(blk + 32u * m, k0, k1);
  }
  for (int m = 0; m < 4; ++m) {
    out[4 * m + 0] = r[m].x;
    out[4 * m + 1] = r[m].y;
    out[4 * m + 2] = r[m].z;
    out[4 * m + 3] = r[m].w;
  }
}

}  // namespace

extern "C" gact_status gact_test_philox_blocks(uint64_t blk, uint64_t seed, int32_t shared_form,
                                               uint32_t* out, void* stream) {
  if (!out) return GACT_ERR_INVALID_ARG;
  philox_blocks_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(blk, seed, shared_form, out);
  return cudaPeekAtLastError() == cudaSuccess ? GACT_OK : GACT_ERR_CUDA;
}
