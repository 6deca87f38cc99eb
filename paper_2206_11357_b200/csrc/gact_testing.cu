// gact_testing.cu — the test-only entry point of include/gact_testing.h: the device Philox
// generator at arbitrary counters (plain and shared-round forms), for the parity tests.
#include "gact_device.cuh"
#include "gact_testing.h"

namespace {

template <int N>
__global__ void philox_blocks_kernel(uint64_t blk, uint64_t seed, int shared_form, uint32_t* out) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint4 r[N];
  if (shared_form) {
    gact::philox4x32_10_xn<N>(blk, k0, k1, r);
  } else {
#pragma unroll
    for (int m = 0; m < N; ++m) r[m] = gact::philox4x32_10(blk + 32u * m, k0, k1);
  }
  for (int m = 0; m < N; ++m) {
    out[4 * m + 0] = r[m].x;
    out[4 * m + 1] = r[m].y;
    out[4 * m + 2] = r[m].z;
    out[4 * m + 3] = r[m].w;
  }
}

}  // namespace

extern "C" gact_status gact_test_philox_blocks(uint64_t blk, uint64_t seed, int32_t shared_form,
                                               int32_t n_blocks, uint32_t* out, void* stream) {
  if (!out || (n_blocks != 4 && n_blocks != 8)) return GACT_ERR_INVALID_ARG;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n_blocks == 4) philox_blocks_kernel<4><<<1, 1, 0, s>>>(blk, seed, shared_form, out);
  else philox_blocks_kernel<8><<<1, 1, 0, s>>>(blk, seed, shared_form, out);
  return cudaPeekAtLastError() == cudaSuccess ? GACT_OK : GACT_ERR_CUDA;
}
