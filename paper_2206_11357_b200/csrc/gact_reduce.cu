// gact_reduce.cu — deterministic ||a - b||^2 (NEXT-3: the sensitivity reduction of Alg. 1,
// c_l = 1/2 ||g0 - g1||^2 / S(b_l)).
//
// Pass 1: a fixed grid of GACT_REDUCE_BLOCKS blocks; block k sums, in binary64, the squared
// differences of a fixed, grid-strided set of 8-element chunks, reduces its 8 warps in a
// fixed tree and writes partials[k]. Pass 2: one warp adds the partials in index order
// (fixed tree). No atomics: bit-reproducible on any GPU.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gact.h"
#include "gact_device.cuh"

namespace gact {
namespace {

constexpr int kRedBlocks = GACT_REDUCE_BLOCKS;

template <int DT>
__device__ __forceinline__ double widen_d(const void* p, int64_t i) {
  if constexpr (DT == DT_F32) return (double)static_cast<const float*>(p)[i];
  else if constexpr (DT == DT_BF16) return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  else return (double)__half2float(static_cast<const __half*>(p)[i]);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int DT>
__global__ void __launch_bounds__(kThreads) sq_diff_partial(const void* a, const void* b, int64_t n,
                                                            double* partials) {
  double acc = 0.0;
  const int64_t chunks = (n + kChunk - 1) / kChunk;
  for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < chunks; c += (int64_t)kRedBlocks * kThreads) {
    const int64_t e = c * kChunk;
    if (e + kChunk <= n) {
      Raw8<DT> ra, rb;
      load8<DT>(ra, a, e);
      load8<DT>(rb, b, e);
      float va[8], vb[8];
      widen8<DT>(ra, va);
      widen8<DT>(rb, vb);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double d = (double)va[j] - (double)vb[j];
        acc = __fma_rn(d, d, acc);
      }
    } else {
      for (int64_t i = e; i < n; ++i) {
        const double d = widen_d<DT>(a, i) - widen_d<DT>(b, i);
        acc = __fma_rn(d, d, acc);
      }
    }
  }
  __shared__ double ws[kWarps];
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kWarps ? ws[threadIdx.x] : 0.0;
    v = warp_sum_d(v);
    if (threadIdx.x == 0) partials[blockIdx.x] = v;
  }
}

__global__ void sq_diff_final(const double* partials, double* out) {
  double v = 0.0;
  for (int k = threadIdx.x; k < kRedBlocks; k += 32) v += partials[k];
  v = warp_sum_d(v);
  if (threadIdx.x == 0) *out = v;
}

}  // namespace
}  // namespace gact

extern "C" gact_status gact_sq_diff_sum(const void* a, const void* b, int32_t dtype, int64_t n,
                                        double* partials, double* out, void* stream) {
  if (n < 0 || dtype < 0 || dtype > 2 || !partials || !out) return GACT_ERR_INVALID_ARG;
  if (n > 0 && (!a || !b)) return GACT_ERR_INVALID_ARG;
  if ((n > 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15)) ||
      (reinterpret_cast<uintptr_t>(partials) & 7) || (reinterpret_cast<uintptr_t>(out) & 7))
    return GACT_ERR_ALIGNMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (dtype) {
    case gact::DT_F32: gact::sq_diff_partial<gact::DT_F32><<<gact::kRedBlocks, gact::kThreads, 0, s>>>(a, b, n, partials); break;
    case gact::DT_BF16: gact::sq_diff_partial<gact::DT_BF16><<<gact::kRedBlocks, gact::kThreads, 0, s>>>(a, b, n, partials); break;
    default: gact::sq_diff_partial<gact::DT_F16><<<gact::kRedBlocks, gact::kThreads, 0, s>>>(a, b, n, partials); break;
  }
  gact::sq_diff_final<<<1, 32, 0, s>>>(partials, out);
  return cudaGetLastError() == cudaSuccess ? GACT_OK : GACT_ERR_CUDA;
}
