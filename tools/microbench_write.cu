// Write bandwidth of streaming stores by width on this GPU (calibrates the dequantize roofline).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_write tools/microbench_write.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int W>  // bytes per store per thread: 16 or 32
__global__ void wr(uint32_t* p, size_t n_words, uint32_t v) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * (W / 4);
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * (W / 4); i < n_words; i += stride) {
    if (W == 16) asm volatile("st.global.cs.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "r"(v) : "memory");
    else asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + i), "r"(v) : "memory");
  }
}
template <int W>
__global__ void wr_plain(uint32_t* p, size_t n_words, uint32_t v) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * (W / 4);
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * (W / 4); i < n_words; i += stride) {
    if (W == 16) asm volatile("st.global.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "r"(v) : "memory");
    else asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + i), "r"(v) : "memory");
  }
}

template <typename K>
void run(const char* name, K k, uint32_t* p, size_t bytes, int blocks) {
  k<<<blocks, 256>>>(p, bytes / 4, 1u);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) k<<<blocks, 256>>>(p, bytes / 4, (uint32_t)r);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s blocks %5d: %7.1f GB/s\n", name, blocks, bytes * 10.0 / (ms * 1e-3) / 1e9);
}

int main() {
  size_t bytes = 1ull << 31;
  uint32_t* p; cudaMalloc(&p, bytes);
  for (int blocks : {148 * 4, 148 * 8, 148 * 32}) {
    run("st.global.cs.v4 (16 B)", wr<16>, p, bytes, blocks);
    run("st.global.cs.v8 (32 B)", wr<32>, p, bytes, blocks);
    run("st.global.v4 (16 B)", wr_plain<16>, p, bytes, blocks);
    run("st.global.v8 (32 B)", wr_plain<32>, p, bytes, blocks);
  }
  return 0;
}
