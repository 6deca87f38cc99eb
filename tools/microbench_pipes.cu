// Issue cost of the instructions the quantize kernel is built from, on this GPU.
// Each kernel runs ITER x UNROLL independent ops per thread over 8 independent chains
// (enough ILP to be throughput-bound); prints warp-instructions per cycle per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITER 4096
#define CH 8

__device__ __forceinline__ void mulw(uint32_t a, uint32_t m, uint32_t& lo, uint32_t& hi) {
  asm volatile("{\n\t.reg .b64 p;\n\tmul.wide.u32 p, %2, %3;\n\tmov.b64 {%0, %1}, p;\n\t}" : "=r"(lo), "=r"(hi) : "r"(a), "r"(m));
}

template <int OP>
__global__ void k(uint32_t* out, uint32_t seed) {
  uint32_t a[CH], b[CH];
  float f[CH];
  unsigned long long f2[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { a[c] = seed * (threadIdx.x + c); b[c] = a[c] ^ 0x1234567u; f[c] = (float)a[c]; f2[c] = ((unsigned long long)a[c] << 32) | b[c]; }
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) { uint32_t lo, hi; mulw(a[c], 0xD2511F53u, lo, hi); a[c] = lo ^ hi; }   // IMAD.WIDE + LOP3
      if (OP == 1) { asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(b[c])); }      // IMAD
      if (OP == 2) { asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(f[(c+1)%CH]), "f"(f[(c+2)%CH])); } // FFMA
      if (OP == 3) { asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(f2[c]) : "l"(f2[(c+1)%CH]), "l"(f2[(c+2)%CH])); } // FFMA2
      if (OP == 4) { asm volatile("add.rm.f32x2 %0, %0, %1;" : "+l"(f2[c]) : "l"(f2[(c+1)%CH])); } // FADD2
      if (OP == 5) { asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b[c]), "r"(a[(c+1)%CH])); } // LOP3
      if (OP == 6) { asm volatile("prmt.b32 %0, %0, %1, 0x7610;" : "+r"(a[c]) : "r"(b[c])); }  // PRMT
      if (OP == 7) { uint32_t lo, hi; mulw(a[c], 0xD2511F53u, lo, hi); a[c] = lo; b[c] ^= hi; } // IMAD.WIDE only
      if (OP == 8) { asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(f[(c+1)%CH]), "f"(f[(c+2)%CH])); } // FMNMX3
      if (OP == 9) { asm volatile("fma.rm.f32x2 %0, %0, %1, %2;" : "+l"(f2[c]) : "l"(f2[(c+1)%CH]), "l"(f2[(c+2)%CH])); } // FFMA2.RM
      if (OP == 10) { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f[c]) : "f"(f[(c+1)%CH])); } // FADD
      if (OP == 11) { asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(f[c]) : "f"(f[(c+3)%CH]), "f"(f[(c+5)%CH])); } // FFMA (acc chain)
      if (OP == 12) { uint32_t lo, hi; mulw(a[c], 0xD2511F53u, lo, hi); a[c] = lo; b[c] ^= hi;
                      asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(f[c]) : "f"(f[(c+3)%CH]), "f"(f[(c+5)%CH]));
                      asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(f[(c+1)%CH]) : "f"(f[(c+3)%CH]), "f"(f[(c+5)%CH])); } // IMAD.WIDE + LOP3 + 2 FFMA
      if (OP == 13) { uint32_t lo, hi; mulw(a[c], 0xD2511F53u, lo, hi); a[c] = lo; b[c] ^= hi;
                      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(f2[c]) : "l"(f2[(c+1)%CH]), "l"(f2[(c+2)%CH])); } // IMAD.WIDE + LOP3 + FFMA2
      if (OP == 14) { uint32_t lo, hi; mulw(a[c], 0xD2511F53u, lo, hi); a[c] = lo; b[c] ^= hi;
                      asm volatile("add.rm.f32x2 %0, %0, %1;" : "+l"(f2[c]) : "l"(f2[(c+1)%CH])); } // IMAD.WIDE + LOP3 + FADD2
      if (OP == 15) { asm volatile("{.reg .b16 l; mov.b32 {l,_}, %1; sub.rn.f32.bf16 %0, l, %0;}" : "+f"(f[c]) : "r"(a[c])); } // FHADD.BF16
      if (OP == 16) { asm volatile("min.bf16x2 %0, %0, %1;" : "+r"(a[c]) : "r"(b[c])); } // HMNMX2.BF16
      if (OP == 17) { asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(b[c]));
                      asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(f[c]) : "f"(f[(c+3)%CH]), "f"(f[(c+5)%CH])); } // IMAD + FFMA
      if (OP == 18) { asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(f2[c]) : "l"(f2[(c+3)%CH]), "l"(f2[(c+5)%CH])); } // FFMA2 acc chain
      if (OP == 19) { asm volatile("add.rm.f32 %0, %0, 0f4B000000;" : "+f"(f[c])); } // FADD imm
      if (OP == 20) { asm volatile("add.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(b[c])); } // VIADD / IADD3
      if (OP == 21) { asm volatile("fma.rm.f64 %0, %0, %1, %2;" : "+l"(f2[c]) : "l"(f2[(c+1)%CH]), "l"(f2[(c+2)%CH])); } // DFMA
      if (OP == 22) { uint32_t lo, hi; mulw(a[c], 0xD2511F53u, lo, hi); a[c] = lo; b[c] ^= hi;
                      asm volatile("add.u32 %0, %0, %1;" : "+r"(b[(c+1)%CH]) : "r"(a[(c+3)%CH])); } // IMAD.WIDE + LOP3 + add
      if (OP == 23) { asm volatile("mov.u32 %0, %1;" : "=r"(a[c]) : "r"(b[(c+1)%CH])); asm volatile("xor.b32 %0, %0, %1;" : "+r"(b[c]) : "r"(a[c])); } // MOV + LOP3
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c] ^ b[c] ^ __float_as_uint(f[c]) ^ (uint32_t)f2[c] ^ (uint32_t)(f2[c] >> 32);
  if (s == 0x12345) out[0] = s;
}

template <int OP>
void run(const char* name, double instr_per_op) {
  uint32_t* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int blocks = sms * 4, threads = 512;
  k<OP><<<blocks, threads>>>(d, 1); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<blocks, threads>>>(d, 1);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double warp_ops = (double)blocks * threads / 32 * ITER * CH * instr_per_op;
  // use the measured SM clock estimate from the driver's max clock (kHz)
  double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-22s %8.3f ms  warp-instr/cycle/SMSP = %.3f  (at %.0f MHz max clock)\n", name, ms, warp_ops / cycles / (sms * 4), clk / 1e3);
}

int main() {
  run<0>("IMAD.WIDE+LOP3", 2); run<7>("IMAD.WIDE+LOP3(b)", 2); run<1>("IMAD", 1); run<2>("FFMA", 1);
  run<3>("FFMA2", 1); run<9>("FFMA2.RM", 1); run<4>("FADD2.RM", 1); run<10>("FADD", 1);
  run<5>("LOP3", 1); run<6>("PRMT", 1); run<8>("FMNMX3", 1);
  run<11>("FFMA acc", 1); run<12>("IMADW+LOP3+2FFMA", 4); run<13>("IMADW+LOP3+FFMA2", 3);
  run<14>("IMADW+LOP3+FADD2", 3); run<15>("FHADD.BF16 (sub)", 1); run<16>("HMNMX2.BF16", 1);
  run<17>("IMAD+FFMA", 2); run<18>("FFMA2 acc", 1); run<19>("FADD imm", 1);
  run<20>("IADD (add.u32)", 1); run<21>("DFMA", 1); run<22>("IMADW+LOP3+add", 3); run<23>("MOV+LOP3", 2);
  return 0;
}
