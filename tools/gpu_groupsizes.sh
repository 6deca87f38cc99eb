#!/bin/bash
# Kernel throughput across group sizes (one 2^28-element tensor).
cd "$(dirname "$0")/.."
for G in 32 64 128 256 512 1024 2048 4096; do for dt in bf16 f32; do
  python tools/prof_kernels.py --bits 4 --dtype $dt --G $G --reps 1 | tail -1
done; done
