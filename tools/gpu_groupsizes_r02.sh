#!/bin/bash
# Quantize / dequantize rates by group size (2^28 elements, b = 4), single-tensor launches.
cd "$(dirname "$0")/.."
for G in 32 64 128 256 512 1024 2048 4096 96 160 224 800 4064; do
  for dt in bf16 f32; do
    python tools/prof_kernels.py --G $G --dtype $dt --bits 4 --reps 1 2>&1 | tail -1
  done
done
