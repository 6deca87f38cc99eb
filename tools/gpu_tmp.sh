#!/bin/bash
cd "$(dirname "$0")/.."
for dt in bf16 f32; do for G in 32 64 128 256 512 1024 2048 4096; do
  python tools/prof_kernels.py --G $G --dtype $dt --bits 4 --reps 1 2>&1 | tail -1
done; done
