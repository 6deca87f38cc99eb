#!/bin/bash
# Per-kernel throughput of each tuning variant in build/var_*/ (experiments only).
cd "$(dirname "$0")/.."
for d in build/var_*; do
  echo "== $d"
  for dt in ${DTS:-bf16 f32}; do for b in ${BITSLIST:-2 4 8}; do
    GACT_LIB_PATH=$d/libgact.so python tools/prof_kernels.py --bits $b --dtype $dt --reps 1 2>&1 | tail -1
  done; done
done
