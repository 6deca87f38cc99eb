#!/bin/bash
cd "$(dirname "$0")/.."
for d in "" build/var_*; do echo "== ${d:-default}"; for dt in f32 bf16; do for b in 2 8; do
  if [ -n "$d" ]; then GACT_LIB_PATH=$d/libgact.so python tools/prof_kernels.py --bits $b --dtype $dt --reps 1 2>&1 | tail -1;
  else python tools/prof_kernels.py --bits $b --dtype $dt --reps 1 2>&1 | tail -1; fi
done; done; done
