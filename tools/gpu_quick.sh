#!/bin/bash
# Quick GPU iteration: parity tests + per-kernel throughput on one 2^28-element tensor
# (+ any tuning variants in build/var_*).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for dt in bf16 f32; do for b in 1 2 4 8; do
  python tools/prof_kernels.py --bits $b --dtype $dt --reps 1 2>&1 | tail -1
done; done
python tools/prof_kernels.py --bits 2 --reps 1 --ref 2>&1 | tail -2
for d in build/var_*; do
  [ -f $d/libgact.so ] || continue
  echo "== $d"
  for dt in bf16 f32; do for b in 2 8; do
    GACT_LIB_PATH=$d/libgact.so python tools/prof_kernels.py --bits $b --dtype $dt --reps 1 2>&1 | tail -1
  done; done
done
