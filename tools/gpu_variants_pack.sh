#!/bin/bash
# Quantize throughput of each build/var_* against the default build (bf16 b = 1/2/4, f32 b = 2),
# two passes interleaved to expose run-to-run noise. Experiments only.
cd "$(dirname "$0")/.."
make oracle > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for pass in 1 2; do
  for d in default build/var_*; do
    lib=paper_2206_11357_b200/libgact.so; [ "$d" != default ] && lib=$d/libgact.so
    for spec in "bf16 1" "bf16 2" "bf16 4" "bf16 8" "f32 2"; do set -- $spec
      echo "$pass $d $(GACT_LIB_PATH=$lib python tools/prof_kernels.py --bits $2 --dtype $1 --reps 1 2>&1 | tail -1)"
    done
  done
done
