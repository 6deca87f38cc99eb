#!/bin/bash
# compute-sanitizer on the kernels added or changed late in round 2: generic group sizes,
# 8-tile small-G units, the shared-round G = 4096 stage.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
for tool in memcheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py -q -p no:cacheprovider \
     -k "generic or every_output or (parity and (64 or 128 or 4096) and bf16) or staged_generic" > gpurun_out/sanitizer_${tool}_r02b.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer_${tool}_r02b.log | tail -2
done
