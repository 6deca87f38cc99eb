#!/bin/bash
# Round-2 warp-pair G = 4096 kernel: full GPU suite, then racecheck / synccheck / memcheck on
# the 2-byte G = 4096 cases (single, batched, edge groups, fuzz).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r02c.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_r02c.log
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -p no:cacheprovider \
     -k "4096 and not f32 and not float32" > gpurun_out/sanitizer_${tool}_r02c.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer_${tool}_r02c.log | tail -2
done
