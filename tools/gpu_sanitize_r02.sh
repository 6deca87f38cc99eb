#!/bin/bash
# compute-sanitizer, round 2: racecheck on the batched shared-memory launches (fp32 G = 2048 /
# 4096 CTA kernel, 2-byte G = 4096 stage) the round-1 race lived in; memcheck / initcheck /
# synccheck on the parity subset that reaches every kernel family with the 8-bit generator.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make oracle > /dev/null
TAG=${1:-r02}
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider \
   -k "batch_large_groups or (batch_equals_single and (2048 or 4096)) or (edge_groups and (2048 or 4096))" > gpurun_out/sanitizer_racecheck_$TAG.log 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_racecheck_$TAG.log | tail -3
for tool in memcheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
     -k "c1_config or tiny_and_ragged or edge_values or batch_large_groups or group_stats_matches or threshold_ties or (edge_groups and bf16)" > gpurun_out/sanitizer_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_${tool}_$TAG.log | tail -2
done
