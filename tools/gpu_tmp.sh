#!/bin/bash
cd "$(dirname "$0")/.."
make oracle >/dev/null
for tool in memcheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
     -k "c1_config or tiny_and_ragged or edge_values or group_stats_matches or threshold_ties or philox_blocks or (quantize_dequantize_parity and (256 or 512 or 1024 or 32))" > gpurun_out/sanitizer_${tool}_r01f.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_${tool}_r01f.log | tail -2
done
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
   -k "(quantize_dequantize_parity and (2048 or 4096)) or group_stats_matches" > gpurun_out/sanitizer_racecheck_r01f.log 2>&1
echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer_racecheck_r01f.log | tail -2
